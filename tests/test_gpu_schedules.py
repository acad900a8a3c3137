"""Race / ordering detection by schedule invariance (compute-sanitizer is closed on the GPU pool, so
its racecheck / synccheck cannot run -- profiles/r02_sanitizer.txt).  The engine's results are
bitwise deterministic by construction (fixed-order reductions, no atomics on data), so every way
of scheduling the same fit must give BITWISE identical traces and factors:
  graph replay (default) | eager launches (CPF_NO_GRAPH=1) | serial fork, no pass-B / LU overlap
  (CPF_SERIAL=1) | no programmatic dependent launch (CPF_PDL=0) | speculative rejection branch
  on / off (CPF_SPEC) | batched instead of progressive triangular inverse (CPF_TRI_PROG=0) |
  repeated runs.
A missing stream / event dependency, an mbarrier or flag race in the LU panels or the tensor-pass
pipelines would show up as a difference under one of these schedules."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SCHEDULES = [
    {},
    {"CPF_NO_GRAPH": "1"},
    {"CPF_SERIAL": "1"},
    {"CPF_PDL": "0"},
    {"CPF_SPEC": "1"},
    {"CPF_SPEC": "0"},
    {"CPF_TRI_PROG": "0"},
    {"CPF_TRI_PROG": "0", "CPF_SPEC": "1"},
    {"CPF_NO_GRAPH": "1", "CPF_SERIAL": "1", "CPF_PDL": "0"},
]

CASES = {
    "c0": ("c0", (20, 20, 20), 5, {}),
    "c2mini": ("c2", (12, 12, 12, 12), 5, {}),
    "c3mini": ("c3", (24, 24, 24), 4, {}),
    "c4mini_int8": ("c4", (20, 20, 40), 4, {"CPF_OZ": "1"}),
    # multi-panel LU (n_B = 3 * 12^2 = 432), DMMA-eligible I1
    "mid": ("c4", (256, 96, 64), 12, {}),
}


@pytest.fixture(scope="module")
def api(engine_lib):
    import paper_1205_2584_b200 as api

    return api


def _run(api, monkeypatch, case, env):
    from paper_1205_2584_b200 import synth

    key, dims, rank, base_env = CASES[case]
    for k, v in {**base_env, **env}.items():
        monkeypatch.setenv(k, v)
    cfg = synth.scaled(synth.CONFIGS[key], dims, rank=rank, max_iters=10, name=case)
    y = synth.make_tensor(cfg, 0)
    tau = synth.tau_for_unit_mu(cfg, 0)
    res = api.fit(y, api.FitConfig(rank=rank, tau=tau, tol=0.0, max_iters=10, seed=0, init="random"))
    for k in {**base_env, **env}:
        monkeypatch.delenv(k, raising=False)
    return [(r.iter, r.relerr, r.mu, r.accepted) for r in res.trace], res.model.as_vector()


@pytest.mark.parametrize("case", sorted(CASES))
def test_bitwise_identical_across_schedules(api, monkeypatch, case):
    base_tr, base_v = _run(api, monkeypatch, case, {})
    again_tr, again_v = _run(api, monkeypatch, case, {})
    assert again_tr == base_tr and np.array_equal(again_v, base_v), "repeat run differs"
    for env in SCHEDULES[1:]:
        tr, v = _run(api, monkeypatch, case, env)
        assert tr == base_tr, f"trace differs under {env}"
        assert np.array_equal(v, base_v), f"factors differ under {env}: max |d| {np.max(np.abs(v - base_v)):.3e}"


@pytest.mark.parametrize("case", ["c0", "c2mini", "c3mini"])
def test_repeated_fits_bitwise(api, monkeypatch, case):
    """Ten repeats with the speculative rejection branch on (its early abandonment reads the
    decision written by another stream's kernel: a torn read once made ~1 in 6 runs diverge)."""
    base_tr, base_v = _run(api, monkeypatch, case, {"CPF_SPEC": "1"})
    for _ in range(9):
        tr, v = _run(api, monkeypatch, case, {"CPF_SPEC": "1"})
        assert tr == base_tr and np.array_equal(v, base_v)


@pytest.mark.parametrize("env", [{}, {"CPF_TRI_ROWS": "0"}])
def test_many_full_c2_fits_do_not_fault(api, monkeypatch, env):
    """Config 2 at full size (n_B = 900: two-CTA cluster panels, speculative branch on), 60 fits in
    one process.  The branch's panels run beside k_decide; before their gate was latched by a single
    thread (lu.cuh panel_gated) about one fit in a hundred hung or faulted on its last iteration,
    when two CTAs of a cluster read `stopped` on either side of k_decide's write."""
    from paper_1205_2584_b200 import synth

    for k, v in env.items():
        monkeypatch.setenv(k, v)
    cfg = synth.CONFIGS["c2"]
    y = synth.make_tensor(cfg, 0)
    tau = synth.tau_for_unit_mu(cfg, 0)
    base = None
    for _ in range(60):
        res = api.fit(y, api.FitConfig(rank=cfg.rank, tau=tau, tol=0.0, max_iters=cfg.max_iters, seed=0, init="random"))
        sig = ([(r.iter, r.relerr, r.mu, r.accepted) for r in res.trace], res.final_relerr)
        if base is None:
            base = sig
        assert sig == base
