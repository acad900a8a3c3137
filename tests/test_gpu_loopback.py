"""The multi-rank engine path EXECUTED: P = 2, 3, 4, 8 slab-sharded ranks on one
B200 through the loopback test transport (comm.cuh: the same allreduce / allgather / broadcast
sites as NCCL, exchanged through device buffers with event ordering and host barriers -- no kernel
waits on another rank's kernel).  Each rank's fit is the public fit(y_slab, ..., distributed=rank,
slab_of=I_N) driven from its own thread.  Checks: every rank returns the same result; against the
single-rank fit the accept/reject sequence, iteration count and stop reason are identical, every
recorded relative error is within 1e-12 and the factors within 1e-10 relative (the only change is
the summation order of the slab partials).  Ragged slabs (20 over 3 ranks = 7/7/6, 50 over 3) and an
empty rank (20 over 8: the last rank owns no slice) are included."""

import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = {
    "c0": ("c0", (20, 20, 20), 5, {}),
    "c2mini": ("c2", (12, 12, 12, 12), 5, {}),
    "c3mini": ("c3", (24, 24, 24), 4, {}),
    "c4mini_int8": ("c4", (20, 20, 40), 4, {"CPF_OZ": "1"}),
    "ragged": ("c4", (32, 24, 50), 6, {}),
}


@pytest.fixture(scope="module")
def api(engine_lib):
    import paper_1205_2584_b200 as api

    return api


def _problem(case):
    from paper_1205_2584_b200 import synth

    key, dims, rank, env = CASES[case]
    cfg = synth.scaled(synth.CONFIGS[key], dims, rank=rank, max_iters=12, name=case)
    return cfg, synth.make_tensor(cfg, 0), synth.tau_for_unit_mu(cfg, 0), env


def _sharded_fit(api, y, conf, world):
    from paper_1205_2584_b200 import _native
    from paper_1205_2584_b200.solver import LoopbackRank, slab_bounds

    group = _native.LoopbackGroup(world)
    out, errs = [None] * world, [None] * world
    i_n = y.shape[-1]

    def run(r):
        try:
            lo, hi = slab_bounds(i_n, world, r)
            out[r] = api.fit(np.asfortranarray(y[..., lo:hi]), conf, distributed=LoopbackRank(group, r), slab_of=i_n)
        except BaseException as exc:  # noqa: BLE001
            errs[r] = exc

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    group.close()
    bad = [(r, e) for r, e in enumerate(errs) if e is not None]
    if bad:
        # report the root cause first: a rank that failed on its own, not one that timed out waiting
        bad.sort(key=lambda re_: "timed out" in str(re_[1]))
        raise AssertionError(f"rank errors: {[(r, repr(e)) for r, e in bad]}") from bad[0][1]
    return out


def _trace(res):
    return [(r.iter, r.relerr, r.mu, r.accepted) for r in res.trace]


def _compare(single, ranks, tag, fac_tol=1e-10, err_tol=1e-12):
    for r, res in enumerate(ranks):
        assert _trace(res) == _trace(ranks[0]), f"{tag}: rank {r} differs from rank 0"
        assert np.array_equal(res.model.as_vector(), ranks[0].model.as_vector())
    res = ranks[0]
    assert res.stop_reason == single.stop_reason
    assert [t.accepted for t in res.trace] == [t.accepted for t in single.trace], tag
    d_err = max(abs(a.relerr - b.relerr) for a, b in zip(res.trace, single.trace))
    v, w = res.model.as_vector(), single.model.as_vector()
    d_fac = float(np.linalg.norm(v - w) / np.linalg.norm(w))
    print(f"{tag}: max |relerr diff| {d_err:.2e}, factor rel diff {d_fac:.2e}")
    assert d_err < err_tol, tag
    assert d_fac < fac_tol, tag


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("world", [2, 3, 4])
def test_sharded_fit_matches_single_rank(api, monkeypatch, case, world):
    cfg, y, tau, env = _problem(case)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    conf = api.FitConfig(rank=cfg.rank, tau=tau, tol=0.0, max_iters=12, seed=0, init="random")
    single = api.fit(y, conf)
    _compare(single, _sharded_fit(api, y, conf, world), f"{case} P={world}")


def test_empty_rank(api):
    """20 slices over 8 ranks: ceil split 3, the last rank owns [20, 20)."""
    cfg, y, tau, _ = _problem("c0")
    conf = api.FitConfig(rank=cfg.rank, tau=tau, tol=0.0, max_iters=12, seed=0, init="random")
    _compare(api.fit(y, conf), _sharded_fit(api, y, conf, 8), "c0 P=8 (empty rank)")


@pytest.mark.parametrize("case", ["c0", "c3mini", "ragged"])
def test_sharded_svd_init(api, case):
    """init='svd' (the reference default) on a sharded tensor: the mode-N unfolding Gram is formed
    across ranks (slab broadcasts), so the default FitConfig works distributed."""
    cfg, y, tau, _ = _problem(case)
    conf = api.FitConfig(rank=cfg.rank, tau=tau, tol=0.0, max_iters=12, seed=0, init="svd")
    # the unfolding Grams' slab sums change order; the eigenvectors move by ~1e-12 (init only)
    _compare(api.fit(y, conf), _sharded_fit(api, y, conf, 3), f"{case} svd P=3", fac_tol=1e-9, err_tol=1e-10)


@pytest.mark.parametrize("variant", ["als", "als-ls"])
def test_sharded_als(api, variant):
    cfg, y, tau, _ = _problem("ragged")
    conf = api.FitConfig(rank=cfg.rank, variant=variant, tol=0.0, max_iters=8, seed=0, init="random")
    _compare(api.fit(y, conf), _sharded_fit(api, y, conf, 3), f"ragged {variant} P=3")


def test_sharded_unfolding_gram_all_modes(api):
    from paper_1205_2584_b200 import _native
    from paper_1205_2584_b200.solver import slab_bounds

    cfg, y, _, _ = _problem("ragged")
    single = _native.Engine(_native.CPF_REAL, y.shape, cfg.rank, 0)
    single.set_tensor_host(y)
    ref = [single.unfolding_gram(n) for n in (1, 2, 3)]
    single.close()
    world = 3
    group = _native.LoopbackGroup(world)
    got = [None] * world

    def run(r):
        lo, hi = slab_bounds(y.shape[-1], world, r)
        e = _native.Engine(_native.CPF_REAL, y.shape, cfg.rank, 0, r, world, loopback=group)
        e.set_tensor_host(np.asfortranarray(y[..., lo:hi]))
        got[r] = [e.unfolding_gram(n) for n in (1, 2, 3)]
        e.close()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    group.close()
    for r in range(world):
        for n in range(3):
            assert np.linalg.norm(got[r][n] - ref[n]) <= 1e-13 * np.linalg.norm(ref[n]), (r, n)
