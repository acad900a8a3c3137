"""Fault injection on the GPU fit (SURVEY §5 failure detection): an exactly singular core system at
iteration t must end the fit the way the reference does -- the LinAlgError inside the loop becomes
stop_reason "error at iteration t: <message>" and the returned model is the last accepted one
(solver.py:349-352; verify.py:117-118).  The hook CPF_TEST_SINGULAR=t zeroes a column of the core
system the engine factors for iteration t (phi.cuh k_test_zero_col), in graph and eager mode, with
and without the speculative rejection branch."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api(engine_lib):
    import paper_1205_2584_b200 as api

    return api


def _problem(cfg_key="c0", dims=(20, 20, 20), rank=5):
    from paper_1205_2584_b200 import synth

    cfg = synth.scaled(synth.CONFIGS[cfg_key], dims, rank=rank, max_iters=12, name="fault")
    return cfg, synth.make_tensor(cfg, 0), synth.tau_for_unit_mu(cfg, 0)


@pytest.mark.parametrize("variant,msg", [("auto", "Singular matrix"),
                                         ("flm-a", "I + Psi K numerically singular: Singular matrix")])
@pytest.mark.parametrize("spec", ["0", "1"])
@pytest.mark.parametrize("graph", ["graph", "eager"])
@pytest.mark.parametrize("t_bad", [1, 5])
def test_singular_core_stops_with_reference_error(api, monkeypatch, variant, msg, spec, graph, t_bad):
    cfg, y, tau = _problem()
    monkeypatch.setenv("CPF_SPEC", spec)
    if graph == "eager":
        monkeypatch.setenv("CPF_NO_GRAPH", "1")
    conf = api.FitConfig(rank=cfg.rank, variant=variant, tau=tau, tol=0.0, max_iters=12, seed=0, init="random")
    clean = api.fit(y, api.FitConfig(rank=cfg.rank, variant=variant, tau=tau, tol=0.0, max_iters=t_bad - 1, seed=0,
                                     init="random")) if t_bad > 1 else None
    monkeypatch.setenv("CPF_TEST_SINGULAR", str(t_bad))
    res = api.fit(y, conf)
    assert res.stop_reason == f"error at iteration {t_bad}: {msg}"
    assert res.iters == t_bad - 1
    if clean is not None:
        got = [(r.iter, r.relerr, r.mu, r.accepted) for r in res.trace]
        ref = [(r.iter, r.relerr, r.mu, r.accepted) for r in clean.trace]
        assert got == ref
        np.testing.assert_array_equal(res.model.as_vector(), clean.model.as_vector())


def test_singular_core_on_int8_passes(api, monkeypatch):
    """The same stop on the int8 tensor-core pass family (config 4's default), forced at this size."""
    cfg, y, tau = _problem()
    monkeypatch.setenv("CPF_OZ", "1")
    monkeypatch.setenv("CPF_TEST_SINGULAR", "3")
    res = api.fit(y, api.FitConfig(rank=cfg.rank, tau=tau, tol=0.0, max_iters=12, seed=0, init="random"))
    assert res.stop_reason == "error at iteration 3: Singular matrix"
    assert res.iters == 2
