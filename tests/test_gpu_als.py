"""GPU parity of the ALS baselines (variants "als" / "als-ls"): the engine's
sweeps (pass A / pass B MTTKRPs, Jacobi pinv_psd, line search by direct residual) through the
drop-in API against fixtures captured from the reference (tests/golden/make_als_golden.py).
Tolerances: pinv_psd 1e-10 relative (Frobenius); single steps 1e-10 relative; fits: every recorded
relative error within 1e-10 absolute, final factors within 1e-9 relative, same stop reason."""

import os

import numpy as np
import pytest

from tests import _golden as G

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def api(engine_lib):
    import paper_1205_2584_b200 as api

    return api


@pytest.mark.parametrize("name", sorted(k for k in G.als_units() if k.startswith("pinv_")))
def test_pinv_psd(api, name):
    c = G.als_units()[name]
    got = api.pinv_psd(c["in"])
    if not np.any(c["out"]):
        assert not np.any(got)
        return
    d = _rel(got, c["out"])
    print(f"{name}: rel diff {d:.2e}")
    assert d < 1e-10


def test_pinv_psd_rejects_large(api):
    with pytest.raises(ValueError):
        api.pinv_psd(np.eye(65))


@pytest.mark.parametrize("name", sorted(k for k in G.als_units() if k.startswith("step")))
def test_als_steps(api, name):
    c = G.als_units()[name]
    dims = tuple(int(x) for x in c["dims"])
    r = int(c["rank"])
    y = api.DenseTensor(c["y"])
    start = api.KruskalModel(G.split_stacked(c["start"], dims, r))
    hist = api.KruskalModel(G.split_stacked(c["hist"], dims, r))
    got = api.als_step(y, start).as_vector()
    assert _rel(got, c["als"]) < 1e-10
    for t in (1, 2, 5):
        got = api.als_line_search_step(y, start, hist, t).as_vector()
        assert _rel(got, c[f"ls_t{t}"]) < 1e-10, t
    got = api.als_line_search_step(y, start, None, 3).as_vector()
    assert _rel(got, c["ls_nohist"]) < 1e-10


def _fit(api, name, c):
    from paper_1205_2584_b200 import synth

    cfg = G.als_config(name, c)
    y = synth.make_tensor(cfg, 0)
    assert synth.tensor_digest(y) == str(c["digest"])
    variant = name.rsplit("_", 1)[1]
    conf = api.FitConfig(rank=cfg.rank, variant=variant, tol=float(c["tol"]), max_iters=int(c["max_iters"]), seed=0,
                         init="random")
    return api.fit(y, conf)


def _check_fit(res, c, name):
    tr = np.array([[r.iter, r.relerr, r.mu, float(r.accepted)] for r in res.trace])
    assert tr.shape == c["trace"].shape, name
    assert res.stop_reason == str(c["stop"])
    d_err = float(np.max(np.abs(tr[:, 1] - c["trace"][:, 1])))
    d_fac = _rel(res.model.as_vector(), c["factors"])
    print(f"{name}: max |relerr diff| {d_err:.2e}, factor rel diff {d_fac:.2e}")
    assert d_err < 1e-10
    assert d_fac < 1e-9


@pytest.mark.parametrize("name", sorted(G.als_fits()))
def test_fit_als(api, name):
    c = G.als_fits()[name]
    _check_fit(_fit(api, name, c), c, name)


@pytest.mark.parametrize("name", sorted(k for k, c in G.als_fits().items() if not bool(c["complex"])))
def test_fit_als_int8_passes(api, name, monkeypatch):
    """The same fits with the int8 tensor-core passes forced (config 4's default pass family)."""
    monkeypatch.setenv("CPF_OZ", "1")
    c = G.als_fits()[name]
    res = _fit(api, name, c)
    _check_fit(res, c, name)


def test_als_rejects_oracle_variant(api):
    with pytest.raises(ValueError):
        api.FitConfig(rank=2, variant="bogus")
    y = api.DenseTensor(np.ones((3, 3, 3)))
    with pytest.raises(ValueError):
        api.fit(y, api.FitConfig(rank=2, variant="dgn-oracle", init="random"))


def test_als_zero_tensor(api):
    y = api.DenseTensor(np.zeros((3, 4, 5)))
    with pytest.raises(ZeroDivisionError):
        api.fit(y, api.FitConfig(rank=2, variant="als", init="random", max_iters=3))
