"""GPU: engine code paths the golden configurations do not reach, each against the CPU oracle on
the same seeded input (identical accept/reject sequence, final fit within 1e-10, factors 1e-9):
the complex register-frame LU panel (N R^2 = 1200 complex128), the substitution solves instead of
the explicit inverse (CPF_NO_INV=1), and the int8 passes on a 4-way tensor."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api(engine_lib):
    import paper_1205_2584_b200 as api

    return api


def _problem(dims, R, complex_, seed):
    rng = np.random.default_rng(seed)
    draw = (lambda s: rng.standard_normal(s) + 1j * rng.standard_normal(s)) if complex_ else rng.standard_normal
    fac = [draw((d, R)) for d in dims]
    x = fac[0]
    for f in fac[1:]:
        x = np.einsum("...r,jr->...jr", x, f)
    x = x.sum(axis=-1)
    noise = draw(dims)
    return np.asfortranarray(x + 0.05 * np.linalg.norm(x) / np.sqrt(x.size) * noise)


def _check(api, y, R, iters=8):
    from oracle import cp_oracle

    complex_ = np.iscomplexobj(y)
    conf = api.FitConfig(rank=R, tau=1e-3, tol=0.0, max_iters=iters, seed=3, init="random")
    res = (api.fit_complex if complex_ else api.fit)(y, conf)
    ref = cp_oracle.fit_lm(y, cp_oracle.OracleConfig(rank=R, tau=1e-3, tol=0.0, max_iters=iters, seed=3))
    assert "".join("A" if t.accepted else "r" for t in res.trace) == ref.accepted
    assert abs(res.final_relerr - ref.final_relerr) < 1e-10
    v, vr = res.model.as_vector(), cp_oracle.stack(ref.factors)
    assert np.linalg.norm(v - vr) <= 1e-9 * np.linalg.norm(vr)


def test_complex_register_frame_panel(api):
    _check(api, _problem((30, 28, 26), 20, True, 5), 20)  # n_B = 1200 complex: k_panel_lu4<cplx>


def test_substitution_solves(api, monkeypatch):
    monkeypatch.setenv("CPF_NO_INV", "1")
    monkeypatch.setenv("CPF_BLK_INV", "0")
    _check(api, _problem((24, 22, 20), 12, False, 6), 12)  # trsv instead of inv(L), inv(U)


@pytest.mark.parametrize("db", [64, 128, 256])
@pytest.mark.parametrize("complex_", [False, True])
def test_block_inverse_substitution(api, monkeypatch, db, complex_):
    """The large-n_B solve path (config 1): inverted diagonal blocks + block steps, forced at
    n_B = 432 with small blocks (7 / 4 / 2 block steps, ragged last block)."""
    monkeypatch.setenv("CPF_NO_INV", "1")
    monkeypatch.setenv("CPF_BLK_DB", str(db))
    _check(api, _problem((24, 22, 20), 12, complex_, 6), 12)


def test_int8_passes_four_way(api, monkeypatch):
    monkeypatch.setenv("CPF_OZ", "1")
    _check(api, _problem((40, 9, 8, 7), 6, False, 7), 6)


@pytest.mark.parametrize("dims,R", [((50, 40), 4), ((6, 5, 4, 5, 7), 3)])
def test_int8_passes_order_2_and_5(api, monkeypatch, dims, R):
    monkeypatch.setenv("CPF_OZ", "1")
    _check(api, _problem(dims, R, False, 8), R)


@pytest.mark.parametrize("env", [{"CPF_TRI_ROWS": "1"}, {"CPF_TRI_ROWS": "1", "CPF_TRI_GROUP": "128"},
                                 {"CPF_TRI_ROWS": "0"}, {"CPF_TRI_ROWS": "0", "CPF_TRI_PROG": "0"},
                                 {"CPF_TRI_ROWS": "1", "CPF_TRI_PROG": "0"}])
@pytest.mark.parametrize("complex_", [False, True])
def test_inverse_forms(api, monkeypatch, env, complex_):
    """Both forms of the explicit triangular inverse (block rows / block pairs), progressive and
    batched, on a multi-panel core system (n_B = 432, ragged last block)."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    _check(api, _problem((24, 22, 20), 12, complex_, 6), 12)
