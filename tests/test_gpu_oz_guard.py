"""GPU: the accuracy guard of the int8 (Ozaki) tensor passes (csrc/tensor_pass_oz.cuh).

The int8 split represents every element in fixed point against its row's (column's) maximum, so an
element far below the maximum loses relative accuracy.  The guard keeps the int8 passes only while
every row of Y and every column of the per-launch operand has peak/rms <= 16; otherwise that pass
runs in fp64 (DMMA).  Adversarial inputs here put the result's mass on such small elements: a spike
per Y row whose operand partner is zero, and a spike in an operand column whose Y partner is zero.
Each test first shows (numpy emulation of the split) that the unguarded int8 result would be off by
far more than fp64 rounding, then that the engine -- int8 passes forced with CPF_OZ=1 -- falls back
and matches the oracle to 1e-13."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DIMS = (300, 12, 512)
R = 4


@pytest.fixture(autouse=True)
def force_ozaki(monkeypatch, engine_lib):
    monkeypatch.setenv("CPF_OZ", "1")


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _split_rows(y_rows: np.ndarray) -> np.ndarray:
    """The split's representation of each row (last axis contracted): rint(|y| 2^F) 2^-F, F = 56 - e."""
    amax = np.max(np.abs(y_rows), axis=-1, keepdims=True)
    e = np.frexp(np.where(amax > 0, amax, 1.0))[1]
    f = 56 - e
    return np.sign(y_rows) * np.rint(np.ldexp(np.abs(y_rows), f)) * np.ldexp(1.0, -f)


def _mttkrp1(y, a2, a3):
    return np.einsum("imc,mr,cr->ir", y, a2, a3)


def _engine(y, factors):
    from paper_1205_2584_b200 import _native

    eng = _native.Engine(_native.CPF_REAL, y.shape, R)
    eng.set_tensor_host(np.asfortranarray(y))
    eng.set_factors(np.concatenate([f.reshape(-1, order="F") for f in factors]))
    return eng


def _check_against_oracle(eng, y, factors):
    from oracle import cp_oracle as O

    for n in range(1, 4):
        got = eng.mttkrp(n).reshape((y.shape[n - 1], R), order="F")
        assert _rel(got, O.mttkrp(y, factors, n)) < 1e-13, f"mode {n}"


def test_spiky_tensor_rows_fall_back_to_fp64():
    from paper_1205_2584_b200 import _native

    rng = np.random.default_rng(41)
    y = 1e-8 * rng.standard_normal(DIMS)
    y[:, :, 7] = 1.0                                       # every pass-A row: one spike (peak/rms ~ sqrt(512))
    factors = [rng.standard_normal((d, R)) for d in DIMS]
    factors[2][7, :] = 0.0                                 # ... whose operand partner is zero
    exact = _mttkrp1(y, factors[1], factors[2])
    emulated = _mttkrp1(_split_rows(y), factors[1], factors[2])
    assert _rel(emulated, exact) > 1e-11, "the adversarial case must defeat an unguarded split"
    eng = _engine(y, factors)
    try:
        assert eng.pass_impl() == _native.PASS_DMMA
        assert eng.pass_guard()[1] is True
        _check_against_oracle(eng, y, factors)
    finally:
        eng.close()


def test_spiky_operand_column_falls_back_per_launch():
    from paper_1205_2584_b200 import _native

    rng = np.random.default_rng(42)
    y = rng.standard_normal(DIMS)
    y[:, :, 11] = 0.0                                       # the operand spike's partner slice is zero
    factors = [rng.standard_normal((d, R)) for d in DIMS]
    factors[2][11, 0] = 1e8                                 # pass-A operand column 0: peak/rms ~ sqrt(512)
    exact = _mttkrp1(y, factors[1], factors[2])
    a3q = _split_rows(factors[2].T).T                       # column-wise split of the operand
    emulated = _mttkrp1(y, factors[1], a3q)
    assert _rel(emulated[:, 0], exact[:, 0]) > 1e-12
    eng = _engine(y, factors)
    try:
        assert eng.pass_impl() == _native.PASS_OZAKI       # Y itself is fine
        got = eng.mttkrp(0)                                 # one pass A + one pass B launch
        fallbacks, rejected = eng.pass_guard()
        assert not rejected
        assert fallbacks == 1                               # pass A fell back, pass B (operand A_2) did not
        _check_against_oracle(eng, y, factors)
        assert got.size == R * sum(DIMS)
    finally:
        eng.close()


def test_regular_data_stays_on_int8():
    from paper_1205_2584_b200 import _native

    rng = np.random.default_rng(43)
    y = rng.standard_normal(DIMS)
    factors = [rng.standard_normal((d, R)) for d in DIMS]
    eng = _engine(y, factors)
    try:
        assert eng.pass_impl() == _native.PASS_OZAKI
        _check_against_oracle(eng, y, factors)
        assert eng.pass_guard() == (0, False)
    finally:
        eng.close()


def test_guard_threshold_matches_documented_envelope():
    # peak/rms of a Gaussian row of length K stays far below 16 (it grows like sqrt(2 ln K));
    # a single spike gives sqrt(K): rejected from K > 256
    rng = np.random.default_rng(0)
    for k in (32, 512, 16384):
        v = rng.standard_normal(k)
        assert np.max(np.abs(v)) / math.sqrt(np.mean(v * v)) < 16
    assert math.sqrt(257) > 16 >= math.sqrt(256)


def test_spiky_tensor_rejected_after_sliced_upload(monkeypatch):
    """The sliced host upload builds the pass-B image behind the slices (Engine::upload_with_split,
    forced here at a small size); a tensor the guard then rejects must drop the images and still
    fit on the fp64 passes like the oracle."""
    import paper_1205_2584_b200 as api
    from oracle import cp_oracle as O
    from paper_1205_2584_b200 import _native

    monkeypatch.setenv("CPF_UPLOAD_SPLIT", "1")
    rng = np.random.default_rng(43)
    y = 1e-3 * rng.standard_normal(DIMS)
    y[:, :, 7] = 1.0
    y = np.asfortranarray(y)
    conf = api.FitConfig(rank=R, tau=1e-3, tol=0.0, max_iters=6, seed=5, init="random")
    res = api.fit(y, conf)
    assert res.pass_impl == _native.PASS_DMMA and res.tensor_guarded
    ref = O.fit_lm(y, O.OracleConfig(rank=R, tau=1e-3, tol=0.0, max_iters=6, seed=5))
    assert "".join("A" if t.accepted else "r" for t in res.trace) == ref.accepted
    assert abs(res.final_relerr - ref.final_relerr) < 1e-10
    # and an ordinary tensor through the same forced path keeps the int8 passes
    y2 = np.asfortranarray(rng.standard_normal(DIMS))
    res2 = api.fit(y2, conf)
    ref2 = O.fit_lm(y2, O.OracleConfig(rank=R, tau=1e-3, tol=0.0, max_iters=6, seed=5))
    assert res2.pass_impl == _native.PASS_OZAKI and not res2.tensor_guarded
    assert "".join("A" if t.accepted else "r" for t in res2.trace) == ref2.accepted
    assert abs(res2.final_relerr - ref2.final_relerr) < 1e-10
