"""Pin the oracle's fast_damped_inverse / materialize_inverse restatement against fixtures
captured from the reference (tests/golden/make_fdi_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import cp_oracle as O
from tests import _golden as G


def _cases():
    z = G._grouped("fdi_cases.npz")
    return {k: v for k, v in z.items() if isinstance(v, dict)}


def test_recorded_bitwise():
    assert bool(G._grouped("fdi_cases.npz")["oracle_bitwise"])


@pytest.mark.parametrize("name", sorted(k for k in _cases() if k.startswith("i")))
def test_oracle_fast_damped_inverse(name):
    c = _cases()[name]
    dims = tuple(int(x) for x in c["dims"])
    fac = G.split_stacked(c["factors"], dims, int(c["rank"]))
    for mu in (1e-6, 1e-2, 1.0, 1e3):
        for path, flag in (("kfree", False), ("kinv", True), ("auto", None)):
            tag = f"{path}_{mu:g}"
            if f"{tag}_error" in c:
                with pytest.raises(np.linalg.LinAlgError):
                    O.fast_damped_inverse(fac, mu, flag)
                continue
            gt, d = O.fast_damped_inverse(fac, mu, flag)
            np.testing.assert_array_equal(np.stack(gt), c[f"{tag}_gt"])
            np.testing.assert_array_equal(d, c[f"{tag}_core"])
            if f"{tag}_dense" in c:
                np.testing.assert_allclose(O.materialize_inverse(gt, d, fac), c[f"{tag}_dense"], rtol=0, atol=1e-12)


def test_oracle_orthonormal_singular_kernel():
    c = _cases()["orth"]
    fac = G.split_stacked(c["factors"], (6, 6, 6), 3)
    with pytest.raises(O.OracleSingularKernel):
        O.fast_damped_inverse(fac, 0.5, True)
    gt, d = O.fast_damped_inverse(fac, 0.5)
    np.testing.assert_array_equal(d, c["auto_0.5_core"])
    with pytest.raises(ValueError):
        O.fast_damped_inverse(fac, 0.0)
