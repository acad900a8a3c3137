"""GPU parity of fast_damped_inverse (hessian.py:232-277): the engine's Gram cache, dense system
assembly, LU and triangular inverses against the reference's own block form
(tests/golden/make_fdi_golden.py).  Tolerances: gamma_tilde 1e-12 and the core grid D 1e-9
relative (Frobenius); the materialised (H + mu I)^{-1} within 1e-8 of the reference's, the
reference's own acceptance bound against the dense inverse (tests/test_hessian.py:155-163)."""

import numpy as np
import pytest

from oracle import cp_oracle as O
from tests import _golden as G

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def _cases():
    z = G._grouped("fdi_cases.npz")
    return {k: v for k, v in z.items() if isinstance(v, dict)}


@pytest.fixture(scope="module")
def api(engine_lib):
    import paper_1205_2584_b200 as api

    return api


@pytest.mark.parametrize("name", sorted(k for k in _cases() if k.startswith("i")))
@pytest.mark.parametrize("mu", [1e-6, 1e-2, 1.0, 1e3])
@pytest.mark.parametrize("path", ["kfree", "kinv", "auto"])
def test_fast_damped_inverse(api, name, mu, path):
    c = _cases()[name]
    dims = tuple(int(x) for x in c["dims"])
    r = int(c["rank"])
    fac = G.split_stacked(c["factors"], dims, r)
    flag = {"kfree": False, "kinv": True, "auto": None}[path]
    tag = f"{path}_{mu:g}"
    if f"{tag}_error" in c:
        with pytest.raises(np.linalg.LinAlgError):
            api.fast_damped_inverse(None, fac, mu, use_kernel_inverse=flag)
        return
    s = api.fast_damped_inverse(None, fac, mu, use_kernel_inverse=flag)
    assert s.scalar_count() == len(dims) * r ** 2 + len(dims) ** 2 * r ** 4
    d = np.block(s.S)
    e_gt = _rel(np.stack(s.gamma_tilde), c[f"{tag}_gt"])
    e_d = _rel(d, c[f"{tag}_core"])
    msg = f"{name} {tag}: gamma_tilde {e_gt:.2e} core {e_d:.2e}"
    if f"{tag}_dense" in c:
        e_m = _rel(O.materialize_inverse(s.gamma_tilde, d, fac), c[f"{tag}_dense"])
        msg += f" materialised {e_m:.2e}"
        assert e_m < 1e-8, msg
    print(msg)
    assert e_gt < 1e-12, msg
    assert e_d < 1e-9, msg


def test_singular_kernel_and_auto_fallback(api):
    c = _cases()["orth"]
    fac = G.split_stacked(c["factors"], (6, 6, 6), 3)
    with pytest.raises(api.SingularKernelError, match="a pairwise Gamma entry vanishes; K is singular"):
        api.fast_damped_inverse(None, fac, 0.5, use_kernel_inverse=True)
    s = api.fast_damped_inverse(None, fac, 0.5)
    assert _rel(np.block(s.S), c["auto_0.5_core"]) < 1e-9
    with pytest.raises(ValueError):
        api.fast_damped_inverse(None, fac, 0.0)
