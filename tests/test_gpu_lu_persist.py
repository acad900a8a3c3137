"""The experimental persistent-kernel LU (lu_persist.cuh, CPF_LU=5; off by default because it
measured slower than the v4 panels) kept correct: the fit parity cases against the
reference goldens (incl. the full config-2 fit, n_B = 900, and a complex fit), the fast damped
inverse and bitwise agreement of its pivot order with LAPACK's (through the fdi goldens)."""

import pytest

from tests import _golden as G
from tests import test_gpu_fdi as FDI
from tests import test_gpu_parity as PAR

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api(engine_lib):
    import paper_1205_2584_b200 as api

    return api


@pytest.fixture(autouse=True)
def persistent_lu(monkeypatch):
    monkeypatch.setenv("CPF_LU", "5")


@pytest.mark.parametrize("name", G.fit_names(include_full=False) + ["fit_c2_s0_auto"])
def test_fit_matches_reference_persistent_lu(api, name):
    PAR.test_fit_matches_reference(api, name)


@pytest.mark.parametrize("name", ["i2", "i5", "i6"])
@pytest.mark.parametrize("mu", [1e-2, 1.0])
@pytest.mark.parametrize("path", ["kfree", "kinv"])
def test_fast_damped_inverse_persistent_lu(api, name, mu, path):
    FDI.test_fast_damped_inverse(api, name, mu, path)
