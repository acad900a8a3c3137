"""The shared-memory cluster LU panel (lu.cuh k_panel_lu + k_row_gather + k_trsm_llnu + k_gemm_sub)
is the engine's path for core systems too large for the register panels (n_B > 8192); forced
here (CPF_PANEL_SMEM=1) on the golden fit cases, real and complex, so it stays correct."""

import pytest

from tests import _golden as G
from tests import test_gpu_parity as PAR

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api(engine_lib):
    import paper_1205_2584_b200 as api

    return api


@pytest.mark.parametrize("name", G.fit_names(include_full=False))
def test_fit_matches_reference_smem_panel(api, name, monkeypatch):
    monkeypatch.setenv("CPF_PANEL_SMEM", "1")
    PAR.test_fit_matches_reference(api, name)
