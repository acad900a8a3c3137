"""Host-side checks that need no GPU: the C-ABI library loads and exports every declared symbol,
API types/validation mirror the reference, and the harness generator is deterministic."""

import re
from pathlib import Path

import numpy as np
import pytest

from tests import _golden as G

ROOT = Path(__file__).resolve().parents[1]


def header_functions():
    text = (ROOT / "include" / "cpfast_b200.h").read_text()
    return sorted(set(re.findall(r"\b(cpf_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol(engine_lib):
    from paper_1205_2584_b200 import _native

    declared = header_functions()
    assert declared, "no functions parsed from the header"
    for name in declared:
        assert hasattr(engine_lib, name), f"{name} not exported"
    assert set(declared) == set(_native.EXPORTED_SYMBOLS)
    assert engine_lib.cpf_abi_version() == 1


def test_engine_fails_loudly_without_gpu(engine_lib):
    from paper_1205_2584_b200 import _native

    if _native.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(Exception):
        _native.Engine(_native.CPF_REAL, (3, 3, 3), 2)


def test_fitconfig_validation_mirrors_reference():
    from paper_1205_2584_b200 import FitConfig

    with pytest.raises(ValueError):
        FitConfig(rank=2, variant="newton")
    with pytest.raises(ValueError):
        FitConfig(rank=0)
    c = FitConfig(rank=3)
    assert (c.variant, c.tau, c.tol, c.max_iters, c.seed, c.init) == ("auto", 1e-3, 1e-8, 1000, 0, "svd")


def test_dgn_oracle_variant_rejected_before_any_device_work():
    """dgn-oracle (the dense desk-scale oracle, hessian.py) is not on the B200 backend; the ALS
    baselines are (tests/test_gpu_als.py)."""
    from paper_1205_2584_b200 import DenseTensor, FitConfig, fit

    y = DenseTensor(np.ones((3, 3, 3)))
    for v in ("dgn-oracle",):
        with pytest.raises(ValueError):
            fit(y, FitConfig(rank=1, variant=v, init="random"))


def test_unknown_init_rejected():
    from paper_1205_2584_b200 import DenseTensor, FitConfig, fit

    with pytest.raises(ValueError):
        fit(DenseTensor(np.ones((3, 3, 3))), FitConfig(rank=1, init="nope"))


def test_fit_complex_kind_check():
    from paper_1205_2584_b200 import DenseTensor, FitConfig, fit_complex

    with pytest.raises(TypeError):
        fit_complex(DenseTensor(np.ones((3, 3))), FitConfig(rank=1, init="random"))


def test_dense_tensor_layout_policy():
    from paper_1205_2584_b200 import DenseTensor

    t = DenseTensor(np.arange(24.0).reshape(2, 3, 4))
    assert t.data.flags["F_CONTIGUOUS"] and t.dims == (2, 3, 4) and t.scalar_kind == "real"
    assert DenseTensor(np.arange(4)).data.dtype == np.float64
    assert DenseTensor(np.ones(3) * 1j).scalar_kind == "complex"


def test_random_init_matches_reference_stream():
    from paper_1205_2584_b200 import random_init

    rng = np.random.default_rng([7, 0])
    m = random_init((3, 4), 2, rng, "complex")
    rng2 = np.random.default_rng([7, 0])
    a = rng2.standard_normal((3, 2))
    a = a + 1j * rng2.standard_normal((3, 2))
    np.testing.assert_array_equal(m.factors[0], a)


@pytest.mark.parametrize("name", G.fit_names(include_full=False))
def test_generator_reproduces_golden_inputs(name):
    from paper_1205_2584_b200 import synth

    d = G.load_fit(name)
    y = synth.make_tensor(G.synth_config(d), d["seed"])
    assert synth.tensor_digest(y) == d["digest"]
    assert synth.tau_for_unit_mu(G.synth_config(d), d["seed"]) == pytest.approx(d["tau"], rel=1e-14)


def test_slab_bounds_cover_last_mode():
    from paper_1205_2584_b200 import slab_bounds

    for dim in (1, 7, 2000, 2001):
        for world in (1, 2, 3, 8):
            spans = [slab_bounds(dim, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == dim
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
