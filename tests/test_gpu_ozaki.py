"""GPU parity of the Ozaki-split int8 tensor passes (csrc/tensor_pass_oz.cuh).

The engine picks them for large real tensors (config 4); CPF_OZ=1 forces them for every real tensor
with R <= 32, so the reference's golden fixtures (small shapes) exercise the same kernels through the
drop-in API: MTTKRP of every mode, relative error, flm_step and whole fits against the reference's
traces.  At config 4's full size there is no reference trace (one reference iteration takes ~20 s
on 16 host cores); there the int8 passes are checked against the engine's fp64 DMMA passes on the
same device-generated tensor: identical accept/reject sequence, relative errors within 1e-10 and
factors within 1e-9 after 20 iterations."""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from tests import _golden as G
from tests import test_gpu_parity as P

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(autouse=True)
def force_ozaki(monkeypatch):
    monkeypatch.setenv("CPF_OZ", "1")


@pytest.fixture(scope="module")
def api(engine_lib):
    import paper_1205_2584_b200 as api

    return api


def _real_small_r(case):
    return (not bool(case.get("complex_", False))) and int(case["rank"]) <= 32


UNIT = sorted(n for n, c in G.unit_cases().items() if not np.iscomplexobj(c["y"]) and int(c["rank"]) <= 32)


def test_engine_reports_ozaki_passes(api):
    from paper_1205_2584_b200 import _native

    eng = _native.Engine(_native.CPF_REAL, (300, 12, 16), 6, 0, 0, 1, None)
    try:
        assert eng.pass_impl() == _native.PASS_OZAKI
    finally:
        eng.close()


@pytest.mark.parametrize("cname", UNIT)
def test_mttkrp_all_modes_ozaki(api, cname):
    P.test_mttkrp_all_modes(api, cname)


@pytest.mark.parametrize("cname", UNIT)
@pytest.mark.parametrize("variant", ["auto", "flm-b"])
@pytest.mark.parametrize("mu", [1e-4, 10.0])
def test_flm_step_ozaki(api, cname, variant, mu):
    P.test_flm_step(api, cname, variant, mu, 2)


FITS = [n for n in G.fit_names(include_full=False) if _real_small_r(G.load_fit(n))]


@pytest.mark.parametrize("name", FITS)
def test_fit_matches_reference_ozaki(api, name):
    P.test_fit_matches_reference(api, name)


@pytest.mark.parametrize("key", sorted(k for k in G.ensemble() if not np.iscomplexobj(G.ensemble()[k]["y"])))
def test_ensemble_fit_ozaki(api, key):
    P.test_ensemble_fit(api, key)


C4_SCRIPT = r"""
import sys, os, json, numpy as np
sys.path.insert(0, %r)
import torch
from paper_1205_2584_b200 import _native, synth
cfg = synth.CONFIGS["c4"]
_native.load()
y = synth.device_tensor(cfg, 0, device="cuda:0", slab=(0, cfg.dims[-1]))
torch.cuda.synchronize()
init = np.concatenate([f.reshape(-1, order="F") for f in synth.init_factors(cfg, 0)])
tau = synth.tau_for_unit_mu(cfg, 0)
out = {}
for oz in ("0", "1"):
    os.environ["CPF_OZ"] = oz
    eng = _native.Engine(_native.CPF_REAL, cfg.dims, cfg.rank, 0, 0, 1, None)
    eng.set_tensor_device(y.data_ptr(), y.numel())
    eng.set_factors(init)
    impl = eng.pass_impl()
    eng.fit_begin("auto", tau, 0.0, 20)
    eng.fit_step(20)
    tr = eng.trace(20)
    out[oz] = {"impl": impl, "seq": "".join("A" if t[3] else "r" for t in tr),
               "err": [float(t[1]) for t in tr], "vec": [float(v) for v in eng.get_factors()]}
    eng.close()
print(json.dumps(out))
""" % str(ROOT)


@pytest.mark.slow
def test_config4_ozaki_matches_dmma(engine_lib):
    env = dict(os.environ)
    r = subprocess.run([sys.executable, "-c", C4_SCRIPT], capture_output=True, text=True, env=env, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    import json

    from paper_1205_2584_b200 import _native

    out = json.loads(r.stdout.strip().splitlines()[-1])
    dm, oz = out["0"], out["1"]
    assert dm["impl"] == _native.PASS_DMMA and oz["impl"] == _native.PASS_OZAKI
    assert len(oz["seq"]) == 20 and oz["seq"] == dm["seq"]
    np.testing.assert_allclose(oz["err"], dm["err"], rtol=0, atol=1e-10)
    a, b = np.array(oz["vec"]), np.array(dm["vec"])
    assert np.linalg.norm(a - b) <= 1e-9 * np.linalg.norm(b)


@pytest.mark.parametrize("key", ["e0_flm-a", "e3_auto"])
def test_int8_passes_are_bitwise_deterministic(api, key):
    """Fixed-order reductions everywhere: repeated fits give identical bits (guards the TMEM
    accumulator initialisation -- every column block must be written before it is accumulated)."""
    e = G.ensemble()[key]
    variant = key.split("_", 1)[1]
    y = api.DenseTensor(e["y"])
    runs = []
    for _ in range(4):
        conf = api.FitConfig(rank=int(e["rank"]), variant=variant, tol=1e-10, max_iters=40, seed=int(e["seed"]),
                             init="random")
        r = api.fit(y, conf)
        runs.append(([(t.relerr, t.mu, t.accepted) for t in r.trace], r.model.as_vector()))
    for tr, v in runs[1:]:
        assert tr == runs[0][0]
        assert np.array_equal(v, runs[0][1])
