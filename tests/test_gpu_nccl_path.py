"""The multi-rank engine code path (NCCL allreduce of pass-A partials, allgather + reorder of the
pass-B rows, scalar allreduces, NCCL inside the captured CUDA graph) exercised on ONE GPU with a
1-rank communicator (CPF_FORCE_NCCL=1), compared with the single-rank path.  Multi-GPU boxes are not
available this round; the host side of N>1 is covered by tests/test_dist_gloo.py."""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

SCRIPT = r"""
import sys, json, numpy as np
sys.path.insert(0, %r)
import paper_1205_2584_b200 as api
from paper_1205_2584_b200 import synth
out = {}
for name, dims, R in [("c4_wide", (300, 12, 16), 6), ("c2_mini", (12, 12, 12, 12), 5), ("c3_mini", (24, 24, 24), 4)]:
    base = {"c4_wide": "c4", "c2_mini": "c2", "c3_mini": "c3"}[name]
    cfg = synth.scaled(synth.CONFIGS[base], dims, rank=R, max_iters=12, name=name)
    y = synth.make_tensor(cfg, 0)
    res = api.fit(y, api.FitConfig(rank=R, tau=synth.tau_for_unit_mu(cfg, 0), tol=0.0, max_iters=12, seed=0, init="random"))
    out[name] = {"seq": "".join("A" if r.accepted else "r" for r in res.trace),
                 "err": [r.relerr for r in res.trace],
                 "vec": [complex(v).real for v in res.model.as_vector()] + [complex(v).imag for v in res.model.as_vector()]}
print(json.dumps(out))
""" % str(ROOT)


def _run(env_extra):
    env = dict(os.environ)
    env.update(env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    import json

    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("oz", ["0", "1"])
def test_forced_nccl_path_matches_single_rank(engine_lib, oz):
    # oz=1: the int8 Ozaki tensor passes (forced for every real case) under the multi-rank path --
    # config 4's default at scale (allreduce of their M_1/Z partials, allgather of M_N rows)
    plain = _run({"CPF_FORCE_NCCL": "0", "CPF_OZ": oz})
    nccl = _run({"CPF_FORCE_NCCL": "1", "CPF_OZ": oz})
    for name in plain:
        assert plain[name]["seq"] == nccl[name]["seq"]
        np.testing.assert_allclose(nccl[name]["err"], plain[name]["err"], rtol=0, atol=1e-13)
        a, b = np.array(plain[name]["vec"]), np.array(nccl[name]["vec"])
        assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(a)
