"""Per-iteration section times of a config-4 fit: eager, profiled (CPF_MARKS=2) or graph replay (CPF_MARKS=3):
[rotated order: branch launch + fork (pass B || this step's core system)] | candidate | normalise +
pass A + trial fit + decide | commit | [classic order: fork] + join of the speculated branch."""
import os as _os
_os.environ.setdefault("CPF_DEBUG", "1")  # engine knobs are read only under CPF_DEBUG=1
import os
import sys

os.environ.setdefault("CPF_MARKS", "2")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1205_2584_b200 import _native, synth

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
_native.load()
y = synth.device_tensor(cfg, 0, device="cuda:0", slab=(0, cfg.dims[-1]))
torch.cuda.synchronize()
eng = _native.Engine(_native.CPF_COMPLEX if cfg.complex_ else _native.CPF_REAL, cfg.dims, cfg.rank, 0, 0, 1, None)
eng.set_tensor_device(y.data_ptr(), y.numel())
eng.set_factors(np.concatenate([f.reshape(-1, order="F") for f in synth.init_factors(cfg, 0)]))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
eng.fit_begin("auto", synth.tau_for_unit_mu(cfg, 0), 0.0, n)
if os.environ["CPF_MARKS"] != "3":
    eng.profile(True)
eng.fit_step(n)
if os.environ["CPF_MARKS"] != "3":
    eng.phase_times()
print("accept sequence:", "".join("A" if t[3] else "r" for t in eng.trace(n)))
eng.close()
