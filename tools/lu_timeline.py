"""LU timeline of one config-4 iteration in graph replay (cpf_debug_lu_trace): per panel step the
start/end of the panel kernel (stream s) and of the trailing U12 / GEMM (stream s2), in us from
the first panel's start."""
import os as _os
_os.environ.setdefault("CPF_DEBUG", "1")  # engine knobs are read only under CPF_DEBUG=1
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1205_2584_b200 import _native, synth

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
lib = _native.load()
lib.cpf_debug_lu_trace.argtypes = [ctypes.c_int, ctypes.c_void_p]
y = synth.device_tensor(cfg, 0, device="cuda:0", slab=(0, cfg.dims[-1]))
torch.cuda.synchronize()
eng = _native.Engine(_native.CPF_COMPLEX if cfg.complex_ else _native.CPF_REAL, cfg.dims, cfg.rank, 0, 0, 1, None)
eng.set_tensor_device(y.data_ptr(), y.numel())
eng.set_factors(np.concatenate([f.reshape(-1, order="F") for f in synth.init_factors(cfg, 0)]))
skip = int(os.environ.get("SKIP", "4"))
eng.fit_begin("auto", synth.tau_for_unit_mu(cfg, 0), 0.0, skip + 2)
eng.fit_step(skip)
buf = (ctypes.c_ulonglong * (3 * 512 * 2 + 1024))()
lib.cpf_debug_lu_trace(1, None)
eng.fit_step(1)
lib.cpf_debug_lu_trace(0, buf)
raw = np.frombuffer(buf, dtype=np.uint64)
a = raw[:3 * 512 * 2].reshape(3, 512, 2).astype(np.float64)
clk = raw[3 * 512 * 2:].reshape(512, 2).astype(np.float64)
valid = a[0, :, 1] > 0
valid[256:] = False
t0 = a[0, valid, 0].min()
print("step   panel[start end dur]        u12[start end]      gemm[start end]   (us)")
for k in np.nonzero(valid)[0]:
    row = [(a[j, k, 0] - t0) / 1e3 if a[j, k, 1] > 0 else float("nan") for j in range(3)]
    ends = [(a[j, k, 1] - t0) / 1e3 if a[j, k, 1] > 0 else float("nan") for j in range(3)]
    mhz = (clk[k, 1] - clk[k, 0]) / (a[0, k, 1] - a[0, k, 0]) * 1e3 if a[0, k, 1] > a[0, k, 0] else float("nan")
    print(f"{k:4d}  {row[0]:8.1f} {ends[0]:8.1f} {ends[0]-row[0]:6.1f}   {row[1]:8.1f} {ends[1]:8.1f}   {row[2]:8.1f} {ends[2]:8.1f}  SM {mhz:6.0f} MHz")
print("triangular-inverse merges launched after LU step k (stream s4): [first start, last end] us")
for k in range(256, 512):
    if a[1, k, 1] > 0:
        print(f"  step {k - 256:3d}: {(a[1, k, 0] - t0) / 1e3:8.1f} {(a[1, k, 1] - t0) / 1e3:8.1f}")
print("accept sequence:", "".join("A" if t[3] else "r" for t in eng.trace(skip + 1)))
eng.close()
