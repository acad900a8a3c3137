"""Timeline of the persistent LU (lu_persist.cuh) inside one fit iteration (cpf_debug_lu_trace):
per 16-column step the panel CTA's [wait begin, publish end], [load end, column loop end] and the
helpers' look-ahead task [first start, last end], in us from the first step; plus the LU phase time
of eagerly launched iterations.  Usage: python tools/lp_timeline.py [N R]  (default 3 20 ->
n_B = 1200, the config-4 core system; the tensor is a small random one: the LU does not depend
on it)."""
import os as _os
_os.environ.setdefault("CPF_DEBUG", "1")  # engine knobs are read only under CPF_DEBUG=1
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_1205_2584_b200 import _native

N = int(sys.argv[1]) if len(sys.argv) > 1 else 3
R = int(sys.argv[2]) if len(sys.argv) > 2 else 20
dims = (64,) * N
rng = np.random.default_rng(0)
y = np.asfortranarray(rng.standard_normal(dims))
lib = _native.load()
lib.cpf_debug_lu_trace.argtypes = [ctypes.c_int, ctypes.c_void_p]
eng = _native.Engine(_native.CPF_REAL, dims, R, 0)
eng.set_tensor_host(y)
eng.set_factors(rng.standard_normal(R * sum(dims)))
eng.fit_begin("auto", 1e-3, 0.0, 40)
eng.fit_step(3)
eng.profile(True)
eng.phase_times()
eng.fit_step(5)
ms, cnt = eng.phase_times()
eng.profile(False)
print(f"n_B = {N * R * R}: LU phase (LU + triangular inverses) {ms[2] / max(1, cnt[2]):.3f} ms per launch-group "
      f"({ms[2]:.3f} ms over {cnt[2]} groups in 5 eager iterations)")
buf = (ctypes.c_ulonglong * (3 * 512 * 2 + 1024))()
lib.cpf_debug_panel_cycles.argtypes = [ctypes.c_void_p]
c0 = (ctypes.c_longlong * 24)()
lib.cpf_debug_panel_cycles(c0)
lib.cpf_debug_lu_trace(1, None)
eng.fit_step(1)
lib.cpf_debug_lu_trace(0, buf)
c1 = (ctypes.c_longlong * 24)()
lib.cpf_debug_panel_cycles(c1)
names = ["wait", "load", "argmax+stage", "barrier", "cta-argmax+book", "elimination", "chunk flush", "publish"]
d = [c1[i] - c0[i] for i in range(8)]
print("panel CTA warp 0 cycles (one LU):", ", ".join(f"{nm} {v}" for nm, v in zip(names, d)), f"| total {sum(d)}")
hn = ["wait-panel", "setup", "wait-owner", "U12(A)", "update(A)", "fence(A)", "U12+store(B)", "update(B)", "fence(B)"]
hd = [c1[8 + i] - c0[8 + i] for i in range(9)]
print("helper 0 cycles:", ", ".join(f"{nm} {v}" for nm, v in zip(hn, hd)))
raw = np.frombuffer(buf, dtype=np.uint64)
a = raw[:3 * 512 * 2].reshape(3, 512, 2).astype(np.float64)
valid = a[0, :, 1] > 0
if valid.any():
    t0 = a[0, valid, 0].min()
    print("step  panel[wait-begin  publish]  cols[load-end  loop-end]  helpersA[start end]  (us)")
    for k in np.nonzero(valid)[0]:
        f = lambda j, e: (a[j, k, e] - t0) / 1e3 if a[j, k, 1] > 0 else float("nan")
        print(f"{k:4d}  {f(0,0):8.1f} {f(0,1):8.1f}   {f(1,0):8.1f} {f(1,1):8.1f}   {f(2,0):8.1f} {f(2,1):8.1f}")
eng.close()
