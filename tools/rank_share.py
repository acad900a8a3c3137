"""Measured per-rank share of a P-GPU config-4 run, on one GPU: the engine on rank 0's slab
(1000 x 1000 x 2000/P; slab sharding of mode 3) runs exactly the kernels one
rank runs -- minus the two NCCL collectives per iteration (a 320 KB allreduce + the M_N row
allgather, ~10-30 us over NVLink 5).  Times are device time per iteration over 20 graph replays
after 3 warm-up iterations.  The slab's own accept/reject pattern differs from the full problem's,
so this bounds the per-rank cost, it is not a scaling measurement."""
import os as _os
_os.environ.setdefault("CPF_DEBUG", "1")  # engine knobs are read only under CPF_DEBUG=1
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1205_2584_b200 import _native, synth

cfg = synth.CONFIGS["c4"]
_native.load()
init = synth.init_factors(cfg, 0)
tau = synth.tau_for_unit_mu(cfg, 0)
base = None
for P in (1, 2, 4, 8):
    c = cfg.dims[-1] // P
    y = synth.device_tensor(cfg, 0, device="cuda:0", slab=(0, c))
    torch.cuda.synchronize()
    dims = tuple(cfg.dims[:-1]) + (c,)
    eng = _native.Engine(_native.CPF_REAL, dims, cfg.rank, 0, 0, 1, None)
    eng.set_tensor_device(y.data_ptr(), y.numel())
    eng.set_factors(np.concatenate([f.reshape(-1, order="F") for f in init[:-1]] + [init[-1][:c].reshape(-1, order="F")]))
    eng.fit_begin("auto", tau, 0.0, 23)
    eng.fit_step(3)
    stream = torch.cuda.ExternalStream(eng.stream_handle)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    st = eng.fit_step(20)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / max(st.iter - 3, 1)
    seq = "".join("A" if t[3] else "r" for t in eng.trace(23))[3:]
    base = base or ms
    print(f"P={P}: rank share 1000x1000x{c}: {ms:.3f} ms/iteration ({1e3 / ms:.1f} it/s), "
          f"speed-up over P=1 {base / ms:.2f}x, efficiency {base / ms / P:.2f}; decisions {seq}", flush=True)
    eng.close()
    del y
    torch.cuda.empty_cache()
