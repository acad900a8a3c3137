"""Per-column phase cycles of the LU panel (build with CPF_NVCC_DEFS=-DCPF_PANEL_TIMING): CTA 0,
thread 0, summed over all panels of the run, divided by the columns processed."""
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
y = synth.device_tensor(cfg, 0, device="cuda:0", slab=(0, cfg.dims[-1]))
torch.cuda.synchronize()
eng = _native.Engine(_native.CPF_COMPLEX if cfg.complex_ else _native.CPF_REAL, cfg.dims, cfg.rank, 0, 0, 1, None)
eng.set_tensor_device(y.data_ptr(), y.numel())
eng.set_factors(np.concatenate([f.reshape(-1, order="F") for f in synth.init_factors(cfg, 0)]))
eng.fit_begin("auto", synth.tau_for_unit_mu(cfg, 0), 0.0, 5)
eng.fit_step(5)
buf = (ctypes.c_longlong * 24)()
lib.cpf_debug_panel_cycles(buf)
c = np.array(buf[:], dtype=np.float64)
npanels = c[7]
nb = cfg.rank * cfg.rank * len(cfg.dims)
cols = npanels / max(1, (nb + 31) // 32) * nb
names = ["argmax(warp)", "pkt push", "mbar wait", "winner", "eliminate", "stage+sync"]
print(f"panels {npanels:.0f}, columns ~{cols:.0f}")
for i, nmx in enumerate(names):
    print(f"  {nmx:14s} {c[i] / cols:8.0f} cycles/column")
print(f"  total          {c[:6].sum() / cols:8.0f}")
seg = c[8:12] / npanels
print(f"per panel (cycles): load+sync {seg[0]:.0f}, column loop {seg[1]:.0f}, write-back+sync {seg[2]:.0f}, whole {seg[3]:.0f}")
sub = c[12:15] / npanels
print(f"  fused load (CTA 0, per panel incl. the first): gather+A12 {sub[0]:.0f}, U12 {sub[1]:.0f}, row update {sub[2]:.0f}")
eng.close()
