import ctypes, sys, numpy as np
sys.path.insert(0, '.')
import torch
from paper_1205_2584_b200 import synth, _native
_native.LIB_PATH = __import__('pathlib').Path('tools/dbg/libtiming.so')
lib = _native.load()
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else 'c4']
y = synth.device_tensor(cfg, 0, device='cuda:0'); torch.cuda.synchronize()
eng = _native.Engine(_native.CPF_REAL, cfg.dims, cfg.rank, 0)
eng.set_tensor_device(y.data_ptr(), y.numel())
eng.set_factors(np.concatenate([f.reshape(-1, order='F') for f in synth.init_factors(cfg, 0)]))
eng.fit_begin('auto', synth.tau_for_unit_mu(cfg, 0), 0.0, 2)
eng.fit_step(1)
out = (ctypes.c_longlong * 8)()
lib.cpf_debug_panel_cycles(out)
n = out[7]
names = ['argmax', 'publish', 'cluster.sync', 'winner', 'eliminate', 'stage+syncthreads']
print('panels', n, 'cycles per COLUMN by phase:', {names[i]: round(out[i] / max(n, 1) / 32) for i in range(6)})
