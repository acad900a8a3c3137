"""Run a short fit on a BASELINE config (device-generated tensor) -- for ncu / nsight captures."""
import os as _os
_os.environ.setdefault("CPF_DEBUG", "1")  # engine knobs are read only under CPF_DEBUG=1
import sys, numpy as np
sys.path.insert(0, '.')
import torch
from paper_1205_2584_b200 import synth, _native, build
build.build()
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else 'c2']
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
y = synth.device_tensor(cfg, 0, device='cuda:0')
torch.cuda.synchronize()
eng = _native.Engine(_native.CPF_COMPLEX if cfg.complex_ else _native.CPF_REAL, cfg.dims, cfg.rank, 0)
eng.set_tensor_device(y.data_ptr(), y.numel())
eng.set_factors(np.concatenate([f.reshape(-1, order='F') for f in synth.init_factors(cfg, 0)]))
eng.fit_begin('auto', synth.tau_for_unit_mu(cfg, 0), 0.0, iters)
st = eng.fit_step(iters)
print('iters', st.iter, 'relerr', st.relerr, 'launches', eng.launch_count())
