import time, sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_1205_2584_b200 import synth
from paper_1205_2584_b200.solver import FitConfig, fit
for name in ("c2", "c4"):
    cfg = synth.CONFIGS[name]
    y = synth.device_tensor(cfg, 0, device="cuda:0", slab=(0, cfg.dims[-1]))
    host = torch.empty(y.shape, dtype=y.dtype, pin_memory=True); host.copy_(y); del y; torch.cuda.empty_cache()
    arr = np.reshape(host.numpy().T, tuple(cfg.dims[:-1]) + (cfg.dims[-1],), order="F")
    tau = synth.tau_for_unit_mu(cfg, 0)
    for i in range(3):
        t0 = time.perf_counter()
        r = fit(arr, FitConfig(rank=cfg.rank, tau=tau, tol=0.0, max_iters=20, seed=0, init="random"), slab_of=cfg.dims[-1])
        t1 = time.perf_counter()
        print(name, i, "%.3f s" % (t1 - t0), r.iters, "it/s %.1f" % (r.iters / (t1 - t0)), flush=True)
    del host, arr
