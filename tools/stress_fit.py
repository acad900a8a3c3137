"""Repeated fits of a BASELINE config in one process: every fit must return the same trace and final
error bit for bit, and none may fault or hang.  Found the speculative branch's cluster-panel gate
race (round 2): two CTAs of a panel reading `stopped` themselves while k_decide wrote it on the
fit's last iteration -- about one fit in a hundred hung or died with a launch failure.
usage: python tools/stress_fit.py c2 300   (wrap in `timeout`: the failure mode was a hang)"""
import os, sys, time
os.environ.setdefault("CPF_DEBUG", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1205_2584_b200 import FitConfig, fit, fit_complex, synth
key = sys.argv[1]; n = int(sys.argv[2])
cfg = synth.CONFIGS[key]
y = synth.make_tensor(cfg, 0)
tau = synth.tau_for_unit_mu(cfg, 0)
fitter = fit_complex if cfg.complex_ else fit
base = None
t0 = time.time()
for i in range(n):
    res = fitter(y, FitConfig(rank=cfg.rank, tau=tau, tol=0.0, max_iters=cfg.max_iters, seed=0, init="random"), device=0)
    sig = ("".join("A" if r.accepted else "r" for r in res.trace), res.final_relerr)
    if i % 25 == 0: print("fit", i, flush=True)
    if base is None: base = sig
    elif sig != base: print("DIFF at", i, sig, base)
print(key, "ok", n, "fits", base[0], base[1], f"{time.time()-t0:.1f}s")
