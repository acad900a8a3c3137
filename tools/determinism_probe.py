"""Run the same fit several times and report whether traces / factors are bitwise identical."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from tests import _golden as G
import paper_1205_2584_b200 as api

key = sys.argv[1] if len(sys.argv) > 1 else "e0_flm-a"
e = G.ensemble()[key]
variant = key.split("_", 1)[1]
y = api.DenseTensor(e["y"])
outs = []
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 6):
    conf = api.FitConfig(rank=int(e["rank"]), variant=variant, tol=1e-10, max_iters=40, seed=int(e["seed"]), init="random")
    r = api.fit(y, conf)
    outs.append((tuple((t.relerr, t.mu, t.accepted) for t in r.trace), r.model.as_vector().copy()))
base = outs[0]
for i, (tr, v) in enumerate(outs):
    same_tr = tr == base[0]
    diff = float(np.max(np.abs(v - base[1])))
    first = next((k for k, (a, b) in enumerate(zip(tr, base[0])) if a != b), None)
    print(f"run {i}: trace identical {same_tr} (first diff at {first}), max |factor diff| {diff:.3e}, iters {len(tr)}")
print("dims", e["y"].shape, "rank", int(e["rank"]))
