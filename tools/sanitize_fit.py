"""Small fits for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): config-0 and a
C2 mini (4-way, 12^4, R=5) through the public fit(), graph replay and eager (CPF_NO_GRAPH=1)
modes chosen by the caller's environment, plus the int8 passes (CPF_OZ=1) when asked.
Usage: compute-sanitizer --tool racecheck python tools/sanitize_fit.py [c0|c2mini|c3mini|als]"""
import os as _os
_os.environ.setdefault("CPF_DEBUG", "1")  # engine knobs are read only under CPF_DEBUG=1

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_1205_2584_b200 import FitConfig, fit, synth  # noqa: E402


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "c0"
    shapes = {"c0": ("c0", (20, 20, 20), 5), "c2mini": ("c2", (12, 12, 12, 12), 5),
              "c3mini": ("c3", (24, 24, 24), 4), "c4mini": ("c4", (20, 20, 40), 4), "als": ("c0", (20, 20, 20), 5)}
    key, dims, rank = shapes[which]
    cfg = synth.scaled(synth.CONFIGS[key], dims, rank=rank, max_iters=6, name=which)
    y = synth.make_tensor(cfg, 0)
    tau = synth.tau_for_unit_mu(cfg, 0)
    variant = "als-ls" if which == "als" else "auto"
    res = fit(y, FitConfig(rank=rank, variant=variant, tau=tau, tol=0.0, max_iters=6, seed=0, init="random"))
    print(f"{which}: {res.iters} iterations, stop {res.stop_reason}, relerr {res.final_relerr:.12f}")


if __name__ == "__main__":
    main()
