"""Golden collinear instances and a small Monte-Carlo grid from the REFERENCE (run in the build
container, where /root/reference is importable; outputs committed):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_grid_golden.py
"""

import hashlib
import json
from pathlib import Path

import numpy as np

from cpfast.bench import run_grid, summarize, write_csv, write_summary_csv
from cpfast.synth import CollinearSpec, add_noise, gen_collinear

OUT = Path(__file__).resolve().parent
cases = {}
for name, (dims, r, nu, snr, seed, kind) in {
    "real3": ((7, 6, 5), 3, 0.4, 25.0, 3, "real"),
    "cplx3": ((5, 6, 4), 2, 0.9, None, 1, "complex"),
    "real4": ((4, 5, 3, 4), 3, 0.2, 10.0, 0, "real"),
}.items():
    truth, x = gen_collinear(CollinearSpec(dims, r, nu, snr, seed, kind))
    y = add_noise(x, snr, seed)
    cases[name] = {"dims": list(dims), "rank": r, "nu": nu, "snr_db": snr, "seed": seed, "kind": kind,
                   "x_sha": hashlib.sha256(np.asfortranarray(x.data).tobytes(order="F")).hexdigest(),
                   "y_sha": hashlib.sha256(np.asfortranarray(y.data).tobytes(order="F")).hexdigest(),
                   "f_sha": [hashlib.sha256(np.ascontiguousarray(f).tobytes()).hexdigest() for f in truth.factors]}
json.dump(cases, open(OUT / "grid_instances.json", "w"), indent=1)
recs = run_grid((6, 6, 6), (2,), (0.3, 0.9), (None, 30.0), ("auto", "flm-b"), 2, init="random")
write_csv(OUT / "grid_reference.csv", recs)
write_summary_csv(OUT / "grid_reference_summary.csv", summarize(recs))
print("wrote grid goldens:", len(recs), "records")
