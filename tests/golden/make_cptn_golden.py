"""Golden CPTN files and MedSAE scores from the REFERENCE implementation (run in the build
container, where /root/reference is importable; the outputs are committed, the reference is not).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_cptn_golden.py
"""

import json
from pathlib import Path

import numpy as np

from cpfast import cptn
from cpfast.bench import RunRecord, write_csv
from cpfast.kruskal import KruskalModel
from cpfast.synth import medsae_pair
from cpfast.tensor import DenseTensor

OUT = Path(__file__).resolve().parent
rng = np.random.default_rng(1205)
real = rng.standard_normal((3, 4, 5))
cplx = rng.standard_normal((2, 3, 2)) + 1j * rng.standard_normal((2, 3, 2))
cptn.write_tensor(OUT / "cptn_real.cptn", DenseTensor(real))
cptn.write_tensor(OUT / "cptn_complex.cptn", DenseTensor(cplx))
cptn.write_matrix(OUT / "cptn_matrix.cptn", rng.standard_normal((4, 2)))
cptn.write_metadata(OUT / "cptn_meta.meta", {"dims": "3,4,5", "R": 2, "nu": 0.5, "snr_db": "inf"})

truth = KruskalModel([rng.standard_normal((6, 3)) for _ in range(3)])
est = KruskalModel([f[:, [2, 0, 1]] * 1.7 + 1e-3 * rng.standard_normal(f.shape) for f in truth.factors])
exact = KruskalModel([f[:, [1, 2, 0]] * -2.0 for f in truth.factors])
scores = {"perturbed": medsae_pair(truth, est), "exact": medsae_pair(truth, exact)}
np.savez(OUT / "medsae_case.npz", **{f"truth{n}": f for n, f in enumerate(truth.factors)},
         **{f"est{n}": f for n, f in enumerate(est.factors)}, **{f"exact{n}": f for n, f in enumerate(exact.factors)})
json.dump({k: {"first_db": v["first_db"], "rest_db": v["rest_db"]} for k, v in scores.items()},
          open(OUT / "medsae_case.json", "w"), indent=1)
write_csv(OUT / "record_case.csv", [RunRecord(3, float("nan"), 4, None, "auto", 17, 12, 123.456, 0.0123456789,
                                              -45.5, None, "tol"),
                                    RunRecord(0, 0.5, 2, float("inf"), "flm-b", 0, 0, 0.0, float("nan"), None, None,
                                              "error")])
print("wrote cptn/medsae/record goldens")
