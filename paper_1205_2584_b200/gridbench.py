"""Monte-Carlo benchmark runner (reference: cpfast/bench.py:65-155, the existing caller of the fit
path) on the B200 fit: one record per (cell x seed x algorithm) in a deterministic order, the
same CSV contract (records.CSV_COLUMNS) and per-cell summary.

Inputs are the reference's collinear swamp instances (cpfast/synth.py:23-99): per mode a_1 = u_1,
a_r = u_1 + nu u_r (r >= 2) for the orthonormal columns u of a seeded QR (``default_rng([seed, 0])``),
the noise-free tensor as A_1 (A_N kr ... kr A_2)^T folded column-major, plus white Gaussian noise
at the requested SNR from ``default_rng([seed, 1])``.  Restated call for call so the tensors are
the reference's own bytes on the same NumPy/LAPACK (pinned by tests/golden/make_grid_golden.py).
This is host-side harness code: the fits it drives run in the engine.
"""

from __future__ import annotations

import csv
import math
import statistics
from dataclasses import dataclass
from functools import reduce

import numpy as np

from .records import RunRecord, _cell, record_from_result, write_csv  # noqa: F401  (re-exported)
from .solver import FitConfig, fit
from .tensor import COMPLEX, REAL, DenseTensor, KruskalModel


@dataclass
class CollinearSpec:
    dims: tuple
    rank: int
    nu: float
    snr_db: float | None = None
    seed: int = 0
    scalar_kind: str = REAL

    def __post_init__(self):
        self.dims = tuple(int(d) for d in self.dims)
        if self.nu <= 0:
            raise ValueError("nu must be positive")
        if self.rank > min(self.dims):
            raise ValueError(f"rank {self.rank} exceeds smallest dimension {min(self.dims)}")


def _kr(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Column-wise Kronecker product (I x R, K x R) -> (I K) x R, b's index fastest."""
    return (a[:, None, :] * b[None, :, :]).reshape(a.shape[0] * b.shape[0], a.shape[1])


def gen_collinear(spec: CollinearSpec):
    """(truth model, noise-free tensor) of the collinear swamp instance."""
    rng = np.random.default_rng([spec.seed, 0])
    factors = []
    for d in spec.dims:
        g = rng.standard_normal((d, spec.rank))
        if spec.scalar_kind == COMPLEX:
            g = g + 1j * rng.standard_normal((d, spec.rank))
        u = np.linalg.qr(g)[0]
        a = u.copy()
        a[:, 1:] = u[:, [0]] + spec.nu * u[:, 1:]
        factors.append(a)
    a1 = factors[0] * np.ones(spec.rank, dtype=factors[0].dtype)[None, :]
    w = reduce(_kr, [factors[k] for k in reversed(range(1, len(factors)))])
    x = (a1 @ w.T).reshape(spec.dims, order="F")
    return KruskalModel(factors), DenseTensor(x)


def add_noise(tensor: DenseTensor, snr_db: float | None, seed: int) -> DenseTensor:
    """White Gaussian noise at ``snr_db`` (None / inf: unchanged); complex noise circular."""
    if snr_db is None or math.isinf(snr_db):
        return tensor
    ynorm = tensor.norm()
    if ynorm == 0.0:
        raise ZeroDivisionError("cannot calibrate noise for a zero tensor")
    sigma = ynorm / math.sqrt(tensor.size * 10.0 ** (snr_db / 10.0))
    rng = np.random.default_rng([seed, 1])
    noise = rng.standard_normal(tensor.dims)
    if tensor.scalar_kind == COMPLEX:
        noise = (noise + 1j * rng.standard_normal(tensor.dims)) / math.sqrt(2.0)
    return DenseTensor(tensor.data + sigma * noise)


def run_single(dims, rank: int, nu: float, snr_db, algo: str, seed: int, scalar_kind: str = REAL,
               tau: float = 1e-3, tol: float = 1e-8, max_iters: int = 1000, init: str = "svd", device=None):
    """One cell instance on the engine: (record, truth, fitted model)."""
    spec = CollinearSpec(dims, rank, nu, snr_db, seed, scalar_kind)
    truth, tensor = gen_collinear(spec)
    tensor = add_noise(tensor, snr_db, seed)
    config = FitConfig(rank=rank, variant=algo, tau=tau, tol=tol, max_iters=max_iters, seed=seed, init=init)
    result = fit(tensor, config, device=device)
    return record_from_result(result, truth, seed, nu, rank, snr_db, algo), truth, result.model


def run_grid(dims, ranks, nus, snrs, algos, seeds: int, scalar_kind: str = REAL, **fit_kwargs) -> list:
    """All (nu, R, snr) x seed x algo cells in the reference's order; a failing cell (e.g. an
    algorithm the B200 backend does not run) becomes an 'error' record, as in the reference."""
    records = []
    for nu in nus:
        for rank in ranks:
            for snr_db in snrs:
                for seed in range(seeds):
                    for algo in algos:
                        try:
                            rec = run_single(dims, rank, nu, snr_db, algo, seed, scalar_kind, **fit_kwargs)[0]
                        except Exception:
                            rec = RunRecord(seed, nu, rank, snr_db, algo, 0, 0, 0.0, float("nan"), None, None, "error")
                        records.append(rec)
    return records


def summarize(records) -> list:
    """Per (nu, R, snr, algo) cell: runs, errors, medians of iterations / relerr / MedSAE."""
    cells = {}
    for rec in records:
        cells.setdefault((rec.nu, rec.R, rec.snr_db, rec.algo), []).append(rec)

    def med(vals):
        vals = [v for v in vals if v is not None]
        return statistics.median(vals) if vals else ""

    rows = []
    for key in sorted(cells, key=lambda k: tuple(map(str, k))):
        group = cells[key]
        ok = [r for r in group if r.stop_reason != "error"]
        rows.append({"nu": key[0], "R": key[1], "snr_db": key[2], "algo": key[3], "runs": len(group),
                     "errors": len(group) - len(ok),
                     "median_iters": med([r.iters for r in ok]),
                     "median_relerr": med([r.final_relerr for r in ok]),
                     "median_medsae_first_db": med([r.medsae_first_db for r in ok]),
                     "median_medsae_rest_db": med([r.medsae_rest_db for r in ok])})
    return rows


SUMMARY_COLUMNS = ("nu", "R", "snr_db", "algo", "runs", "errors", "median_iters", "median_relerr",
                   "median_medsae_first_db", "median_medsae_rest_db")


def write_summary_csv(path, rows) -> None:
    with open(path, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(SUMMARY_COLUMNS)
        w.writerows([_cell(row[c]) for c in SUMMARY_COLUMNS] for row in rows)
