"""Run records, their CSV form and the MedSAE score -- what the reference's ``fit`` CLI writes
(cpfast/bench.py:16-66, 98-124, 190-196; cpfast/synth.py:174-245).  Host-side bookkeeping around
the fit path; the scoring compares a fitted model with the generating factors.
"""

from __future__ import annotations

import csv
import math
from dataclasses import dataclass, fields

import numpy as np

CSV_COLUMNS = ("seed", "nu", "R", "snr_db", "algo", "iters", "accepted_iters", "time_ms", "final_relerr",
               "medsae_first_db", "medsae_rest_db", "stop_reason")
MEDSAE_FLOOR_DB = -300.0


@dataclass
class RunRecord:
    seed: int
    nu: float
    R: int
    snr_db: float | None
    algo: str
    iters: int
    accepted_iters: int
    time_ms: float
    final_relerr: float
    medsae_first_db: float | None
    medsae_rest_db: float | None
    stop_reason: str

    def __post_init__(self):
        if not (self.iters >= self.accepted_iters >= 0):
            raise ValueError("need iters >= accepted_iters >= 0")

    def row(self) -> list:
        return [_cell(getattr(self, f.name)) for f in fields(self)]


def _cell(value) -> str:
    """CSV cell: empty for None, 'inf' for infinities, repr() for floats (exact round trip)."""
    if value is None:
        return ""
    if isinstance(value, float):
        return "inf" if math.isinf(value) else repr(value)
    return str(value)


def component_angles(truth, estimate) -> np.ndarray:
    """(N, R) angles between truth components and their Hungarian-matched estimates; matching
    maximises the product over modes of normalised |inner products|; cosines within 1e-14 of 1
    count as exact alignment."""
    from scipy.optimize import linear_sum_assignment

    if truth.rank != estimate.rank:
        raise ValueError("rank mismatch between truth and estimate")
    unit = lambda f: f / np.linalg.norm(f, axis=0, keepdims=True)  # noqa: E731
    score = np.ones((truth.rank, truth.rank))
    for ft, fe in zip(truth.factors, estimate.factors):
        score = score * np.abs(unit(ft).conj().T @ unit(fe))
    perm = linear_sum_assignment(-score)[1]
    out = np.zeros((truth.order, truth.rank))
    for n, (ft, fe) in enumerate(zip(truth.factors, estimate.factors)):
        fe = fe[:, perm]
        cos = np.abs(np.sum(ft.conj() * fe, axis=0)) / (np.linalg.norm(ft, axis=0) * np.linalg.norm(fe, axis=0))
        cos = np.clip(cos, 0.0, 1.0)
        out[n] = np.arccos(np.where(cos > 1.0 - 1e-14, 1.0, cos))
    return out


def medsae(angle_runs) -> dict:
    """Median (over runs) squared angular error per component in dB, floored at -300 dB;
    first_db = component 1 averaged over modes, rest_db = components 2.. (None for R = 1)."""
    sq = np.median(np.stack([np.asarray(a) ** 2 for a in angle_runs]), axis=0)
    db = np.full(sq.shape, MEDSAE_FLOOR_DB)
    pos = sq > 0
    db[pos] = np.maximum(10.0 * np.log10(sq[pos]), MEDSAE_FLOOR_DB)
    return {"first_db": float(np.mean(db[:, 0])),
            "rest_db": float(np.mean(db[:, 1:])) if db.shape[1] > 1 else None,
            "per_component": db}


def medsae_pair(truth, estimate) -> dict:
    return medsae([component_angles(truth, estimate)])


def record_from_result(result, truth, seed, nu, rank, snr_db, algo) -> RunRecord:
    stop = result.stop_reason if result.stop_reason in ("tol", "max_iters", "mu_overflow") else "error"
    scores = medsae_pair(truth, result.model) if truth is not None else None
    return RunRecord(seed=seed, nu=nu, R=rank, snr_db=snr_db, algo=algo, iters=result.iters,
                     accepted_iters=result.accepted_iters, time_ms=result.time_ms,
                     final_relerr=result.final_relerr,
                     medsae_first_db=scores["first_db"] if scores else None,
                     medsae_rest_db=scores["rest_db"] if scores else None, stop_reason=stop)


def write_csv(path, records) -> None:
    with open(path, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(CSV_COLUMNS)
        w.writerows(rec.row() for rec in records)
