"""Helpers to load the golden fixtures captured from the reference (tests/golden/make_golden.py)."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def fit_names(include_full: bool = True):
    names = json.loads((GOLDEN / "manifest.json").read_text())["fits"]
    if not include_full:
        names = [n for n in names if not n.split("_")[1] in ("c1", "c2", "c3") or "mini" in n]
    return [n for n in names if (GOLDEN / f"{n}.npz").exists()]


def load_fit(name: str) -> dict:
    z = np.load(GOLDEN / f"{name}.npz", allow_pickle=False)
    d = {k: z[k] for k in z.files}
    for k in ("rank", "seed", "max_iters"):
        d[k] = int(d[k])
    for k in ("tau", "tol", "congruence", "snr_db", "time_ms"):
        d[k] = float(d[k])
    for k in ("complex_", "bottleneck", "oracle_bitwise"):
        d[k] = bool(d[k])
    d["variant"] = str(d["variant"])
    d["digest"] = str(d["digest"])
    d["stop_reason"] = str(d["stop_reason"])
    d["dims"] = tuple(int(x) for x in d["dims"])
    return d


def synth_config(d: dict):
    from paper_1205_2584_b200 import synth

    return synth.SynthConfig("golden", d["dims"], d["rank"], d["congruence"], d["snr_db"], d["complex_"],
                             d["bottleneck"], d["max_iters"], d["tol"])


def unit_cases() -> dict:
    z = np.load(GOLDEN / "unit_cases.npz", allow_pickle=False)
    cases: dict = {}
    for key in z.files:
        cname, field = key.split("__", 1)
        cases.setdefault(cname, {})[field] = z[key]
    return cases


def ensemble() -> dict:
    z = np.load(GOLDEN / "ensemble_fits.npz", allow_pickle=False)
    out: dict = {}
    for key in z.files:
        cname, field = key.split("__", 1)
        out.setdefault(cname, {})[field] = z[key]
    return out


def accept_seq(trace: np.ndarray) -> str:
    return "".join("A" if a else "r" for a in trace[:, 3])


def split_stacked(vec, dims, rank):
    out, off = [], 0
    for d in dims:
        out.append(np.asarray(vec[off: off + d * rank]).reshape((d, rank), order="F"))
        off += d * rank
    return out


def _grouped(fname: str) -> dict:
    z = np.load(GOLDEN / fname, allow_pickle=False)
    out: dict = {}
    for key in z.files:
        if "__" not in key:
            out[key] = z[key]
            continue
        cname, field = key.split("__", 1)
        out.setdefault(cname, {})[field] = z[key]
    return out


def als_fits() -> dict:
    """ALS / ALS-ls fits captured from the reference (tests/golden/make_als_golden.py)."""
    return {k: v for k, v in _grouped("als_fits.npz").items() if isinstance(v, dict)}


def als_units() -> dict:
    return _grouped("als_units.npz")


def als_config(name: str, case: dict):
    """SynthConfig of an ALS fit fixture (name = '<config>_<variant>')."""
    from paper_1205_2584_b200 import synth

    base = name.rsplit("_", 1)[0]
    key = base.split("_")[0]
    dims = tuple(int(x) for x in case["dims"])
    return synth.scaled(synth.CONFIGS[key], dims, rank=int(case["rank"]), max_iters=int(case["max_iters"]), name=base)
