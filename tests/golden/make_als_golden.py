"""Golden fixtures for the ALS baselines (variants "als" / "als-ls"), captured
by running the REFERENCE implementation in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_als_golden.py

Writes
* ``als_fits.npz``  -- ``cpfast.fit`` traces and final factors with variant "als" and "als-ls" on
  the config-0 instance (seed 0) and the C1-C4 minis (inputs from paper_1205_2584_b200/synth.py, so
  the GPU box regenerates them byte-identically; digest recorded);
* ``als_units.npz`` -- ``cpfast.kruskal.pinv_psd`` on Hermitian PSD matrices (full rank, rank
  deficient, complex, with zero and negative-rounding eigenvalues), and ``als_step`` /
  ``als_line_search_step`` (with and without history, t = 1, 2, 5) on small real / complex instances.

Every output is also replayed through ``oracle/cp_oracle.py`` and the fixture records whether the
replay is bit-identical (``oracle_bitwise``).
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import cpfast  # noqa: E402  (the reference)
from cpfast.kruskal import KruskalModel as RefModel  # noqa: E402
from cpfast.kruskal import als_line_search_step as ref_als_ls, als_step as ref_als_step  # noqa: E402
from cpfast.kruskal import pinv_psd as ref_pinv  # noqa: E402
from cpfast.tensor import DenseTensor as RefTensor  # noqa: E402

from oracle import cp_oracle  # noqa: E402
from paper_1205_2584_b200 import synth  # noqa: E402


def stacked(factors):
    return np.concatenate([np.asarray(f).reshape(-1, order="F") for f in factors])


def fit_cases(out: dict):
    cases = [
        (synth.scaled(synth.CONFIGS["c0"], (20, 20, 20), rank=5, max_iters=60, name="c0"), 1e-10),
        (synth.scaled(synth.CONFIGS["c1"], (30, 30, 30), rank=6, max_iters=25, name="c1_mini"), 0.0),
        (synth.scaled(synth.CONFIGS["c2"], (12, 12, 12, 12), rank=5, max_iters=25, name="c2_mini"), 0.0),
        (synth.scaled(synth.CONFIGS["c3"], (24, 24, 24), rank=4, max_iters=25, name="c3_mini"), 0.0),
        (synth.scaled(synth.CONFIGS["c4"], (20, 20, 40), rank=4, max_iters=20, name="c4_mini"), 0.0),
    ]
    for cfg, tol in cases:
        y = synth.make_tensor(cfg, 0)
        for variant in ("als", "als-ls"):
            conf = cpfast.FitConfig(rank=cfg.rank, variant=variant, tol=tol, max_iters=cfg.max_iters, seed=0,
                                    init="random")
            t0 = time.monotonic()
            res = cpfast.fit(RefTensor(y), conf)
            wall = time.monotonic() - t0
            o = cp_oracle.fit_als(y, cp_oracle.OracleConfig(rank=cfg.rank, variant=variant, tol=tol,
                                                             max_iters=cfg.max_iters, seed=0))
            tr = np.array([[r.iter, r.relerr, r.mu, float(r.accepted)] for r in res.trace])
            otr = np.array([[t, e, m, float(a)] for (t, e, m, a) in o.trace])
            bitwise = tr.shape == otr.shape and bool(np.array_equal(tr, otr)) and bool(
                np.array_equal(stacked(res.model.factors), cp_oracle.stack(o.factors)))
            key = f"{cfg.name}_{variant}"
            out.update({
                f"{key}__dims": np.array(cfg.dims), f"{key}__rank": cfg.rank, f"{key}__complex": cfg.complex_,
                f"{key}__tol": tol, f"{key}__max_iters": cfg.max_iters, f"{key}__digest": synth.tensor_digest(y),
                f"{key}__trace": tr, f"{key}__stop": res.stop_reason, f"{key}__factors": stacked(res.model.factors),
                f"{key}__oracle_bitwise": bitwise,
            })
            print(f"{key}: iters={res.iters} stop={res.stop_reason} relerr={res.final_relerr:.12g} "
                  f"wall={wall:.2f}s oracle_bitwise={bitwise}", flush=True)
    return [k.split("__")[0] for k in out if k.endswith("__trace")]


def unit_cases(out: dict):
    rng = np.random.default_rng([2025, 7])
    mats = {}
    for r in (1, 2, 5, 7, 20, 40):
        a = rng.standard_normal((3 * r + 2, r))
        mats[f"full_r{r}"] = a.T @ a
    for r in (3, 6, 17):
        a = rng.standard_normal((3 * r, r)) + 1j * rng.standard_normal((3 * r, r))
        mats[f"cfull_r{r}"] = a.conj().T @ a
    a = rng.standard_normal((8, 4))
    mats["deficient_r8"] = a @ a.T                  # rank 4 of 8: truncated eigenvalues
    a = rng.standard_normal((6, 3)) + 1j * rng.standard_normal((6, 3))
    mats["cdeficient_r6"] = a @ a.conj().T
    mats["zero_r3"] = np.zeros((3, 3))
    g = rng.standard_normal((9, 5))
    mats["hadamard_r5"] = (g.T @ g) * (np.ones((5, 5)) * 0.9 + 0.1 * np.eye(5)) * (1e3 * np.eye(5) + 1.0)
    bitwise = True
    for name, m in mats.items():
        p = ref_pinv(m)
        out[f"pinv_{name}__in"] = m
        out[f"pinv_{name}__out"] = p
        bitwise &= bool(np.array_equal(p, cp_oracle.pinv_psd(m)))
    specs = [((5, 6, 7), 3, False), ((4, 5, 3), 2, True), ((4, 3, 5, 2), 2, False), ((6, 5), 3, True)]
    for k, (dims, r, cplx) in enumerate(specs):
        rng = np.random.default_rng([k, 91])

        def draw():
            fac = []
            for d in dims:
                a = rng.standard_normal((d, r))
                if cplx:
                    a = a + 1j * rng.standard_normal((d, r))
                fac.append(a)
            return fac

        truth, start, hist = draw(), draw(), draw()
        noise = rng.standard_normal(dims) + (1j * rng.standard_normal(dims) if cplx else 0)
        y = np.asfortranarray(cp_oracle.reconstruct(truth) + 0.05 * noise)
        yt = RefTensor(y)
        key = f"step{k}"
        out[f"{key}__y"] = y
        out[f"{key}__dims"] = np.array(dims)
        out[f"{key}__rank"] = r
        out[f"{key}__start"] = stacked(start)
        out[f"{key}__hist"] = stacked(hist)
        s = ref_als_step(yt, RefModel([f.copy() for f in start]))
        out[f"{key}__als"] = stacked(s.factors)
        bitwise &= bool(np.array_equal(stacked(s.factors), cp_oracle.stack(cp_oracle.als_step(y, start))))
        for t in (1, 2, 5):
            ls = ref_als_ls(yt, RefModel([f.copy() for f in start]), RefModel([f.copy() for f in hist]), t)
            out[f"{key}__ls_t{t}"] = stacked(ls.factors)
            o = cp_oracle.als_line_search_step(y, start, hist, t)
            bitwise &= bool(np.array_equal(stacked(ls.factors), cp_oracle.stack(o)))
        ls0 = ref_als_ls(yt, RefModel([f.copy() for f in start]), None, 3)
        out[f"{key}__ls_nohist"] = stacked(ls0.factors)
    out["oracle_bitwise"] = bitwise
    print(f"als units: {len(mats)} pinv matrices, {len(specs)} step instances, oracle_bitwise={bitwise}")
    return list(mats)


def main():
    fits = {}
    fit_cases(fits)
    np.savez_compressed(HERE / "als_fits.npz", **fits)
    units = {}
    unit_cases(units)
    np.savez_compressed(HERE / "als_units.npz", **units)


if __name__ == "__main__":
    main()
