"""Generate the golden fixtures in tests/golden/ by running the REFERENCE implementation.

Run in the build container (the reference is not on the GPU box):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--full]

Every fixture stores the reference's own outputs (cpfast from /root/reference/pkg/src, unmodified)
on inputs produced by the deterministic generator in paper_1205_2584_b200/synth.py (BLAS-free, so
the GPU box regenerates byte-identical inputs; each fixture records the input digest).  The
decision margins per iteration (err_sq, cand_sq) come from the repo's oracle, which this script
first checks reproduces the reference trace exactly.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import cpfast  # noqa: E402  (the reference)
from cpfast.kruskal import KruskalModel as RefModel, build_gram_cache, mttkrp as ref_mttkrp  # noqa: E402
from cpfast.kruskal import normalize_equal_energy as ref_nee, relative_error as ref_relerr  # noqa: E402
from cpfast.solver import flm_step as ref_flm_step  # noqa: E402
from cpfast.tensor import DenseTensor as RefTensor  # noqa: E402

from oracle import cp_oracle  # noqa: E402
from paper_1205_2584_b200 import synth  # noqa: E402


def stacked(factors):
    return np.concatenate([np.asarray(f).reshape(-1, order="F") for f in factors])


def run_fit_case(cfg: synth.SynthConfig, seed: int, variant: str = "auto", out_name: str | None = None):
    y = synth.make_tensor(cfg, seed)
    tau = synth.tau_for_unit_mu(cfg, seed)
    conf = cpfast.FitConfig(rank=cfg.rank, variant=variant, tau=tau, tol=cfg.tol, max_iters=cfg.max_iters,
                            seed=seed, init="random")
    t0 = time.monotonic()
    res = cpfast.fit(RefTensor(y), conf)
    wall = time.monotonic() - t0
    # oracle replay: same trace bit-for-bit?  (gives the per-iteration margins)
    o = cp_oracle.fit_lm(y, cp_oracle.OracleConfig(rank=cfg.rank, variant=variant, tau=tau, tol=cfg.tol,
                                                    max_iters=cfg.max_iters, seed=seed, init="random"))
    ref_tr = np.array([[r.iter, r.relerr, r.mu, float(r.accepted)] for r in res.trace])
    or_tr = np.array([[t, e, m, float(a)] for (t, e, m, a) in o.trace])
    oracle_bitwise = ref_tr.shape == or_tr.shape and bool(np.array_equal(ref_tr, or_tr))
    det = np.array(o.detail) if o.detail else np.zeros((0, 3))
    name = out_name or f"fit_{cfg.name}_s{seed}_{variant}"
    np.savez_compressed(
        HERE / f"{name}.npz",
        dims=np.array(cfg.dims), rank=cfg.rank, complex_=cfg.complex_, seed=seed, tau=tau, tol=cfg.tol,
        max_iters=cfg.max_iters, variant=variant, digest=synth.tensor_digest(y),
        congruence=cfg.congruence, snr_db=cfg.snr_db, bottleneck=cfg.bottleneck,
        trace=ref_tr, stop_reason=res.stop_reason, factors=stacked(res.model.factors),
        time_ms=res.time_ms, margins=det, oracle_bitwise=oracle_bitwise,
    )
    acc = "".join("A" if r.accepted else "r" for r in res.trace)
    print(f"{name}: iters={res.iters} stop={res.stop_reason} relerr={res.final_relerr:.12g} "
          f"wall={wall:.2f}s oracle_bitwise={oracle_bitwise} seq={acc}", flush=True)
    return name


def unit_cases():
    """Building-block goldens on small instances (real and complex, N = 2, 3, 4)."""
    specs = [((4, 5, 6), 2, False), ((3, 4, 5), 2, True), ((5, 4), 3, False), ((3, 4, 2, 3), 2, False),
             ((4, 3, 5, 2), 2, True), ((6, 5, 7), 3, False), ((2, 3), 1, True)]
    cases = {}
    for k, (dims, r, cplx) in enumerate(specs):
        rng = np.random.default_rng([k, 77])
        fac = []
        for d in dims:
            a = rng.standard_normal((d, r))
            if cplx:
                a = a + 1j * rng.standard_normal((d, r))
            a /= np.linalg.norm(a, axis=0, keepdims=True)
            fac.append(a)
        noise = rng.standard_normal(dims)
        if cplx:
            noise = noise + 1j * rng.standard_normal(dims)
        x = cp_oracle.reconstruct(fac)
        y = np.asfortranarray(x + 0.1 * noise)
        model = RefModel([f.copy() for f in fac])
        yt = RefTensor(y)
        rec = {"y": y, "factors": stacked(fac), "dims": np.array(dims), "rank": r}
        rec["mttkrp"] = stacked([ref_mttkrp(yt, model, n) for n in range(1, len(dims) + 1)])
        cache = build_gram_cache(model)
        rec["grams"] = np.concatenate([c.reshape(-1, order="F") for c in cache.C])
        rec["relerr"] = ref_relerr(yt, model)
        rec["nee"] = stacked(ref_nee(model).factors)
        for mu in (1e-4, 0.1, 10.0):
            for variant in ("auto", "flm-a", "flm-b"):
                for refine in (0, 2):
                    key = f"step_{variant}_{mu:g}_{refine}"
                    try:
                        rec[key] = stacked(ref_flm_step(yt, model, mu, variant, refine_steps=refine).factors)
                    except np.linalg.LinAlgError as exc:
                        rec[key + "_error"] = str(exc)
        cases[f"case{k}"] = rec
    flat = {}
    for cname, rec in cases.items():
        for key, val in rec.items():
            flat[f"{cname}__{key}"] = val
    np.savez_compressed(HERE / "unit_cases.npz", **flat)
    print(f"unit_cases: {len(cases)} instances")


def ensemble_fits():
    """Tiny acceptance-style instances: N in {2,3,4}, I_n in [2,6], R in [1,3], real and complex."""
    out = {}
    for k in range(16):
        rng = np.random.default_rng([k, 55])
        cplx = bool(k % 2)
        n_modes = int(rng.integers(2, 5))
        dims = tuple(int(rng.integers(2, 7)) for _ in range(n_modes))
        r = int(rng.integers(1, 4))
        fac = []
        for d in dims:
            a = rng.standard_normal((d, r)) + (1j * rng.standard_normal((d, r)) if cplx else 0)
            a /= np.linalg.norm(a, axis=0, keepdims=True)
            fac.append(a)
        noise = rng.standard_normal(dims) + (1j * rng.standard_normal(dims) if cplx else 0)
        y = np.asfortranarray(cp_oracle.reconstruct(fac) + 0.1 * noise)
        for variant in ("auto", "flm-a"):
            conf = cpfast.FitConfig(rank=r, variant=variant, tol=1e-10, max_iters=40, seed=k, init="random")
            res = cpfast.fit(RefTensor(y), conf)
            key = f"e{k}_{variant}"
            out[f"{key}__y"] = y
            out[f"{key}__rank"] = r
            out[f"{key}__seed"] = k
            out[f"{key}__trace"] = np.array([[t.iter, t.relerr, t.mu, float(t.accepted)] for t in res.trace])
            out[f"{key}__stop"] = res.stop_reason
            out[f"{key}__factors"] = stacked(res.model.factors)
    np.savez_compressed(HERE / "ensemble_fits.npz", **out)
    print("ensemble_fits: 16 instances x 2 variants")


def main():
    full = "--full" in sys.argv
    unit_cases()
    ensemble_fits()
    names = []
    for seed in (0, 1, 2):
        names.append(run_fit_case(synth.CONFIGS["c0"], seed))
    names.append(run_fit_case(synth.CONFIGS["c0"], 0, "flm-a"))
    minis = [
        synth.scaled(synth.CONFIGS["c1"], (30, 30, 30), rank=6, max_iters=30, name="c1_mini"),
        synth.scaled(synth.CONFIGS["c2"], (12, 12, 12, 12), rank=5, max_iters=30, name="c2_mini"),
        synth.scaled(synth.CONFIGS["c3"], (24, 24, 24), rank=4, max_iters=30, name="c3_mini"),
        synth.scaled(synth.CONFIGS["c4"], (20, 20, 40), rank=4, max_iters=20, name="c4_mini"),
    ]
    for cfg in minis:
        names.append(run_fit_case(cfg, 0))
    if full:
        for key in ("c1", "c2", "c3"):
            names.append(run_fit_case(synth.CONFIGS[key], 0))
    (HERE / "manifest.json").write_text(json.dumps({"fits": names}, indent=1))


if __name__ == "__main__":
    main()
