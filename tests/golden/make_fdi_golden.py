"""Golden fixtures for fast_damped_inverse (hessian.py:232-277), captured by
running the REFERENCE implementation in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_fdi_golden.py

``fdi_cases.npz``: per instance (real / complex unit-column models, N = 2, 3, 4, R = 1..10 so the
core system n_B = N R^2 spans 2..300), per mu in the reference's verification grid
(verify.py:43 MU_GRID) and per path (K-free / K^{-1} / auto): gamma_tilde, the stacked core grid
D, and the dense (H + mu I)^{-1} (materialize_inverse) for reference.  Plus an orthonormal model
whose K is singular: the K^{-1} path raises SingularKernelError, auto falls back to K-free.
Each entry is replayed through the oracle restatement (oracle_bitwise records agreement)."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

from cpfast.hessian import SingularKernelError, fast_damped_inverse, materialize_inverse  # noqa: E402
from cpfast.kruskal import KruskalModel, build_gram_cache, random_init  # noqa: E402

from oracle import cp_oracle  # noqa: E402

MU_GRID = (1e-6, 1e-2, 1.0, 1e3)


def unit_model(rng, dims, rank, kind):
    m = random_init(dims, rank, rng, kind)
    for f in m.factors:
        f /= np.linalg.norm(f, axis=0, keepdims=True)
    return m


def core(sinv):
    return np.block(sinv.S)


def main():
    out = {}
    bitwise = True
    specs = [((3, 4, 2), 2, "real"), ((3, 4, 2), 2, "complex"), ((5, 6), 3, "real"), ((2, 3, 2, 3), 2, "complex"),
             ((6, 5, 7), 4, "real"), ((8, 9, 7), 10, "real"), ((5, 6, 4), 6, "complex"), ((4, 4, 4), 1, "real")]
    for k, (dims, r, kind) in enumerate(specs):
        rng = np.random.default_rng([k, 33])
        m = unit_model(rng, dims, r, kind)
        cache = build_gram_cache(m)
        key = f"i{k}"
        out[f"{key}__dims"] = np.array(dims)
        out[f"{key}__rank"] = r
        out[f"{key}__factors"] = np.concatenate([f.reshape(-1, order="F") for f in m.factors])
        for mu in MU_GRID:
            for path, flag in (("kfree", False), ("kinv", True), ("auto", None)):
                tag = f"{key}__{path}_{mu:g}"
                try:
                    s = fast_damped_inverse(cache, m.factors, mu, use_kernel_inverse=flag)
                except SingularKernelError as exc:
                    out[f"{tag}_error"] = str(exc)
                    continue
                out[f"{tag}_gt"] = np.stack(s.gamma_tilde)
                out[f"{tag}_core"] = core(s)
                if sum(dims) * r <= 400:
                    out[f"{tag}_dense"] = materialize_inverse(s, m.factors)
                o = cp_oracle.fast_damped_inverse(m.factors, mu, flag)
                bitwise &= bool(np.array_equal(core(s), o[1])) and all(
                    np.array_equal(a, b) for a, b in zip(s.gamma_tilde, o[0]))
    # orthonormal factors: pairwise Gammas are identity-like, K singular
    rng = np.random.default_rng(5)
    fac = []
    for d in (6, 6, 6):
        q, _ = np.linalg.qr(rng.standard_normal((d, 3)))
        fac.append(q)
    m = KruskalModel(fac)
    cache = build_gram_cache(m)
    out["orth__dims"] = np.array((6, 6, 6))
    out["orth__rank"] = 3
    out["orth__factors"] = np.concatenate([f.reshape(-1, order="F") for f in m.factors])
    try:
        fast_damped_inverse(cache, m.factors, 0.5, use_kernel_inverse=True)
        out["orth__kinv_error"] = ""
    except SingularKernelError as exc:
        out["orth__kinv_error"] = str(exc)
    s = fast_damped_inverse(cache, m.factors, 0.5)
    out["orth__auto_0.5_gt"] = np.stack(s.gamma_tilde)
    out["orth__auto_0.5_core"] = core(s)
    out["oracle_bitwise"] = bitwise
    np.savez_compressed(HERE / "fdi_cases.npz", **out)
    print(f"fdi cases: {len(specs)} instances x {len(MU_GRID)} mu x 3 paths + orthonormal; oracle_bitwise={bitwise}; "
          f"K^-1 on orthonormal: {out['orth__kinv_error']!r}")


if __name__ == "__main__":
    main()
