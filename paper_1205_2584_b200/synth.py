"""Seeded synthetic inputs for the five BASELINE configurations (harness, not product code).

BASELINE.json's configs use a congruence construction that the reference package does not
ship:  A_n = Q_n chol(C_n)^T with Q_n an orthonormalised Gaussian draw and
C_n = (1-c) I + c 11^T, X = sum_r a1_r o ... o aN_r, Y = X + sigma N with sigma calibrated to
the SNR exactly like the reference's ``add_noise`` (cpfast/synth.py:81-99; noise stream
``default_rng([seed, 1])``).  The truth stream is ``default_rng([seed, 100])`` -- NOT
``[seed, 0]``, which the fit itself uses for its initial factors (finding 5).

The host path is written to be bit-reproducible on any IEEE-754 machine: no BLAS/LAPACK call
(Gram-Schmidt and Cholesky with ``math.fsum`` inner products, outer products accumulated
elementwise in a fixed order), so the GPU box regenerates exactly the bytes the golden traces
were captured on.  ``device_tensor`` builds the 16 GB config-4 tensor directly in HBM (same
factors; noise from a seeded torch generator) for the throughput benchmark.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class SynthConfig:
    name: str
    dims: tuple
    rank: int
    congruence: float
    snr_db: float
    complex_: bool = False
    bottleneck: bool = False      # config 2: mode-1 C[0,1] = 0.99, log-uniform magnitudes
    max_iters: int = 50
    tol: float = 0.0


CONFIGS = {
    "c0": SynthConfig("c0", (20, 20, 20), 5, 0.8, 30.0, max_iters=200, tol=1e-10),
    "c1": SynthConfig("c1", (200, 200, 200), 40, 0.9, 20.0, max_iters=50),
    "c2": SynthConfig("c2", (80, 80, 80, 80), 15, 0.5, 25.0, bottleneck=True, max_iters=50),
    "c3": SynthConfig("c3", (256, 256, 256), 10, 0.85, 20.0, complex_=True, max_iters=30),
    "c4": SynthConfig("c4", (1000, 1000, 2000), 20, 0.7, 20.0, max_iters=20),
}


def scaled(cfg: SynthConfig, dims, rank=None, max_iters=None, name=None) -> SynthConfig:
    """A reduced-size variant of a config (same construction) for fast parity tests."""
    return SynthConfig(name or f"{cfg.name}_mini", tuple(dims), rank or cfg.rank, cfg.congruence, cfg.snr_db,
                       cfg.complex_, cfg.bottleneck, max_iters or cfg.max_iters, cfg.tol)


def _fsum_c(values) -> complex | float:
    v = np.asarray(values)
    if np.iscomplexobj(v):
        return complex(math.fsum(v.real.tolist()), math.fsum(v.imag.tolist()))
    return math.fsum(v.tolist())


def _orthonormal(g: np.ndarray) -> np.ndarray:
    """Classical Gram-Schmidt applied twice, exact-sum inner products (deterministic)."""
    q = np.array(g, copy=True)
    n, r = q.shape
    for j in range(r):
        v = q[:, j].copy()
        for _ in range(2):
            for k in range(j):
                coef = _fsum_c(np.conj(q[:, k]) * v)
                v = v - coef * q[:, k]
        nrm = math.sqrt(math.fsum((np.abs(v) ** 2).tolist()))
        q[:, j] = v / nrm
    return q


def _cholesky(c: np.ndarray) -> np.ndarray:
    r = c.shape[0]
    L = np.zeros_like(c)
    for i in range(r):
        for j in range(i + 1):
            s = math.fsum([L[i, k] * L[j, k] for k in range(j)])
            if i == j:
                L[i, i] = math.sqrt(c[i, i] - s)
            else:
                L[i, j] = (c[i, j] - s) / L[j, j]
    return L


def congruence_matrix(rank: int, c: float, pair: float | None = None) -> np.ndarray:
    m = (1.0 - c) * np.eye(rank) + c * np.ones((rank, rank))
    if pair is not None and rank >= 2:
        m[0, 1] = m[1, 0] = pair
    return m


def truth_factors(cfg: SynthConfig, seed: int = 0) -> list:
    rng = np.random.default_rng([seed, 100])
    factors = []
    for n, d in enumerate(cfg.dims):
        g = rng.standard_normal((d, cfg.rank))
        if cfg.complex_:
            g = (g + 1j * rng.standard_normal((d, cfg.rank))) / math.sqrt(2.0)
        q = _orthonormal(g)
        cmat = congruence_matrix(cfg.rank, cfg.congruence, 0.99 if (cfg.bottleneck and n == 0) else None)
        L = _cholesky(cmat)
        a = np.zeros_like(q)
        for j in range(cfg.rank):          # A = Q L^T, fixed accumulation order
            col = np.zeros(d, dtype=q.dtype)
            for k in range(j + 1):
                col = col + q[:, k] * L[j, k]
            a[:, j] = col
        factors.append(a)
    if cfg.bottleneck:
        mags = 10.0 ** rng.uniform(0.0, 3.0, cfg.rank)
        factors[-1] = factors[-1] * mags[None, :]
    return factors


def reconstruct_exact(factors) -> np.ndarray:
    """sum_r outer products, accumulated elementwise in r order (no BLAS), Fortran order."""
    dims = tuple(f.shape[0] for f in factors)
    dtype = np.result_type(*factors)
    x = np.zeros(dims, dtype=dtype, order="F")
    for r in range(factors[0].shape[1]):
        t = factors[0][:, r]
        for f in factors[1:]:
            t = np.multiply.outer(t, f[:, r])
        x += t
    return x


_FSUM_CHUNK = 1 << 22


def frob_exact(x: np.ndarray) -> float:
    """Frobenius norm with exact (fsum) accumulation; above 2^22 elements the exact sums of
    2^22-element chunks (Fortran order) are fsum-ed -- still machine independent, without a
    J-element Python list."""
    flat = x.ravel(order="F") if x.flags.f_contiguous else x.ravel(order="K")
    if flat.size <= _FSUM_CHUNK:
        a = np.abs(flat) ** 2 if np.iscomplexobj(flat) else flat * flat
        return math.sqrt(math.fsum(a.tolist()))
    parts = []
    for lo in range(0, flat.size, _FSUM_CHUNK):
        blk = flat[lo:lo + _FSUM_CHUNK]
        a = np.abs(blk) ** 2 if np.iscomplexobj(blk) else blk * blk
        parts.append(math.fsum(a.tolist()))
    return math.sqrt(math.fsum(parts))


def make_tensor(cfg: SynthConfig, seed: int = 0) -> np.ndarray:
    """Y = X + sigma N (Fortran order), add_noise semantics of cpfast/synth.py:81-99."""
    x = reconstruct_exact(truth_factors(cfg, seed))
    ynorm = frob_exact(x)
    j = x.size
    sigma = ynorm / math.sqrt(j * 10.0 ** (cfg.snr_db / 10.0))
    rng = np.random.default_rng([seed, 1])
    noise = rng.standard_normal(cfg.dims)
    if cfg.complex_:
        noise = (noise + 1j * rng.standard_normal(cfg.dims)) / math.sqrt(2.0)
    return np.asfortranarray(x + sigma * noise)


def init_factors(cfg: SynthConfig, seed: int = 0) -> list:
    """The fit's own initial factors (random_init from default_rng([seed, 0]), kruskal.py:217-224)."""
    rng = np.random.default_rng([seed, 0])
    out = []
    for d in cfg.dims:
        a = rng.standard_normal((d, cfg.rank))
        if cfg.complex_:
            a = a + 1j * rng.standard_normal((d, cfg.rank))
        out.append(a)
    return out


def tau_for_unit_mu(cfg: SynthConfig, seed: int = 0) -> float:
    """tau giving mu0 = 1 (BASELINE's "mu0 = 1"): 1 / max(1, max Re diag C^(N)) of
    normalize_unit_modes(normalize_equal_energy(init)) -- computed from column norms."""
    init = init_factors(cfg, seed)
    n_modes = len(init)
    norms = np.array([[math.sqrt(math.fsum((np.abs(f[:, r]) ** 2).tolist())) for r in range(cfg.rank)]
                      for f in init])
    target = np.prod(norms, axis=0) ** (1.0 / n_modes)   # equal energy: every mode norm = target
    diag = (target ** n_modes) ** 2                      # unit modes 1..N-1, all magnitude in mode N
    return 1.0 / max(1.0, float(np.max(diag)))


def tensor_digest(y: np.ndarray) -> str:
    return hashlib.sha256(np.asfortranarray(y).tobytes(order="F")).hexdigest()[:16]


def device_tensor(cfg: SynthConfig, seed: int = 0, device="cuda", slab=None):
    """Build Y (or the mode-N slab [lo, hi)) directly on the GPU with torch (input synthesis only).

    X from the deterministic host truth factors; noise from torch's seeded generator (a different
    stream than numpy's -- used only for throughput runs, never for golden parity).
    """
    import torch

    fac = truth_factors(cfg, seed)
    dtype = torch.complex128 if cfg.complex_ else torch.float64
    lo, hi = slab if slab is not None else (0, cfg.dims[-1])
    ts = [torch.as_tensor(f, dtype=dtype, device=device) for f in fac]
    ts[-1] = ts[-1][lo:hi]
    # X stored column-major: build as reversed-dims C-order tensor = Fortran order of dims
    lead = 1
    for d in cfg.dims[:-1]:
        lead *= d
    # KR of modes 1..N-1 (mode 1 fastest): rows = lead, cols = R
    kr = ts[0]
    for t in ts[1:-1]:
        kr = (t[:, None, :] * kr[None, :, :]).reshape(-1, cfg.rank)
    y = torch.empty((hi - lo, lead), dtype=dtype, device=device)   # row c holds Y[:, ..., c] contiguous
    chunk = max(1, (1 << 27) // max(lead, 1))
    gen = torch.Generator(device=device)
    gen.manual_seed(int(seed) * 1000003 + 17)
    # ||X||^2 from the Grams (exact in exact arithmetic) for sigma
    grams = [f.conj().T @ f for f in [torch.as_tensor(a, dtype=dtype, device=device) for a in fac]]
    g = grams[0]
    for m in grams[1:]:
        g = g * m
    xnorm = float(torch.sqrt(g.sum().real))
    j = 1
    for d in cfg.dims:
        j *= d
    sigma = xnorm / math.sqrt(j * 10.0 ** (cfg.snr_db / 10.0))
    for c0 in range(0, hi - lo, chunk):
        c1 = min(hi - lo, c0 + chunk)
        blk = ts[-1][c0:c1] @ kr.T                 # (c, lead)
        if cfg.complex_:
            nr = torch.randn(blk.shape, generator=gen, device=device, dtype=torch.float64)
            ni = torch.randn(blk.shape, generator=gen, device=device, dtype=torch.float64)
            blk = blk + sigma * torch.complex(nr, ni) / math.sqrt(2.0)
        else:
            blk = blk + sigma * torch.randn(blk.shape, generator=gen, device=device, dtype=torch.float64)
        y[c0:c1] = blk
    return y   # memory layout == column-major Y slab
