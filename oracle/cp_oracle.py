"""CPU oracle for the fast damped Gauss-Newton (fLM) CP solver -- TEST INFRASTRUCTURE ONLY.

This module is a NumPy restatement of the reference package ``cpfast`` (the
pure-Python/NumPy implementation that accompanies arXiv:1205.2584).  It exists
for exactly three consumers:

* ``tests/``            -- the checker the CUDA path is compared against;
* ``__graft_entry__.smoke()`` -- a tiny on-GPU sanity check against this oracle;
* ``bench.py``          -- the ``cpu_baseline`` leg and the ``--impl reference`` arm
                           (the reference CPU algorithm timed on the host cores).

The product path (``paper_1205_2584_b200``) never imports anything from here.

Citations below are to ``/root/reference/pkg/src/cpfast/<file>.py:<line>``.
The arithmetic follows the reference call for call (same NumPy/LAPACK
operations in the same order: explicit ``inv`` for B, ``inv`` for the damped
Gamma blocks, direct residual norms) so that it reproduces the reference
trajectory to rounding level; ``tests/test_oracle_golden.py`` pins it against
golden traces captured from the reference itself (``tests/golden/``).

Layout conventions (reference ``tensor.py:1-6``, ``kruskal.py:70-72``): tensors
are column-major (mode-1 index fastest), factors are I_n x R and vectorise
column-major; modes are 1-based in the public helpers.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from functools import reduce

import numpy as np
import scipy.linalg

MU_OVERFLOW = 1e30          # solver.py:47
RHO_DENOM_GUARD = 1e-30     # solver.py:48
LM_VARIANTS = ("flm-a", "flm-b", "auto")


class OracleSingularKernel(np.linalg.LinAlgError):
    """Mirror of ``hessian.SingularKernelError`` (hessian.py:34-35)."""


# ----------------------------------------------------------------------------
# Tensor layout helpers (tensor.py)
# ----------------------------------------------------------------------------

def fortran_tensor(y) -> np.ndarray:
    """Column-major float64/complex128 copy policy of DenseTensor (tensor.py:45-55)."""
    data = getattr(y, "data", y)
    arr = np.asfortranarray(data)
    if arr.dtype not in (np.float64, np.complex128):
        arr = arr.astype(np.complex128 if np.iscomplexobj(arr) else np.float64)
    return arr


def unfold(y: np.ndarray, n: int) -> np.ndarray:
    """Mode-n unfolding, remaining modes ascending (tensor.py:81-86)."""
    moved = np.moveaxis(y, n - 1, 0)
    return moved.reshape((y.shape[n - 1], -1), order="F")


def fold(mat: np.ndarray, n: int, dims) -> np.ndarray:
    """Inverse of unfold (tensor.py:89-95)."""
    dims = tuple(int(d) for d in dims)
    shape = (dims[n - 1],) + dims[: n - 1] + dims[n:]
    return np.moveaxis(np.asarray(mat).reshape(shape, order="F"), 0, n - 1)


def khatri_rao_pair(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Column-wise Kronecker, a's row index slowest (tensor.py:111-121)."""
    return (a[:, None, :] * b[None, :, :]).reshape(a.shape[0] * b.shape[0], a.shape[1])


def khatri_rao_skip(factors, n: int) -> np.ndarray:
    """KR over modes N..1 skipping mode n (descending order, tensor.py:124-136)."""
    chain = [factors[k] for k in range(len(factors) - 1, -1, -1) if k != n - 1]
    return reduce(khatri_rao_pair, chain)


def commutation(i: int, j: int) -> np.ndarray:
    """P with P vec(X^T) = vec(X) for I x J X (tensor.py:153-162)."""
    size = i * j
    out = np.zeros((size, size))
    idx = np.arange(size)
    out[idx, (idx // i) + j * (idx % i)] = 1.0
    return out


# ----------------------------------------------------------------------------
# Kruskal-model kernels (kruskal.py)
# ----------------------------------------------------------------------------

def reconstruct(factors) -> np.ndarray:
    """Dense X from factors (weights are always None on the fit path; kruskal.py:85-89)."""
    dims = tuple(f.shape[0] for f in factors)
    # the reference scales mode 1 by the (unit) weights first; the product's memory layout
    # decides the BLAS path, so keep it for rounding-identical results
    a1 = factors[0] * np.ones(factors[0].shape[1], dtype=factors[0].dtype)[None, :]
    mat = a1 @ khatri_rao_skip(factors, 1).T
    return np.asfortranarray(fold(mat, 1, dims))   # DenseTensor(...) stores Fortran order


def relative_error(y: np.ndarray, factors) -> float:
    """||Y - X|| / ||Y|| with a full reconstruction (kruskal.py:159-167)."""
    y = fortran_tensor(y)
    ynorm = float(np.linalg.norm(y))
    if ynorm == 0.0:
        raise ZeroDivisionError("relative error undefined for a zero tensor")
    return float(np.linalg.norm(y - reconstruct(factors))) / ynorm


def mttkrp(y: np.ndarray, factors, n: int) -> np.ndarray:
    """M_n = Y_(n) conj(KR_{k!=n}) (kruskal.py:126-135)."""
    return unfold(y, n) @ khatri_rao_skip(factors, n).conj()


@dataclass
class Grams:
    """C^(n), Gamma^(n), Gamma^(n,m), Gamma (kruskal.py:92-123)."""

    C: list
    excl: list
    pair: list
    full: np.ndarray


def gram_cache(factors) -> Grams:
    """Gram matrices and their Hadamard products (kruskal.py:107-123)."""
    nm = len(factors)
    rank = factors[0].shape[1]
    C = [a.conj().T @ a for a in factors]

    def hadamard_without(skip):
        kept = [C[k] for k in range(nm) if k not in skip]
        return reduce(np.multiply, kept) if kept else np.ones((rank, rank), dtype=C[0].dtype)

    excl = [hadamard_without({n}) for n in range(nm)]
    pair = [[excl[n] if n == m else hadamard_without({n, m}) for m in range(nm)] for n in range(nm)]
    return Grams(C, excl, pair, hadamard_without(set()))


def normalize_equal_energy(factors) -> list:
    """Equal per-mode column energy, phase folded into the last mode (kruskal.py:170-198)."""
    out = [np.asarray(a).copy() for a in factors]  # C-order copies, as ndarray.copy()
    nm = len(out)
    rank = out[0].shape[1]
    weights = np.ones(rank, dtype=out[0].dtype)
    for r in range(rank):
        norms = np.array([np.linalg.norm(a[:, r]) for a in out])
        if np.any(norms == 0.0):
            raise ZeroDivisionError(f"component {r} has a zero-norm vector")
        target = (np.abs(weights[r]) * np.prod(norms)) ** (1.0 / nm)
        wphase = weights[r] / np.abs(weights[r]) if weights[r] != 0 else 1.0
        for n in range(nm):
            out[n][:, r] *= target / norms[n]
        out[-1][:, r] *= wphase
        if nm >= 2:
            lead = out[0][:, r]
            top = lead[np.argmax(np.abs(lead))]
            phase = top / np.abs(top) if top != 0 else 1.0
            out[0][:, r] /= phase
            out[-1][:, r] *= phase
    return out


def normalize_unit_modes(factors) -> list:
    """Unit columns in modes 1..N-1, magnitude moved to mode N (kruskal.py:201-214)."""
    out = [np.asarray(a).copy() for a in factors]  # C-order copies, as ndarray.copy()
    rank = out[0].shape[1]
    for r in range(rank):
        scale = 1.0
        for n in range(len(out) - 1):
            nrm = np.linalg.norm(out[n][:, r])
            if nrm == 0.0:
                raise ZeroDivisionError(f"component {r} has a zero-norm vector")
            out[n][:, r] /= nrm
            scale = scale * nrm
        out[-1][:, r] *= scale
    return out


def random_init(dims, rank: int, rng, is_complex: bool) -> list:
    """N(0,1) factors, complex = re + i*im drawn per factor (kruskal.py:217-224)."""
    out = []
    for d in dims:
        a = rng.standard_normal((d, rank))
        if is_complex:
            a = a + 1j * rng.standard_normal((d, rank))
        out.append(a)
    return out


def stack(factors) -> np.ndarray:
    """Concatenated column-major vectorisations (kruskal.py:70-72)."""
    return np.concatenate([a.reshape(-1, order="F") for a in factors])


def unstack(vec: np.ndarray, dims, rank: int) -> list:
    """Inverse of ``stack`` (kruskal.py:75-82)."""
    out, off = [], 0
    for d in dims:
        out.append(np.asarray(vec[off: off + d * rank]).reshape((d, rank), order="F"))
        off += d * rank
    return out


def gradient_from_mttkrps(factors, g: Grams, M) -> np.ndarray:
    """g_n = vec(M_n - A^(n) Gamma^(n)^T) (solver.py:251-256, kruskal.py:138-156)."""
    return np.concatenate([(M[n] - factors[n] @ g.excl[n].T).reshape(-1, order="F")
                           for n in range(len(factors))])


# ----------------------------------------------------------------------------
# Hessian structure (hessian.py)
# ----------------------------------------------------------------------------

def kernel_is_invertible(g: Grams, rtol: float = 1e-10) -> bool:
    """Magnitude proxy over the off-diagonal Gamma^(n,m) (hessian.py:81-94)."""
    nm = len(g.C)
    mags = [np.abs(g.pair[n][m]) for n in range(nm) for m in range(nm) if n != m]
    top = max(x.max() for x in mags)
    if top == 0.0:
        return False
    return all(x.min() > rtol * top for x in mags)


def kernel_matrix(g: Grams) -> np.ndarray:
    """K with blocks (1-delta) P_R diag(vec Gamma^(n,m)) (hessian.py:62-78)."""
    nm = len(g.C)
    r = g.full.shape[0]
    p = commutation(r, r)
    rows = []
    for n in range(nm):
        row = []
        for m in range(nm):
            if n == m:
                row.append(np.zeros((r * r, r * r), dtype=g.full.dtype))
            else:
                row.append(p * g.pair[n][m].reshape(-1, order="F")[None, :])
        rows.append(row)
    return np.block(rows)


def kernel_inverse(g: Grams) -> np.ndarray:
    """Closed-form K^{-1}: (1/(N-1) - delta) diag(vec(C_n*C_m/Gamma)) P_R (hessian.py:97-119)."""
    nm = len(g.C)
    if nm < 2:
        raise ValueError("kernel inverse needs at least two modes")
    if not kernel_is_invertible(g):
        raise OracleSingularKernel("a pairwise Gamma entry vanishes; K is singular")
    r = g.full.shape[0]
    p = commutation(r, r)
    rows = []
    for n in range(nm):
        row = []
        for m in range(nm):
            coeff = 1.0 / (nm - 1) - (1.0 if n == m else 0.0)
            d = (g.C[n] * g.C[m] / g.full).reshape(-1, order="F")
            row.append(coeff * d[:, None] * p)
        rows.append(row)
    return np.block(rows)


def psi_diag_blocks(g: Grams, mu: float) -> list:
    """(Gamma^(n) + mu I)^{-1} kron C^(n) -- NOT transposed (hessian.py:185-193)."""
    r = g.full.shape[0]
    return [np.kron(np.linalg.inv(g.excl[n] + mu * np.eye(r)), g.C[n]) for n in range(len(g.C))]


def b_core(g: Grams, mu: float, use_kernel_inverse: bool) -> np.ndarray:
    """B_mu = (K^{-1} + Psi)^{-1}  or  K (I + Psi K)^{-1} (hessian.py:196-211)."""
    psi = scipy.linalg.block_diag(*psi_diag_blocks(g, mu))
    k = kernel_matrix(g)
    eye = np.eye(k.shape[0])
    if use_kernel_inverse:
        return np.linalg.inv(kernel_inverse(g) + psi)
    try:
        return k @ np.linalg.solve(eye + psi @ k, eye)
    except np.linalg.LinAlgError as exc:
        raise OracleSingularKernel(f"I + Psi K numerically singular: {exc}")


def fast_damped_inverse(factors, mu: float, use_kernel_inverse=None):
    """(gamma_tilde list, core grid D) of the structured (H + mu I)^{-1} (hessian.py:232-277):
    K^{-1} path D = inv(Sb K~ Sb + blkdiag((Gamma_n + mu I) kron C_n)); K-free path
    D = blkdiag(Gt kron I) K solve(Sb + Chat K, I)."""
    if mu <= 0:
        raise ValueError("mu must be positive")
    g = gram_cache(factors)
    if use_kernel_inverse is None:
        use_kernel_inverse = kernel_is_invertible(g)
    r = g.full.shape[0]
    eye = np.eye(r)
    gamma_tilde = [np.linalg.inv(x + mu * eye) for x in g.excl]
    damped = [g.excl[n] + mu * eye for n in range(len(factors))]
    sb = scipy.linalg.block_diag(*[np.kron(x, eye) for x in damped])
    if use_kernel_inverse:
        diag = scipy.linalg.block_diag(*[np.kron(x, c) for x, c in zip(damped, g.C)])
        d = np.linalg.inv(sb @ kernel_inverse(g) @ sb + diag)
    else:
        chat = scipy.linalg.block_diag(*[np.kron(eye, c) for c in g.C])
        k = kernel_matrix(g)
        gt = scipy.linalg.block_diag(*[np.kron(x, eye) for x in gamma_tilde])
        try:
            d = gt @ k @ np.linalg.solve(sb + chat @ k, np.eye(k.shape[0]))
        except np.linalg.LinAlgError as exc:
            raise OracleSingularKernel(f"Sb + Chat K numerically singular: {exc}")
    return gamma_tilde, d


def materialize_inverse(gamma_tilde, core, factors) -> np.ndarray:
    """Dense (H + mu I)^{-1} from the block form (hessian.py:278-297; test scaffolding)."""
    r = gamma_tilde[0].shape[0]
    r2 = r * r
    nm = len(factors)
    eye_r = np.eye(r)
    rows = []
    for n in range(nm):
        row = []
        for m in range(nm):
            zn = np.kron(eye_r, factors[n])
            zm = np.kron(eye_r, factors[m])
            block = -zn @ core[n * r2:(n + 1) * r2, m * r2:(m + 1) * r2] @ zm.conj().T
            if n == m:
                block = block + np.kron(gamma_tilde[n], np.eye(factors[n].shape[0]))
            row.append(block)
        rows.append(row)
    return np.block(rows)


def core_matrix(g: Grams, mu: float, variant: str) -> np.ndarray:
    """Variant dispatch (solver.py:143-148)."""
    if variant == "auto":
        variant = "flm-b" if kernel_is_invertible(g) else "flm-a"
    if variant == "flm-b" and not kernel_is_invertible(g):
        raise OracleSingularKernel("flm-b requested but K is singular")
    return b_core(g, mu, variant == "flm-b")


def _blocks(vec: np.ndarray, factors) -> list:
    out, off = [], 0
    for a in factors:
        out.append(vec[off: off + a.size].reshape(a.shape, order="F"))
        off += a.size
    return out


def apply_damped_hessian(g: Grams, factors, vec: np.ndarray, mu: float) -> np.ndarray:
    """(H + mu I) v through G + Z K Z^H (hessian.py:311-326)."""
    x = _blocks(vec, factors)
    w = [a.conj().T @ xn for a, xn in zip(factors, x)]
    out = []
    for n in range(len(factors)):
        acc = x[n] @ g.excl[n].T + mu * x[n]
        terms = [(g.pair[n][m] * w[m]).T for m in range(len(factors)) if m != n]
        if terms:
            acc = acc + factors[n] @ sum(terms)
        out.append(acc.reshape(-1, order="F"))
    return np.concatenate(out)


def apply_damped_inverse(g: Grams, factors, b: np.ndarray, vec: np.ndarray, mu: float) -> np.ndarray:
    """(H + mu I)^{-1} v by the binomial inverse with core B (hessian.py:329-348)."""
    r = g.full.shape[0]
    x = _blocks(vec, factors)
    gti = [np.linalg.inv(e.T + mu * np.eye(r)) for e in g.excl]
    t = [xn @ gi for xn, gi in zip(x, gti)]
    wv = np.concatenate([(a.conj().T @ tn).reshape(-1, order="F") for a, tn in zip(factors, t)])
    yv = b @ wv
    r2 = r * r
    out = []
    for n in range(len(factors)):
        yn = yv[n * r2:(n + 1) * r2].reshape((r, r), order="F")
        out.append((t[n] - factors[n] @ yn @ gti[n]).reshape(-1, order="F"))
    return np.concatenate(out)


# ----------------------------------------------------------------------------
# fLM step (solver.py)
# ----------------------------------------------------------------------------

def damped_factor(M_n: np.ndarray, g: Grams, n0: int, mu: float) -> np.ndarray:
    """A_mu^(n) = M_n (Gamma^(n)^T + mu I)^{-1} (solver.py:107-119); n0 is 0-based."""
    r = M_n.shape[1]
    return M_n @ np.linalg.inv(g.excl[n0].T + mu * np.eye(r))


def projected_residual(factors, g: Grams, damped, mu: float) -> np.ndarray:
    """w blocks vec(A^H A_mu - C Gamma^T (Gamma^T + mu I)^{-1}) (solver.py:122-140)."""
    r = factors[0].shape[1]
    parts = []
    for n in range(len(factors)):
        gt = g.excl[n].T
        gti = np.linalg.inv(gt + mu * np.eye(r))
        parts.append((factors[n].conj().T @ damped[n] - g.C[n] @ gt @ gti).reshape(-1, order="F"))
    return np.concatenate(parts)


def frontal_slices(f: np.ndarray, nm: int, r: int) -> list:
    """F_n = reshape_F(f block n) (solver.py:151-156)."""
    return [f[n * r * r:(n + 1) * r * r].reshape((r, r), order="F") for n in range(nm)]


def factored_update(factors, damped, F, g: Grams, mu: float) -> list:
    """A_mu + A (I - (F_n + Gamma^T) (Gamma^T + mu I)^{-1}) (solver.py:172-186)."""
    r = factors[0].shape[1]
    eye = np.eye(r)
    out = []
    for n in range(len(factors)):
        gt = g.excl[n].T
        gti = np.linalg.inv(gt + mu * eye)
        out.append(damped[n] + factors[n] @ (eye - (F[n] + gt) @ gti))
    return out


def flm_candidate(factors, mu: float, variant: str, g: Grams, M, refine_steps: int = 2,
                  y: np.ndarray | None = None) -> list:
    """One fLM candidate with structured refinement (solver.py:189-226)."""
    if g is None:
        g = gram_cache(factors)
    if M is None:
        M = [mttkrp(y, factors, n) for n in range(1, len(factors) + 1)]
    nm = len(factors)
    r = factors[0].shape[1]
    damped = [damped_factor(M[n], g, n, mu) for n in range(nm)]
    w = projected_residual(factors, g, damped, mu)
    b = core_matrix(g, mu, variant)
    F = frontal_slices(b @ w, nm, r)
    cand = factored_update(factors, damped, F, g, mu)
    if refine_steps:
        grad = gradient_from_mttkrps(factors, g, M)
        base = stack(factors)
        delta = stack(cand) - base
        for _ in range(refine_steps):
            resid = grad - apply_damped_hessian(g, factors, delta, mu)
            delta = delta + apply_damped_inverse(g, factors, b, resid, mu)
        cand = unstack(base + delta, [a.shape[0] for a in factors], r)
    return cand


def mu_initial(g_unit: Grams, tau: float) -> float:
    """tau * max(1, max Re diag C^(N)) (solver.py:229-235)."""
    return float(tau * max(1.0, np.max(np.real(np.diag(g_unit.C[-1])))))


def nielsen(mu: float, growth: float, rho: float):
    """Nielsen gain-ratio schedule (solver.py:238-248) -> (mu, growth, accepted)."""
    if rho > 0:
        return mu * max(1.0 / 3.0, 1.0 - (2.0 * rho - 1.0) ** 3), 2.0, True
    return mu * growth, 2.0 * growth, False


def gain_ratio(prev_sq: float, cand_sq: float, delta: np.ndarray, grad: np.ndarray, mu: float,
               sign: float = 1.0) -> float:
    """rho = (prev - cand) / Re<delta, g + mu delta> with the 1e-30 guard (solver.py:259-263).
    ``sign = -1`` is a test hook (negated denominator, see OracleConfig.negate_denom_at)."""
    denom = sign * np.real(np.vdot(delta, grad + mu * delta))
    if abs(denom) < RHO_DENOM_GUARD:
        return -1.0
    return (prev_sq - cand_sq) / denom


# ----------------------------------------------------------------------------
# The LM loop (solver.py:278-291, 319-384)
# ----------------------------------------------------------------------------

@dataclass
class OracleConfig:
    """Same fields/defaults as FitConfig (solver.py:62-76); only the LM variants."""

    rank: int
    variant: str = "auto"
    tau: float = 1e-3
    tol: float = 1e-8
    max_iters: int = 1000
    seed: int = 0
    init: str = "random"
    # test hook, not reference behaviour: negate the gain-ratio denominator at this iteration so a
    # worse candidate gets rho > 0 -- the "rho > 0 but cand_err >= err" rejection of solver.py:361
    # (mirrors the engine's CPF_TEST_NEGDENOM)
    negate_denom_at: int = 0


@dataclass
class OracleResult:
    factors: list
    trace: list                      # (iter, relerr, mu, accepted)
    stop_reason: str
    time_ms: float = 0.0
    detail: list = field(default_factory=list)   # per-iteration (err_sq, cand_sq, rho, denom)

    @property
    def iters(self) -> int:
        return len(self.trace)

    @property
    def accepted(self) -> str:
        return "".join("A" if t[3] else "r" for t in self.trace)

    @property
    def final_relerr(self) -> float:
        return self.trace[-1][1] if self.trace else float("nan")


def fit_lm(y, cfg: OracleConfig, init_factors=None, on_iter=None, phases=None) -> OracleResult:
    """The damped Gauss-Newton loop, semantics of solver.py:319-384 (Appendix A of SURVEY).

    ``phases`` (bench.py's CPU reference arm): a list that receives, per iteration, the seconds spent
    in the J-independent step (candidate, gradient, decision) and in the tensor-sized work
    (relative_error of the candidate, and on accept the N MTTKRPs) -- the split bench.py uses to
    extrapolate a bounded slab sample to the full tensor.  It does not change the arithmetic."""
    t0 = time.monotonic()
    y = fortran_tensor(y)
    if cfg.variant not in LM_VARIANTS:
        raise ValueError(f"oracle covers the LM variants only, got {cfg.variant!r}")
    rng = np.random.default_rng([cfg.seed, 0])
    if init_factors is not None:
        start = [np.array(a, copy=True) for a in init_factors]
    elif cfg.init == "random":
        start = random_init(y.shape, cfg.rank, rng, np.iscomplexobj(y))
    else:
        raise ValueError(f"oracle supports init='random' only, got {cfg.init!r}")
    A = normalize_equal_energy(start)
    ynorm = float(np.linalg.norm(y))
    if ynorm == 0.0:
        raise ZeroDivisionError("cannot fit a zero tensor")
    mu = mu_initial(gram_cache(normalize_unit_modes(A)), cfg.tau)
    growth = 2.0
    g = gram_cache(A)
    M = [mttkrp(y, A, n) for n in range(1, len(A) + 1)]
    err = relative_error(y, A)
    err_sq = (err * ynorm) ** 2
    trace, deltas, detail = [], [], []
    stop = "max_iters"
    if on_iter is not None:
        on_iter(0)
    clock = time.perf_counter
    for t in range(1, cfg.max_iters + 1):
        c0 = clock()
        try:
            cand = flm_candidate(A, mu, cfg.variant, g, M)
        except np.linalg.LinAlgError as exc:
            return OracleResult(A, trace, f"error at iteration {t}: {exc}",
                                (time.monotonic() - t0) * 1e3, detail)
        delta = stack(cand) - stack(A)
        c1 = clock()
        cand_err = relative_error(y, cand)
        c2 = clock()
        t_tensor = c2 - c1
        cand_sq = (cand_err * ynorm) ** 2
        grad = gradient_from_mttkrps(A, g, M)
        rho = gain_ratio(err_sq, cand_sq, delta, grad, mu, -1.0 if t == cfg.negate_denom_at else 1.0)
        mu, growth, ok = nielsen(mu, growth, rho)
        detail.append((err_sq, cand_sq, rho))
        if ok and cand_err < err:
            A = normalize_equal_energy(cand)
            g = gram_cache(A)
            c3 = clock()
            M = [mttkrp(y, A, n) for n in range(1, len(A) + 1)]
            t_tensor += clock() - c3
            deltas.append(abs(err - cand_err))
            err, err_sq = cand_err, cand_sq
            accepted = True
        else:
            deltas.append(0.0)
            accepted = False
        trace.append((t, err, mu, accepted))
        if phases is not None:
            total = clock() - c0
            phases.append((total - t_tensor, t_tensor))
        if on_iter is not None:
            on_iter(t)
        if len(deltas) >= 10 and all(d < cfg.tol for d in deltas[-10:]):
            stop = "tol"
            break
        if mu > MU_OVERFLOW:
            stop = "mu_overflow"
            break
    return OracleResult(A, trace, stop, (time.monotonic() - t0) * 1e3, detail)


# ----------------------------------------------------------------------------
# ALS baselines (kruskal.py:245-293, solver.py:294-316)
# ----------------------------------------------------------------------------

def pinv_psd(gamma: np.ndarray) -> np.ndarray:
    """Eigen-decomposition pseudo-inverse, eigenvalues <= eps R lambda_max dropped (kruskal.py:245-254)."""
    w, v = np.linalg.eigh(gamma)
    r = gamma.shape[0]
    cutoff = np.finfo(np.float64).eps * r * max(w.max(initial=0.0), 0.0)
    inv_w = np.where(w > cutoff, 1.0 / np.where(w > cutoff, w, 1.0), 0.0)
    return (v * inv_w[None, :]) @ v.conj().T


def als_step(y: np.ndarray, factors) -> list:
    """One sweep in ascending mode order, A_n = M_n pinv_psd(Gamma^(n))^T (kruskal.py:257-265)."""
    out = [np.asarray(a).copy() for a in factors]
    for n in range(len(out)):
        g = gram_cache(out)
        out[n] = mttkrp(y, out, n + 1) @ pinv_psd(g.excl[n]).T
    return out


def als_line_search_step(y: np.ndarray, factors, history, t: int = 1) -> list:
    """Sweep, then A_prev + s (A_als - A_prev) for s in {1.1, t^(1/3)}, best relative error
    (kruskal.py:268-293); plain sweep without history."""
    stepped = als_step(y, factors)
    if history is None:
        return stepped
    best, best_err = stepped, relative_error(y, stepped)
    for s in (1.1, float(t) ** (1.0 / 3.0)):
        cand = [hp + s * (ha - hp) for hp, ha in zip(history, stepped)]
        err = relative_error(y, cand)
        if err < best_err:
            best, best_err = cand, err
    return best


def fit_als(y, cfg: "OracleConfig", init_factors=None) -> "OracleResult":
    """_fit_als (solver.py:294-316): relative error recorded per sweep, mu = 0, every step
    "accepted"; stop on the 10-delta tolerance window."""
    t0 = time.monotonic()
    y = fortran_tensor(y)
    rng = np.random.default_rng([cfg.seed, 0])
    if init_factors is not None:
        model = [np.array(a, copy=True) for a in init_factors]
    elif cfg.init == "random":
        model = random_init(y.shape, cfg.rank, rng, np.iscomplexobj(y))
    else:
        raise ValueError(f"oracle supports init='random' only, got {cfg.init!r}")
    err = relative_error(y, model)
    trace, deltas = [], []
    history = None
    stop = "max_iters"
    for t in range(1, cfg.max_iters + 1):
        prev = model
        if cfg.variant == "als-ls":
            model = als_line_search_step(y, model, history, t)
        else:
            model = als_step(y, model)
        history = prev
        new_err = relative_error(y, model)
        trace.append((t, new_err, 0.0, True))
        deltas.append(abs(err - new_err))
        err = new_err
        if len(deltas) >= 10 and all(d < cfg.tol for d in deltas[-10:]):
            stop = "tol"
            break
    return OracleResult(model, trace, stop, (time.monotonic() - t0) * 1e3, [])


# ----------------------------------------------------------------------------
# Dense dGN oracle (hessian.py:46-60, 122-148, 175-182) for step equivalence
# ----------------------------------------------------------------------------

def _mode_commutation(dims, n: int) -> np.ndarray:
    lead = int(np.prod(dims[: n - 1], dtype=np.int64))
    trail = int(np.prod(dims[n:], dtype=np.int64))
    return np.kron(np.eye(trail), commutation(lead, dims[n - 1]))


def jacobian(factors) -> np.ndarray:
    dims = tuple(a.shape[0] for a in factors)
    cols = []
    for n in range(1, len(factors) + 1):
        w = khatri_rao_skip(factors, n)
        cols.append(_mode_commutation(dims, n) @ np.kron(w, np.eye(dims[n - 1])))
    return np.hstack(cols)


def dense_damped_step(y: np.ndarray, factors, mu: float) -> np.ndarray:
    """Solve (J^H J + mu I) d = J^H vec(Y - X) densely (desk-scale only)."""
    y = fortran_tensor(y)
    j = jacobian(factors)
    resid = (y - reconstruct(factors)).reshape(-1, order="F")
    h = j.conj().T @ j
    return np.linalg.solve(h + mu * np.eye(h.shape[0]), j.conj().T @ resid)
