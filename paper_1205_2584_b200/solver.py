"""Drop-in fast damped Gauss-Newton (fLM) CP solver entry points, executed by the B200 engine.

Mirrors ``cpfast.solver`` (cpfast/solver.py) and ``cpfast.complexcp`` (cpfast/complexcp.py):
``FitConfig`` / ``IterRecord`` / ``FitResult`` have the same fields, defaults and validation;
``fit`` / ``fit_complex`` / ``flm_step`` / ``mttkrp`` / ``relative_error`` have the same arguments,
return types and error behaviour.  Every numerical step runs in hand-written sm_100a kernels
behind the C ABI (include/cpfast_b200.h); the host only draws the seeded initial factors
(bit-identical to the reference's ``default_rng([seed, 0])`` stream, kruskal.py:217-224) and
assembles the result.  There is no CPU fallback.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .tensor import COMPLEX, REAL, DenseTensor, KruskalModel, as_dense, as_model, model_from_vector, require_same_kind

VARIANTS = ("flm-a", "flm-b", "auto", "als", "als-ls", "dgn-oracle")   # solver.py:44
LM_VARIANTS = ("flm-a", "flm-b", "auto")
MU_OVERFLOW = 1e30                                                       # solver.py:47
RHO_DENOM_GUARD = 1e-30                                                  # solver.py:48
# iterations per fit_step call: the engine polls its device-side stop flag every 4 graph replays
# internally, so a fixed-length fit (tol = 0) runs in one call; with a tolerance, one call per
# iteration keeps the trace exact without gated replays after the stop
POLL_EVERY = 1
_TIMING = bool(__import__("os").environ.get("CPF_FIT_TIMING"))


@dataclass
class FitConfig:
    """Same fields, defaults and validation as cpfast.solver.FitConfig (solver.py:62-76)."""

    rank: int
    variant: str = "auto"
    tau: float = 1e-3
    tol: float = 1e-8
    max_iters: int = 1000
    seed: int = 0
    init: str = "svd"

    def __post_init__(self):
        if self.variant not in VARIANTS:
            raise ValueError(f"unknown variant {self.variant!r}")
        if self.rank < 1:
            raise ValueError("rank must be >= 1")


@dataclass
class IterRecord:
    iter: int
    relerr: float
    mu: float
    accepted: bool


@dataclass
class FitResult:
    model: KruskalModel
    trace: list
    stop_reason: str
    time_ms: float = 0.0
    launches: int = field(default=0, repr=False)
    # engine diagnostics (no reference counterpart): tensor-pass implementation (_native.PASS_*),
    # int8-pass launches that ran in fp64 under the accuracy guard, tensor rejected by the guard
    pass_impl: int = field(default=-1, repr=False)
    pass_fallbacks: int = field(default=0, repr=False)
    tensor_guarded: bool = field(default=False, repr=False)

    @property
    def iters(self) -> int:
        return len(self.trace)

    @property
    def accepted_iters(self) -> int:
        return sum(1 for rec in self.trace if rec.accepted)

    @property
    def final_relerr(self) -> float:
        return self.trace[-1].relerr if self.trace else float("nan")


def _kind_code(arr) -> int:
    return _native.CPF_COMPLEX if np.iscomplexobj(arr) else _native.CPF_REAL


def random_init(dims, rank: int, rng, scalar_kind: str = "real") -> KruskalModel:
    """N(0,1) factors drawn exactly like kruskal.py:217-224 (host RNG, bit-identical)."""
    factors = []
    for d in dims:
        a = rng.standard_normal((d, rank))
        if scalar_kind == COMPLEX:
            a = a + 1j * rng.standard_normal((d, rank))
        factors.append(a)
    return KruskalModel(factors)


class _Dims:
    """dims + scalar kind of the (possibly sharded) tensor, for the host-side init draw."""

    def __init__(self, dims, kind):
        self.dims, self.scalar_kind = tuple(dims), kind


def _init_model(y, config: FitConfig, rng, eng=None) -> KruskalModel:
    if config.init == "random":
        return random_init(y.dims, config.rank, rng, y.scalar_kind)
    if config.init == "svd":
        if eng is None:
            raise ValueError("init='svd' needs the tensor bound to the engine")
        return svd_init(eng, y.dims, config.rank, rng, y.scalar_kind)
    raise ValueError(f"unknown init {config.init!r}")


def _eigh_descending(g: np.ndarray):
    """Eigen-decomposition of a small Hermitian unfolding Gram on the GPU (cuSOLVER syevd/heevd
    through torch -- library code, off the per-iteration path; the Gram itself is formed by the
    engine); eigenvalues descending.  No CPU fallback: without a CUDA device this raises."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("init='svd' needs a CUDA device (the engine has no CPU fallback)")
    w, v = torch.linalg.eigh(torch.from_numpy(np.ascontiguousarray(g)).cuda())
    w, v = w.cpu().numpy(), v.cpu().numpy()
    return w[::-1], v[:, ::-1]


def svd_init(eng, dims, rank: int, rng, scalar_kind: str = "real") -> KruskalModel:
    """Leading mode-n left singular vectors (kruskal.py:227-242), computed as the leading
    eigenvectors of the unfolding Gram Y_(n) Y_(n)^H formed on the GPU (cpf_engine_unfolding_gram);
    extra columns (R > rank of the unfolding) are unit-norm draws from ``rng`` exactly as in the
    reference.  Singular vectors are only defined up to sign/phase: each column is normalised so its
    largest-magnitude entry is real positive (LAPACK's gesdd convention is implementation-defined)."""
    total = int(np.prod(dims, dtype=np.int64))
    factors = []
    for n, d in enumerate(dims):
        g = eng.unfolding_gram(n + 1)
        g = 0.5 * (g + g.conj().T)
        _, v = _eigh_descending(g)
        k = min(rank, d, total // d)
        u = np.array(v[:, :k])
        for r in range(k):
            top = u[np.argmax(np.abs(u[:, r])), r]
            u[:, r] = u[:, r] / (top / abs(top))
        cols = [u]
        if k < rank:
            extra = rng.standard_normal((d, rank - k))
            if scalar_kind == COMPLEX:
                extra = extra + 1j * rng.standard_normal(extra.shape)
            extra = extra / np.linalg.norm(extra, axis=0, keepdims=True)
            cols.append(extra.astype(u.dtype))
        dtype = np.complex128 if scalar_kind == COMPLEX else np.float64
        factors.append(np.hstack(cols).astype(dtype))
    return KruskalModel(factors)


def _stop_reason(st) -> str:
    if st.stopped == _native.STOP_TOL:
        return "tol"
    if st.stopped == _native.STOP_MU_OVERFLOW:
        return "mu_overflow"
    if st.stopped == _native.STOP_ERROR:
        return f"error at iteration {st.err_iter}: {_native.ERR_MESSAGE.get(st.err_code, 'numerical error')}"
    return "max_iters"


class _Dist:
    """Slab-sharding context for multi-GPU fits (one process per GPU, torch.distributed group)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def unique_id(self) -> bytes:
        obj = [_native.nccl_unique_id() if self.rank == 0 else None]
        self.dist.broadcast_object_list(obj, src=0, group=self.group)
        return obj[0]


class LoopbackRank:
    """``distributed=`` handle of the loopback TEST transport: rank ``rank`` of a
    ``_native.LoopbackGroup`` -- several ranks' engines in one process on one GPU, each fit driven
    from its own thread, exchanging through device buffers (include/cpfast_b200.h)."""

    def __init__(self, group, rank: int):
        self.group, self.rank, self.world = group, int(rank), group.world


def _engine_for(kind: int, dims, rank: int, dev: int, distributed):
    if distributed is None:
        return _native.Engine(kind, dims, rank, dev)
    if isinstance(distributed, LoopbackRank):
        return _native.Engine(kind, dims, rank, dev, distributed.rank, distributed.world, loopback=distributed.group)
    ctx = distributed if isinstance(distributed, _Dist) else _Dist(distributed if distributed is not True else None)
    uid = ctx.unique_id() if ctx.world > 1 else None
    return _native.Engine(kind, dims, rank, dev, ctx.rank, ctx.world, uid)


def slab_bounds(dim_n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous slab of the last mode owned by ``rank`` (ceil split, same rule as the engine)."""
    per = -(-dim_n // world)
    lo = min(dim_n, per * rank)
    return lo, min(dim_n, lo + per)


def _make_engine(y: DenseTensor, rank: int, device, distributed, slab_of=None):
    dims = y.dims if slab_of is None else tuple(y.dims[:-1]) + (int(slab_of),)
    if len(dims) < 2:
        raise ValueError("the fLM solver needs a tensor of order >= 2")
    dev = 0 if device is None else int(device)
    eng = _engine_for(_kind_code(y.data), dims, rank, dev, distributed)
    lo, hi = eng.slab
    if slab_of is None:
        eng.set_tensor_host(y.data[..., lo:hi])
    else:
        if y.dims[-1] != hi - lo:
            raise ValueError(f"local slab has {y.dims[-1]} slices, this rank owns [{lo}, {hi})")
        eng.set_tensor_host(y.data)
    return eng


ALS_VARIANTS = ("als", "als-ls")


def _check_lm(config: FitConfig):
    if config.variant not in LM_VARIANTS + ALS_VARIANTS:
        raise ValueError(f"variant {config.variant!r} is not supported on the B200 backend "
                         "(the fast damped Gauss-Newton variants 'auto', 'flm-a', 'flm-b' and the "
                         "ALS baselines 'als', 'als-ls')")
    if config.init not in ("svd", "random"):
        raise ValueError(f"unknown init {config.init!r}")


def _stop_on_tol(err_deltas, tol) -> bool:
    """solver.py:274-275."""
    return len(err_deltas) >= 10 and all(d < tol for d in err_deltas[-10:])


def _run_als(eng, gdims, scalar_kind: str, config: FitConfig, rng) -> FitResult:
    """_fit_als (solver.py:294-316) on an engine whose tensor is bound: every sweep, line search
    and relative error runs on the device (cpf_engine_als_step); the host keeps the reference's
    10-delta tolerance window.  Closes the engine."""
    try:
        init = _init_model(_Dims(gdims, scalar_kind), config, rng, eng)
        eng.set_factors(init.as_vector())
        err = eng.relative_error()
        trace, deltas = [], []
        stop_reason = "max_iters"
        line_search = config.variant == "als-ls"
        for t in range(1, config.max_iters + 1):
            new_err = eng.als_step(line_search, t)
            trace.append(IterRecord(t, new_err, 0.0, True))
            deltas.append(abs(err - new_err))
            err = new_err
            if _stop_on_tol(deltas, config.tol):
                stop_reason = "tol"
                break
        model = model_from_vector(eng.get_factors(), gdims, config.rank)
        fallbacks, rejected = eng.pass_guard()
        result = FitResult(model, trace, stop_reason, launches=eng.launch_count(), pass_impl=eng.pass_impl(),
                           pass_fallbacks=fallbacks, tensor_guarded=rejected)
    finally:
        eng.close()
    return result


def _run_fit(eng, gdims, scalar_kind: str, config: FitConfig, rng) -> FitResult:
    """The LM loop on an engine whose tensor is bound (solver.py:319-384); closes the engine.
    ALS variants go to _run_als (solver.py:285-288 dispatch)."""
    if config.variant in ALS_VARIANTS:
        return _run_als(eng, gdims, scalar_kind, config, rng)
    try:
        tt = [time.monotonic()]
        init = _init_model(_Dims(gdims, scalar_kind), config, rng, eng)
        eng.set_factors(init.as_vector())
        tt.append(time.monotonic())
        st = eng.fit_begin(config.variant, config.tau, config.tol, config.max_iters)
        tt.append(time.monotonic())
        first = True
        while st.stopped == _native.STOP_RUNNING:
            st = eng.fit_step(config.max_iters if config.tol == 0.0 else max(1, min(POLL_EVERY, config.max_iters)))
            if first:
                tt.append(time.monotonic())
                first = False
        tt.append(time.monotonic())
        recs = eng.trace(config.max_iters)
        if _TIMING:
            import sys as _sys

            _sys.stderr.write("[fit timing] init %.1f | fit_begin (upload wait + preamble) %.1f | first step "
                              "(graph capture) %.1f | remaining steps %.1f ms\n"
                              % tuple(1e3 * (tt[i + 1] - tt[i]) for i in range(len(tt) - 1))
                              if len(tt) == 5 else "")
        trace = [IterRecord(t, e, m, a) for (t, e, m, a) in recs]
        model = model_from_vector(eng.get_factors(), gdims, config.rank)
        fallbacks, rejected = eng.pass_guard()
        result = FitResult(model, trace, _stop_reason(st), launches=eng.launch_count(), pass_impl=eng.pass_impl(),
                           pass_fallbacks=fallbacks, tensor_guarded=rejected)
        if st.stopped == _native.STOP_ERROR and st.err_code == _native.ERR_ZERO_COLUMN:
            raise ZeroDivisionError("a component of the accepted candidate has a zero-norm vector")
    finally:
        eng.close()
    return result


def fit(y, config: FitConfig, *, device=None, distributed=None, slab_of=None) -> FitResult:
    """Decompose ``y`` with the fLM damped Gauss-Newton loop (solver.py:278-291, 319-384).

    ``distributed``: None (single GPU), True (default torch.distributed group) or a process group;
    the tensor is then slab-sharded along its last mode across the group's ranks, every rank
    returns the same result.  ``slab_of``: when given (the global size of the last mode), ``y``
    holds only this rank's slab of the last mode (``slab_bounds``), so no rank needs the whole
    tensor in host memory.
    """
    t0 = time.monotonic()
    _check_lm(config)
    y = as_dense(y)
    gdims = y.dims if slab_of is None else tuple(y.dims[:-1]) + (int(slab_of),)
    rng = np.random.default_rng([config.seed, 0])
    eng = _make_engine(y, config.rank, device, distributed, slab_of)
    t1 = time.monotonic()
    result = _run_fit(eng, gdims, y.scalar_kind, config, rng)
    result.time_ms = (time.monotonic() - t0) * 1e3
    if _TIMING:
        import sys as _sys

        _sys.stderr.write(f"[fit timing] engine + tensor upload {1e3 * (t1 - t0):.1f} ms, "
                          f"init + LM loop + download {1e3 * (time.monotonic() - t1):.1f} ms\n")
    return result


def fit_file(path, config: FitConfig, *, device=None, distributed=None, complex_only: bool = False) -> FitResult:
    """``fit`` of a CPTN tensor file (cli.py:115-118 reads it with cptn.read_tensor first): the
    engine streams its slab of the file straight into device memory (``cpf_engine_load_cptn``),
    so neither the whole tensor nor a host copy of it is ever materialised.  Same result, errors
    and ``time_ms`` convention as ``fit`` (the file read is inside the timed region)."""
    from . import cptn

    t0 = time.monotonic()
    _check_lm(config)
    h = cptn.read_header(path)
    if len(h.dims) < 2:
        raise ValueError("the fLM solver needs a tensor of order >= 2")
    if complex_only and h.kind != 1:
        raise TypeError("expected a complex tensor")
    kind = _native.CPF_COMPLEX if h.kind else _native.CPF_REAL
    dev = 0 if device is None else int(device)
    eng = _engine_for(kind, h.dims, config.rank, dev, distributed)
    try:
        cptn.load_to_engine(eng, path, h)
    except BaseException:
        eng.close()
        raise
    rng = np.random.default_rng([config.seed, 0])
    result = _run_fit(eng, h.dims, COMPLEX if h.kind else REAL, config, rng)
    result.time_ms = (time.monotonic() - t0) * 1e3
    return result


def fit_complex(y, config: FitConfig, **kw) -> FitResult:
    """Complex fit: identical damping, stopping and normalisation (complexcp.py:51-54)."""
    y = as_dense(y)
    if y.scalar_kind != COMPLEX:
        raise TypeError("expected a complex tensor")
    return fit(y, config, **kw)


def _model_engine(y: DenseTensor, model: KruskalModel, device):
    if y.dims != model.dims:
        raise ValueError(f"tensor dims {y.dims} do not match model {model.dims}")
    require_same_kind(y.data, *model.factors)
    eng = _make_engine(y, model.rank, device, None)
    dtype = np.complex128 if np.iscomplexobj(y.data) else np.float64
    eng.set_factors(np.concatenate([np.asarray(f, dtype=dtype).reshape(-1, order="F") for f in model.factors]))
    return eng


def mttkrp(y, model, n: int, *, device=None) -> np.ndarray:
    """M_n = Y_(n) conj(KR_{k != n}) (kruskal.py:126-135), n is 1-based."""
    y, model = as_dense(y), as_model(model)
    if not 1 <= n <= model.order:
        raise ValueError(f"mode {n} out of range for order-{model.order} tensor")
    eng = _model_engine(y, model, device)
    try:
        out = eng.mttkrp(n)
    finally:
        eng.close()
    return out.reshape((model.dims[n - 1], model.rank), order="F")


def relative_error(y, model, *, device=None) -> float:
    """||Y - X|| / ||Y|| (kruskal.py:159-167), weights folded into mode 1."""
    y, model = as_dense(y), as_model(model)
    if model.weights is not None:
        f0 = model.factors[0] * model.weights[None, :]
        model = KruskalModel([f0] + list(model.factors[1:]))
    eng = _model_engine(y, model, device)
    try:
        return eng.relative_error()
    finally:
        eng.close()


def flm_step(y, model, mu: float, variant: str = "auto", cache=None, mttkrps=None, refine_steps: int = 2,
             *, device=None) -> KruskalModel:
    """One fLM candidate with structured refinement (solver.py:189-226).

    ``cache``/``mttkrps`` are accepted for signature compatibility; the engine recomputes them on
    the device from ``model`` (they are pure functions of it).  Numerical failures raise like the
    reference (numpy LinAlgError / SingularKernelError).
    """
    y, model = as_dense(y), as_model(model)
    if variant not in LM_VARIANTS:
        raise ValueError(f"unknown variant {variant!r}")
    eng = _model_engine(y, model, device)
    try:
        vec, code = eng.flm_step(mu, variant, refine_steps)
    finally:
        eng.close()
    if code:
        if code in (_native.ERR_KERNEL_SINGULAR, _native.ERR_PHI1_SINGULAR):
            raise SingularKernelError(_native.ERR_MESSAGE[code])
        raise np.linalg.LinAlgError(_native.ERR_MESSAGE.get(code, "numerical error"))
    return model_from_vector(vec, model.dims, model.rank)


def pinv_psd(gamma, *, device=None) -> np.ndarray:
    """Pseudo-inverse of a Hermitian PSD matrix (kruskal.py:245-254) on the GPU: Jacobi
    eigen-decomposition, eigenvalues below eps * R * lambda_max truncated."""
    return _native.pinv_psd(gamma, 0 if device is None else int(device))


def als_step(y, model, *, device=None) -> KruskalModel:
    """One ALS sweep, factors updated in ascending mode order (kruskal.py:257-265)."""
    y, model = as_dense(y), as_model(model)
    eng = _model_engine(y, model, device)
    try:
        eng.als_step(False, 1)
        vec = eng.get_factors()
    finally:
        eng.close()
    return model_from_vector(vec, model.dims, model.rank)


def als_line_search_step(y, model, history, t: int = 1, *, device=None) -> KruskalModel:
    """ALS sweep with extrapolation against the previous iterate (kruskal.py:268-293): candidates
    A_prev + s (A_als - A_prev), s in {1.1, t^(1/3)}, scored by relative error; plain ALS when
    ``history`` is None."""
    y, model = as_dense(y), as_model(model)
    eng = _model_engine(y, model, device)
    try:
        if history is not None:
            history = as_model(history)
            dtype = np.complex128 if np.iscomplexobj(y.data) else np.float64
            eng.set_history(np.concatenate([np.asarray(f, dtype=dtype).reshape(-1, order="F")
                                            for f in history.factors]))
        eng.als_step(True, t)
        vec = eng.get_factors()
    finally:
        eng.close()
    return model_from_vector(vec, model.dims, model.rank)


@dataclass
class StructuredInverse:
    """Block form of (H + mu I)^{-1} (hessian.py:214-229): gamma_tilde[n] = (Gamma^(n) + mu I)^{-1},
    S[n][m] the R^2 x R^2 blocks of the core grid."""

    gamma_tilde: list
    S: list
    mu: float

    def scalar_count(self) -> int:
        n = len(self.gamma_tilde)
        r2 = self.gamma_tilde[0].size
        return n * r2 + sum(b.size for row in self.S for b in row)


def fast_damped_inverse(cache, factors, mu: float, use_kernel_inverse=None, *, device=None) -> StructuredInverse:
    """Structured (H + mu I)^{-1} from the low-rank adjustment (hessian.py:232-277), on the GPU.

    ``cache`` is accepted for signature compatibility; the engine recomputes the Gram cache from
    ``factors`` on the device (it is a pure function of them).  ``use_kernel_inverse=None`` picks
    the explicit-K^{-1} path exactly when the kernel invertibility proxy holds.  Errors as the
    reference: ValueError for mu <= 0, SingularKernelError for a singular K (K^{-1} path requested)
    or a singular K-free system, LinAlgError("Singular matrix") otherwise."""
    if mu <= 0:
        raise ValueError("mu must be positive")
    model = as_model(factors if isinstance(factors, KruskalModel) else KruskalModel(list(factors)))
    if model.order < 2:
        raise ValueError("kernel inverse needs at least two modes")
    kind = _native.CPF_COMPLEX if model.scalar_kind == COMPLEX else _native.CPF_REAL
    eng = _native.Engine(kind, model.dims, model.rank, 0 if device is None else int(device))
    try:
        eng.set_factors(model.as_vector())
        gt, d, code = eng.fast_damped_inverse(mu, use_kernel_inverse)
    finally:
        eng.close()
    if code in (_native.ERR_KINV_SINGULAR, _native.ERR_SBCK_SINGULAR):
        raise SingularKernelError(_native.ERR_MESSAGE[code])
    if code:
        raise np.linalg.LinAlgError(_native.ERR_MESSAGE.get(code, "numerical error"))
    r2 = model.rank * model.rank
    n_modes = model.order
    S = [[d[n * r2:(n + 1) * r2, m * r2:(m + 1) * r2] for m in range(n_modes)] for n in range(n_modes)]
    return StructuredInverse(gt, S, mu)


class SingularKernelError(np.linalg.LinAlgError):
    """The kernel matrix K is (numerically) singular (hessian.py:34-35)."""
