"""ctypes binding of the C ABI in ``include/cpfast_b200.h`` (libcpfast_b200.so).

This is the reference-side binding a Python host adds over the native engine (see
INTEGRATION.md).  There is deliberately no CPU fallback: if the shared library is missing, or
no CUDA device is visible, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

LIB_NAME = "libcpfast_b200.so"
LIB_DIR = Path(__file__).resolve().parent / "_lib"
LIB_PATH = LIB_DIR / LIB_NAME

# return codes
CPF_OK = 0
CPF_E_ARG = -1
CPF_E_KIND = -2
CPF_E_CUDA = -4
CPF_E_NCCL = -5
CPF_E_ZERODIV = -6
CPF_E_UNSUPPORTED = -7
CPF_E_STATE = -8
CPF_E_FORMAT = -9

CPF_REAL = 0
CPF_COMPLEX = 1

# tensor-pass implementations (cpf_engine_pass_impl)
PASS_FMA = 0
PASS_DMMA = 1
PASS_OZAKI = 2

VARIANT_CODE = {"auto": 0, "flm-a": 1, "flm-b": 2}

STOP_RUNNING = 0
STOP_TOL = 1
STOP_MU_OVERFLOW = 2
STOP_ERROR = 3
STOP_MAX_ITERS = 4

ERR_NONE = 0
ERR_SINGULAR = 1
ERR_KERNEL_SINGULAR = 2
ERR_PHI1_SINGULAR = 3
ERR_ZERO_COLUMN = 4
ERR_NONFINITE = 5
ERR_KINV_SINGULAR = 6
ERR_SBCK_SINGULAR = 7

# messages of the reference's in-loop exceptions (solver.py:349-352; hessian.py:146-147, 210-211;
# numpy.linalg "Singular matrix")
ERR_MESSAGE = {
    ERR_SINGULAR: "Singular matrix",
    ERR_KERNEL_SINGULAR: "flm-b requested but K is singular",
    ERR_PHI1_SINGULAR: "I + Psi K numerically singular: Singular matrix",
    ERR_NONFINITE: "non-finite values in the step",
    ERR_KINV_SINGULAR: "a pairwise Gamma entry vanishes; K is singular",
    ERR_SBCK_SINGULAR: "Sb + Chat K numerically singular: Singular matrix",
}

EXPORTED_SYMBOLS = (
    "cpf_abi_version",
    "cpf_engine_als_step",
    "cpf_engine_set_history",
    "cpf_engine_fast_damped_inverse",
    "cpf_loopback_group_create",
    "cpf_loopback_group_destroy",
    "cpf_engine_create_loopback",
    "cpf_pinv_psd",
    "cpf_device_count",
    "cpf_nccl_unique_id",
    "cpf_engine_create",
    "cpf_engine_destroy",
    "cpf_engine_last_error",
    "cpf_engine_slab",
    "cpf_engine_stream",
    "cpf_engine_set_tensor",
    "cpf_engine_set_factors",
    "cpf_engine_get_factors",
    "cpf_engine_fit_begin",
    "cpf_engine_fit_step",
    "cpf_engine_trace",
    "cpf_engine_mttkrp",
    "cpf_engine_relative_error",
    "cpf_engine_flm_step",
    "cpf_engine_profile",
    "cpf_engine_phase_times",
    "cpf_engine_phase_max",
    "cpf_engine_launch_count",
    "cpf_engine_unfolding_gram",
    "cpf_engine_pass_impl",
    "cpf_engine_pass_guard",
    "cpf_engine_load_cptn",
    "cpf_pool_reserve",
)


class IterRecordC(ctypes.Structure):
    _fields_ = [("iter", ctypes.c_int32), ("accepted", ctypes.c_int32),
                ("relerr", ctypes.c_double), ("mu", ctypes.c_double)]


class StatusC(ctypes.Structure):
    _fields_ = [("stopped", ctypes.c_int32), ("err_code", ctypes.c_int32), ("err_iter", ctypes.c_int32),
                ("iter", ctypes.c_int32), ("last_accepted", ctypes.c_int32), ("err_column", ctypes.c_int32),
                ("relerr", ctypes.c_double), ("mu", ctypes.c_double), ("ynorm", ctypes.c_double)]


class NativeError(RuntimeError):
    """A native-engine failure that maps to no reference exception (CUDA / NCCL)."""


_lock = threading.Lock()
_lib = None


def _declare(lib) -> None:
    P, I, I64, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
    sig = {
        "cpf_abi_version": (I, []),
        "cpf_device_count": (I, [ctypes.POINTER(I)]),
        "cpf_nccl_unique_id": (I, [P]),
        "cpf_engine_create": (I, [ctypes.POINTER(P), I, I, I, ctypes.POINTER(I64), I, I, I, P]),
        "cpf_engine_destroy": (None, [P]),
        "cpf_engine_last_error": (ctypes.c_char_p, [P]),
        "cpf_engine_slab": (I, [P, ctypes.POINTER(I64), ctypes.POINTER(I64)]),
        "cpf_engine_stream": (P, [P]),
        "cpf_engine_set_tensor": (I, [P, P, I64, I]),
        "cpf_engine_set_factors": (I, [P, P]),
        "cpf_engine_get_factors": (I, [P, P]),
        "cpf_engine_fit_begin": (I, [P, I, D, D, I, ctypes.POINTER(StatusC)]),
        "cpf_engine_fit_step": (I, [P, I, ctypes.POINTER(StatusC)]),
        "cpf_engine_trace": (I, [P, ctypes.POINTER(IterRecordC), I, ctypes.POINTER(I)]),
        "cpf_engine_mttkrp": (I, [P, I, P]),
        "cpf_engine_relative_error": (I, [P, ctypes.POINTER(D)]),
        "cpf_engine_flm_step": (I, [P, D, I, I, P, ctypes.POINTER(I)]),
        "cpf_engine_profile": (I, [P, I]),
        "cpf_engine_phase_times": (I, [P, ctypes.POINTER(D), ctypes.POINTER(I64), I]),
        "cpf_engine_phase_max": (I, [P, ctypes.POINTER(D), I]),
        "cpf_engine_launch_count": (I64, [P]),
        "cpf_engine_unfolding_gram": (I, [P, I, P]),
        "cpf_engine_pass_impl": (I, [P]),
        "cpf_engine_pass_guard": (I, [P, ctypes.POINTER(I64), ctypes.POINTER(I)]),
        "cpf_engine_load_cptn": (I, [P, ctypes.c_char_p, I64]),
        "cpf_pool_reserve": (I, [I, I64]),
        "cpf_engine_als_step": (I, [P, I, I, ctypes.POINTER(D)]),
        "cpf_engine_set_history": (I, [P, P]),
        "cpf_pinv_psd": (I, [I, I, I, P, P]),
        "cpf_engine_fast_damped_inverse": (I, [P, D, I, P, P, ctypes.POINTER(I)]),
        "cpf_loopback_group_create": (I, [I, ctypes.POINTER(P)]),
        "cpf_loopback_group_destroy": (None, [P]),
        "cpf_engine_create_loopback": (I, [ctypes.POINTER(P), I, I, I, ctypes.POINTER(I64), I, I, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def load():
    """Load libcpfast_b200.so (built in-tree by ``__graft_entry__.build()``); raise if absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA engine first "
                "(python -c 'import __graft_entry__ as g; g.build()').  There is no CPU fallback."
            )
        # NCCL is resolved by soname.  torch (the device-memory / torch.distributed plumbing) bundles
        # a newer libnccl than the system one; load it first so that one library serves both --
        # the other order leaves the older system NCCL global and a later `import torch` fails
        # (undefined symbol ncclDevCommCreate).
        try:
            import torch  # noqa: F401
        except ImportError:  # pragma: no cover - the engine itself does not need torch
            pass
        lib = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_GLOBAL if hasattr(os, "RTLD_GLOBAL") else 0)
        _declare(lib)
        _lib = lib
        return lib


def pool_reserve(device: int, nbytes: int) -> None:
    """Grow the device memory pool engines allocate from (see cpf_pool_reserve)."""
    rc = load().cpf_pool_reserve(int(device), int(nbytes))
    if rc != CPF_OK:
        raise NativeError(f"cpf_pool_reserve failed ({rc})")


def device_count() -> int:
    n = ctypes.c_int(0)
    load().cpf_device_count(ctypes.byref(n))
    return n.value


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    rc = load().cpf_nccl_unique_id(buf)
    if rc != CPF_OK:
        raise NativeError("ncclGetUniqueId failed")
    return buf.raw


def pinv_psd(gamma: np.ndarray, device: int = 0) -> np.ndarray:
    """pinv_psd (kruskal.py:245-254) of a Hermitian PSD R x R matrix on the GPU (cpf_pinv_psd)."""
    g = np.asarray(gamma)
    if g.ndim != 2 or g.shape[0] != g.shape[1]:
        raise ValueError("pinv_psd needs a square matrix")
    kind = CPF_COMPLEX if np.iscomplexobj(g) else CPF_REAL
    dt = np.complex128 if kind == CPF_COMPLEX else np.float64
    gf = np.asfortranarray(g, dtype=dt)
    out = np.empty(g.shape, dtype=dt, order="F")
    rc = load().cpf_pinv_psd(int(device), kind, g.shape[0], gf.ctypes.data, out.ctypes.data)
    if rc == CPF_E_ARG:
        raise ValueError(f"not supported on the B200 backend: pinv_psd of a {g.shape[0]} x {g.shape[0]} matrix (R <= 64)")
    if rc != CPF_OK:
        raise NativeError(f"cpf_pinv_psd failed ({rc})")
    return out


def _raise_for(rc: int, msg: str):
    if rc == CPF_OK:
        return
    if rc == CPF_E_ARG:
        raise ValueError(msg)
    if rc == CPF_E_KIND:
        raise TypeError(msg)
    if rc == CPF_E_ZERODIV:
        raise ZeroDivisionError(msg)
    if rc == CPF_E_FORMAT:
        from .cptn import FormatError

        raise FormatError(msg)
    if rc == CPF_E_UNSUPPORTED:
        raise ValueError(f"not supported on the B200 backend: {msg}")
    raise NativeError(f"native engine error {rc}: {msg}")


class LoopbackGroup:
    """Test transport: ``world`` engines of this process on one device exchanging through device
    buffers (cpf_loopback_group_create).  Drive each rank's engine from its own thread."""

    def __init__(self, world: int):
        lib = load()
        self._lib = lib
        self.world = int(world)
        h = ctypes.c_void_p()
        rc = lib.cpf_loopback_group_create(self.world, ctypes.byref(h))
        if rc != CPF_OK:
            _raise_for(rc, f"loopback group of {world} ranks")
        self.handle = h

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            self._lib.cpf_loopback_group_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Engine:
    """One native fit context on one GPU (owns device buffers; not thread-safe)."""

    def __init__(self, kind: int, dims, rank: int, device: int = 0, world_rank: int = 0, world_size: int = 1,
                 nccl_uid: bytes | None = None, loopback: LoopbackGroup | None = None):
        lib = load()
        self._lib = lib
        self.kind = kind
        self.dims = tuple(int(d) for d in dims)
        self.rank = int(rank)
        self.dtype = np.complex128 if kind == CPF_COMPLEX else np.float64
        arr = (ctypes.c_int64 * len(self.dims))(*self.dims)
        h = ctypes.c_void_p()
        if loopback is not None:
            rc = lib.cpf_engine_create_loopback(ctypes.byref(h), int(device), int(kind), len(self.dims), arr,
                                                self.rank, int(world_rank), loopback.handle)
        else:
            uid = ctypes.create_string_buffer(nccl_uid, 128) if nccl_uid is not None else None
            rc = lib.cpf_engine_create(ctypes.byref(h), int(device), int(kind), len(self.dims), arr, self.rank,
                                       int(world_rank), int(world_size), uid)
        if rc != CPF_OK:
            msg = lib.cpf_engine_last_error(h).decode() if h.value else "engine creation failed"
            if h.value:
                lib.cpf_engine_destroy(h)
            _raise_for(rc, msg)
        self._h = h

    # -- lifetime
    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.cpf_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int):
        if rc != CPF_OK:
            _raise_for(rc, self._lib.cpf_engine_last_error(self._h).decode())

    # -- data
    @property
    def slab(self) -> tuple[int, int]:
        lo, hi = ctypes.c_int64(), ctypes.c_int64()
        self._check(self._lib.cpf_engine_slab(self._h, ctypes.byref(lo), ctypes.byref(hi)))
        return lo.value, hi.value

    @property
    def stream_handle(self) -> int:
        return int(self._lib.cpf_engine_stream(self._h) or 0)

    def set_tensor_host(self, slab: np.ndarray):
        arr = np.asarray(slab)
        if arr.dtype != self.dtype:
            raise TypeError("tensor dtype does not match the engine kind")
        flat = np.ravel(arr, order="F")  # no copy for a Fortran-contiguous slab
        self._keep = flat
        self._check(self._lib.cpf_engine_set_tensor(self._h, flat.ctypes.data, flat.size, 0))

    def load_cptn(self, path, payload_offset: int):
        self._check(self._lib.cpf_engine_load_cptn(self._h, str(path).encode(), int(payload_offset)))

    def set_tensor_device(self, ptr: int, nelem: int):
        self._check(self._lib.cpf_engine_set_tensor(self._h, ctypes.c_void_p(ptr), int(nelem), 1))

    def set_factors(self, stacked: np.ndarray):
        v = np.ascontiguousarray(stacked, dtype=self.dtype)
        self._check(self._lib.cpf_engine_set_factors(self._h, v.ctypes.data))

    def get_factors(self) -> np.ndarray:
        out = np.empty(self.rank * sum(self.dims), dtype=self.dtype)
        self._check(self._lib.cpf_engine_get_factors(self._h, out.ctypes.data))
        return out

    # -- fit
    def fit_begin(self, variant: str, tau: float, tol: float, max_iters: int) -> StatusC:
        st = StatusC()
        self._check(self._lib.cpf_engine_fit_begin(self._h, VARIANT_CODE[variant], float(tau), float(tol),
                                                   int(max_iters), ctypes.byref(st)))
        return st

    def fit_step(self, n: int) -> StatusC:
        st = StatusC()
        self._check(self._lib.cpf_engine_fit_step(self._h, int(n), ctypes.byref(st)))
        return st

    def trace(self, cap: int):
        buf = (IterRecordC * max(cap, 1))()
        n = ctypes.c_int(0)
        self._check(self._lib.cpf_engine_trace(self._h, buf, int(cap), ctypes.byref(n)))
        return [(buf[i].iter, buf[i].relerr, buf[i].mu, bool(buf[i].accepted)) for i in range(n.value)]

    # -- building blocks
    def mttkrp(self, mode: int) -> np.ndarray:
        if mode == 0:
            out = np.empty(self.rank * sum(self.dims), dtype=self.dtype)
        else:
            out = np.empty(self.rank * self.dims[mode - 1], dtype=self.dtype)
        self._check(self._lib.cpf_engine_mttkrp(self._h, int(mode), out.ctypes.data))
        return out

    def relative_error(self) -> float:
        v = ctypes.c_double()
        self._check(self._lib.cpf_engine_relative_error(self._h, ctypes.byref(v)))
        return v.value

    def flm_step(self, mu: float, variant: str, refine_steps: int):
        out = np.empty(self.rank * sum(self.dims), dtype=self.dtype)
        code = ctypes.c_int(0)
        self._check(self._lib.cpf_engine_flm_step(self._h, float(mu), VARIANT_CODE[variant], int(refine_steps),
                                                  out.ctypes.data, ctypes.byref(code)))
        return out, code.value

    def als_step(self, line_search: bool, t: int) -> float:
        v = ctypes.c_double()
        self._check(self._lib.cpf_engine_als_step(self._h, 1 if line_search else 0, int(t), ctypes.byref(v)))
        return v.value

    def fast_damped_inverse(self, mu: float, use_kernel_inverse):
        """(gamma_tilde (N, R, R), core grid D (N R^2 x N R^2), CPF_ERR_* code)."""
        n, r = len(self.dims), self.rank
        nb = n * r * r
        gt = np.empty(n * r * r, dtype=self.dtype)
        d = np.empty((nb, nb), dtype=self.dtype, order="F")
        code = ctypes.c_int(0)
        uk = -1 if use_kernel_inverse is None else (1 if use_kernel_inverse else 0)
        self._check(self._lib.cpf_engine_fast_damped_inverse(self._h, float(mu), uk, gt.ctypes.data, d.ctypes.data,
                                                             ctypes.byref(code)))
        return [gt[k * r * r:(k + 1) * r * r].reshape((r, r), order="F") for k in range(n)], d, code.value

    def set_history(self, stacked: np.ndarray | None):
        if stacked is None:
            self._check(self._lib.cpf_engine_set_history(self._h, None))
            return
        v = np.ascontiguousarray(stacked, dtype=self.dtype)
        self._check(self._lib.cpf_engine_set_history(self._h, v.ctypes.data))

    # -- profiling
    def profile(self, on: bool):
        self._check(self._lib.cpf_engine_profile(self._h, 1 if on else 0))

    def phase_times(self, n: int = 5):
        ms = (ctypes.c_double * n)()
        cnt = (ctypes.c_int64 * n)()
        self._check(self._lib.cpf_engine_phase_times(self._h, ms, cnt, n))
        return list(ms), list(cnt)

    def phase_max(self, n: int = 5):
        ms = (ctypes.c_double * n)()
        self._check(self._lib.cpf_engine_phase_max(self._h, ms, n))
        return list(ms)

    def unfolding_gram(self, mode: int) -> np.ndarray:
        d = self.dims[mode - 1]  # sharded mode N: every rank receives the full I_N x I_N Gram
        out = np.empty((d, d), dtype=self.dtype, order="F")
        self._check(self._lib.cpf_engine_unfolding_gram(self._h, int(mode), out.ctypes.data))
        return out

    def launch_count(self) -> int:
        return int(self._lib.cpf_engine_launch_count(self._h))

    def pass_impl(self) -> int:
        return int(self._lib.cpf_engine_pass_impl(self._h))

    def pass_guard(self) -> tuple[int, bool]:
        """(int8-pass launches that fell back to fp64 since fit_begin, tensor rejected by the guard)."""
        fb, rej = ctypes.c_int64(0), ctypes.c_int(0)
        self._check(self._lib.cpf_engine_pass_guard(self._h, ctypes.byref(fb), ctypes.byref(rej)))
        return int(fb.value), bool(rej.value)
