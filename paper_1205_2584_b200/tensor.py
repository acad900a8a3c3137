"""Host containers with the reference's conventions (drop-in types).

``DenseTensor`` mirrors ``cpfast.tensor.DenseTensor`` (cpfast/tensor.py:36-73): a frozen
column-major float64 / complex128 array.  ``KruskalModel`` mirrors ``cpfast.kruskal.KruskalModel``
(cpfast/kruskal.py:27-72).  The solver also accepts the reference's own objects (anything with a
``.data`` array, or ``.factors``) and plain ndarrays.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

REAL = "real"
COMPLEX = "complex"


class ScalarKindError(TypeError):
    """Mixed real and complex operands (cpfast/tensor.py:21-22)."""


def kind_of(arr) -> str:
    return COMPLEX if np.iscomplexobj(arr) else REAL


def require_same_kind(*arrays) -> str:
    kinds = {kind_of(np.asarray(a)) for a in arrays}
    if len(kinds) > 1:
        raise ScalarKindError("mixed real/complex operands are not supported")
    return kinds.pop()


@dataclass(frozen=True)
class DenseTensor:
    """N-way float64/complex128 tensor stored column-major (mode-1 index fastest)."""

    data: np.ndarray

    def __post_init__(self):
        arr = np.asfortranarray(self.data)
        if arr.ndim < 1:
            arr = arr.reshape(1)
        if arr.dtype not in (np.float64, np.complex128):
            arr = arr.astype(np.complex128 if np.iscomplexobj(arr) else np.float64)
        object.__setattr__(self, "data", arr)

    @property
    def dims(self) -> tuple:
        return self.data.shape

    @property
    def order(self) -> int:
        return self.data.ndim

    @property
    def size(self) -> int:
        return self.data.size

    @property
    def scalar_kind(self) -> str:
        return kind_of(self.data)

    def norm(self) -> float:
        return float(np.linalg.norm(self.data))


@dataclass
class KruskalModel:
    """Factor matrices A^(n) (I_n x R) with optional component weights."""

    factors: list
    weights: np.ndarray | None = None

    def __post_init__(self):
        self.factors = [np.atleast_2d(np.asarray(f)) for f in self.factors]
        if len({f.shape[1] for f in self.factors}) != 1:
            raise ValueError("all factors must share the same column count")
        if self.weights is not None:
            self.weights = np.asarray(self.weights).reshape(-1)
            if self.weights.shape[0] != self.rank:
                raise ValueError("weights length must equal the rank")

    @property
    def rank(self) -> int:
        return self.factors[0].shape[1]

    @property
    def order(self) -> int:
        return len(self.factors)

    @property
    def dims(self) -> tuple:
        return tuple(f.shape[0] for f in self.factors)

    @property
    def scalar_kind(self) -> str:
        return require_same_kind(*self.factors)

    def copy(self) -> "KruskalModel":
        return KruskalModel([f.copy() for f in self.factors], None if self.weights is None else self.weights.copy())

    def as_vector(self) -> np.ndarray:
        """Concatenated column-major vectorisations (kruskal.py:70-72)."""
        return np.concatenate([f.reshape(-1, order="F") for f in self.factors])


def model_from_vector(vec: np.ndarray, dims, rank: int) -> KruskalModel:
    """Inverse of ``as_vector`` (kruskal.py:75-82)."""
    out, off = [], 0
    for d in dims:
        out.append(np.asarray(vec[off: off + d * rank]).reshape((d, rank), order="F"))
        off += d * rank
    return KruskalModel(out)


def as_dense(y) -> DenseTensor:
    """Accept our DenseTensor, the reference's DenseTensor (duck-typed ``.data``) or an ndarray."""
    if isinstance(y, DenseTensor):
        return y
    data = getattr(y, "data", y)
    return DenseTensor(np.asarray(data))


def as_model(m) -> KruskalModel:
    if isinstance(m, KruskalModel):
        return m
    return KruskalModel(list(m.factors), getattr(m, "weights", None))
