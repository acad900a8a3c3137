"""B200-native fast damped Gauss-Newton (fLM) CP decomposition -- drop-in for ``cpfast``'s solver path.

Public surface mirrors the reference package (cpfast/__init__.py:32-33 and the solver module):
``fit``, ``fit_complex``, ``FitConfig``, ``FitResult``, ``IterRecord``, ``flm_step``, ``mttkrp``,
``relative_error``, ``DenseTensor``, ``KruskalModel``, and the ALS baselines ``als_step``,
``als_line_search_step``, ``pinv_psd`` (variants ``als`` / ``als-ls``).  All numerics run in the sm_100a engine
(``_lib/libcpfast_b200.so``, C ABI in ``include/cpfast_b200.h``).
"""

from .tensor import COMPLEX, REAL, DenseTensor, KruskalModel, ScalarKindError, model_from_vector
from .solver import (
    ALS_VARIANTS,
    LM_VARIANTS,
    MU_OVERFLOW,
    VARIANTS,
    FitConfig,
    FitResult,
    IterRecord,
    SingularKernelError,
    StructuredInverse,
    als_line_search_step,
    als_step,
    fit,
    fit_complex,
    fit_file,
    fast_damped_inverse,
    flm_step,
    mttkrp,
    pinv_psd,
    random_init,
    relative_error,
    slab_bounds,
)

__version__ = "0.1.0"

__all__ = [
    "COMPLEX", "REAL", "DenseTensor", "KruskalModel", "ScalarKindError", "model_from_vector",
    "LM_VARIANTS", "MU_OVERFLOW", "VARIANTS", "FitConfig", "FitResult", "IterRecord",
    "SingularKernelError", "fit", "fit_complex", "fit_file", "flm_step", "mttkrp", "random_init",
    "relative_error", "slab_bounds", "ALS_VARIANTS", "als_step", "als_line_search_step", "pinv_psd",
    "StructuredInverse", "fast_damped_inverse",
]
