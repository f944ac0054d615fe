"""ctypes binding of libpsa.so (include/psa.h).

The product path has no fallback: if the library is missing or CUDA is unavailable, every
entry point raises. Status codes map onto the reference error taxonomy
(pkg/src/pyrattn/errors.py:9-18).
"""

from __future__ import annotations

import ctypes
from ctypes import c_double, c_int, c_int64, c_size_t, c_void_p
from pathlib import Path

from .errors import NumericError, ValidationError

import os

# PSA_LIB_PATH: an alternative build of the same library (instrumented probe builds only)
LIB_PATH = Path(os.environ.get("PSA_LIB_PATH") or Path(__file__).with_name("libpsa.so"))
_lib = None

PSA_OK, PSA_EINVAL, PSA_ENUMERIC, PSA_ECUDA = 0, -2, -4, -5
PSA_IMP_FP64_ONLY = 1

_SIGNATURES = {
    "psa_last_error": (ctypes.c_char_p, []),
    "psa_version": (c_int, []),
    "psa_pyramid_build": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int, c_int, c_int,
                                  c_void_p, c_void_p, c_void_p, c_void_p]),
    "psa_similarity_caps": (c_int, [c_void_p, c_int64, c_int64, c_int, c_int, c_int,
                                    c_void_p, c_void_p, c_void_p]),
    "psa_importance_workspace_bytes": (c_size_t, [c_int64, c_int64, c_int, c_int, c_int, c_int]),
    "psa_importance_sampled": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int, c_int64, c_int,
                                       c_int, c_int, c_void_p, c_void_p, c_int, c_int, c_int,
                                       c_int, c_void_p, c_void_p, c_void_p]),
    "psa_antidiag_workspace_bytes": (c_size_t, [c_int64, c_int64, c_int64, c_int, c_int, c_int]),
    "psa_importance_antidiagonal": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int, c_int64,
                                            c_int, c_int, c_int, c_int, c_int, c_void_p, c_void_p,
                                            c_void_p]),
    "psa_assign_levels": (c_int, [c_void_p, c_int64, c_int, c_int, c_int, c_int, c_int,
                                  c_void_p, c_void_p, c_int, c_void_p, c_int, c_int, c_int, c_int,
                                  c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "psa_mask_to_plan": (c_int, [c_void_p, c_int, c_int64, c_int, c_int, c_int, c_int, c_int,
                                 c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "psa_gather_rows": (c_int, [c_void_p, c_int64, c_int64, c_int, c_void_p, c_void_p, c_void_p]),
    "psa_attn_fwd": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int,
                             c_int, c_int64, c_int, c_int, c_int, c_int, c_void_p, c_void_p,
                             c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
    "psa_attn_fwd_scatter": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64,
                                     c_int, c_int, c_int64, c_int, c_int, c_int, c_int, c_void_p,
                                     c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p,
                                     c_void_p]),
    "psa_attn_bwd_workspace_bytes": (c_size_t, [c_int64, c_int, c_int, c_int64, c_int]),
    "psa_attn_bwd": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                             c_void_p, c_int64, c_int, c_int, c_int64, c_int, c_int, c_int, c_int,
                             c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_void_p,
                             c_void_p, c_void_p]),
    "psa_pyramid_build_gather": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int, c_int, c_int,
                                         c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                         c_void_p, c_void_p]),
    "psa_importance_sampled_rows": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int, c_int64,
                                            c_int, c_int, c_int, c_void_p, c_void_p, c_int, c_int,
                                            c_int, c_int, c_int, c_void_p, c_void_p, c_void_p]),
    "psa_antidiag_workspace_bytes_rows": (c_size_t, [c_int64, c_int64, c_int64, c_int, c_int, c_int,
                                                     c_int]),
    "psa_importance_antidiagonal_rows": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int,
                                                 c_int64, c_int, c_int, c_int, c_int, c_int,
                                                 c_void_p, c_int, c_void_p, c_void_p, c_void_p]),
    "psa_assign_levels_rows": (c_int, [c_void_p, c_int64, c_int, c_int, c_int, c_int, c_int,
                                       c_void_p, c_void_p, c_int, c_void_p, c_int, c_int, c_int,
                                       c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                       c_void_p]),
    "psa_attn_fwd_rows": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int,
                                  c_int, c_int64, c_int, c_int, c_int, c_int, c_void_p, c_void_p,
                                  c_int, c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
}

EXPORTED = tuple(_SIGNATURES)


def load(path: Path | None = None):
    """Load libpsa.so (once) and declare every exported signature."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise RuntimeError(
            f"{p} is missing: the sm_100a kernels are not built (run __graft_entry__.build()); "
            "there is no CPU fallback")
    lib = ctypes.CDLL(str(p))
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc == PSA_OK:
        return
    msg = load().psa_last_error().decode(errors="replace")
    if rc == PSA_EINVAL:
        raise ValidationError(msg)
    if rc == PSA_ENUMERIC:
        raise NumericError(msg)
    raise RuntimeError(f"{what}: {msg}")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None for None)."""
    return None if t is None else t.data_ptr()


def host_doubles(values) -> ctypes.Array:
    arr = (c_double * max(1, len(values)))()
    for i, x in enumerate(values):
        arr[i] = float(x)
    return arr


def host_ints(values) -> ctypes.Array:
    arr = (ctypes.c_int32 * max(1, len(values)))()
    for i, x in enumerate(values):
        arr[i] = int(x)
    return arr
