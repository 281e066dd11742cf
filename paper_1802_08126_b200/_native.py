"""ctypes binding of libpint.so (include/pint.h).

There is no CPU fallback: if the library is missing or no CUDA device is
present, constructing a :class:`Context` raises immediately.  Arrays passed
in may be numpy arrays (host; staged by the library) or CUDA float64 torch
tensors (used in place); outputs follow the input's kind.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import (
    DimensionMismatchError,
    InputError,
    NotSpdError,
    SolverDivergenceError,
)

LIB_PATH = os.environ.get("PINT_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpint.so")

PINT_OK, PINT_INPUT, PINT_DIMENSION, PINT_NOT_SPD, PINT_DIVERGED, PINT_CUDA = range(6)

# Arithmetic of the band kernels for contexts created from now on
# (include/pint.h pint_set_arith): "fast" (FMA, the default) or "exact"
# (bit-identical to the reference's CSR products).  PINT_ARITH sets the
# process default.
_ARITH = os.environ.get("PINT_ARITH", "fast")


def set_arithmetic(mode: str) -> str:
    """Select "fast" or "exact" band-kernel arithmetic for new contexts;
    returns the previous mode."""
    global _ARITH
    if mode not in ("fast", "exact"):
        raise InputError(f"arithmetic must be 'fast' or 'exact', not {mode!r}")
    prev, _ARITH = _ARITH, mode
    return prev


def get_arithmetic() -> str:
    return _ARITH
MG_ATILDE, MG_HTILDE, MG_EULER = 0, 1, 2

_P = ctypes.c_void_p
_D = ctypes.c_double
_I = ctypes.c_int
_DP = ctypes.POINTER(ctypes.c_double)
_IP = ctypes.POINTER(ctypes.c_int)

# name -> (restype, argtypes); mirrors include/pint.h
_SIGNATURES = {
    "pint_abi_version": (_I, []),
    "pint_ctx_create": (_I, [_I, _I, _I, _P, ctypes.POINTER(_P)]),
    "pint_ctx_destroy": (_I, [_P]),
    "pint_last_error": (ctypes.c_char_p, [_P]),
    "pint_sync": (_I, [_P]),
    "pint_set_arith": (_I, [_P, _I]),
    "pint_get_arith": (_I, [_P]),
    "pint_set_stream": (_I, [_P, _P, _I]),
    "pint_problem_set": (_I, [_P, _I, _I, _I, _P, _P, _I, _P, _P, _P, _P, _D]),
    "pint_fold_rhs": (_I, [_P, _P, _P, _P]),
    "pint_apply_K": (_I, [_P, _P, _P]),
    "pint_apply_Kt": (_I, [_P, _P, _P]),
    "pint_apply_Abd": (_I, [_P, _P, _P]),
    "pint_mg_set": (_I, [_P, _I, _I, _P, _I, _P, _P]),
    "pint_mg_set_options": (_I, [_P, _I, _I, _I]),
    "pint_vcycle": (_I, [_P, _I, _I, _P, _P]),
    "pint_atilde_inv": (_I, [_P, _P, _P]),
    "pint_htilde_inv": (_I, [_P, _P, _P]),
    "pint_dst": (_I, [_P, _I, _P, _P]),
    "pint_dst_raw": (_I, [_P, _I, _I, ctypes.c_longlong, _P, _P]),
    "pint_dst_raw_axpy": (_I, [_P, _I, _I, ctypes.c_longlong, _P, _P, _P, _D]),
    "pint_uzawa_begin": (_I, [_P, _P, _P, _P, _DP]),
    "pint_uzawa_step": (_I, [_P, _D, _DP]),
    "pint_uzawa_end": (_I, [_P, _P, _P]),
    "pint_host_prefault": (_I, [_P, _P, ctypes.c_longlong]),
    "pint_host_prefault_join": (_I, [_P]),
    "pint_apply_saddle": (_I, [_P, _P, _P, _P, _P]),
    "pint_lincomb": (_I, [_P, _P, ctypes.c_longlong, _P, _D, _P, _D, _P, _D, _I]),
    "pint_dot": (_I, [_P, _P, _P, ctypes.c_longlong, _DP]),
    "pint_uzawa": (_I, [_P, _P, _P, _P, _D, _D, _I, _I, _P, _IP, _IP, _P]),
    "pint_set_timing": (_I, [_P, _I]),
    "pint_phase_ms": (_I, [_P, _P]),
    "pint_profile": (_I, [_P, _I]),
    "pint_kernel_count": (_I, []),
    "pint_kernel_stat": (_I, [_P, _I, ctypes.POINTER(ctypes.c_char_p), _DP,
                              ctypes.POINTER(ctypes.c_longlong), _DP]),
    "pint_uzawa_run": (_I, [_P, _D, _I, _P, _DP]),
    "pint_set_partition": (_I, [_P, _I, _I, _I, _I]),
    "pint_residual_r1": (_I, [_P, _P, _P, _P, _P]),
    "pint_residual_z": (_I, [_P, _P, _P, _P, _P]),
    "pint_atilde_update": (_I, [_P, _P, _P, _DP]),
    "pint_htilde_modes": (_I, [_P, _P, _P, _DP]),
    "pint_axpy": (_I, [_P, _P, _P, _D, ctypes.c_longlong]),
    "pint_launch_count": (ctypes.c_longlong, [_P]),
    "pint_field_set": (_I, [_P, _I, _I, _P]),
    "pint_field_assemble": (_I, [_P, _I, _I, _P]),
    "pint_field_separable": (_I, [_P, _I, _P, _P]),
    "pint_field_aref": (_I, [_P, _I, _P]),
    "pint_mg_set_field": (_I, [_P, _I, _I, _P, _D, _P]),
    "pint_sequential_euler": (_I, [_P, _P, _P, _P, _D, _I, _IP, _DP]),
    "pint_s_norm": (_I, [_P, _P, _P, _D, _I, _DP]),
    "pint_uzawa_s_error": (_I, [_P, _P, _D, _I, _DP]),
    "pint_abd_inverse": (_I, [_P, _P, _P, _D, _I]),
}

_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libpint.so once; raises if it was not built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build the CUDA library first "
            "(python -c 'import __graft_entry__ as g; g.build()')"
        )
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)


def _is_tensor(x) -> bool:
    return type(x).__module__.startswith("torch")


def as_buffer(x, shape=None):
    """(pointer, keep-alive object) for a float64 host or device array."""
    if _is_tensor(x):
        import torch

        if x.dtype != torch.float64 or not x.is_cuda:
            raise InputError("device arrays must be float64 CUDA tensors")
        t = x.contiguous()
        if shape is not None and tuple(t.shape) != tuple(shape):
            raise DimensionMismatchError(f"expected shape {tuple(shape)}, got {tuple(t.shape)}")
        return t.data_ptr(), t
    a = np.ascontiguousarray(x, dtype=np.float64)
    if shape is not None and a.shape != tuple(shape):
        raise DimensionMismatchError(f"expected shape {tuple(shape)}, got {a.shape}")
    return a.ctypes.data, a


def empty_like_kind(x, shape):
    if _is_tensor(x):
        import torch

        return torch.empty(shape, dtype=torch.float64, device=x.device)
    return np.empty(shape, dtype=np.float64)


def ptr_of(out):
    if _is_tensor(out):
        return out.data_ptr()
    return out.ctypes.data


class Context:
    """One libpint context (one CUDA device, one stream)."""

    def __init__(self, device: int | None = None):
        self.lib = load_library()
        if device is None:
            device = 0
            try:
                import torch

                if torch.cuda.is_available():
                    device = torch.cuda.current_device()
            except ImportError:
                pass
        h = _P()
        st = self.lib.pint_ctx_create(int(device), 0, 1, None, ctypes.byref(h))
        if st != PINT_OK:
            raise RuntimeError(
                f"libpint: cannot create a context on CUDA device {device} (status {st}); "
                "the GPU path has no CPU fallback"
            )
        self.h = h
        self.device = int(device)
        self.arith = _ARITH
        self.call("pint_set_arith", 1 if _ARITH == "exact" else 0)

    def close(self):
        if getattr(self, "h", None):
            self.lib.pint_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, status: int) -> None:
        if status == PINT_OK:
            return
        msg = (self.lib.pint_last_error(self.h) or b"").decode()
        if status == PINT_DIMENSION:
            raise DimensionMismatchError(msg)
        if status == PINT_INPUT:
            raise InputError(msg)
        if status == PINT_NOT_SPD:
            raise NotSpdError(msg)
        if status == PINT_DIVERGED:
            raise SolverDivergenceError(msg)
        raise RuntimeError(f"libpint CUDA failure: {msg}")

    def call(self, name: str, *args) -> None:
        self.check(getattr(self.lib, name)(self.h, *args))

    def launches(self) -> int:
        return int(self.lib.pint_launch_count(self.h))

    def kernel_stats(self) -> dict:
        """{name: (total_ms, launches, algorithmic_bytes)} from profiling mode."""
        out = {}
        for k in range(self.lib.pint_kernel_count()):
            name = ctypes.c_char_p()
            ms, nb = ctypes.c_double(), ctypes.c_double()
            cnt = ctypes.c_longlong()
            self.call("pint_kernel_stat", k, ctypes.byref(name), ctypes.byref(ms),
                      ctypes.byref(cnt), ctypes.byref(nb))
            out[name.value.decode()] = (ms.value, cnt.value, nb.value)
        return out
