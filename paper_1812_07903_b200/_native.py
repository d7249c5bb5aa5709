"""ctypes binding of liblevsketch_b200.so (the C ABI in include/levsketch_b200.h).

The product path has no CPU fallback: if the shared library is missing or no
CUDA device is visible, every compute entry point raises.  ``build()`` in
``__graft_entry__`` (or ``make -C paper_1812_07903_b200/csrc``) produces the
library in-tree.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import torch

from . import errors

LIB_PATH = Path(__file__).resolve().parent / "liblevsketch_b200.so"

LVSK_F32, LVSK_F64, LVSK_BF16 = 0, 1, 2
FLAG_NONFINITE, FLAG_NEGATIVE, FLAG_BADINDEX = 1, 2, 4

_ERRORS = {
    1: errors.ConfigurationError,
    2: errors.DimensionMismatchError,
    3: errors.FormatError,
    4: errors.CapacityError,
    5: errors.UnsupportedFamilyError,
    6: errors.DegenerateInputError,
    7: errors.IncompatibleSketchError,
    8: RuntimeError,
}

_DTYPE = {torch.float32: LVSK_F32, torch.float64: LVSK_F64, torch.bfloat16: LVSK_BF16}


class HashBlock(C.Structure):
    _fields_ = [("a", C.c_uint64), ("b", C.c_uint64), ("sign_key", C.c_uint64), ("offset", C.c_int64), ("size", C.c_int64)]


_P, _I64, _I32, _U64, _D, _SZ = C.c_void_p, C.c_int64, C.c_int32, C.c_uint64, C.c_double, C.c_size_t

_SIGS = {
    "lvsk_last_error": (C.c_char_p, []),
    "lvsk_abi_version": (_I32, []),
    "lvsk_set_inflight": (_I32, [_I32]),
    "lvsk_get_inflight": (_I32, []),
    "lvsk_hashed_workspace_bytes": (_SZ, [_I64, _I32, _I64]),
    "lvsk_hashed_sketch": (
        _I32,
        [_P, _I32, _I64, _I64, _I64, _U64, C.POINTER(HashBlock), _I32, _D, _P, _P, _P, _P, _I64, _P, _SZ, _P, _P],
    ),
    "lvsk_hash_rows": (_I32, [_P, _I64, C.POINTER(HashBlock), _I32, _P, _P, _P]),
    "lvsk_merge_compensated": (_I32, [_P, _P, _P, _P, _P, _P, _I64, _P]),
    "lvsk_fold_compensated": (_I32, [_P, _P, _P, _I64, _P]),
    "lvsk_srht_workspace_bytes": (_SZ, [_I64, _I64, _I32, _I64]),
    "lvsk_srht": (_I32, [_P, _I32, _I64, _I64, _I64, _I64, _P, _P, _I64, _D, _P, _P, _SZ, _P, _P]),
    "lvsk_srht_rows": (_I32, [_P, _I64, _I64, _I64, _I64, _I64, _P, _P, _I64, _D, _P, _P, _SZ, _P, _P]),
    "lvsk_gaussian_workspace_bytes": (_SZ, [_I64, _I64, _I64, _I32]),
    "lvsk_gaussian_sketch": (_I32, [_P, _I32, _I64, _I64, _I64, _U64, _U64, _I64, _P, _I32, _P, _SZ, _P, _P]),
    "lvsk_gaussian_entries": (_I32, [_U64, _I64, _U64, _I64, _P, _P]),
    "lvsk_rowsumsq_gemm": (_I32, [_P, _I32, _I64, _I64, _I64, _P, _P, _I64, _P, _P, _P]),
    "lvsk_leverage_tf32x3": (_I32, [_P, _I64, _I64, _I64, _P, _P, _P, _I64, _P, _P, _P]),
    "lvsk_leverage_bf16": (_I32, [_P, _I64, _I64, _I64, _P, _I64, _I64, _P, _P, _P]),
    "lvsk_hashed_csr_workspace_bytes": (_SZ, [_I64, _I32, _I64]),
    "lvsk_hashed_sketch_csr": (
        _I32,
        [_P, _P, _P, _I32, _I64, _I64, _U64, C.POINTER(HashBlock), _I32, _D, _P, _P, _P, _P, _I64, _P, _SZ, _P, _P],
    ),
    "lvsk_rowsumsq_csr": (_I32, [_P, _P, _P, _I32, _I64, _I64, _P, _I64, _P, _P, _P]),
    "lvsk_rowsumsq_csr_prep_bytes": (_SZ, [_I64, _I64]),
    "lvsk_rowsumsq_csr_prepare": (_I32, [_P, _I64, _I64, _P, _SZ, _P]),
    "lvsk_rowsumsq_csr_prepared": (_I32, [_P, _P, _P, _I32, _I64, _I64, _P, _I64, _P, _SZ, _P, _P, _P]),
    "lvsk_normalize_workspace_bytes": (_SZ, [_I64]),
    "lvsk_normalize_scores": (_I32, [_P, _I64, _P, _P, _P, _SZ, _P, _P]),
    "lvsk_sum_f64": (_I32, [_P, _I64, _P, _P, _SZ, _P]),
    "lvsk_split_fold": (_I32, [_P, _I64, _I64, _I32, _I64, _P, _P, _P, _P]),
    "lvsk_chol_fold_workspace_bytes": (_SZ, [_I64, _I64]),
    "lvsk_gram_workspace_bytes": (_SZ, [_I64, _I64]),
    "lvsk_syrk_workspace_bytes": (_SZ, [_I64, _I64]),
    "lvsk_syrk_f64": (_I32, [_P, _I64, _I64, _I64, _P, _I64, _P, _SZ, _P]),
    "lvsk_gram_f64": (_I32, [_P, _I64, _I64, _I64, _P, _I64, _P, _SZ, _P, _P]),
    "lvsk_gaussian_tables": (_I32, [_P, _I64]),
    "lvsk_chol_fold": (_I32, [_P, _I64, _I64, _P, _I64, _P, _P, _D, _P, _P, _SZ, _P]),
    "lvsk_argsort_workspace_bytes": (_SZ, [_I64]),
    "lvsk_argsort_f64": (_I32, [_P, _I64, _I32, _P, _P, _SZ, _P]),
    "lvsk_merge_runs_workspace_bytes": (_SZ, [_I64, _I32]),
    "lvsk_merge_argsort_runs": (_I32, [_P, _P, C.POINTER(C.c_int64), _I32, _I32, _P, _P, _SZ, _P, _P]),
}

_lib = None


def lib():
    """The loaded library (raises ImportError loudly if it was never built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} not found: build the sm_100a kernels first "
                "(python -c 'import __graft_entry__ as g; g.build()' or make -C paper_1812_07903_b200/csrc)"
            )
        handle = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGS)


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = lib().lvsk_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, RuntimeError)(f"{what}: {msg}" if what else msg)


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("levsketch_b200 needs a CUDA device (B200 / sm_100a); no CPU fallback exists")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def host_numpy(t: torch.Tensor):
    """Device tensor -> numpy array backed by pinned host memory.  The D2H is a
    direct DMA (4x a pageable copy for 8 MB vectors), and the array handed
    back to the caller travels back to the device at DMA speed too when it is
    passed to the next stage (scores -> distribution -> plan)."""
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t)
    return h.numpy()


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def dtype_code(t: torch.Tensor) -> int:
    try:
        return _DTYPE[t.dtype]
    except KeyError:
        raise errors.FormatError(f"unsupported element type {t.dtype}") from None


class Workspace:
    """Grow-only device scratch buffers reused across calls (the C ABI never
    allocates).  One buffer per (thread, device, stream): kernels queued on
    different streams, devices or host threads never share scratch memory,
    so the ABI's reentrancy holds at the Python layer too.  The caching
    allocator orders a replaced buffer's reuse after the work queued on its
    stream."""

    MAX_KEYS = 32

    def __init__(self):
        self._bufs: dict = {}

    def get(self, nbytes: int) -> torch.Tensor:
        import threading

        nbytes = max(int(nbytes), 256)
        dev = device()
        key = (threading.get_ident(), dev.index, torch.cuda.current_stream(dev).cuda_stream)
        buf = self._bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            if buf is None and len(self._bufs) >= self.MAX_KEYS:
                self._bufs.pop(next(iter(self._bufs)))  # oldest key
            buf = torch.empty(nbytes, dtype=torch.uint8, device=dev)
            self._bufs[key] = buf
        return buf


_ws = Workspace()


def workspace(nbytes: int) -> torch.Tensor:
    return _ws.get(nbytes)


class Flags:
    """One device int32 for kernel-side data errors (non-finite, negative...)."""

    def __init__(self):
        self.t = torch.zeros(1, dtype=torch.int32, device=device())

    @property
    def p(self) -> int:
        return self.t.data_ptr()

    def read(self) -> int:
        return int(self.t.item())


def hash_blocks(blocks) -> C.Array:
    arr = (HashBlock * len(blocks))()
    for i, (a, b, key, off, size) in enumerate(blocks):
        arr[i] = HashBlock(a, b, key, off, size)
    return arr


if os.environ.get("LVSK_EAGER_LOAD"):
    lib()
