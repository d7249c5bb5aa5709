"""CSR row blocks on the device (extension G2: BASELINE config 4).

The reference only accepts dense rows (matrix.py:30-39); on sparse data its
semantics are those of ``consume_rows`` on the densified rows
(sketch.py:289-312).  ``CSRMatrix`` carries a canonical CSR matrix
(int64 row pointers, int32 strictly increasing column indices per row,
float32/float64 values) on the device; the K2 / K6 kernels in csrc/csr.cu
sketch and score it without densifying, bit-exactly equal to the dense path.
Accepted inputs: ``CSRMatrix``, scipy.sparse CSR matrices, or a tuple
``(indptr, indices, data, (n, d))`` of numpy arrays / torch tensors.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .errors import DimensionMismatchError, FormatError


class CSRMatrix:
    def __init__(self, indptr, indices, data, shape):
        dev = N.device()
        self.indptr = _as(indptr, torch.int64, dev)
        self.indices = _as(indices, torch.int32, dev)
        d = data if isinstance(data, torch.Tensor) else np.asarray(data)
        dt = torch.float32 if (getattr(d, "dtype", None) in (np.float32, torch.float32)) else torch.float64
        self.data = _as(data, dt, dev)
        self.shape = (int(shape[0]), int(shape[1]))
        if self.indptr.dim() != 1 or self.indptr.numel() != self.shape[0] + 1:
            raise DimensionMismatchError(f"indptr has {self.indptr.numel()} entries, expected {self.shape[0] + 1}")
        if self.shape[0] < 1 or self.shape[1] < 1:
            raise FormatError(f"CSR matrix must be non-empty, got shape {self.shape}")
        if self.indices.numel() != self.data.numel():
            raise DimensionMismatchError("indices and data lengths differ")

    @property
    def n(self) -> int:
        return self.shape[0]

    @property
    def d(self) -> int:
        return self.shape[1]

    @property
    def nnz(self) -> int:
        return int(self.indices.numel())

    def rows(self, lo: int, hi: int) -> "CSRMatrix":
        """Row block [lo, hi) sharing storage (the kernels rebase on indptr[0])."""
        sub = CSRMatrix.__new__(CSRMatrix)
        sub.indptr = self.indptr[lo : hi + 1]
        base = int(sub.indptr[0])
        sub.indices = self.indices[base:]
        sub.data = self.data[base:]
        sub.shape = (hi - lo, self.shape[1])
        return sub

    def to_dense(self) -> torch.Tensor:
        out = torch.zeros(self.shape, dtype=self.data.dtype, device=self.data.device)
        base = int(self.indptr[0])
        counts = (self.indptr[1:] - self.indptr[:-1]).to(torch.int64)
        rows = torch.repeat_interleave(torch.arange(self.n, device=out.device), counts)
        nnz = int(counts.sum())
        out[rows, self.indices[:nnz].to(torch.int64)] = self.data[:nnz]
        _ = base
        return out

    @classmethod
    def from_any(cls, obj):
        if isinstance(obj, CSRMatrix):
            return obj
        if hasattr(obj, "indptr") and hasattr(obj, "indices") and hasattr(obj, "data") and hasattr(obj, "shape"):
            if getattr(obj, "format", "csr") != "csr":
                obj = obj.tocsr()
            m = obj.copy()
            m.sort_indices()
            m.sum_duplicates()
            return cls(m.indptr.astype(np.int64), m.indices.astype(np.int32), m.data, m.shape)
        if isinstance(obj, tuple) and len(obj) == 4:
            return cls(*obj)
        return None


def _as(x, dtype, dev):
    if isinstance(x, torch.Tensor):
        t = x.detach()
    else:
        t = torch.from_numpy(np.ascontiguousarray(x))
    return t.to(dev, dtype).contiguous()


def is_csr(obj) -> bool:
    return CSRMatrix.from_any(obj) is not None if not isinstance(obj, (np.ndarray, torch.Tensor, list)) else False


def csr_code(m: CSRMatrix) -> int:
    return N.LVSK_F32 if m.data.dtype == torch.float32 else N.LVSK_F64


def csr_prepare(Mf: torch.Tensor) -> torch.Tensor | None:
    """The bf16 operand images of M's hot column window for the prepared K6
    pass (``lvsk_rowsumsq_csr_prepare``), or None when the pass does not apply
    (r != 128).  Built once per fold; ``Mf`` is the contiguous float32 d x r M."""
    d, r = Mf.shape
    nbytes = int(N.lib().lvsk_rowsumsq_csr_prep_bytes(d, r))
    if nbytes == 0 or Mf.data_ptr() % 16:
        return None
    prep = torch.empty(nbytes, dtype=torch.uint8, device=Mf.device)
    N.check(N.lib().lvsk_rowsumsq_csr_prepare(Mf.data_ptr(), d, r, prep.data_ptr(), nbytes, N.stream_ptr()),
            "csr leverage operand")
    return prep


def csr_scores(m: CSRMatrix, M: torch.Tensor, out: torch.Tensor | None = None, flags=None) -> torch.Tensor:
    """K6: ||x_i M||^2 for CSR rows (fp32 M gathers, fp32 accumulation)."""
    if M.shape[0] != m.d:
        raise DimensionMismatchError(f"basis has {M.shape[0]} rows, expected {m.d}")
    Mf = M.to(torch.float32).contiguous()
    out = torch.empty(m.n, dtype=torch.float64, device=Mf.device) if out is None else out
    own = flags is None
    flags = flags or N.Flags()
    prep = csr_prepare(Mf)
    if prep is not None:  # r = 128: the hot column window on tcgen05 (K6-TC v2)
        N.check(N.lib().lvsk_rowsumsq_csr_prepared(m.indptr.data_ptr(), m.indices.data_ptr(), m.data.data_ptr(),
                                                   csr_code(m), m.n, m.d, Mf.data_ptr(), Mf.shape[1], prep.data_ptr(),
                                                   prep.numel(), out.data_ptr(), flags.p, N.stream_ptr()),
                "csr leverage pass")
    else:
        N.check(N.lib().lvsk_rowsumsq_csr(m.indptr.data_ptr(), m.indices.data_ptr(), m.data.data_ptr(), csr_code(m),
                                          m.n, m.d, Mf.data_ptr(), Mf.shape[1], out.data_ptr(), flags.p,
                                          N.stream_ptr()),
                "csr leverage pass")
    if own:
        _raise_flags(flags.read())
    return out


def _raise_flags(f: int) -> None:
    if f & N.FLAG_BADINDEX:
        raise FormatError("CSR rows need strictly increasing column indices in [0, d)")
    if f & N.FLAG_NONFINITE:
        raise FormatError("CSR matrix contains non-finite entries")
