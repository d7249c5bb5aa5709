"""Out-of-core leverage scores: two streaming passes over row blocks.

SURVEY.md section 8(f) row 2 (next after the hot path): the reference reads
the whole matrix into memory (matrix.py:120-133 LVSK binary, 141-179 CSV)
and then sketches it in chunks through ``consume_rows`` (sketch.py:289-312).
Here the rows stay on the host (an LVSK file is memory-mapped, or any array /
block iterator is used) and only a block at a time lives in HBM:

* pass 1 - each block is copied to a pinned staging buffer, sent to the device
  on a copy stream while the previous block is sketched (``consume_rows`` with
  its global row offset, so the state is the same one a single call makes:
  bit-identical for the hashed families);
* the small fold (``sketch_fold``) on the finished sketch;
* pass 2 - the blocks stream again through the leverage pass (K5) and the
  scores come back into one pinned host array.

n is bounded by host memory / the file, not by HBM. Scores equal those of
``leverage_sketched_trunc`` on the whole matrix (row-independent second pass).
"""

from __future__ import annotations

import time
from pathlib import Path

import numpy as np
import torch

from . import _native as N
from .errors import ConfigurationError, DimensionMismatchError, FormatError
from .leverage import LeverageResult, jl_device, scores_device, sketch_fold
from .matrix import _HEADER, BINARY_VERSION, MAGIC
from .sketch import SketchSpec, SketchState, consume_rows

_DTYPES = {torch.float64: np.float64, torch.float32: np.float32}


def open_lvsk(path) -> np.ndarray:
    """Memory-map an LVSK binary matrix (reference matrix.py:120-133 layout:
    header <4sIQQ magic, version, n, d> then n*d little-endian float64)."""
    path = Path(path)
    with open(path, "rb") as f:
        head = f.read(_HEADER.size)
    if len(head) != _HEADER.size:
        raise FormatError(f"{path}: truncated header")
    magic, version, n, d = _HEADER.unpack(head)
    if magic != MAGIC:
        raise FormatError(f"{path}: bad magic {magic!r}")
    if version != BINARY_VERSION:
        raise FormatError(f"{path}: unsupported version {version}")
    if path.stat().st_size < _HEADER.size + 8 * n * d:
        raise FormatError(f"{path}: expected {n * d} values")
    return np.memmap(path, dtype="<f8", mode="r", offset=_HEADER.size, shape=(n, d))


class _Stager:
    """Two pinned host buffers + a copy stream: block i+1 is copied while block
    i is consumed; ``get`` returns the device block for the current stream."""

    def __init__(self, rows: int, d: int, dtype: torch.dtype, dev: torch.device):
        self.host = [torch.empty((rows, d), dtype=dtype, pin_memory=True) for _ in range(2)]
        self.dev = [torch.empty((rows, d), dtype=dtype, device=dev) for _ in range(2)]
        self.copy = torch.cuda.Stream(device=dev)
        self.done = [torch.cuda.Event(), torch.cuda.Event()]
        self.free = [torch.cuda.Event(), torch.cuda.Event()]
        self.np_dtype = _DTYPES[dtype]
        for e in self.free:
            e.record(torch.cuda.current_stream())

    def put(self, slot: int, block: np.ndarray) -> None:
        m = block.shape[0]
        self.free[slot].synchronize()  # the device buffer and the pinned buffer are reusable
        np.copyto(self.host[slot][:m].numpy(), block, casting="same_kind")
        with torch.cuda.stream(self.copy):
            self.dev[slot][:m].copy_(self.host[slot][:m], non_blocking=True)
            self.done[slot].record(self.copy)

    def get(self, slot: int, m: int) -> torch.Tensor:
        torch.cuda.current_stream().wait_event(self.done[slot])
        return self.dev[slot][:m]

    def release(self, slot: int) -> None:
        self.free[slot].record(torch.cuda.current_stream())


def _blocks(a, block_rows: int):
    n = a.shape[0]
    for r0 in range(0, n, block_rows):
        yield r0, np.asarray(a[r0 : min(n, r0 + block_rows)])


def leverage_streamed(a, spec: SketchSpec, sv_tol: float | None, *, block_rows: int = 1 << 18,
                      dtype: torch.dtype = torch.float64, jl_dim: int | None = None, jl_seed: int = 0,
                      rank: int | None = None) -> LeverageResult:
    """Sketched (truncated) leverage scores of a host-resident matrix in two
    streaming passes.  ``a``: an LVSK path, a numpy array or memmap (n x d).
    ``dtype``: the device arithmetic type of the rows (float64 keeps the
    reference's arithmetic; float32 halves the transfer)."""
    t0 = time.perf_counter()
    if isinstance(a, (str, Path)):
        a = open_lvsk(a)
    if not hasattr(a, "shape") or len(a.shape) != 2:
        raise DimensionMismatchError("need a 2-D matrix")
    if dtype not in _DTYPES:
        raise ConfigurationError(f"unsupported block dtype {dtype}")
    if block_rows < 1:
        raise ConfigurationError(f"block_rows must be positive, got {block_rows}")
    n, d = a.shape
    if d != spec.d:
        raise DimensionMismatchError(f"matrix has {d} columns, spec expects {spec.d}")
    dev = N.device()
    rows = min(block_rows, n)
    st = _Stager(rows, d, dtype, dev)

    # pass 1: sketch
    state = SketchState(spec, n)
    it = _blocks(a, rows)
    pending = next(it, None)
    slot = 0
    if pending is not None:
        st.put(slot, pending[1])
    while pending is not None:
        r0, blk = pending
        nxt = next(it, None)
        if nxt is not None:
            st.put(slot ^ 1, nxt[1])
        consume_rows(state, st.get(slot, blk.shape[0]), r0)
        st.release(slot)
        pending, slot = nxt, slot ^ 1

    # fold
    pi = None if jl_dim is None else jl_device(jl_seed, d, jl_dim)
    M, eff = sketch_fold(state.data_device, sv_tol, rank, pi)

    # pass 2: leverage pass, scores back into one pinned host array
    scores = torch.empty(n, dtype=torch.float64, pin_memory=True)
    out = torch.empty(rows, dtype=torch.float64, device=dev)
    it = _blocks(a, rows)
    pending = next(it, None)
    slot = 0
    if pending is not None:
        st.put(slot, pending[1])
    while pending is not None:
        r0, blk = pending
        m = blk.shape[0]
        nxt = next(it, None)
        if nxt is not None:
            st.put(slot ^ 1, nxt[1])
        scores_device(st.get(slot, m), M, out=out[:m])
        scores[r0 : r0 + m].copy_(out[:m])  # synchronous: `out` is reused by the next block
        st.release(slot)
        pending, slot = nxt, slot ^ 1
    return LeverageResult(scores=scores.numpy(), method="sketch" if sv_tol is None else "sketch_trunc",
                          effective_rank=eff, eps=spec.eps, spec=spec, sv_tol=sv_tol,
                          wall_time_s=time.perf_counter() - t0)


__all__ = ["leverage_streamed", "open_lvsk"]
