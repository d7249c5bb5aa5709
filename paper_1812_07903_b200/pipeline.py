"""Preallocated device-resident leverage pipeline (the bench / serving path).

One ``run(X)`` is the whole hot path of reference leverage_sketched_trunc +
scores_to_distribution + make_plan("dec") (leverage.py:115-132,
order.py:51-100) on a CUDA-resident X:

    sketch (K1 | K3 | K4) -> fold SX -> fp64 factorisation (cuSOLVER)
    -> truncate + fold M -> K5 leverage pass -> normalise -> K7 argsort

All buffers and workspaces are allocated once in the constructor; the only
host synchronisations per run are the factorisation's (cuSOLVER returns
its spectrum to pick the truncation rank) and the final flag check.
"""

from __future__ import annotations

import math
import os

import numpy as np
import torch

from . import _native as N
from .errors import FormatError, UncertifiedFoldError
from .leverage import FoldGraph, KernelOperands, jl_device, sketch_fold
from .csr import CSRMatrix, csr_code, csr_prepare
from .sketch import GAUSSIAN, SRHT, SketchSpec, SketchState, sketch_rows

STAGES = ("sketch", "factor", "leverage", "order")
# LVSK_NVTX=1: one NVTX range per stage (sketch / factor / leverage / order) for
# Nsight timelines (SURVEY §5 tracing); off by default (host cost per range)
_NVTX = os.environ.get("LVSK_NVTX", "0") == "1"


class LeveragePipeline:
    def __init__(self, spec: SketchSpec, n: int, d: int, dtype=torch.float32, sv_tol: float = 1e-6,
                 jl_dim: int | None = None, jl_seed: int = 0, rank: int | None = None, order: bool = True,
                 row0: int = 0, factor_method: str = "auto"):
        if d != spec.d:
            raise ValueError(f"spec.d={spec.d} but d={d}")
        self.spec, self.n, self.d, self.dtype = spec, n, d, dtype
        self.sv_tol, self.rank, self.order, self.row0 = sv_tol, rank, order, row0
        self.factor_method = factor_method
        self.k = sketch_rows(spec)
        dev = N.device()
        self.dev = dev
        self.state = SketchState(spec, n, mem_cap=1 << 62)
        self.sx = torch.empty((self.k, d), dtype=torch.float64, device=dev)
        code = {torch.float32: N.LVSK_F32, torch.float64: N.LVSK_F64, torch.bfloat16: N.LVSK_BF16}[dtype]
        self.code = code
        L = N.lib()
        if spec.family == SRHT:
            wsb = L.lvsk_srht_workspace_bytes(self.state._m, d, code, self.k)
        elif spec.family == GAUSSIAN:
            wsb = L.lvsk_gaussian_workspace_bytes(n, d, self.k, code)
        else:
            wsb = max(L.lvsk_hashed_workspace_bytes(n, spec.s, self.k), L.lvsk_hashed_csr_workspace_bytes(n, spec.s, self.k))
        self.ws_sketch = torch.empty(max(wsb, 256), dtype=torch.uint8, device=dev)
        self.scores = torch.empty(n, dtype=torch.float64, device=dev)
        self.p = torch.empty(n, dtype=torch.float64, device=dev)
        self.total = torch.empty(1, dtype=torch.float64, device=dev)
        self.idx = torch.empty(n, dtype=torch.int64, device=dev)
        self.ws_norm = torch.empty(max(L.lvsk_normalize_workspace_bytes(n), 256), dtype=torch.uint8, device=dev)
        self.ws_sort = torch.empty(max(L.lvsk_argsort_workspace_bytes(n), 256), dtype=torch.uint8, device=dev)
        self.flags = torch.zeros(1, dtype=torch.int32, device=dev)
        self.pi = None if jl_dim is None else jl_device(jl_seed, d, jl_dim)
        # a dtype/alignment witness for choosing the K5 kernel (real X has the same layout)
        self._x_like = torch.empty((1, d), dtype=dtype, device=dev)
        self._fold_graph = None
        self._cert_pending = False
        self._cert_fails_seen = 0  # certificate failures already accounted for by check()
        self._last_X = None
        self._m32 = None
        self._m32_src = None
        self._m32_prep = None
        self.effective_rank = None
        # keep_state: also write the compensated pair (hi, lo) of the sketch
        # (multi-rank merges need it); otherwise K1 writes the folded SX only
        self.keep_state = False
        self.events = {s: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for s in STAGES}

    # -- stages ------------------------------------------------------------
    def _sketch(self, X) -> None:
        L, st, s = N.lib(), N.stream_ptr(), self.state
        fam = self.spec.family
        if isinstance(X, CSRMatrix):
            # a fresh state each run: NULL (hi_in, lo_in) = zeros, no memset and no state read;
            # without keep_state K2 writes the folded SX straight away (no state pair, no fold pass)
            keep = self.keep_state
            N.check(L.lvsk_hashed_sketch_csr(X.indptr.data_ptr(), X.indices.data_ptr(), X.data.data_ptr(),
                                             csr_code(X), X.n, X.d, self.row0, s._blocks, self.spec.s, s._scale,
                                             None, None, s._hi.data_ptr() if keep else self.sx.data_ptr(),
                                             s._lo.data_ptr() if keep else None,
                                             self.k, self.ws_sketch.data_ptr(), self.ws_sketch.numel(),
                                             self.flags.data_ptr(), st), "csr sketch")
            if keep:
                N.check(L.lvsk_fold_compensated(s._hi.data_ptr(), s._lo.data_ptr(), self.sx.data_ptr(),
                                                self.sx.numel(), st), "fold")
            return
        ldx = X.stride(0)
        if fam == SRHT:
            N.check(L.lvsk_srht(X.data_ptr(), self.code, self.n, self.d, ldx, s._m, s._signs_dev.data_ptr(),
                                s._sample_dev.data_ptr(), self.k, math.sqrt(self.k), self.sx.data_ptr(),
                                self.ws_sketch.data_ptr(), self.ws_sketch.numel(), self.flags.data_ptr(), st), "srht")
        elif fam == GAUSSIAN:
            N.check(L.lvsk_gaussian_sketch(X.data_ptr(), self.code, self.n, self.d, ldx, self.row0, self.spec.seed,
                                           self.k, self.sx.data_ptr(), 0, self.ws_sketch.data_ptr(),
                                           self.ws_sketch.numel(), self.flags.data_ptr(), st), "gaussian")
        elif self.keep_state:  # a fresh state each run: NULL (hi_in, lo_in) = zeros, no memset and no state read
            N.check(L.lvsk_hashed_sketch(X.data_ptr(), self.code, self.n, self.d, ldx, self.row0, s._blocks,
                                         self.spec.s, s._scale, None, None, s._hi.data_ptr(),
                                         s._lo.data_ptr(), self.k, self.ws_sketch.data_ptr(), self.ws_sketch.numel(),
                                         self.flags.data_ptr(), st), "hashed sketch")
            N.check(L.lvsk_fold_compensated(s._hi.data_ptr(), s._lo.data_ptr(), self.sx.data_ptr(), self.sx.numel(), st),
                    "fold")
        else:  # only SX is needed: K1 writes the folded hi + lo straight into it (no state pair, no fold pass)
            N.check(L.lvsk_hashed_sketch(X.data_ptr(), self.code, self.n, self.d, ldx, self.row0, s._blocks,
                                         self.spec.s, s._scale, None, None, self.sx.data_ptr(), None, self.k,
                                         self.ws_sketch.data_ptr(), self.ws_sketch.numel(), self.flags.data_ptr(), st),
                    "hashed sketch")

    def _factor(self) -> None:
        k, d = self.sx.shape
        # a certificate still pending from an earlier run(check=False) is not
        # dropped: the KF kernel counts failures on the device (cert_fail) and
        # check() raises if any run other than the last one was uncertified
        if (self.factor_method == "auto" and self.pi is not None and self.rank is None and k >= d
                and os.environ.get("LVSK_NO_GRAPH", "0") != "1"):
            if self._fold_graph is None:
                self._fold_graph = FoldGraph(self.sx, self.sv_tol, self.pi, self._x_like)
            # optimistic: the leverage pass runs on R^-1 Pi right away and the
            # certificate is verified in check(); a failed certificate redoes
            # the fold (spectral route) and the passes after it
            self._fold_graph.replay()
            self._cert_pending = True
            self.ops = self._fold_graph.ops
            self.r = self.ops.r
            self.effective_rank = d
            return
        M, self.effective_rank = sketch_fold(self.sx, self.sv_tol, self.rank, self.pi, self.factor_method)
        self.set_fold(M)

    def cert_failures(self) -> int:
        """Runs whose optimistic Cholesky fold failed its certificate (device count)."""
        return int(self._fold_graph.cert_fail.item()) if self._fold_graph is not None else 0

    def _verify_fold(self) -> None:
        if not self._cert_pending:
            return
        self._cert_pending = False
        fails = self.cert_failures()
        last_ok = self._fold_graph.certified()
        earlier = fails - self._cert_fails_seen - (0 if last_ok else 1)
        self._cert_fails_seen = fails
        if earlier > 0:
            raise UncertifiedFoldError(
                f"{earlier} earlier run(check=False) result(s) came from a Cholesky fold whose certificate failed; "
                "call check() after each run (or run(check=True)) when the sketch may be ill-conditioned")
        if last_ok:
            return
        M, self.effective_rank = sketch_fold(self.sx, self.sv_tol, self.rank, self.pi, "qr")
        self.set_fold(M)
        # the optimistic passes ran on an uncertified (possibly non-finite) fold;
        # their flags are void — the leverage pass re-checks X itself
        self.flags.zero_()
        self._leverage(self._last_X)
        if self.order:
            self._order()

    def set_fold(self, M: torch.Tensor) -> None:
        self.ops = KernelOperands(M, self._x_like)
        self.r = M.shape[1]

    def _leverage(self, X) -> None:
        if isinstance(X, CSRMatrix):
            # the fold graph rewrites its operands in place on every replay: M is new each run
            replayed = self._fold_graph is not None and self.ops is self._fold_graph.ops
            if self._m32 is None or self._m32_src is not self.ops or replayed:
                self._m32 = (self.ops.a.T.double() + self.ops.b.T.double()).to(torch.float32).contiguous() \
                    if self.ops.tc else self.ops.a.to(torch.float32).contiguous()
                self._m32_src = self.ops
                self._m32_prep = csr_prepare(self._m32)
            if self._m32_prep is not None:
                N.check(N.lib().lvsk_rowsumsq_csr_prepared(X.indptr.data_ptr(), X.indices.data_ptr(),
                                                           X.data.data_ptr(), csr_code(X), X.n, X.d,
                                                           self._m32.data_ptr(), self._m32.shape[1],
                                                           self._m32_prep.data_ptr(), self._m32_prep.numel(),
                                                           self.scores.data_ptr(), self.flags.data_ptr(),
                                                           N.stream_ptr()), "csr leverage pass")
                return
            N.check(N.lib().lvsk_rowsumsq_csr(X.indptr.data_ptr(), X.indices.data_ptr(), X.data.data_ptr(),
                                              csr_code(X), X.n, X.d, self._m32.data_ptr(), self._m32.shape[1],
                                              self.scores.data_ptr(), self.flags.data_ptr(), N.stream_ptr()),
                    "csr leverage pass")
            return
        self.ops.run(X, self.scores, self.flags.data_ptr())

    def _order(self) -> None:
        L, st = N.lib(), N.stream_ptr()
        N.check(L.lvsk_normalize_scores(self.scores.data_ptr(), self.n, self.p.data_ptr(), self.total.data_ptr(),
                                        self.ws_norm.data_ptr(), self.ws_norm.numel(), self.flags.data_ptr(), st),
                "normalize")
        N.check(L.lvsk_argsort_f64(self.p.data_ptr(), self.n, 1, self.idx.data_ptr(), self.ws_sort.data_ptr(),
                                   self.ws_sort.numel(), st), "argsort")

    # -- public --------------------------------------------------------------
    def run(self, X: torch.Tensor, timing: bool = False, check: bool = True):
        """Full pass over device-resident X (n x d, self.dtype).  Returns
        (scores, order) CUDA tensors (order is None when order=False)."""
        if isinstance(X, CSRMatrix):
            if X.shape != (self.n, self.d):
                raise ValueError(f"expected a ({self.n}, {self.d}) CSR matrix")
        elif X.shape != (self.n, self.d) or X.dtype != self.dtype or X.stride(1) != 1:
            raise ValueError(f"expected a ({self.n}, {self.d}) {self.dtype} row-major CUDA tensor")
        self.flags.zero_()
        self._last_X = X
        ev = self.events
        steps = [("sketch", lambda: self._sketch(X)), ("factor", self._factor), ("leverage", lambda: self._leverage(X))]
        if self.order:
            steps.append(("order", self._order))
        nvtx = _NVTX
        for name, fn in steps:
            if nvtx:
                torch.cuda.nvtx.range_push(f"levsketch.{name}")
            if timing:
                ev[name][0].record()
            fn()
            if timing:
                ev[name][1].record()
            if nvtx:
                torch.cuda.nvtx.range_pop()
        if check:
            self.check()
        return self.scores, (self.idx if self.order else None)

    def stage_ms(self) -> dict:
        torch.cuda.synchronize()
        out = {}
        for name in STAGES:
            a, b = self.events[name]
            try:
                out[name] = a.elapsed_time(b)
            except RuntimeError:
                pass
        return out

    def check(self) -> None:
        """Verify the fold certificate of the last run (redoing the fold and the
        passes after it if it failed), raise UncertifiedFoldError if an earlier
        unchecked run used an uncertified fold, and raise on flagged input
        errors."""
        self._verify_fold()
        f = int(self.flags.item())
        if f & N.FLAG_BADINDEX:
            raise FormatError("CSR rows need strictly increasing column indices in [0, d)")
        if f & N.FLAG_NONFINITE:
            raise FormatError("matrix contains non-finite entries")

    def launches_per_run(self, csr: bool = False) -> int:
        """Kernels this library launches per run() (host-side count; csr: the
        input is a CSRMatrix — K2 adds the row-metadata pass and never uses
        the cooperative grouping)."""
        fam = self.spec.family
        radix = lambda items, bits: 3 * max(1, (bits + 7) // 8)  # noqa: E731
        if fam == SRHT:
            m = self.state._m
            L = int(math.log2(m))
            cb = 8 if L <= 8 else min(L, 16)
            chunks = max(1, -(-self.n // (1 << cb)))
            sk = 1 + radix(self.k, 8) + 1 + 2 * chunks
        elif fam == GAUSSIAN:
            # fp32 X on the tensor cores: split3 + one K4-TC launch over the stacked planes + reduce
            # (csrc/gaussian.cu f32_tc; LVSK_NO_TC is a test-only switch)
            planes = 3 * (-(-self.n // 64) * 64) * (-(-self.d // 8) * 8) * 2
            sk = 3 if (self.code == N.LVSK_F32 and self.k >= 64 and self.n >= 256 and planes <= 3 << 30
                       and "LVSK_NO_TC" not in os.environ) else 2
        else:
            # grouping: one cooperative counting sort (k <= 4096, s <= 64; csrc/sketch_hashed.cu)
            # or keygen + radix passes + bucket bounds; then the gather (K1) and the hi+lo fold
            coop = self.k <= 4096 and self.spec.s <= 64 and not os.environ.get("LVSK_GROUP_RADIX") and not csr
            group = 1 if coop else 1 + radix(self.n * self.spec.s, max(1, (self.k - 1).bit_length())) + 1
            sk = group + (1 if csr else 0) + 1 + (1 if self.keep_state else 0)
        lev = 1
        k, d = self.sx.shape
        # the Gram (KG: colmax, colexp, slice, gram_i8; KD: syrk [+ its slice reduce]),
        # KF (chol_fold_kernel) and the K5 operand split (split_fold_kernel)
        fold = 0
        if self.pi is not None and self.rank is None and k >= d:
            from .leverage import use_kg
            gram = 4 if use_kg(k, d) else (2 if N.lib().lvsk_syrk_workspace_bytes(k, d) > 0 else 1)
            fold = gram + 2
        # normalise (2-stage sum + divide), then K7: one cooperative kernel up to 8M keys
        coop_sort = self.n <= (8 << 20) and not os.environ.get("LVSK_ARGSORT_CLASSIC")
        order_ = (3 + (1 if coop_sort else 1 + radix(self.n, 64))) if self.order else 0
        return sk + fold + lev + order_


class BatchRunner:
    """Independent passes (batches) kept in flight on ``slots`` streams.

    Each slot owns a ``LeveragePipeline`` (its own sketch state, fold graph,
    scores and order buffers) and a CUDA stream; ``submit(X)`` runs one full
    pass over X on the next slot, so the latency-bound stages of one pass (the
    fold: KD + KF; the order: K7) run beside the HBM-bound stages (K1 / K3 /
    K4 / K5) of the next one.  The C library is told how many passes are in
    flight (``lvsk_set_inflight``) so its cooperative kernels leave SMs to the
    other stream; results are bit-identical to ``LeveragePipeline.run``.  A
    slot is reused only after its stream finished the previous pass (stream
    order), and ``result(i)`` / ``drain()`` synchronise with it.  No reference
    counterpart (the reference runs one pass at a time on the host)."""

    def __init__(self, *args, slots: int = 2, **kwargs):
        if slots < 1:
            raise ValueError("slots must be >= 1")
        self.pipes = [LeveragePipeline(*args, **kwargs) for _ in range(slots)]
        self.streams = [torch.cuda.Stream(device=self.pipes[0].dev) for _ in range(slots)]
        self.slots = slots
        self._next = 0
        self._done = [None] * slots
        N.check(N.lib().lvsk_set_inflight(slots), "set_inflight")

    def submit(self, X, timing: bool = False) -> int:
        """Run one pass over X (device-resident; the caller keeps X alive and
        unmodified until the slot's pass completed) on the next slot; returns
        the slot index.  Inputs written on the caller's stream are visible."""
        i = self._next
        self._next = (i + 1) % self.slots
        st = self.streams[i]
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            self.pipes[i].run(X, timing=timing, check=False)
            ev = torch.cuda.Event()
            ev.record()
        self._done[i] = ev
        return i

    def drain(self) -> None:
        """Make the caller's stream wait for every pass in flight."""
        cur = torch.cuda.current_stream()
        for ev in self._done:
            if ev is not None:
                cur.wait_event(ev)

    def result(self, slot: int):
        """(scores, order) of the slot's last pass after its certificate check
        (redoing the fold if it failed, as LeveragePipeline.check)."""
        self.drain()
        p = self.pipes[slot]
        with torch.cuda.stream(self.streams[slot]):
            p.check()
        torch.cuda.current_stream().wait_stream(self.streams[slot])
        return p.scores, (p.idx if p.order else None)

    def check(self) -> None:
        for i in range(self.slots):
            self.result(i)

    def close(self) -> None:
        """Back to one pass in flight (the library-wide hint)."""
        self.drain()
        N.check(N.lib().lvsk_set_inflight(1), "set_inflight")
