"""Row-partitioned distributed sketching in the coordinator model, on GPUs.

Drop-in for the reference module (pkg/src/levsketch/dist.py:26-151).  The
reference's workers are threads exchanging in-memory values; here a worker
is one CUDA rank (one process per GPU, ``torch.distributed`` over NCCL /
NVLink):

* each rank sketches its contiguous partition with GLOBAL row indices
  (identical hash assignments to a serial pass, dist.py:106-107);
* boundary #1 (dist.py:114-118): the compensated (hi, lo) partials are cut
  into world row slices and exchanged all-to-all; rank q folds ``merge`` over
  slice q in ascending rank order (the reference's exact TwoSum fold, so the
  merged sketch equals the reference's bit-for-bit — an NCCL sum would
  reassociate) and the merged slices are all-gathered (Gaussian partials,
  plain sums, are all-gathered and added in rank order);
* one rank factorises; boundary #2 (dist.py:125): the d x r fold M is
  broadcast;
* scores stay rank-local (concatenation order = rank order, dist.py:128);
  ``run_distributed`` all-gathers them only because its contract returns the
  full vector.

Without an initialised process group (or with ``workers`` != world size) the
partitions run one after another on the local device — the reference's
"simulate ranks and compare to serial" mode.

The coordination logic is written against a small ``ops`` interface so the
multi-process path is exercised on CPU (gloo) in tests with the oracle as
the compute; the product binds :class:`DeviceOps` (CUDA kernels only).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as tdist

from . import _native as N
from .errors import ConfigurationError, UnsupportedFamilyError
from .leverage import LeverageResult, factor_device, jl_device, scores_device, sketch_fold
from .matrix import device_matrix
from .sketch import COUNTSKETCH, GAUSSIAN, OSNAP, SketchSpec, SketchState, consume_rows, merge

DIST_FAMILIES = (COUNTSKETCH, OSNAP, GAUSSIAN)  # gaussian: extension (linear, mergeable)


@dataclass
class Partition:
    worker_id: int
    lo: int
    hi: int
    rows: object  # the worker's block (device tensor view)


@dataclass
class CoordinatorReport:
    merged: SketchState
    basis_sigma: np.ndarray
    basis_vt: np.ndarray
    workers: int
    per_worker_times: list[float]
    merge_time: float
    svd_time: float
    score_time: float
    bytes_communicated: int
    per_worker_rows: list[int] = field(default_factory=list)

    def to_json_dict(self) -> dict:
        return {
            "workers": self.workers,
            "per_worker_times_s": self.per_worker_times,
            "merge_time_s": self.merge_time,
            "svd_time_s": self.svd_time,
            "score_time_s": self.score_time,
            "bytes_communicated": self.bytes_communicated,
            "per_worker_rows": self.per_worker_rows,
            "sketch": {
                "family": self.merged.spec.family,
                "k": self.merged.k,
                "d": self.merged.d,
                "eps": self.merged.spec.eps,
                "seed": self.merged.spec.seed,
            },
        }


def partition_rows(n: int, w: int) -> list[tuple[int, int]]:
    """[0, n) as w contiguous ranges, sizes differing by at most 1 (dist.py:66-79)."""
    if w < 1:
        raise ConfigurationError(f"need at least one worker, got {w}")
    if w > n:
        raise ConfigurationError(f"cannot split {n} rows across {w} workers")
    base, rem = divmod(n, w)
    out, lo = [], 0
    for p in range(w):
        hi = lo + base + (1 if p < rem else 0)
        out.append((lo, hi))
        lo = hi
    return out


# ---------------------------------------------------------------------------
# compute interface


class DeviceOps:
    """CUDA implementation of the per-rank compute steps."""

    def __init__(self, spec: SketchSpec, n_total: int, sv_tol: float, jl_dim=None, jl_seed=0, rank=None,
                 mem_cap_bytes=None):
        self.spec, self.n, self.sv_tol = spec, n_total, sv_tol
        self.jl_dim, self.jl_seed, self.rank, self.mem_cap = jl_dim, jl_seed, rank, mem_cap_bytes

    def sketch(self, rows, row0: int) -> SketchState:
        st = SketchState(self.spec, self.n, mem_cap=self.mem_cap)
        return consume_rows(st, rows, row0)

    @staticmethod
    def payload(state: SketchState) -> list[torch.Tensor]:
        return [state._acc] if state.spec.family == GAUSSIAN else [state._hi, state._lo]

    def from_payload(self, tensors, rows_consumed: int) -> SketchState:
        st = SketchState(self.spec, self.n)
        if self.spec.family == GAUSSIAN:
            st._acc = tensors[0]
        else:
            st._hi, st._lo = tensors
        st.rows_consumed = rows_consumed
        return st

    merge = staticmethod(merge)

    @staticmethod
    def merge_arrays(h1, l1, h2, l2):
        """(h1, l1) <- TwoSum merge with (h2, l2) on raw row slices (in place)."""
        N.check(N.lib().lvsk_merge_compensated(h1.data_ptr(), l1.data_ptr(), h2.data_ptr(), l2.data_ptr(),
                                               h1.data_ptr(), l1.data_ptr(), h1.numel(), N.stream_ptr()), "merge")
        return h1, l1

    def factor(self, merged: SketchState):
        sx = merged.data_device
        pi = None if self.jl_dim is None else jl_device(self.jl_seed, self.spec.d, self.jl_dim)
        M, _ = sketch_fold(sx, self.sv_tol, self.rank, pi)
        # the coordinator report carries the spectrum (reference dist.py:378-381)
        _, vt, s_host = factor_device(sx, self.sv_tol, self.rank, "svd")
        return M, s_host, vt.cpu().numpy()

    @staticmethod
    def scores(rows, M) -> torch.Tensor:
        from .csr import CSRMatrix, csr_scores

        return csr_scores(rows, M) if isinstance(rows, CSRMatrix) else scores_device(rows, M)

    @staticmethod
    def sync():
        torch.cuda.synchronize()


def _fold_in_order(ops, states):
    merged = states[0]
    for st in states[1:]:
        merged = ops.merge(merged, st)
    return merged


def coordinate(ops, local_rows, row0: int, rank: int, world: int, counts: list[int], group=None):
    """One rank's share of the coordinator protocol (boundaries #1/#2 as
    collectives).  Returns (local scores, merged state, sigma, vt, timings)."""
    t0 = time.perf_counter()
    state = ops.sketch(local_rows, row0)
    ops.sync()
    t_sketch = time.perf_counter() - t0

    t0 = time.perf_counter()
    mine = ops.payload(state)
    if len(mine) == 2 and world > 1:  # hashed (hi, lo): sliced rank-ordered merge, then gather
        h, l = sliced_merge(mine[0], mine[1], rank, world, ops.merge_arrays, group)
        k = mine[0].shape[0]
        merged = ops.from_payload([gather_row_slices(h, k, world, group), gather_row_slices(l, k, world, group)],
                                  sum(counts))
    else:
        gathered = [[torch.empty_like(t) for _ in range(world)] for t in mine]
        for slot, t in enumerate(mine):
            tdist.all_gather(gathered[slot], t.contiguous(), group=group)
        states = [ops.from_payload([gathered[s][p] for s in range(len(mine))], counts[p]) for p in range(world)]
        merged = _fold_in_order(ops, states)
    ops.sync()
    t_merge = time.perf_counter() - t0

    t0 = time.perf_counter()
    if rank == 0:
        M, s_host, vt_host = ops.factor(merged)
        shape = torch.tensor([M.shape[0], M.shape[1]], dtype=torch.int64)
    else:
        M = None
        shape = torch.zeros(2, dtype=torch.int64)
    shape = shape.to(mine[0].device)
    tdist.broadcast(shape, 0, group=group)
    if rank != 0:
        M = torch.empty((int(shape[0]), int(shape[1])), dtype=torch.float64, device=mine[0].device)
    tdist.broadcast(M, 0, group=group)
    if rank != 0:
        s_host = vt_host = None
    ops.sync()
    t_svd = time.perf_counter() - t0

    t0 = time.perf_counter()
    local = ops.scores(local_rows, M)
    ops.sync()
    t_score = time.perf_counter() - t0
    return local, merged, s_host, vt_host, (t_sketch, t_merge, t_svd, t_score)


def exchange_row_slices(t: torch.Tensor, rank: int, world: int, group=None) -> torch.Tensor:
    """all_to_all of a (k, d) partial: rank q receives row slice q
    (partition_rows(k, world)) of every rank's t, stacked in rank order as
    (world, rows_q, d) — the reduce-scatter layout of a sketch merge, with
    (world - 1) / world of one state per rank on the wire instead of an
    all-gather's (world - 1) states."""
    k, d = t.shape
    bounds = partition_rows(k, world)
    lo, hi = bounds[rank]
    out = torch.empty((world, hi - lo, d), dtype=t.dtype, device=t.device)
    tdist.all_to_all_single(out.view(-1), t.contiguous().view(-1), [(hi - lo) * d] * world,
                            [(b - a) * d for a, b in bounds], group=group)
    return out


def gather_row_slices(sl: torch.Tensor, k: int, world: int, group=None) -> torch.Tensor:
    """Inverse of the slicing: every rank gets the full (k, d) from its slices."""
    bounds = partition_rows(k, world)
    rows = max(b - a for a, b in bounds)
    d = sl.shape[1]
    if k % world == 0 and sl.is_contiguous():  # equal slices: gathered in place, rank order = row order
        out = torch.empty((k, d), dtype=sl.dtype, device=sl.device)
        tdist.all_gather_into_tensor(out, sl, group=group)
        return out
    buf = torch.zeros((rows, d), dtype=sl.dtype, device=sl.device)
    buf[: sl.shape[0]] = sl
    outs = [torch.empty_like(buf) for _ in range(world)]
    tdist.all_gather(outs, buf, group=group)
    return torch.cat([outs[q][: b - a] for q, (a, b) in enumerate(bounds)], dim=0)


def sliced_merge(hi: torch.Tensor, lo: torch.Tensor, rank: int, world: int, merge_arrays, group=None):
    """Rank q's row slice of merge_0..world-1(hi, lo): slice q of every rank's
    partial arrives by one all-to-all and is merged in rank order with the
    reference's TwoSum (merge_arrays), so each slice holds the same bits as
    the all-gather-then-fold merge (reference dist.py:114-118)."""
    his = exchange_row_slices(hi, rank, world, group)
    los = exchange_row_slices(lo, rank, world, group)
    h, l = his[0].clone(), los[0].clone()
    for q in range(1, world):
        h, l = merge_arrays(h, l, his[q], los[q])
    return h, l


def sliced_hashed_merge(hi: torch.Tensor, lo: torch.Tensor, rank: int, world: int, group=None) -> torch.Tensor:
    """Merged float64 sketch SX = fold(merge(hi, lo)) on every rank: the
    merged slice is folded (hi + lo) before the all-gather, so one k x d
    float64 array crosses the wire instead of the pair."""
    h, l = sliced_merge(hi, lo, rank, world, DeviceOps.merge_arrays, group)
    sx = torch.empty_like(h)
    N.check(N.lib().lvsk_fold_compensated(h.data_ptr(), l.data_ptr(), sx.data_ptr(), sx.numel(), N.stream_ptr()),
            "fold")
    return gather_row_slices(sx, hi.shape[0], world, group)


def gather_scores(local: torch.Tensor, counts: list[int], group=None) -> torch.Tensor:
    """Concatenate rank-local score vectors in rank order (uneven sizes)."""
    world = len(counts)
    mx = max(counts)
    buf = torch.zeros(mx, dtype=local.dtype, device=local.device)
    buf[: local.numel()] = local
    outs = [torch.empty_like(buf) for _ in range(world)]
    tdist.all_gather(outs, buf, group=group)
    return torch.cat([outs[p][: counts[p]] for p in range(world)])


def run_distributed(
    a,
    spec: SketchSpec,
    workers: int,
    sv_tol: float,
    max_threads: int | None = None,
    mem_cap_bytes: int | None = None,
    *,
    jl_dim: int | None = None,
    jl_seed: int = 0,
    rank: int | None = None,
    group=None,
) -> tuple[LeverageResult, CoordinatorReport]:
    """Truncated sketched scores over ``workers`` row partitions; identical to
    leverage_sketched_trunc(a, spec, sv_tol) for any worker count
    (reference dist.py:82-151).  ``max_threads`` is accepted for API parity;
    device partitions do not use host threads."""
    if spec.family not in DIST_FAMILIES:
        raise UnsupportedFamilyError(f"distributed sketching supports countsketch and osnap, not {spec.family!r}")
    X = device_matrix(a)
    n = X.shape[0]
    ranges = partition_rows(n, workers)
    ops = DeviceOps(spec, n, sv_tol, jl_dim, jl_seed, rank, mem_cap_bytes)
    counts = [hi - lo for lo, hi in ranges]
    multi = tdist.is_available() and tdist.is_initialized() and tdist.get_world_size(group) == workers
    if multi:
        me = tdist.get_rank(group)
        lo, hi = ranges[me]
        local, merged, s_host, vt_host, (t_sk, t_mg, t_svd, t_sc) = coordinate(
            ops, X[lo:hi], lo, me, workers, counts, group
        )
        t_all = torch.tensor([t_sk], dtype=torch.float64, device=X.device)
        times = [torch.empty_like(t_all) for _ in range(workers)]
        tdist.all_gather(times, t_all, group=group)
        per_worker = [float(t.item()) for t in times]
        scores = gather_scores(local, counts, group)
        # every rank reports the coordinator's spectrum
        s_host, vt_host = _broadcast_host(s_host, vt_host, group, X.device)
    else:
        per_worker = []
        states = []
        for p, (lo, hi) in enumerate(ranges):
            t0 = time.perf_counter()
            states.append(ops.sketch(X[lo:hi], lo))
            torch.cuda.synchronize()
            per_worker.append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        merged = _fold_in_order(ops, states)
        torch.cuda.synchronize()
        t_mg = time.perf_counter() - t0
        t0 = time.perf_counter()
        M, s_host, vt_host = ops.factor(merged)
        t_svd = time.perf_counter() - t0
        t0 = time.perf_counter()
        scores = torch.cat([ops.scores(X[lo:hi], M) for lo, hi in ranges])
        torch.cuda.synchronize()
        t_sc = time.perf_counter() - t0
    result = LeverageResult(
        scores=N.host_numpy(scores),
        method="sketch_trunc",
        effective_rank=int(s_host.shape[0]),
        eps=spec.eps,
        spec=spec,
        sv_tol=sv_tol,
    )
    report = CoordinatorReport(
        merged=merged,
        basis_sigma=s_host,
        basis_vt=vt_host,
        workers=workers,
        per_worker_times=per_worker,
        merge_time=t_mg,
        svd_time=t_svd,
        score_time=t_sc,
        bytes_communicated=workers * merged.payload_bytes,
        per_worker_rows=counts,
    )
    return result, report


def _broadcast_host(s_host, vt_host, group, dev):
    obj = [None if s_host is None else (s_host, vt_host)]
    tdist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def run_sharded(local_rows, row0: int, n_total: int, spec: SketchSpec, sv_tol: float, *, jl_dim=None, jl_seed=0,
                rank=None, group=None):
    """Production multi-GPU entry: each rank passes ONLY its own rows
    (global indices row0..), gets back its rank-local scores (float64 CUDA
    tensor) plus the merged sketch and the coordinator's spectrum."""
    if spec.family not in DIST_FAMILIES:
        raise UnsupportedFamilyError(f"distributed sketching supports countsketch and osnap, not {spec.family!r}")
    from .csr import CSRMatrix

    m = None if isinstance(local_rows, (np.ndarray, torch.Tensor, list)) else CSRMatrix.from_any(local_rows)
    X = m if m is not None else device_matrix(local_rows)  # CSR row blocks: K2 sketch + K6 scores
    world = tdist.get_world_size(group)
    me = tdist.get_rank(group)
    cnt = torch.tensor([m.n if m is not None else X.shape[0]], dtype=torch.int64, device=N.device())
    allc = [torch.empty_like(cnt) for _ in range(world)]
    tdist.all_gather(allc, cnt, group=group)
    counts = [int(c.item()) for c in allc]
    ops = DeviceOps(spec, n_total, sv_tol, jl_dim, jl_seed, rank)
    local, merged, s_host, vt_host, timings = coordinate(ops, X, row0, me, world, counts, group)
    return local, merged, s_host, vt_host, timings


__all__ = ["CoordinatorReport", "Partition", "partition_rows", "run_distributed", "run_sharded", "coordinate"]
