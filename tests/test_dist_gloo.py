"""Multi-process coordinator path on CPU: world_size 2 over gloo.

Exercises paper_1812_07903_b200.dist.coordinate / gather_scores (the code the
NCCL ranks run) with the CPU oracle plugged in as the compute, and checks
the result equals the serial reference pipeline bit-for-bit (hashed sketch +
rank-ordered TwoSum fold) and the distributed contract (partitioning,
uneven shards, M broadcast, rank-order concatenation)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import levsketch_oracle as O


class _State:
    def __init__(self, hi, lo, rows_consumed):
        self.hi, self.lo, self.rows_consumed = hi, lo, rows_consumed


class OracleOps:
    """Same interface as dist.DeviceOps, computed by the CPU oracle."""

    def __init__(self, family, k, seed, s, d, sv_tol, pi):
        self.hp = O.HashParams(family, seed, k, s)
        self.k, self.d, self.sv_tol, self.pi = k, d, sv_tol, pi

    def sketch(self, rows, row0):
        hi = np.zeros((self.k, self.d))
        lo = np.zeros_like(hi)
        O.hashed_consume(hi, lo, self.hp, rows.numpy(), row0)
        return _State(torch.from_numpy(hi), torch.from_numpy(lo), rows.shape[0])

    @staticmethod
    def payload(st):
        return [st.hi, st.lo]

    @staticmethod
    def from_payload(tensors, rows_consumed):
        return _State(tensors[0], tensors[1], rows_consumed)

    @staticmethod
    def merge(a, b):
        h, l = O.merge_hashed(a.hi.numpy(), a.lo.numpy(), b.hi.numpy(), b.lo.numpy())
        return _State(torch.from_numpy(h), torch.from_numpy(l), a.rows_consumed + b.rows_consumed)

    @staticmethod
    def merge_arrays(h1, l1, h2, l2):
        h, l = O.merge_hashed(h1.numpy(), l1.numpy(), h2.numpy(), l2.numpy())
        return torch.from_numpy(h), torch.from_numpy(l)

    def factor(self, merged):
        sx = (merged.hi + merged.lo).numpy()
        _, s, vt = O.thin_svd(sx)
        s, vt = O.truncate(s, vt, self.sv_tol)
        M, _ = O.fold_r(sx, self.sv_tol, self.pi)
        return torch.from_numpy(np.ascontiguousarray(M)), s, vt

    @staticmethod
    def scores(rows, M):
        return torch.from_numpy(O.row_scores(rows.numpy(), M.numpy()))

    @staticmethod
    def sync():
        pass


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, x, family, k, seed, s, sv_tol, pi, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1812_07903_b200.dist import coordinate, gather_scores, partition_rows

        n = x.shape[0]
        ranges = partition_rows(n, world)
        counts = [hi - lo for lo, hi in ranges]
        lo, hi = ranges[rank]
        ops = OracleOps(family, k, seed, s, x.shape[1], sv_tol, pi)
        local, merged, s_host, vt, _ = coordinate(ops, torch.from_numpy(x[lo:hi]), lo, rank, world, counts)
        full = gather_scores(local, counts)
        out_q.put((rank, full.numpy(), (merged.hi + merged.lo).numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("family,s,n", [("countsketch", 1, 1001), ("osnap", 3, 777)])
def test_two_rank_coordinator_equals_serial(family, s, n):
    rng = np.random.default_rng(n)
    d, k, seed, sv_tol = 12, 200, 4, 1e-3
    x = rng.standard_normal((n, d)) @ np.diag(np.linspace(3, 0.5, d))
    pi = O.jl_matrix(1, d, 6)
    ref_scores, _, ref_sx = O.pipeline_hashed(x, family, k, seed, s, sv_tol, pi)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, x, family, k, seed, s, sv_tol, pi, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, scores, sx in results:
        assert np.array_equal(sx, ref_sx), rank  # TwoSum fold in rank order == serial, bit-exact here
        np.testing.assert_allclose(scores, ref_scores, rtol=1e-10)
        assert scores.shape == (n,)


def _slice_worker(rank, world, port, x, k, seed, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1812_07903_b200.dist import exchange_row_slices, gather_row_slices, partition_rows

        n, d = x.shape
        lo_r, hi_r = partition_rows(n, world)[rank]
        hp = O.HashParams("countsketch", seed, k, 1)
        hi = np.zeros((k, d))
        lo = np.zeros_like(hi)
        O.hashed_consume(hi, lo, hp, x[lo_r:hi_r], lo_r)
        his = exchange_row_slices(torch.from_numpy(hi), rank, world)
        los = exchange_row_slices(torch.from_numpy(lo), rank, world)
        h, l = his[0].numpy(), los[0].numpy()
        for q in range(1, world):  # rank-ordered TwoSum merge of this rank's row slice
            h, l = O.merge_hashed(h, l, his[q].numpy(), los[q].numpy())
        full = gather_row_slices(torch.from_numpy(h + l), k, world)
        out_q.put((rank, full.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("k", [101, 102])
def test_sliced_merge_layout_equals_serial_three_ranks(k):
    """The reduce-scatter layout bench.py's multi-GPU path uses
    (dist.exchange_row_slices / gather_row_slices over 3 ranks — uneven row
    slices, and equal ones gathered in place): merging each slice in rank
    order and gathering the folded slices gives the serial sketch bit for
    bit."""
    rng = np.random.default_rng(9)
    n, d, seed = 901, 7, 3
    x = rng.standard_normal((n, d))
    hp = O.HashParams("countsketch", seed, k, 1)
    ref_hi = np.zeros((k, d))
    ref_lo = np.zeros_like(ref_hi)
    O.hashed_consume(ref_hi, ref_lo, hp, x, 0)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slice_worker, args=(r, 3, port, x, k, seed, q)) for r in range(3)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, full in results:
        assert np.array_equal(full, ref_hi + ref_lo), rank
