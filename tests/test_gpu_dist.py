"""run_sharded (the production multi-GPU entry, dist.py) through the CUDA
kernels: 3 ranks on cuda:0 over gloo (host-staged collectives — no rank's
kernel waits on another's), uneven row partitions, dense and CSR rows.
The merged sketch must equal the oracle's rank-ordered partition merge
(reference dist.py:104-118) bit for bit on dense rows."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import levsketch_oracle as O

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, x, csr, family, k, s, sv_tol, pi_r, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1812_07903_b200 as P
        from paper_1812_07903_b200.dist import gather_scores, partition_rows

        n, d = x.shape
        ranges = partition_rows(n, world)
        lo, hi = ranges[rank]
        spec = P.SketchSpec(family, eps=0.5, d=d, seed=5, rows_override=k, osnap_s=s)
        if csr:
            import scipy.sparse as sp

            m = sp.csr_matrix(x[lo:hi])
            rows = (m.indptr.astype(np.int64), m.indices.astype(np.int32), m.data.astype(np.float32), m.shape)
        else:
            rows = torch.from_numpy(x[lo:hi]).cuda()
        local, merged, *_ = P.run_sharded(rows, lo, n, spec, sv_tol, jl_dim=pi_r)
        full = gather_scores(local, [b - a for a, b in ranges])
        out_q.put((rank, full.cpu().numpy(), merged.data_device.cpu().numpy()))
    finally:
        dist.destroy_process_group()


def _run(x, csr, family, k, s, sv_tol, pi_r, world=3):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, x, csr, family, k, s, sv_tol, pi_r, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return results


def test_run_sharded_dense_countsketch_bit_exact_merge():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    rng = np.random.default_rng(21)
    n, d, k = 30_001, 48, 512
    x = ((rng.standard_normal((n, 8)) @ rng.standard_normal((8, d))) + 0.5 * rng.standard_normal((n, d)))
    x = x.astype(np.float32).astype(np.float64)
    pi = O.jl_matrix(0, d, 16)
    ref_scores, _, ref_sx = O.pipeline_hashed(x, "countsketch", k, 5, 1, 1e-6, pi, workers=3)
    for rank, scores, sx in _run(x.astype(np.float32), False, "countsketch", k, None, 1e-6, 16):
        assert np.array_equal(sx, ref_sx), rank
        np.testing.assert_allclose(scores, ref_scores, rtol=1e-4, atol=1e-12)


def test_run_sharded_csr_osnap():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    rng = np.random.default_rng(22)
    n, d, k = 20_003, 64, 1024
    x = rng.standard_normal((n, d)) * (rng.random((n, d)) < 0.15)
    x[::97] = 0.0  # empty rows
    x = x.astype(np.float32).astype(np.float64)
    pi = O.jl_matrix(0, d, 16)
    ref_scores, _, ref_sx = O.pipeline_hashed(x, "osnap", k, 5, 3, 1e-6, pi, workers=3)
    for rank, scores, sx in _run(x.astype(np.float32), True, "osnap", k, 3, 1e-6, 16):
        np.testing.assert_allclose(sx, ref_sx, rtol=0, atol=1e-12 * np.abs(ref_sx).max())  # K2: order-free atomics
        np.testing.assert_allclose(scores, ref_scores, rtol=1e-4, atol=1e-12)
