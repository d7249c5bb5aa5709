"""BatchRunner (independent passes in flight on separate streams): every
slot's scores and order are bit-identical to LeveragePipeline.run on the
same batch, although the library runs KF / K7 with fewer CTAs while passes
are in flight (lvsk_set_inflight)."""

import pytest
import torch

import paper_1812_07903_b200 as P
from paper_1812_07903_b200 import _native as N

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("family,dtype,n,d,k", [
    ("countsketch", torch.float32, 60000, 512, 2048),
    ("osnap", torch.float32, 30000, 256, 1024),
    ("gaussian", torch.float32, 20000, 256, 1024),
    ("gaussian", torch.bfloat16, 20000, 640, 1024),
    ("srht", torch.float32, 40000, 256, 1024),
])
def test_batch_runner_matches_serial(family, dtype, n, d, k):
    g = torch.Generator(device="cuda").manual_seed(n + d)
    batches = [torch.randn(n, d, device="cuda", generator=g).to(dtype) * (1 + b) for b in range(3)]
    spec = P.SketchSpec(family, eps=0.5, d=d, seed=3, rows_override=k, osnap_s=4 if family == "osnap" else None)
    ref = P.LeveragePipeline(spec, n, d, dtype, sv_tol=1e-6, jl_dim=64)
    want = []
    for X in batches:
        s, o = ref.run(X)
        want.append((s.clone(), o.clone()))
    runner = P.BatchRunner(spec, n, d, dtype, sv_tol=1e-6, jl_dim=64, slots=2)
    try:
        assert N.lib().lvsk_get_inflight() == 2
        # slot i % 2 gets batch i % 3: each slot's last pass is known
        last = {}
        for i in range(7):
            slot = runner.submit(batches[i % 3])
            last[slot] = i % 3
        for slot, b in last.items():
            s, o = runner.result(slot)
            assert torch.equal(s, want[b][0]), (slot, b)
            assert torch.equal(o, want[b][1]), (slot, b)
    finally:
        runner.close()
    assert N.lib().lvsk_get_inflight() == 1


def test_batch_runner_rejects_bad_slots():
    spec = P.SketchSpec("countsketch", eps=0.5, d=64, seed=0, rows_override=256)
    with pytest.raises(ValueError):
        P.BatchRunner(spec, 1000, 64, torch.float32, slots=0)


def test_csr_pipeline_rebuilds_its_operand_per_batch():
    """The CSR leverage pass takes a float32 copy of M and (r = 128) its
    prepared bf16 operand images; the fold graph rewrites M in place on every
    replay, so both must be rebuilt per run: different CSR batches through one
    pipeline give the scores of a fresh pipeline on each batch."""
    import numpy as np

    from paper_1812_07903_b200.csr import CSRMatrix

    n, d, k, r = 6000, 256, 1024, 128

    def batch(seed):
        rng = np.random.default_rng(seed)
        nnz = 24
        cols = np.sort(np.stack([rng.choice(d, size=nnz, replace=False) for _ in range(n)]), axis=1)
        vals = rng.lognormal(0.0, 1.0, size=(n, nnz)) * (1.0 + seed)
        vals[:, : nnz // 2] *= 1.0 + 3.0 * rng.random((1, nnz // 2))  # batch-specific column weights
        indptr = np.arange(n + 1, dtype=np.int64) * nnz
        return CSRMatrix(indptr, cols.reshape(-1).astype(np.int32), vals.reshape(-1).astype(np.float32), (n, d))

    spec = P.SketchSpec("osnap", eps=0.5, d=d, seed=5, rows_override=k, osnap_s=4)
    batches = [batch(s) for s in range(3)]
    pipe = P.LeveragePipeline(spec, n, d, torch.float32, sv_tol=1e-6, jl_dim=r)
    for X in batches + batches[::-1]:
        got, _ = pipe.run(X)
        fresh = P.LeveragePipeline(spec, n, d, torch.float32, sv_tol=1e-6, jl_dim=r)
        want, _ = fresh.run(X)
        assert torch.equal(got, want)
