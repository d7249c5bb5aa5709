"""Config-level parity: the five BASELINE.json configs, generated exactly as
BASELINE defines them (paper_1812_07903_b200/synth.py — the same inputs the
bench measures), through the product path against the CPU oracle.

north_star's acceptance criteria, per config:
  * hash buckets, signs and SRHT sample bit-exact (hashed states are
    bit-identical to the reference's compensated accumulators);
  * sketches and leverage scores within 1e-4 per-row relative error for the
    fp32 configs, 2e-2 for the bf16 config (C5);
  * Kendall tau >= 0.999 between the device scores and the oracle's;
  * the "dec" order of the device scores is the stable argsort
    (reference order.py:89-90) bit-for-bit.
Contract: /root/reference/pkg/tests/test_acceptance.py:50-324, order.py:89-90.

C1-C3 run at full size against the oracle end to end.  C4 (4e6 CSR rows)
and C5 (8e6 bf16 rows) run the full matrix on the device; the oracle checks
(a) sketch row windows at the full (k, d, s) and large global row offsets,
(b) a full-size checksum of the C4 sketch, (c) the fold recomputed in
float64 from the device sketch and the scores of a random row sample.
Results are also written to gpurun_out/parity_<config>.json when that
directory exists (copied under profiles/)."""

from __future__ import annotations

import json
import math
import os
from pathlib import Path

import numpy as np
import pytest
import torch
from scipy.stats import kendalltau

import paper_1812_07903_b200 as P
from paper_1812_07903_b200 import _native as N
from paper_1812_07903_b200 import synth as S
from oracle import levsketch_oracle as O

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-4
BF16_TOL = 2e-2
TAU_MIN = 0.999
OUT = Path(__file__).resolve().parent.parent / "gpurun_out"


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)
    yield
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def spec_of(name):
    c = S.CONFIGS[name]
    return P.SketchSpec(c["family"], eps=0.5, d=c["d"], seed=0, rows_override=c["k"], osnap_s=c["s"])


def rel_rows(got, ref):
    """Per-row relative error of a k x d sketch (row norms)."""
    num = np.linalg.norm(got - ref, axis=1)
    den = np.maximum(np.linalg.norm(ref, axis=1), 1e-300)
    return float((num / den).max())


def check_scores(name, got, ref, tol, extra=None):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape
    assert np.isfinite(got).all() and (got >= 0).all()
    rel = np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300)
    tau = float(kendalltau(got, ref).statistic)
    rec = {"config": name, "rows_compared": int(got.size), "score_max_rel": float(rel.max()),
           "score_median_rel": float(np.median(rel)), "kendall_tau": tau, "tol": tol, **(extra or {})}
    if OUT.is_dir():
        (OUT / f"parity_{name}.json").write_text(json.dumps(rec, indent=1))
    print(json.dumps(rec))
    assert rel.max() <= tol, rec
    assert tau >= TAU_MIN, rec
    return rec


def check_order(scores):
    """dec of the device scores: bit-exact stable argsort (order.py:89-90)."""
    p = P.scores_to_distribution(scores)
    plan = P.make_plan(p, P.OrderingPolicy("dec"))
    assert np.array_equal(plan.indices, np.argsort(-np.asarray(p), kind="stable"))


# ---------------------------------------------------------------------------


def test_c1_gaussian_full():
    name = "c1"
    c = S.CONFIGS[name]
    X = S.generate(name)
    x = X.double().cpu().numpy()
    spec = spec_of(name)
    res = P.leverage_sketched_trunc(X, spec, c["sv_tol"], jl_dim=c["r"])
    sx = P.apply_sketch(X, spec).data
    sx_o = O.gaussian_sketch(x, c["k"], 0)
    sk = rel_rows(sx, sx_o)
    assert sk <= FP32_TOL
    ref, r_o, _ = O.leverage_from_sketch(x, sx_o, c["sv_tol"], O.jl_matrix(0, c["d"], c["r"]))
    assert res.effective_rank == r_o
    check_scores(name, res.scores, ref, FP32_TOL, {"sketch_row_max_rel": sk, "rank": r_o})
    check_order(res.scores)


def test_c2_countsketch_full():
    name = "c2"
    c = S.CONFIGS[name]
    X = S.generate(name)
    spec = spec_of(name)
    res = P.leverage_sketched_trunc(X, spec, c["sv_tol"], jl_dim=c["r"])
    st = P.apply_sketch(X, spec)
    x = X.double().cpu().numpy()
    ref, r_o, sx_o = O.pipeline_hashed(x, "countsketch", c["k"], 0, 1, c["sv_tol"], O.jl_matrix(0, c["d"], c["r"]),
                                       workers=threads())
    # the compensated state (hi + lo) is the reference's, bit for bit: every
    # bucket and sign of the 1e6 rows is right
    assert np.array_equal(st.data, sx_o)
    # buckets / signs of the last rows through the C ABI
    hp = O.HashParams("countsketch", 0, c["k"], 1)
    idx = np.arange(c["n"] - 4096, c["n"], dtype=np.int64)
    blocks = N.hash_blocks([(hp.a[0], hp.b[0], hp.sign_keys[0], hp.offsets[0], hp.sizes[0])])
    it = torch.from_numpy(idx).cuda()
    bk = torch.empty((1, idx.size), dtype=torch.int64, device="cuda")
    sg = torch.empty((1, idx.size), dtype=torch.float64, device="cuda")
    N.check(N.lib().lvsk_hash_rows(it.data_ptr(), idx.size, blocks, 1, bk.data_ptr(), sg.data_ptr(), N.stream_ptr()))
    assert np.array_equal(bk.cpu().numpy()[0], O.block_buckets(hp, idx.astype(np.uint64), 0))
    assert np.array_equal(sg.cpu().numpy()[0], O.sign_of(idx.astype(np.uint64), hp.sign_keys[0]))
    assert res.effective_rank == r_o
    check_scores(name, res.scores, ref, FP32_TOL, {"sketch": "bit-exact", "rank": r_o})
    check_order(res.scores)


def test_c3_srht_full():
    name = "c3"
    c = S.CONFIGS[name]
    X = S.generate(name)
    spec = spec_of(name)
    cap = 16 << 30  # the SRHT buffer exceeds the reference's 4 GiB default (G8)
    res = P.leverage_sketched_trunc(X, spec, c["sv_tol"], mem_cap_bytes=cap, jl_dim=c["r"])
    st = P.apply_sketch(X, spec, mem_cap=cap)
    signs, sample = O.srht_signs_sample(0, c["n"], c["k"])
    assert np.array_equal(st._sample, sample)
    assert np.array_equal(st._signs, signs)
    sx = st.data
    x = X.double().cpu().numpy()
    sx_o = O.srht_sketch(x, c["k"], 0)
    sk = rel_rows(sx, sx_o)
    assert sk <= FP32_TOL
    ref, r_o, _ = O.leverage_from_sketch(x, sx_o, c["sv_tol"], O.jl_matrix(0, c["d"], c["r"]))
    assert res.effective_rank == r_o
    check_scores(name, res.scores, ref, FP32_TOL, {"sketch_row_max_rel": sk, "signs_sample": "bit-exact"})
    check_order(res.scores)


def _csr_host(m):
    import scipy.sparse as sp

    ip = m.indptr.cpu().numpy()
    ip = ip - ip[0]
    nnz = int(ip[-1])
    return sp.csr_matrix((m.data[:nnz].cpu().numpy().astype(np.float64), m.indices[:nnz].cpu().numpy(), ip),
                         shape=m.shape)


def test_c4_osnap_csr():
    name = "c4"
    c = S.CONFIGS[name]
    n, d, k, s = c["n"], c["d"], c["k"], c["s"]
    m = S.generate(name)
    assert abs(m.nnz / n - 80) < 0.5  # ~80 nonzeros per row (exactly 80 distinct columns)
    spec = spec_of(name)
    st = P.apply_sketch(m, spec)
    sx = st.data_device
    hp = O.HashParams("osnap", 0, k, s)
    # (a) row windows at the full (k, d, s) with large global offsets, against
    # the reference hashing on the densified rows (the compensated state)
    win = {}
    for lo in (n - 20_000, 2_000_000 + 13):
        hi = lo + 20_000
        sub = S.generate(name, lo=lo, hi=hi)
        w = P.consume_rows(P.SketchState(spec, n), sub, lo)
        xd = _csr_host(sub).toarray()
        h_o = np.zeros((k, d))
        l_o = np.zeros((k, d))
        O.hashed_consume(h_o, l_o, hp, xd, lo)
        e = rel_rows(w.data, h_o + l_o)
        assert e <= 1e-12, (lo, e)
        win[lo] = e
    # (b) full-size checksum: v^T SX w = sum_i sum_j v[b_j(i)] s_j(i)/sqrt(s) (x_i . w)
    rng = np.random.default_rng(4)
    v = rng.standard_normal(k)
    wv = rng.standard_normal(d)
    xw = _csr_host(m) @ wv
    idx = np.arange(n, dtype=np.uint64)
    coef = np.zeros(n)
    for j in range(s):
        coef += v[O.block_buckets(hp, idx, j)] * O.sign_of(idx, hp.sign_keys[j]) * hp.scale
    chk_o = float(coef @ xw)
    chk = float(v @ sx.cpu().numpy() @ wv)
    assert abs(chk - chk_o) <= 1e-9 * (np.abs(coef) @ np.abs(xw)), (chk, chk_o)
    # (c) the product scores (public API) vs the fold recomputed in float64
    # from the device sketch, on a random sample of 200k rows
    res = P.leverage_sketched_trunc(m, spec, c["sv_tol"], jl_dim=c["r"])
    M_o, r_o = O.fold_r(sx.cpu().numpy(), c["sv_tol"], O.jl_matrix(0, d, c["r"]))
    assert res.effective_rank == r_o
    rows = np.sort(rng.choice(n, size=200_000, replace=False))
    xs = _csr_host(m)[rows]
    u = xs @ M_o
    ref = np.einsum("ij,ij->i", u, u)
    check_scores(name, res.scores[rows], ref, FP32_TOL,
                 {"window_sketch_row_max_rel": max(win.values()), "checksum_rel": abs(chk - chk_o) / abs(chk_o),
                  "nnz": m.nnz, "rank": r_o})
    check_order(res.scores)


def test_c5_gaussian_bf16():
    name = "c5"
    c = S.CONFIGS[name]
    n, d, k = c["n"], c["d"], c["k"]
    X = S.generate(name)
    spec = spec_of(name)
    # (a) sketch windows at large global offsets: Z X_w / sqrt(k) in float64
    win = {}
    for lo in (n - 20_000, 3_000_017):
        hi = lo + 20_000
        w = P.consume_rows(P.SketchState(spec, n), X[lo:hi], lo)
        xw = X[lo:hi].double().cpu().numpy()
        ref_w = O.gaussian_z(0, k, lo, hi - lo).astype(np.float64) @ xw / math.sqrt(k)
        e = rel_rows(w.data, ref_w)
        assert e <= FP32_TOL, (lo, e)  # fp32 accumulation of exact bf16 products
        win[lo] = e
    # (b) the whole pipeline on the device; fold recomputed in float64 from its sketch
    res = P.leverage_sketched_trunc(X, spec, c["sv_tol"], jl_dim=c["r"], rank=c["rank"])
    sx = P.apply_sketch(X, spec).data
    M_o, r_o = O.fold_r(sx, c["sv_tol"], O.jl_matrix(0, d, c["r"]), rank=c["rank"])
    assert res.effective_rank == r_o == c["rank"]
    rng = np.random.default_rng(5)
    rows = np.sort(rng.choice(n, size=200_000, replace=False))
    xs = X[torch.from_numpy(rows).cuda()].double().cpu().numpy()
    u = xs @ M_o
    ref = np.einsum("ij,ij->i", u, u)
    check_scores(name, res.scores[rows], ref, BF16_TOL, {"window_sketch_row_max_rel": max(win.values()),
                                                          "rank": r_o})
    check_order(res.scores)


def test_c2_sharded_ranks_equal_serial():
    """The multi-GPU partitioning (dist.partition_rows, global row offsets,
    rank-ordered merge) reproduces the serial C2 state bit for bit and its
    scores exactly: simulated ranks on one device (reference test_dist.py:47-61)."""
    name = "c2"
    c = S.CONFIGS[name]
    X = S.generate(name)
    spec = spec_of(name)
    serial = P.leverage_sketched_trunc(X, spec, c["sv_tol"], jl_dim=c["r"])
    for w in (2, 8):
        res, report = P.run_distributed(X, spec, workers=w, sv_tol=c["sv_tol"], jl_dim=c["r"])
        assert np.array_equal(res.scores, serial.scores), w
        assert report.bytes_communicated > 0
