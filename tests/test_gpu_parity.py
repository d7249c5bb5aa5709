"""GPU parity: the CUDA product path (through the C ABI / drop-in API) against
the reference's golden vectors and the CPU oracle.  Needs a B200."""

import math
import os

import numpy as np
import pytest
import torch

import paper_1812_07903_b200 as P
from paper_1812_07903_b200 import _native as N
from paper_1812_07903_b200 import errors
from oracle import levsketch_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, scope="module")
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


# ---------------------------------------------------------------------------
# hashing: bit-exact buckets / signs (reference sketch.py:151-159)


def test_hash_rows_kat(golden, golden_meta):
    for ci, m in enumerate(golden_meta["hash"]):
        hp = O.HashParams(m["family"], m["seed"], m["k"], m["s"])
        blocks = N.hash_blocks([(hp.a[j], hp.b[j], hp.sign_keys[j], hp.offsets[j], hp.sizes[j]) for j in range(hp.s)])
        idx = dev(golden[f"hash{ci}_idx"].view(np.int64))
        n = idx.numel()
        bk = torch.empty((hp.s, n), dtype=torch.int64, device="cuda")
        sg = torch.empty((hp.s, n), dtype=torch.float64, device="cuda")
        N.check(N.lib().lvsk_hash_rows(idx.data_ptr(), n, blocks, hp.s, bk.data_ptr(), sg.data_ptr(), N.stream_ptr()))
        assert np.array_equal(bk.cpu().numpy(), golden[f"hash{ci}_buckets"])
        assert np.array_equal(sg.cpu().numpy(), golden[f"hash{ci}_signs"])


# ---------------------------------------------------------------------------
# K1 hashed sketch: bit-exact compensated state (sketch.py:173-191, 260-266)


def test_hashed_sketch_bit_exact_f64(golden, golden_meta):
    for ci, m in enumerate(golden_meta["sketch"]):
        x = golden[f"sk{ci}_x"]
        spec = P.SketchSpec(m["family"], eps=0.5, d=m["d"], seed=m["seed"], rows_override=m["k"],
                            osnap_s=m["s"] if m["family"] == "osnap" else None)
        st = P.apply_sketch(x, spec)
        assert np.array_equal(st._hi.cpu().numpy(), golden[f"sk{ci}_hi"]), ci
        assert np.array_equal(st._lo.cpu().numpy(), golden[f"sk{ci}_lo"]), ci
        assert np.array_equal(st.data, golden[f"sk{ci}_data"])
        cut = m["cut"]
        s1 = P.consume_rows(P.SketchState(spec, m["n"]), x[:cut], 0)
        assert np.array_equal(s1._hi.cpu().numpy(), golden[f"sk{ci}_part1_hi"])
        assert np.array_equal(s1._lo.cpu().numpy(), golden[f"sk{ci}_part1_lo"])
        s2 = P.consume_rows(P.SketchState(spec, m["n"]), x[cut:], cut)
        assert np.array_equal(P.merge(s1, s2).data, golden[f"sk{ci}_merged"])


def test_hashed_sketch_bit_exact_f32_and_bf16(golden, golden_meta):
    for ci, m in enumerate(golden_meta["fp32_sketch"]):
        x = golden[f"f32sk{ci}_x"]
        spec = P.SketchSpec(m["family"], eps=0.5, d=m["d"], seed=m["seed"], rows_override=m["k"],
                            osnap_s=m["s"] if m["family"] == "osnap" else None)
        assert np.array_equal(P.apply_sketch(dev(x), spec).data, golden[f"f32sk{ci}_data"])
        # bf16 inputs: the reference would see the same values upcast
        xb = torch.from_numpy(x).to(torch.bfloat16)
        ref_hi, ref_lo = O.hashed_sketch(xb.float().numpy(), m["family"], m["k"], m["seed"], m["s"])
        assert np.array_equal(P.apply_sketch(xb.cuda(), spec).data, ref_hi + ref_lo)


def test_hashed_ragged_and_strided():
    rng = np.random.default_rng(3)
    for n, d in ((1, 1), (7, 3), (33, 5), (1000, 130), (513, 257)):
        x = rng.standard_normal((n, d + 3)).astype(np.float32)
        view = torch.from_numpy(x).cuda()[:, 1 : d + 1]  # misaligned, strided rows
        for fam, s, k in (("countsketch", 1, 17), ("osnap", 3, 31)):
            if k < s:
                continue
            spec = P.SketchSpec(fam, eps=0.5, d=d, seed=5, rows_override=k, osnap_s=s if fam == "osnap" else None)
            hi, lo = O.hashed_sketch(x[:, 1 : d + 1], fam, k, 5, s)
            assert np.array_equal(P.apply_sketch(view, spec).data, hi + lo), (n, d, fam)


@pytest.mark.parametrize("k,s,n", [(4096, 1, 200_003), (4096, 4, 300_001), (4095, 2, 30_000), (6000, 1, 40_000),
                                   (1, 1, 999), (37, 37, 2_000)])
def test_hashed_grouping_paths(monkeypatch, k, s, n):
    """K1's bucket grouping: the cooperative counting sort (k <= 4096, s <= 64;
    ragged item ranges over the CTAs, items cached in shared memory or rehashed
    when a CTA holds more than 7168, one bucket) and the
    radix fallback (k > 4096, or forced) give the oracle's state bit for bit."""
    rng = np.random.default_rng(k + s)
    d = 24
    x = rng.standard_normal((n, d)).astype(np.float32)
    fam = "countsketch" if s == 1 else "osnap"
    spec = P.SketchSpec(fam, eps=0.5, d=d, seed=9, rows_override=k, osnap_s=s if s > 1 else None)
    hi, lo = O.hashed_sketch(x, fam, k, 9, s)
    assert np.array_equal(P.apply_sketch(dev(x), spec).data, hi + lo)
    monkeypatch.setenv("LVSK_GROUP_RADIX", "1")
    assert np.array_equal(P.apply_sketch(dev(x), spec).data, hi + lo)


def test_stream_update_and_order_independence(golden, golden_meta):
    m = golden_meta["sketch"][0]
    x = golden["sk0_x"]
    spec = P.SketchSpec(m["family"], eps=0.5, d=m["d"], seed=m["seed"], rows_override=m["k"])
    st = P.SketchState(spec, m["n"])
    for i in range(60):
        P.stream_update(st, i, x[i])
    hi, lo = O.hashed_sketch(x[:60], m["family"], m["k"], m["seed"], 1)
    assert np.array_equal(st.data, hi + lo)
    with pytest.raises(errors.DimensionMismatchError):
        P.stream_update(st, 0, np.zeros(m["d"] + 1))
    with pytest.raises(errors.DimensionMismatchError):
        P.stream_update(st, m["n"], np.zeros(m["d"]))


def test_merge_rules():
    spec = P.SketchSpec("countsketch", eps=0.5, d=16, seed=1)
    with pytest.raises(errors.IncompatibleSketchError):
        P.merge(P.SketchState(spec, 10), P.SketchState(P.SketchSpec("countsketch", eps=0.5, d=16, seed=2), 10))
    with pytest.raises(errors.IncompatibleSketchError):
        P.merge(P.SketchState(spec, 10), P.SketchState(spec, 11))
    a = np.random.default_rng(10).standard_normal((10, 16))
    with pytest.raises(errors.IncompatibleSketchError):
        P.merge(P.apply_sketch(a, spec), P.apply_sketch(a, spec))
    s = P.apply_sketch(a, spec)
    assert np.array_equal(P.merge(s, P.SketchState(spec, 10)).data, s.data)


def test_nonfinite_rejected_and_state_untouched():
    spec = P.SketchSpec("countsketch", eps=0.5, d=4, seed=1, rows_override=8)
    st = P.consume_rows(P.SketchState(spec, 20), np.ones((5, 4)), 0)
    before = st.data.copy()
    bad = np.ones((5, 4))
    bad[2, 1] = np.inf
    with pytest.raises(errors.FormatError):
        P.consume_rows(st, bad, 5)
    assert np.array_equal(st.data, before) and st.rows_consumed == 5
    with pytest.raises(errors.FormatError):
        P.leverage_sketched_trunc(torch.tensor(bad, device="cuda", dtype=torch.float32), spec, 0.0)


@pytest.mark.parametrize("family", ["countsketch", "osnap", "gaussian", "csr"])
def test_nonfinite_first_block_leaves_zero_state(family):
    """A rejected FIRST block (the state is still zero and updated in place)
    must not poison the state: a retry with clean rows equals a fresh state
    (the reference validates before touching anything,
    matrix.py:30-39)."""
    rng = np.random.default_rng(3)
    d, n = 24, 40
    clean = rng.standard_normal((n, d))
    bad = clean.copy()
    bad[7, 3] = np.nan
    fam = "osnap" if family == "csr" else family
    spec = P.SketchSpec(fam, eps=0.5, d=d, seed=2, rows_override=16, osnap_s=3 if fam == "osnap" else None)
    if family == "csr":
        import scipy.sparse as sp

        clean_in, bad_in = sp.csr_matrix(clean), sp.csr_matrix(bad)
    else:
        clean_in, bad_in = clean, bad
    st = P.SketchState(spec, n)
    with pytest.raises(errors.FormatError):
        P.consume_rows(st, bad_in, 0)
    assert st.rows_consumed == 0 and not np.any(st.data)
    P.consume_rows(st, clean_in, 0)
    ref = P.consume_rows(P.SketchState(spec, n), clean_in, 0)
    assert np.array_equal(st.data, ref.data)


def test_srht_whole_matrix_is_transformed_eagerly():
    """SRHT consume of the whole matrix: the product is formed inside the
    call (no reference to the caller's rows is kept, errors raise from the
    call itself, as the reference's consume_rows does)."""
    rng = np.random.default_rng(4)
    n, d, k = 1000, 16, 64
    x = rng.standard_normal((n, d)).astype(np.float32)
    spec = P.SketchSpec("srht", eps=0.5, d=d, seed=3, rows_override=k)
    X = torch.from_numpy(x).cuda()
    st = P.apply_sketch(X, spec)
    ref = O.srht_sketch(x.astype(np.float64), k, 3)
    X.mul_(2.0)  # the caller edits its array afterwards
    assert np.linalg.norm(st.data - ref) <= 2e-6 * np.linalg.norm(ref)
    X[5, 5] = float("inf")
    with pytest.raises(errors.FormatError):
        P.consume_rows(P.SketchState(spec, n), X, 0)
    # a fully consumed state merges with an empty one (linearity of the transform)
    m = P.merge(st, P.SketchState(spec, n))
    assert np.array_equal(m.data, st.data)
    with pytest.raises(errors.IncompatibleSketchError):
        P.merge(st, st)


def test_capacity_and_srht_config():
    with pytest.raises(errors.ConfigurationError):
        P.SketchState(P.SketchSpec("srht", eps=0.5, d=8, rows_override=64), 10)
    with pytest.raises(errors.CapacityError):
        P.SketchState(P.SketchSpec("srht", eps=0.5, d=64, rows_override=16), 100_000, mem_cap=1_000_000)


def test_explicit_matrix_matches_oracle():
    for fam, s in (("countsketch", 1), ("osnap", 3)):
        spec = P.SketchSpec(fam, eps=0.5, d=16, seed=5, osnap_s=s if fam == "osnap" else None, rows_override=40)
        assert np.array_equal(P.sketch_matrix(spec, 150), O.explicit_hashed_matrix(fam, 40, 5, s, 150))
    spec = P.SketchSpec("srht", eps=0.5, d=8, seed=17, rows_override=32)
    np.testing.assert_allclose(P.sketch_matrix(spec, 64), O.explicit_srht_matrix(32, 17, 64), atol=1e-12)


# ---------------------------------------------------------------------------
# K3 SRHT (sketch.py:248-257, 364-385)


def test_srht_matches_reference(golden, golden_meta):
    for ci, m in enumerate(golden_meta["srht"]):
        spec = P.SketchSpec("srht", eps=0.5, d=m["d"], seed=m["seed"], rows_override=m["k"])
        st = P.srht_apply(spec, golden[f"srht{ci}_x"])
        assert np.array_equal(st._signs, golden[f"srht{ci}_signs"])
        assert np.array_equal(st._sample, golden[f"srht{ci}_sample"])
        ref = golden[f"srht{ci}_data"]
        np.testing.assert_allclose(st.data, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())
        # fp32 inputs against the float64 oracle on the same (rounded) values
        x32 = golden[f"srht{ci}_x"].astype(np.float32)
        ref32 = O.srht_sketch(x32, m["k"], m["seed"])
        got = P.srht_apply(spec, dev(x32)).data
        assert np.linalg.norm(got - ref32) <= 1e-5 * np.linalg.norm(ref32)


@pytest.mark.parametrize("n,d,k", [(2**16, 8, 512), (3 * 2**15 + 17, 33, 512), (2**17, 256, 512),
                                   (2**20 + 3, 4, 512), (2**14 + 17, 100, 4096), (5000, 68, 4097),
                                   (3000, 64, 300), (2048, 4096, 64)])
def test_srht_multi_chunk(n, d, k):
    """fp32 X: the one-pass sampled kernel (srht_sampled.cu; d % 4 == 0,
    k <= 4096) and the two-pass kernels (srht.cu) against explicit rows of H."""
    rng = np.random.default_rng(n)
    x = rng.standard_normal((n, d)).astype(np.float32)
    spec = P.SketchSpec("srht", eps=0.5, d=d, seed=7, rows_override=k)
    got = P.srht_apply(spec, dev(x)).data
    S_rows = O.srht_signs_sample(7, O.next_pow2(n), k)
    # oracle via explicit rows of H for the sampled indices (float64)
    signs, sample = S_rows
    ref = np.zeros((k, d))
    xs = signs[:n, None] * x.astype(np.float64)
    idx = np.arange(n, dtype=np.uint64)
    for t0 in range(0, k, 64):
        v = sample[t0 : t0 + 64, None].astype(np.uint64) & idx[None, :]
        par = np.zeros_like(v)
        while v.any():
            par ^= v & np.uint64(1)
            v >>= np.uint64(1)
        ref[t0 : t0 + 64] = (1.0 - 2.0 * par.astype(np.float64)) @ xs
    ref /= math.sqrt(k)
    assert np.linalg.norm(got - ref) <= 2e-6 * np.linalg.norm(ref)
    # deterministic: a second call is bit-identical
    assert np.array_equal(P.srht_apply(spec, dev(x)).data, got)


def test_srht_sampled_vs_two_pass(monkeypatch):
    """The one-pass kernel and the two-pass kernels agree on C3-shaped input."""
    n, d, k = 2**18, 64, 4096
    x = np.random.default_rng(3).standard_normal((n, d)).astype(np.float32)
    spec = P.SketchSpec("srht", eps=0.5, d=d, seed=5, rows_override=k)
    a = P.srht_apply(spec, dev(x)).data
    monkeypatch.setenv("LVSK_SRHT_V2", "1")
    b = P.srht_apply(spec, dev(x)).data
    assert np.linalg.norm(a - b) <= 1e-6 * np.linalg.norm(b)
    # both against the oracle's float64 transform (reference sketch.py:248-257)
    ref = O.srht_sketch(x.astype(np.float64), k, 5)
    assert np.linalg.norm(a - ref) <= 2e-6 * np.linalg.norm(ref)
    assert np.linalg.norm(b - ref) <= 2e-6 * np.linalg.norm(ref)


def test_fwht_kats(golden):
    assert np.array_equal(P.fwht([1.0, 0.0, 0.0, 0.0]), [1.0, 1.0, 1.0, 1.0])
    assert np.array_equal(P.fwht([1.0, 1.0, 1.0, 1.0]), [4.0, 0.0, 0.0, 0.0])
    np.testing.assert_allclose(P.fwht(golden["fwht_x"]), golden["fwht_y"], rtol=1e-13, atol=1e-12)
    x = np.random.default_rng(11).standard_normal(64)
    np.testing.assert_allclose(P.fwht(P.fwht(x)), 64 * x, atol=1e-9)
    with pytest.raises(errors.ConfigurationError):
        P.fwht(np.ones(6))


# ---------------------------------------------------------------------------
# K4 Gaussian (extension; oracle-pinned generator)


def test_gaussian_entries_bit_exact():
    for seed, k, row0, n in ((0, 64, 0, 1000), (12345, 37, 2**32 - 5, 300), (2**40 + 3, 8, 10**9, 64)):
        Z = torch.empty((k, n), dtype=torch.float32, device="cuda")
        N.check(N.lib().lvsk_gaussian_entries(seed, k, row0, n, Z.data_ptr(), N.stream_ptr()))
        assert np.array_equal(Z.cpu().numpy(), O.gaussian_z(seed, k, row0, n)), (seed, k, row0)


def test_gaussian_entries_bit_exact_at_ks_sample_size():
    """The 1.2e7 entries the CPU distribution test (test_oracle_golden.py:
    KS vs bf16_rn(N(0,1)), moments, per-column law) runs on, generated by the
    device generator: bit-identical, so the distribution result is the
    kernel's."""
    k, n, row0 = 4096, 3000, 5_000_000
    Z = torch.empty((k, n), dtype=torch.float32, device="cuda")
    N.check(N.lib().lvsk_gaussian_entries(0, k, row0, n, Z.data_ptr(), N.stream_ptr()))
    assert np.array_equal(Z.cpu().numpy(), O.gaussian_z(0, k, row0, n))


def test_gaussian_sketch_matches_oracle():
    rng = np.random.default_rng(1)
    for n, d, k, dt in ((3000, 40, 256, torch.float32), (2000, 130, 100, torch.float64), (1500, 64, 128, torch.bfloat16)):
        x = rng.standard_normal((n, d))
        X = torch.from_numpy(x).to(dt).cuda()
        xv = X.double().cpu().numpy()
        spec = P.SketchSpec("gaussian", eps=0.5, d=d, seed=9, rows_override=k)
        got = P.apply_sketch(X, spec).data
        ref = O.gaussian_sketch(xv, k, 9)
        tol = 1e-12 if dt == torch.float64 else 2e-6
        assert np.linalg.norm(got - ref) <= tol * np.linalg.norm(ref), dt
        # row offset: two halves consumed separately == one pass
        st = P.SketchState(spec, n)
        P.consume_rows(st, X[: n // 2], 0)
        P.consume_rows(st, X[n // 2 :], n // 2)
        assert np.linalg.norm(st.data - ref) <= tol * np.linalg.norm(ref)


@pytest.mark.parametrize("n,d,k", [(20000, 256, 1024), (3001, 100, 200), (700, 520, 64), (2100, 1000, 256)])
def test_gaussian_fp32_tensor_core_vs_simt(n, d, k, monkeypatch):
    """fp32 X through the exact three-plane bf16 split on tcgen05 (default:
    the planes stacked with a 64-row-padded period, one K4-TC launch whose
    splits straddle plane boundaries; d = 1000 takes the CTA-pair kernel) vs
    the SIMT split-K GEMM (LVSK_NO_TC=1) vs the float64 oracle."""
    x = np.random.default_rng(n).standard_normal((n, d)).astype(np.float32)
    X = torch.from_numpy(x).cuda()
    spec = P.SketchSpec("gaussian", eps=0.5, d=d, seed=4, rows_override=k)
    tc = P.apply_sketch(X, spec).data
    ref = O.gaussian_sketch(x.astype(np.float64), k, 4)
    assert np.linalg.norm(tc - ref) <= 2e-6 * np.linalg.norm(ref)
    monkeypatch.setenv("LVSK_NO_TC", "1")
    simt = P.apply_sketch(X, spec).data
    assert np.linalg.norm(simt - ref) <= 2e-6 * np.linalg.norm(ref)


@pytest.mark.parametrize("variant", ["3", "2", "1", "0"])
@pytest.mark.parametrize("n,d,k,ldx,row0", [(5000, 1024, 300, 1024, 0), (3001, 200, 128, 208, 7),
                                            (700, 520, 256, 520, 2**33 + 5), (64, 64, 8, 64, 0),
                                            (4100, 1024, 250, 1032, 2**35 + 1), (2000, 700, 512, 704, 3)])
def test_gaussian_tc_bf16_vs_oracle(n, d, k, ldx, row0, variant, monkeypatch):
    """K4-TC (tcgen05, bf16 X as the MN-major B operand, Z generated in smem)
    against the oracle's exact Z X / sqrt(k): ragged k / d (TMA zero fill),
    two 512-column slabs, strided rows, a large global row offset — for every
    kernel variant (LVSK_K4_VARIANT: 3 = CTA pair x shared Z tiles, 2 = Z
    tiles shared by the slab pair, 1 = X multicast, 0 = plain)."""
    monkeypatch.setenv("LVSK_K4_VARIANT", variant)
    rng = np.random.default_rng(n + d)
    buf = torch.from_numpy(rng.standard_normal((n, ldx))).to(torch.bfloat16).cuda()
    X = buf[:, :d]
    xv = X.double().cpu().numpy()
    L = N.lib()
    ws = torch.empty(int(L.lvsk_gaussian_workspace_bytes(n, d, k, N.LVSK_BF16)), dtype=torch.uint8, device="cuda")
    SX = torch.empty((k, d), dtype=torch.float64, device="cuda")
    flags = N.Flags()
    N.check(L.lvsk_gaussian_sketch(X.data_ptr(), N.LVSK_BF16, n, d, ldx, row0, 77, k, SX.data_ptr(), 0,
                                   ws.data_ptr(), ws.numel(), flags.p, N.stream_ptr()), "gaussian tc")
    assert flags.read() == 0
    ref = O.gaussian_z(77, k, row0, n).astype(np.float64) @ xv / math.sqrt(k)
    got = SX.cpu().numpy()
    assert np.linalg.norm(got - ref) <= 2e-6 * np.linalg.norm(ref)
    assert np.abs(got - ref).max() <= 1e-5 * np.abs(ref).max()
    # accumulate = 1 adds onto the state; non-finite input raises the flag
    N.check(L.lvsk_gaussian_sketch(X.data_ptr(), N.LVSK_BF16, n, d, ldx, row0, 77, k, SX.data_ptr(), 1,
                                   ws.data_ptr(), ws.numel(), flags.p, N.stream_ptr()), "gaussian tc")
    assert np.linalg.norm(SX.cpu().numpy() - 2 * ref) <= 2e-6 * np.linalg.norm(2 * ref)
    buf[n // 2, 3] = float("inf")
    N.check(L.lvsk_gaussian_sketch(X.data_ptr(), N.LVSK_BF16, n, d, ldx, row0, 77, k, SX.data_ptr(), 0,
                                   ws.data_ptr(), ws.numel(), flags.p, N.stream_ptr()), "gaussian tc")
    assert flags.read() & N.FLAG_NONFINITE


# ---------------------------------------------------------------------------
# K5 leverage pass vs a float64 torch reference


@pytest.mark.parametrize("n,d,r", [(1, 1, 1), (1000, 64, 64), (5000, 512, 64), (3001, 100, 128), (777, 37, 13), (4096, 256, 100)])
@pytest.mark.parametrize("dt", [torch.float32, torch.float64, torch.bfloat16])
def test_rowsumsq_vs_fp64(n, d, r, dt):
    g = torch.Generator(device="cpu").manual_seed(n + d + r)
    X = torch.randn(n, d, generator=g, dtype=torch.float64)
    M = torch.randn(d, r, generator=g, dtype=torch.float64) / math.sqrt(d)
    Xd = X.to(dt).cuda()
    ref = ((Xd.double() @ M.cuda()) ** 2).sum(1)
    got = P.leverage.scores_device(Xd, M.cuda())
    rel = ((got - ref).abs() / ref.clamp_min(1e-300)).max().item()
    assert rel < (1e-12 if dt == torch.float64 else 5e-5), rel  # fp32 accumulation over d terms


@pytest.mark.parametrize("n,d,r", [(300, 32, 64), (70_001, 512, 64), (4096, 256, 128), (5000, 96, 100), (1024, 20, 7)])
def test_tcgen05_leverage_vs_fp64(n, d, r):
    """tcgen05 3xTF32 kernel against a float64 reference (fp32-level accuracy)."""
    g = torch.Generator(device="cpu").manual_seed(7 * n + r)
    X = (torch.randn(n, d, generator=g, dtype=torch.float64) * 3).to(torch.float32).cuda()
    M = (torch.randn(d, r, generator=g, dtype=torch.float64) / math.sqrt(d)).cuda()
    ref = ((X.double() @ M) ** 2).sum(1)
    mt_hi, mt_lo = P.leverage.split_m_tf32(M)
    hb = mt_hi.to(torch.bfloat16).contiguous()
    flags = N.Flags()
    for variant in (None, hb):  # v1 (x_lo as TF32) and v2 (x_lo as BF16, r <= 64)
        out = torch.full((n,), -1.0, dtype=torch.float64, device="cuda")
        rc = N.lib().lvsk_leverage_tf32x3(X.data_ptr(), n, d, X.stride(0), mt_hi.data_ptr(), mt_lo.data_ptr(),
                                          N.ptr(variant), r, out.data_ptr(), flags.p, N.stream_ptr())
        N.check(rc)
        assert flags.read() == 0
        rel = ((out - ref).abs() / ref).max().item()
        assert rel < 2e-5, (rel, variant is None)
    # the SIMT kernel agrees too
    simt = torch.empty_like(out)
    a, b = P.leverage.split_m(M, torch.float32)
    N.check(N.lib().lvsk_rowsumsq_gemm(X.data_ptr(), N.LVSK_F32, n, d, X.stride(0), a.data_ptr(), b.data_ptr(), r,
                                       simt.data_ptr(), flags.p, N.stream_ptr()))
    assert ((simt - ref).abs() / ref).max().item() < 2e-5


def test_tcgen05_nonfinite_and_strided():
    n, d, r = 1000, 64, 64
    base = torch.randn(n, d + 4, device="cuda", dtype=torch.float32)
    X = base[:, :d]  # row stride 68 floats (16-byte multiple)
    M = torch.randn(d, r, device="cuda", dtype=torch.float64) / 8
    got = P.leverage.scores_device(X, M)
    ref = ((X.double() @ M) ** 2).sum(1)
    assert ((got - ref).abs() / ref).max().item() < 2e-5
    X2 = X.clone()
    X2[17, 3] = float("nan")
    with pytest.raises(errors.FormatError):
        P.leverage.scores_device(X2, M)


def test_cholesky_fold_equals_qr_fold_and_oracle():
    g = torch.Generator(device="cuda").manual_seed(3)
    sx = torch.randn(2048, 256, device="cuda", dtype=torch.float64, generator=g)
    sx[:, :10] *= 50.0
    pi = P.leverage.jl_device(0, 256, 64)
    m_ch = P.leverage.cholesky_fold(sx, 1e-6, pi)
    assert m_ch is not None
    m_qr, r = P.leverage.qr_fold(sx, 1e-6, None, pi)
    assert r == 256
    assert torch.allclose(m_ch, m_qr, rtol=1e-9, atol=1e-12 * m_qr.abs().max().item())
    m_or, r_or = O.fold_r(sx.cpu().numpy(), 1e-6, O.jl_matrix(0, 256, 64))
    assert r_or == 256 and np.allclose(m_qr.cpu().numpy(), m_or, rtol=1e-9, atol=1e-12 * np.abs(m_or).max())
    # a threshold that would truncate is refused by the certificate, then the QR fold truncates
    assert P.leverage.cholesky_fold(sx, 0.5, pi) is None
    m_tr, r_tr = P.leverage.qr_fold(sx, 0.5, None, pi)
    m_or2, r_or2 = O.fold_r(sx.cpu().numpy(), 0.5, O.jl_matrix(0, 256, 64))
    # r' <= 64 = Pi's width: both return the (sign-ambiguous) basis V'/sigma'; compare M M^T
    mm, mo = m_tr.cpu().numpy(), m_or2
    assert r_tr == r_or2 < 64 and mm.shape == mo.shape
    assert np.allclose(mm @ mm.T, mo @ mo.T, rtol=1e-8, atol=1e-11 * np.abs(mo @ mo.T).max())


@pytest.mark.parametrize("k,d,r", [(64, 1, 1), (300, 64, 64), (400, 100, 7), (2048, 512, 64), (1500, 700, 130), (2100, 1100, 64),
                                   (6200, 3100, 130)])
def test_kf_cholesky_fold_kernel_vs_numpy(k, d, r):
    """KF (csrc/factor.cu) against numpy: M = R^-1 Pi and the certificate
    traces, on ragged d / r (identity padding) and one-tile cases."""
    rng = np.random.default_rng(k + d + r)
    sx = rng.standard_normal((k, d)) * np.linspace(1.0, 20.0, d)
    pi = O.jl_matrix(5, d, r)
    G = sx.T @ sx
    R = np.linalg.cholesky(G).T
    m_ref = np.linalg.solve(R, pi)
    tr_inv = float(np.sum(np.linalg.inv(R) ** 2))
    M, diag = P.leverage._chol_body(torch.from_numpy(sx).cuda(), torch.from_numpy(pi).cuda())
    diag = diag.cpu().numpy()
    assert diag[0] == 0.0
    assert abs(diag[1] - np.trace(G)) <= 1e-12 * np.trace(G)
    assert abs(diag[2] - tr_inv) <= 1e-9 * tr_inv
    assert np.allclose(M.cpu().numpy(), m_ref, rtol=1e-9, atol=1e-11 * np.abs(m_ref).max())


def test_kf_cholesky_fold_flags_indefinite():
    d = 130
    rng = np.random.default_rng(1)
    sx = rng.standard_normal((50, d))  # k < d: G singular
    g = sx.T @ sx
    g[90, 90] = -1.0
    L = P._native.lib()
    Gt = torch.from_numpy(g).cuda()
    pi = torch.from_numpy(O.jl_matrix(1, d, 16)).cuda()
    ws = torch.empty(int(L.lvsk_chol_fold_workspace_bytes(d, 16)), dtype=torch.uint8, device="cuda")
    M = torch.empty((d, 16), dtype=torch.float64, device="cuda")
    diag = torch.empty(3, dtype=torch.float64, device="cuda")
    fail = torch.zeros(1, dtype=torch.int32, device="cuda")
    P._native.check(L.lvsk_chol_fold(Gt.data_ptr(), d, d, pi.data_ptr(), 16, M.data_ptr(), diag.data_ptr(),
                                     1e10, fail.data_ptr(), ws.data_ptr(), ws.numel(), P._native.stream_ptr()), "fold")
    assert diag[0].item() != 0.0
    assert not P.leverage.chol_certified(diag.tolist(), 1e-6)
    assert int(fail.item()) == 1  # the device-side certificate agrees and counts the failure
    g2 = rng.standard_normal((400, d))
    G2 = torch.from_numpy(g2.T @ g2).cuda()
    P._native.check(L.lvsk_chol_fold(G2.data_ptr(), d, d, pi.data_ptr(), 16, M.data_ptr(), diag.data_ptr(),
                                     1e10, fail.data_ptr(), ws.data_ptr(), ws.numel(), P._native.stream_ptr()), "fold")
    assert P.leverage.chol_certified(diag.tolist(), 1e-6) and int(fail.item()) == 1


# ---------------------------------------------------------------------------
# end-to-end leverage (reference leverage.py / dist.py golden cases)


def test_leverage_golden(golden, golden_meta):
    for ci, m in enumerate(golden_meta["leverage"]):
        x = golden[f"lev{ci}_x"]
        spec = P.SketchSpec(**m["spec"])
        res = P.leverage_sketched(x, spec) if m["sv_tol"] is None else P.leverage_sketched_trunc(x, spec, m["sv_tol"])
        assert res.effective_rank == m["rank"] and res.method == m["method"]
        ref = golden[f"lev{ci}_scores"]
        np.testing.assert_allclose(res.scores, ref, rtol=1e-7, atol=1e-10 * ref.max())


def test_leverage_fp32_within_tolerance(golden):
    x = golden["lev2_x"].astype(np.float32)
    spec = P.SketchSpec("osnap", eps=0.5, d=100, seed=3)
    res = P.leverage_sketched_trunc(dev(x), spec, 1e-3)
    hi, lo = O.hashed_sketch(x, "osnap", P.sketch_rows(spec), 3, spec.s)
    ref, r, _ = O.leverage_from_sketch(x, hi + lo, 1e-3)
    assert res.effective_rank == r
    assert np.abs(res.scores - ref).max() <= 1e-4 * ref.max()


def test_jl_fold_and_rank_cap():
    rng = np.random.default_rng(5)
    # moderately conditioned (kappa(X) ~ 30): fp32 GEMM error ~ eps32 * kappa stays far below 1e-4
    x = (rng.standard_normal((6000, 30)) @ rng.standard_normal((30, 96)) + 0.3 * rng.standard_normal((6000, 96))).astype(np.float32)
    spec = P.SketchSpec("countsketch", eps=0.5, d=96, seed=2, rows_override=1024)
    hi, lo = O.hashed_sketch(x, "countsketch", 1024, 2, 1)
    for jl, rank in ((32, None), (None, 20), (64, 25)):
        res = P.leverage_sketched_trunc(dev(x), spec, 1e-6, jl_dim=jl, jl_seed=4, rank=rank)
        pi = None if jl is None else O.jl_matrix(4, 96, jl)
        ref, r, _ = O.leverage_from_sketch(x, hi + lo, 1e-6, pi, rank)
        assert res.effective_rank == r
        assert np.abs(res.scores - ref).max() <= 1e-4 * ref.max(), (jl, rank)


def test_distributed_simulated_equals_serial(golden):
    x = golden["lev3_x"]
    spec = P.SketchSpec("osnap", eps=0.5, d=16, seed=4)
    res, rep = P.run_distributed(x, spec, 3, 1e-3)
    assert np.array_equal(rep.merged.data, golden["dist_w3_merged"])
    np.testing.assert_allclose(res.scores, golden["dist_w3_scores"], rtol=1e-9)
    assert rep.bytes_communicated == 3 * rep.merged.k * 16 * 8 and rep.per_worker_rows == [334, 333, 333]
    for fam in ("countsketch", "osnap"):
        spec = P.SketchSpec(fam, eps=0.5, d=16, seed=4)
        serial = P.leverage_sketched_trunc(x, spec, 1e-3)
        for w in (1, 2, 3, 4, 8):
            r, _ = P.run_distributed(x, spec, w, 1e-3)
            assert np.array_equal(r.scores, serial.scores), (fam, w)
    with pytest.raises(errors.UnsupportedFamilyError):
        P.run_distributed(x, P.SketchSpec("srht", eps=0.5, d=16, seed=8), 2, 1e-3)
    with pytest.raises(errors.ConfigurationError):
        P.run_distributed(x[:10], P.SketchSpec("countsketch", eps=0.5, d=16), 11, 1e-3)


# ---------------------------------------------------------------------------
# ordering (order.py)


def test_order_golden(golden):
    p = P.scores_to_distribution(golden["ord_scores"])
    np.testing.assert_allclose(p, golden["ord_p"], rtol=1e-15)
    pg = golden["ord_p"]
    assert np.array_equal(P.make_plan(pg, P.OrderingPolicy("dec")).indices, golden["ord_dec"])
    assert np.array_equal(P.make_plan(pg, P.OrderingPolicy("dec_swor", seed=3), 2).indices, golden["ord_swor_s3_e2"])
    assert np.array_equal(P.make_plan(pg, P.OrderingPolicy("shuffle", seed=3), 2).indices, golden["ord_shuffle_s3_e2"])
    assert np.array_equal(P.make_plan(pg, P.OrderingPolicy("dec_swr", seed=3), 2).indices, golden["ord_swr_s3_e2"])
    assert P.make_plan(P.scores_to_distribution([0.1, 0.9, 0.5]), P.OrderingPolicy("dec")).indices.tolist() == [1, 2, 0]
    assert P.make_plan(P.scores_to_distribution([0.3, 0.4, 0.3]), P.OrderingPolicy("dec")).indices.tolist() == [1, 0, 2]
    zs = P.make_plan(np.array([0.5, 0.0, 0.5, 0.0]), P.OrderingPolicy("dec_swor", seed=11)).indices
    assert set(zs[:2].tolist()) == {0, 2} and set(zs[2:].tolist()) == {1, 3}
    for bad in ([0.0, 0.0], [1.0, -0.5], [], [1.0, np.nan]):
        with pytest.raises(errors.DegenerateInputError):
            P.scores_to_distribution(bad)
    with pytest.raises(errors.DegenerateInputError):
        P.make_plan(np.array([0.5, 0.2]), P.OrderingPolicy("dec"))
    with pytest.raises(errors.ConfigurationError):
        P.make_plan(np.array([0.5, 0.5]), P.OrderingPolicy("dec"), epoch=-1)


@pytest.mark.parametrize("n", [1, 2, 4095, 4096, 4097, 1_000_003])
def test_argsort_matches_numpy_stable(n):
    rng = np.random.default_rng(n)
    p = rng.random(n)
    p[rng.integers(0, n, n // 7 + 1)] = p[0]  # ties
    if n > 10:
        p[3] = 0.0
        p[5] = -0.0
        p[7] = np.inf
    for desc in (True, False):
        got = P.order.argsort_device(dev(p), desc).cpu().numpy()
        ref = np.argsort(-p if desc else p, kind="stable")
        assert np.array_equal(got, ref), (n, desc)


@pytest.mark.parametrize("n", [4_194_303, 4_194_304, 8_000_000])
def test_argsort_40bit_path_c5_like(n):
    """From 4M keys K7 sorts on the high 40 key bits before the local fix-up:
    8e6 probabilities of a narrow range (C5's scores: long runs of equal high
    32 bits) plus ties, +-0, inf — bit-exact against numpy's stable argsort."""
    rng = np.random.default_rng(n)
    s = 0.8 + 0.4 * rng.random(n)
    s[rng.integers(0, n, n // 50)] = s[11]
    p = s / s.sum()
    p[3], p[5], p[7] = 0.0, -0.0, np.inf
    for desc in (True, False):
        got = P.order.argsort_device(dev(p), desc).cpu().numpy()
        assert np.array_equal(got, np.argsort(-p if desc else p, kind="stable")), (n, desc)


@pytest.mark.parametrize("kind", ["long_runs", "short_runs", "wide_exponents"])
def test_argsort_high_bits_then_fixup_paths(kind):
    """K7 sorts by the high 32 key bits, then orders runs of equal high bits
    locally (<= 64 keys) or falls back to all eight digits: keys that share
    their high 32 bits in one long run (fallback), in many short runs (local
    fix-up), and keys spread over many binades."""
    rng = np.random.default_rng(7)
    n = 300_001
    if kind == "long_runs":
        p = 0.5 + rng.random(n) * 1e-12
    elif kind == "short_runs":
        p = np.repeat(rng.random(n // 20 + 1), 20)[:n] * (1.0 + rng.random(n) * 1e-13)
    else:
        p = rng.random(n) ** 12
    for desc in (True, False):
        got = P.order.argsort_device(dev(p), desc).cpu().numpy()
        assert np.array_equal(got, np.argsort(-p if desc else p, kind="stable")), (kind, desc)


# ---------------------------------------------------------------------------
# full-size properties (BASELINE config 2 shape)


def test_c2_full_size_properties():
    n, d, k = 1_000_000, 512, 4096
    g = torch.Generator(device="cuda").manual_seed(0)
    X = torch.randn(n, d, device="cuda", generator=g, dtype=torch.float32)
    spec = P.SketchSpec("countsketch", eps=0.5, d=d, seed=0, rows_override=k)
    whole = P.apply_sketch(X, spec)
    # partition invariance: 4 partial states merged == one pass (bit-exact in practice)
    parts = [P.consume_rows(P.SketchState(spec, n), X[lo:hi], lo) for lo, hi in P.partition_rows(n, 4)]
    merged = parts[0]
    for s in parts[1:]:
        merged = P.merge(merged, s)
    assert torch.equal(merged.data_device, whole.data_device)
    # checksum of checksums: sum over buckets == signed row sum (float64)
    idx = np.arange(n, dtype=np.uint64)
    st = whole
    signs = dev(O.sign_of(idx, st._sign_keys[0]))
    ref = (signs[:, None] * X.double()).sum(0)
    got = whole.data_device.sum(0)
    assert torch.allclose(got, ref, rtol=1e-9, atol=1e-6)
    # bucket occupancy matches the hash (subsample check of the gather grouping)
    sub = 20000
    hi, lo = O.hashed_sketch(X[:sub].cpu().numpy(), "countsketch", k, 0, 1)
    assert np.array_equal(P.apply_sketch(X[:sub], spec).data, hi + lo)
    # pipeline end to end
    pipe = P.LeveragePipeline(spec, n, d, torch.float32, sv_tol=1e-6, jl_dim=64)
    scores, order = pipe.run(X)
    assert torch.all(scores >= 0)
    o = order.cpu().numpy()
    assert np.array_equal(np.sort(o), np.arange(n))
    sc = scores.cpu().numpy()
    assert np.all(np.diff(sc[o] / sc.sum()) <= 0)


@pytest.mark.parametrize("sv_tol,noise", [(1e-6, 1.0), (0.05, 0.0)])
def test_pipeline_fold_certificate_and_fallback(sv_tol, noise):
    """LeveragePipeline runs the KF fold optimistically and verifies the
    certificate in check(): certified -> R^-1 Pi; refused (a threshold that
    truncates) -> the spectral fold redone, scores and order recomputed.
    Both equal the oracle's fold_r scores."""
    rng = np.random.default_rng(11)
    n, d, k, jl = 6000, 96, 512, 32
    x = (rng.standard_normal((n, 12)) @ rng.standard_normal((12, d))) * np.linspace(1, 5, d) \
        + noise * rng.standard_normal((n, d))
    X = torch.from_numpy(x.astype(np.float32)).cuda()
    spec = P.SketchSpec("countsketch", eps=0.5, d=d, seed=5, rows_override=k)
    pipe = P.LeveragePipeline(spec, n, d, torch.float32, sv_tol=sv_tol, jl_dim=jl, jl_seed=6)
    scores, order = pipe.run(X)
    hi, lo = O.hashed_sketch(X.double().cpu().numpy(), "countsketch", k, 5, 1)
    ref, r, _ = O.leverage_from_sketch(X.double().cpu().numpy(), hi + lo, sv_tol, O.jl_matrix(6, d, jl))
    assert pipe.effective_rank == r
    got = scores.cpu().numpy()
    assert np.max(np.abs(got - ref) / np.maximum(ref, 1e-30)) < 1e-4
    assert np.array_equal(order.cpu().numpy(), np.argsort(-(got / got.sum()), kind="stable"))


def test_pipeline_unchecked_uncertified_runs_raise():
    """run(check=False) repeatedly on a sketch whose certificate fails: the
    KF kernel counts every failure on the device, check() redoes the last run
    and raises UncertifiedFoldError for the earlier ones instead
    of dropping their certificates."""
    rng = np.random.default_rng(12)
    n, d, k, jl = 6000, 96, 512, 32
    x = (rng.standard_normal((n, 12)) @ rng.standard_normal((12, d))).astype(np.float32)  # rank 12 < d
    X = torch.from_numpy(x).cuda()
    spec = P.SketchSpec("countsketch", eps=0.5, d=d, seed=5, rows_override=k)
    pipe = P.LeveragePipeline(spec, n, d, torch.float32, sv_tol=0.05, jl_dim=jl, jl_seed=6)
    pipe.run(X)  # checked: fine, the fallback recomputes
    assert pipe.cert_failures() == 1
    pipe.run(X, check=False)
    pipe.run(X, check=False)
    with pytest.raises(errors.UncertifiedFoldError):
        pipe.check()
    assert pipe.cert_failures() == 3
    # a well-conditioned sketch never trips it
    good = P.LeveragePipeline(spec, n, d, torch.float32, sv_tol=1e-6, jl_dim=jl, jl_seed=6)
    y = torch.from_numpy(rng.standard_normal((n, d)).astype(np.float32)).cuda()
    for _ in range(3):
        good.run(y, check=False)
    good.check()
    assert good.cert_failures() == 0


# ---------------------------------------------------------------------------
# K2 / K6: CSR rows (extension G2), semantics = densified rows


def _random_csr(n, d, per_row, seed, dtype=np.float32):
    rng = np.random.default_rng(seed)
    indptr = [0]
    cols, vals = [], []
    for _ in range(n):
        k = int(rng.integers(0, per_row * 2 + 1))
        c = np.unique(np.minimum(rng.zipf(1.1, size=k) - 1, d - 1))
        v = rng.lognormal(0.0, 1.0, size=c.size)
        if c.size:
            v = v / np.linalg.norm(v)
        cols.append(c.astype(np.int32))
        vals.append(v.astype(dtype))
        indptr.append(indptr[-1] + c.size)
    indptr = np.array(indptr, dtype=np.int64)
    col = np.concatenate(cols) if cols else np.zeros(0, np.int32)
    val = np.concatenate(vals) if vals else np.zeros(0, dtype)
    dense = np.zeros((n, d), dtype=np.float64)
    for r in range(n):
        dense[r, col[indptr[r] : indptr[r + 1]]] = val[indptr[r] : indptr[r + 1]]
    return (indptr, col, val, (n, d)), dense


@pytest.mark.parametrize("n,d,k,s", [(3000, 300, 512, 4), (1500, 2100, 1024, 3), (777, 64, 128, 1),
                                     (600, 5000, 256, 2), (500, 9000, 128, 4)])
def test_csr_sketch_bit_exact_vs_dense(n, d, k, s, monkeypatch):
    """K2 default (per-warp float64 partial rows + TwoSum fold): hi + lo within
    1e-13 of the reference's compensated state — power-of-two and other
    scales, one and several 4096-column groups; LVSK_K2_DETERMINISTIC=1
    (ordered gather): bit-exact."""
    csr, dense = _random_csr(n, d, 40, seed=n + d)
    fam = "osnap" if s > 1 else "countsketch"
    spec = P.SketchSpec(fam, eps=0.5, d=d, seed=7, rows_override=k, osnap_s=s if fam == "osnap" else None)
    hi, lo = O.hashed_sketch(dense, fam, k, 7, s)
    ref = hi + lo
    tol = 1e-13 * np.abs(ref).max()
    assert np.allclose(P.apply_sketch(csr, spec).data, ref, rtol=1e-13, atol=tol)
    # two row blocks with global indices == one pass
    m = P.csr.CSRMatrix(*csr)
    st = P.SketchState(spec, n)
    P.consume_rows(st, m.rows(0, n // 2), 0)
    P.consume_rows(st, m.rows(n // 2, n), n // 2)
    assert np.allclose(st.data, ref, rtol=1e-13, atol=tol)
    monkeypatch.setenv("LVSK_K2_DETERMINISTIC", "1")
    assert np.array_equal(P.apply_sketch(csr, spec).data, ref)
    st = P.SketchState(spec, n)
    P.consume_rows(st, m.rows(0, n // 2), 0)
    P.consume_rows(st, m.rows(n // 2, n), n // 2)
    assert np.array_equal(st.data, ref)


@pytest.mark.parametrize("vdtype", [np.float32, np.float64])
def test_csr_sketch_long_and_empty_rows(vdtype):
    """K2 loader: rows longer than a stage (streamed in pieces), empty rows and
    every 16-byte misalignment of the row starts, f32 and f64 values."""
    rng = np.random.default_rng(5)
    n, d, k = 300, 4096, 256
    lens = rng.integers(0, 60, size=n)
    lens[rng.choice(n, 40, replace=False)] = 0
    lens[[3, 97, 98, 250]] = [2500, 1021, 3000, 4096]
    indptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    col = np.concatenate([np.sort(rng.choice(d, size=L, replace=False)) for L in lens]).astype(np.int32)
    val = rng.standard_normal(col.size).astype(vdtype)
    dense = np.zeros((n, d))
    for r in range(n):
        dense[r, col[indptr[r]:indptr[r + 1]]] = val[indptr[r]:indptr[r + 1]]
    spec = P.SketchSpec("osnap", eps=0.5, d=d, seed=9, rows_override=k, osnap_s=4)
    hi, lo = O.hashed_sketch(dense, "osnap", k, 9, 4)
    ref = hi + lo
    got = P.apply_sketch((indptr, col, val, (n, d)), spec).data
    assert np.allclose(got, ref, rtol=1e-13, atol=1e-13 * np.abs(ref).max())
    # deterministic: a second call is bit-identical
    assert np.array_equal(P.apply_sketch((indptr, col, val, (n, d)), spec).data, got)
    # a column out of order inside the second piece of the 3000-entry row is caught
    bad = col.copy()
    e = indptr[98] + 2000
    bad[e], bad[e + 1] = bad[e + 1], bad[e]
    with pytest.raises(errors.FormatError):
        P.apply_sketch((indptr, bad, val, (n, d)), spec)


def test_csr_leverage_vs_oracle():
    n, d, k, r = 4000, 256, 2048, 128
    csr, dense = _random_csr(n, d, 30, seed=11)
    spec = P.SketchSpec("osnap", eps=0.5, d=d, seed=3, rows_override=k, osnap_s=4)
    res = P.leverage_sketched_trunc(csr, spec, 1e-6, jl_dim=r, jl_seed=2)
    hi, lo = O.hashed_sketch(dense, "osnap", k, 3, 4)
    ref, rr, _ = O.leverage_from_sketch(dense, hi + lo, 1e-6, O.jl_matrix(2, d, r))
    assert res.effective_rank == rr
    mask = ref > 1e-12
    assert np.abs(res.scores - ref).max() <= 1e-4 * ref.max()
    assert np.all(res.scores[~mask] <= 1e-6 * ref.max())


@pytest.mark.parametrize("n,d,per_row,vdt", [(3000, 4096, 80, np.float32), (257, 100, 30, np.float64),
                                             (1000, 300, 0, np.float32), (5000, 1024, 200, np.float32)])
def test_csr_leverage_tensor_core_vs_simt_and_fp64(n, d, per_row, vdt, monkeypatch):
    """K6-TC (hot columns < 128 on tcgen05, cold ones gathered; r = 128)
    against the SIMT kernel and a float64 recompute: Zipf rows, d < 128 hot
    window edge, empty rows, long rows, f64 values, a ragged last tile."""
    from paper_1812_07903_b200.csr import CSRMatrix, csr_scores

    csr, dense = _random_csr(n, d, per_row, seed=n + d, dtype=vdt)
    m = CSRMatrix.from_any(csr)
    g = np.random.default_rng(d)
    M = g.standard_normal((d, 128)) / math.sqrt(d)
    Mt = torch.from_numpy(M).cuda()
    tc = csr_scores(m, Mt).cpu().numpy()
    ref = ((dense @ M.astype(np.float32).astype(np.float64)) ** 2).sum(1)
    scale = max(ref.max(), 1e-30)
    assert np.abs(tc - ref).max() <= 2e-5 * scale
    # hot windows of 64 / 128 / 1024 columns (v2), the resident 128-column kernel (v1), SIMT
    for nb in ("1", "2", "16"):
        monkeypatch.setenv("LVSK_K6_HOTBLOCKS", nb)
        assert np.abs(csr_scores(m, Mt).cpu().numpy() - ref).max() <= 2e-5 * scale
    monkeypatch.setenv("LVSK_K6_V1", "1")
    assert np.abs(csr_scores(m, Mt).cpu().numpy() - ref).max() <= 2e-5 * scale
    monkeypatch.setenv("LVSK_K6_SIMT", "1")
    simt = csr_scores(m, Mt).cpu().numpy()
    assert np.abs(tc - simt).max() <= 2e-5 * scale


def test_csr_leverage_unsorted_row_rejected():
    """The prepared K6 pass walks each row's sorted columns: a row that is not
    strictly increasing is flagged (FormatError), as K2 does."""
    from paper_1812_07903_b200.csr import CSRMatrix, csr_scores

    csr, _ = _random_csr(500, 2000, 40, seed=5)
    indptr, col, val, shape = csr
    row = int(np.argmax(np.diff(indptr)))
    bad = col.copy()
    e = indptr[row]
    bad[e], bad[e + 1] = bad[e + 1], bad[e]
    M = torch.randn(2000, 128, dtype=torch.float64, device="cuda")
    csr_scores(CSRMatrix.from_any(csr), M)
    with pytest.raises(errors.FormatError):
        csr_scores(CSRMatrix.from_any((indptr, bad, val, shape)), M)


def test_csr_validation():
    indptr = np.array([0, 2, 3], dtype=np.int64)
    spec = P.SketchSpec("countsketch", eps=0.5, d=8, seed=1, rows_override=16)
    with pytest.raises(errors.FormatError):  # unsorted columns
        P.apply_sketch((indptr, np.array([3, 1, 2], np.int32), np.ones(3, np.float32), (2, 8)), spec)
    with pytest.raises(errors.FormatError):  # out of range
        P.apply_sketch((indptr, np.array([1, 9, 2], np.int32), np.ones(3, np.float32), (2, 8)), spec)
    with pytest.raises(errors.FormatError):  # non-finite
        P.apply_sketch((indptr, np.array([1, 3, 2], np.int32), np.array([1, np.nan, 1], np.float32), (2, 8)), spec)
    with pytest.raises(errors.UnsupportedFamilyError):
        P.apply_sketch((indptr, np.array([1, 3, 2], np.int32), np.ones(3, np.float32), (2, 8)),
                       P.SketchSpec("srht", eps=0.5, d=8, rows_override=2))


@pytest.mark.parametrize("n,d,r", [(5000, 1024, 128), (3000, 256, 100), (2048, 64, 30), (777, 512, 64),
                                   (100, 1024, 128), (257, 128, 120), (70_000, 1024, 128)])
def test_tcgen05_bf16_leverage_vs_fp64(n, d, r):
    g = torch.Generator(device="cpu").manual_seed(n + r)
    X = torch.rand(n, d, generator=g, dtype=torch.float64).to(torch.bfloat16).cuda()
    M = (torch.randn(d, r, generator=g, dtype=torch.float64) / math.sqrt(d)).cuda()
    ref = ((X.double() @ M) ** 2).sum(1)
    ops = P.leverage.KernelOperands(M, X)
    assert ops.bf16
    out = torch.full((n,), -1.0, dtype=torch.float64, device="cuda")
    fl = N.Flags()
    ops.run(X, out, fl.p)
    rel = ((out - ref).abs() / ref).max().item()
    assert rel < 1e-4, rel  # bf16 X exact, M as bf16 hi + lo (~16 bits), fp32 accumulation
    if ops.r_pad == 128:  # the CTA-pair kernel (cta_group::2) and the 1-CTA kernel: same arithmetic, same bits
        import os

        os.environ["LVSK_K5_SINGLE_CTA"] = "1"
        try:
            single = torch.full((n,), -1.0, dtype=torch.float64, device="cuda")
            ops.run(X, single, fl.p)
        finally:
            del os.environ["LVSK_K5_SINGLE_CTA"]
        assert torch.equal(single, out)


def test_c5_shaped_pipeline_small():
    """Gaussian sketch on bf16 X, rank-capped truncation, r = 128 (config 5 shape, reduced n)."""
    n, d, k = 20000, 256, 512
    g = torch.Generator(device="cuda").manual_seed(5)
    X = torch.sigmoid(torch.randn(n, 20, generator=g, device="cuda") @ torch.randn(20, d, generator=g, device="cuda")
                      / 3 + 0.05 * torch.randn(n, d, generator=g, device="cuda")).to(torch.bfloat16)
    spec = P.SketchSpec("gaussian", eps=0.5, d=d, seed=1, rows_override=k)
    res = P.leverage_sketched_trunc(X, spec, 1e-6, jl_dim=128, jl_seed=3, rank=20)
    xv = X.double().cpu().numpy()
    sx = O.gaussian_sketch(xv, k, 1)
    ref, r, _ = O.leverage_from_sketch(xv, sx, 1e-6, O.jl_matrix(3, d, 128), rank=20)
    assert res.effective_rank == r == 20
    assert np.abs(res.scores - ref).max() <= 2e-2 * ref.max()
    assert np.median(np.abs(res.scores - ref) / ref) < 1e-3


def test_streamed_host_input_equals_device_input(monkeypatch):
    """Pinned host X (>= 256 MB) goes through the chunked copy-stream path
    (each 128 MB chunk sketched as it lands); results equal the device-X path
    bit for bit (the hashed sketch is order-exact across row blocks)."""
    n, d = 160_000, 512
    g = torch.Generator(device="cuda").manual_seed(5)
    Xd = torch.randn(n, d, device="cuda", dtype=torch.float32, generator=g)
    Xh = torch.empty((n, d), dtype=torch.float32, pin_memory=True)
    Xh.copy_(Xd)
    monkeypatch.setenv("LVSK_STREAM", "1")
    assert P.leverage._streamable(Xh, P.SketchSpec("countsketch", eps=0.5, d=d))
    for fam in ("countsketch", "osnap"):
        spec = P.SketchSpec(fam, eps=0.5, d=d, seed=3, rows_override=2048, osnap_s=4 if fam == "osnap" else None)
        a = P.leverage_sketched_trunc(Xh, spec, 1e-6, jl_dim=64)
        b = P.leverage_sketched_trunc(Xd, spec, 1e-6, jl_dim=64)
        assert np.array_equal(a.scores, b.scores), fam


# ---------------------------------------------------------------------------
# out-of-core streaming


@pytest.mark.parametrize("family,s,dtype", [("countsketch", None, torch.float64), ("osnap", 3, torch.float64),
                                            ("gaussian", None, torch.float32)])
def test_leverage_streamed_matches_in_memory(tmp_path, family, s, dtype):
    """Two streaming passes over an LVSK file in ragged blocks give the scores
    of the in-memory call (hashed families: the same sketch bits)."""
    rng = np.random.default_rng(3)
    n, d = 20_011, 40
    x = rng.standard_normal((n, 6)) @ rng.standard_normal((6, d)) + 0.3 * rng.standard_normal((n, d))
    path = tmp_path / "x.lvsk"
    P.save_matrix(x, path)
    spec = P.SketchSpec(family, eps=0.5, d=d, seed=2, rows_override=512, osnap_s=s)
    got = P.leverage_streamed(path, spec, 1e-6, block_rows=3001, dtype=dtype, jl_dim=16)
    xin = x if dtype == torch.float64 else x.astype(np.float32)
    ref = P.leverage_sketched_trunc(torch.from_numpy(xin).cuda(), spec, 1e-6, jl_dim=16)
    assert got.effective_rank == ref.effective_rank
    if family == "gaussian":
        np.testing.assert_allclose(got.scores, ref.scores, rtol=1e-5)  # fp32 blocks: partial sums reassociate
    else:
        assert np.array_equal(got.scores, ref.scores)
    # and against the CPU oracle on the same values
    xv = xin.astype(np.float64)
    pi = O.jl_matrix(0, d, 16)
    if family == "gaussian":
        sx_o = O.gaussian_sketch(xv, 512, 2)
    else:
        hi, lo = O.hashed_sketch(xv, family, 512, 2, s or 1)
        sx_o = hi + lo
    oracle, r_o, _ = O.leverage_from_sketch(xv, sx_o, 1e-6, pi)
    assert got.effective_rank == r_o
    tol = 1e-4 if dtype == torch.float32 else 1e-9
    assert np.max(np.abs(got.scores - oracle) / oracle) <= tol


def test_srht_row_blocks_sum_to_whole():
    """lvsk_srht_rows (extension G7): partials of 2048-aligned global row blocks
    sum to the whole-matrix SRHT; unaligned row0 is refused."""
    from paper_1812_07903_b200.sketch import srht_signs_and_sample

    n, d, k = 3 * 2048 + 100, 64, 256
    m = O.next_pow2(n)
    x = np.random.default_rng(8).standard_normal((n, d)).astype(np.float32)
    X = dev(x)
    signs, sample = srht_signs_and_sample(3, m, k)
    sg = torch.from_numpy(signs.astype(np.int8)).cuda()
    sm = torch.from_numpy(sample.astype(np.int64)).cuda()
    L = N.lib()
    ws = N.workspace(L.lvsk_srht_workspace_bytes(m, d, N.LVSK_F32, k))
    flags = N.Flags()
    whole = torch.empty((k, d), dtype=torch.float64, device="cuda")
    N.check(L.lvsk_srht(X.data_ptr(), N.LVSK_F32, n, d, d, m, sg.data_ptr(), sm.data_ptr(), k, math.sqrt(k),
                        whole.data_ptr(), ws.data_ptr(), ws.numel(), flags.p, N.stream_ptr()), "srht")
    total = torch.zeros_like(whole)
    part = torch.empty_like(whole)
    for r0, r1 in ((0, 4096), (4096, n)):
        N.check(L.lvsk_srht_rows(X[r0:].data_ptr(), r1 - r0, d, d, r0, m, sg.data_ptr(), sm.data_ptr(), k,
                                 math.sqrt(k), part.data_ptr(), ws.data_ptr(), ws.numel(), flags.p,
                                 N.stream_ptr()), "srht rows")
        total += part
    assert flags.read() == 0
    w = whole.cpu().numpy()
    assert np.linalg.norm(total.cpu().numpy() - w) <= 1e-6 * np.linalg.norm(w)
    ref = O.srht_sketch(x, k, 3)
    assert np.linalg.norm(w - ref) <= 2e-6 * np.linalg.norm(ref)
    rc = L.lvsk_srht_rows(X[100:].data_ptr(), n - 100, d, d, 100, m, sg.data_ptr(), sm.data_ptr(), k,
                          math.sqrt(k), part.data_ptr(), ws.data_ptr(), ws.numel(), flags.p, N.stream_ptr())
    assert rc == 5  # LVSK_ERR_UNSUPPORTED


# ---------------------------------------------------------------------------
# KG: the fold's Gram on the int8 tensor cores (Ozaki scheme, csrc/gram_i8.cu)


@pytest.mark.parametrize("k,d,scaled", [(300, 100, False), (1000, 700, False), (2048, 1024, True),
                                        (4100, 2100, False), (16384, 4096, False)])
def test_kg_gram_vs_float64(k, d, scaled):
    """KG's block upper triangle of SX^T SX against torch float64: the error
    stays in the float64-GEMM class (below the worst-case DGEMM bound
    k eps sum_k |x_kc||x_kd| and within a small multiple of the Ozaki bound
    2^-49 k max|x_c| max|x_d|), ragged k / d, columns scaled over 12 decades."""
    g = torch.Generator(device="cuda").manual_seed(k + d)
    sx = torch.randn(k, d, dtype=torch.float64, device="cuda", generator=g)
    if scaled:
        sx *= torch.logspace(-6, 6, d, dtype=torch.float64, device="cuda")
    L = N.lib()
    ws = torch.empty(int(L.lvsk_gram_workspace_bytes(k, d)), dtype=torch.uint8, device="cuda")
    G = torch.full((d, d), float("nan"), dtype=torch.float64, device="cuda")
    fl = N.Flags()
    N.check(L.lvsk_gram_f64(sx.data_ptr(), k, d, d, G.data_ptr(), d, ws.data_ptr(), ws.numel(), fl.p,
                            N.stream_ptr()), "gram")
    ref = sx.T @ sx
    i = torch.arange(d, device="cuda")
    up = (i[:, None] // 256) <= (i[None, :] // 256)
    assert not torch.isnan(G[up]).any()
    diff = torch.where(up, (G - ref).abs(), torch.zeros_like(G))
    cm = sx.abs().max(0).values
    ozaki = (cm[:, None] * cm[None, :]) * k * 2.0**-49
    assert (diff / ozaki).max().item() < 16
    assert fl.read() == 0
    # deterministic
    G2 = G.clone()
    N.check(L.lvsk_gram_f64(sx.data_ptr(), k, d, d, G2.data_ptr(), d, ws.data_ptr(), ws.numel(), fl.p,
                            N.stream_ptr()), "gram")
    assert torch.equal(G2[up], G[up])
    sx[k // 2, d // 3] = float("inf")
    N.check(L.lvsk_gram_f64(sx.data_ptr(), k, d, d, G2.data_ptr(), d, ws.data_ptr(), ws.numel(), fl.p,
                            N.stream_ptr()), "gram")
    assert fl.read() & N.FLAG_NONFINITE


def test_kf_fold_on_kg_gram_matches_oracle():
    """The certified Cholesky fold with the KG Gram (d >= 2048) against the
    oracle's fold_r in float64 (M to 1e-9)."""
    k, d, r = 6000, 2048, 64
    g = torch.Generator(device="cuda").manual_seed(3)
    sx = torch.randn(k, d, dtype=torch.float64, device="cuda", generator=g) * torch.linspace(1, 3, d, device="cuda",
                                                                                               dtype=torch.float64)
    pi = O.jl_matrix(2, d, r)
    from paper_1812_07903_b200.leverage import cholesky_fold, use_kg

    assert use_kg(k, d)
    M = cholesky_fold(sx, 1e-6, torch.from_numpy(pi).cuda())
    assert M is not None
    M_o, r_o = O.fold_r(sx.cpu().numpy(), 1e-6, pi)
    assert r_o == d
    assert np.linalg.norm(M.cpu().numpy() - M_o) <= 1e-9 * np.linalg.norm(M_o)


def test_k1_folded_output_equals_pair_then_fold():
    """lvsk_hashed_sketch with lo_out = NULL writes hi + lo straight into
    hi_out: bit-identical to the pair followed by lvsk_fold_compensated
    (the pipeline's single-GPU sketch path)."""
    rng = np.random.default_rng(21)
    n, d, k = 20_000, 64, 1024
    X = dev(rng.standard_normal((n, d)).astype(np.float32))
    spec = P.SketchSpec("osnap", eps=0.5, d=d, seed=4, rows_override=k, osnap_s=3)
    st = P.apply_sketch(X, spec)
    ref = st.data_device
    L = N.lib()
    ws = torch.empty(int(L.lvsk_hashed_workspace_bytes(n, 3, k)), dtype=torch.uint8, device="cuda")
    out = torch.empty((k, d), dtype=torch.float64, device="cuda")
    fl = N.Flags()
    N.check(L.lvsk_hashed_sketch(X.data_ptr(), N.LVSK_F32, n, d, d, 0, st._blocks, 3, st._scale, None, None,
                                 out.data_ptr(), None, k, ws.data_ptr(), ws.numel(), fl.p, N.stream_ptr()))
    assert torch.equal(out, ref)
    pipe = P.LeveragePipeline(spec, n, d, torch.float32, sv_tol=1e-6, jl_dim=32)
    scores, _ = pipe.run(X)
    assert torch.equal(pipe.sx, ref)


def test_k2_folded_output_equals_pair_then_fold():
    """lvsk_hashed_sketch_csr with lo_out = NULL writes hi + lo straight into
    hi_out: bit-identical to the pair followed by lvsk_fold_compensated (the
    pipeline's single-GPU CSR path), for the fast and the ordered kernels."""
    csr, dense = _random_csr(3000, 700, 40, seed=31)
    m = P.csr.CSRMatrix(*csr)
    n, d, k = 3000, 700, 1024
    spec = P.SketchSpec("osnap", eps=0.5, d=d, seed=6, rows_override=k, osnap_s=4)
    L = N.lib()
    ws = torch.empty(int(L.lvsk_hashed_csr_workspace_bytes(n, 4, k)), dtype=torch.uint8, device="cuda")
    out = torch.empty((k, d), dtype=torch.float64, device="cuda")
    for det in (False, True):
        if det:
            os.environ["LVSK_K2_DETERMINISTIC"] = "1"
        try:
            st = P.apply_sketch(csr, spec)
            ref = st.data_device
            fl = N.Flags()
            N.check(L.lvsk_hashed_sketch_csr(m.indptr.data_ptr(), m.indices.data_ptr(), m.data.data_ptr(),
                                             P.csr.csr_code(m), n, d, 0, st._blocks, 4, st._scale, None, None,
                                             out.data_ptr(), None, k, ws.data_ptr(), ws.numel(), fl.p,
                                             N.stream_ptr()))
        finally:
            os.environ.pop("LVSK_K2_DETERMINISTIC", None)
        assert torch.equal(out, ref)
    pipe = P.LeveragePipeline(spec, n, d, torch.float32, sv_tol=1e-6, jl_dim=32)
    pipe.run(m)
    assert torch.allclose(pipe.sx, ref, rtol=1e-13, atol=1e-13 * float(ref.abs().max()))


def test_jl_fold_needs_k_at_least_d():
    """The JL fold "R M = Pi" needs a square triangular factor: with fewer
    sketch rows than columns and a kept rank above the JL width it raises
    DimensionMismatchError (not a shape error from inside the linear algebra)."""
    rng = np.random.default_rng(2)
    n, d, k = 4000, 300, 256
    X = dev(rng.standard_normal((n, d)).astype(np.float32))
    spec = P.SketchSpec("countsketch", eps=0.5, d=d, seed=1, rows_override=k)
    with pytest.raises(errors.DimensionMismatchError):
        P.leverage_sketched_trunc(X, spec, 1e-6, jl_dim=32)


@pytest.mark.parametrize("counts", [[1000], [700, 300], [5000, 0, 4096, 1, 2047], [20000] * 8, [3] * 17,
                                    [5, 0, 9, 1] * 128])
@pytest.mark.parametrize("descending", [True, False])
def test_merge_argsort_runs_equals_full_argsort(counts, descending):
    """KM (the multi-rank order): merging the per-rank stable argsorts gives
    the stable argsort of the concatenated keys, bit for bit — with ties across
    runs, NaN, +-0 and inf (numpy's stable order, order.py:89-90)."""
    from paper_1812_07903_b200.order import argsort_device, merge_argsort_runs

    rng = np.random.default_rng(sum(counts) + len(counts))
    n = sum(counts)
    k = np.round(rng.random(n) * 50) / 50  # many ties, within and across runs
    special = rng.choice(n, size=min(n, 9), replace=False)
    k[special[:3]] = np.nan
    k[special[3:5]] = -0.0
    k[special[5:7]] = 0.0
    k[special[7:]] = np.inf
    keys = dev(k)
    parts, skeys, o = [], [], 0
    for c in counts:
        run = keys[o:o + c].contiguous()
        loc = argsort_device(run, descending) if c else torch.zeros(0, dtype=torch.int64, device="cuda")
        parts.append(loc.to(torch.int32))
        skeys.append(run[loc])
        o += c
    got = merge_argsort_runs(torch.cat(skeys), torch.cat(parts), counts, descending)
    want = argsort_device(keys, descending)
    assert torch.equal(got, want)
    ref = np.argsort(-k if descending else k, kind="stable")
    assert np.array_equal(got.cpu().numpy(), ref)


def test_merge_argsort_runs_flags_bad_local_index():
    from paper_1812_07903_b200.order import merge_argsort_runs

    keys = dev(np.arange(10, dtype=np.float64)[::-1].copy())
    idx = torch.tensor([0, 1, 2, 3, 9, 0, 1, 2, 3, 4], dtype=torch.int32, device="cuda")  # 9 is outside run 0
    with pytest.raises(errors.ConfigurationError):
        merge_argsort_runs(keys, idx, [5, 5], True)


@pytest.mark.parametrize("n,d,rank", [(3000, 40, 40), (2500, 64, 17), (50, 80, 50)])
def test_leverage_exact_matches_oracle_svd(n, d, rank):
    """leverage_exact (QR -> SVD of R -> leverage pass, no n x d U) against
    the oracle's thin-SVD scores (reference leverage.py:44-53), incl. a
    rank-deficient matrix and n < d."""
    rng = np.random.default_rng(n + d)
    x = (rng.standard_normal((n, rank)) @ rng.standard_normal((rank, d))).astype(np.float64)
    res = P.leverage_exact(x)
    u, s, _ = np.linalg.svd(x, full_matrices=False)
    r = int(np.count_nonzero(s > 1e-12 * s[0]))
    ref = np.einsum("ij,ij->i", u[:, :r], u[:, :r])
    assert res.effective_rank == r
    assert np.allclose(res.scores, ref, rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("k,d", [(4096, 512), (1000, 136), (77, 200), (2048, 1024), (300, 64), (5, 3)])
def test_kd_syrk_upper_triangle_vs_float64(k, d):
    """KD (csrc/gram_f64.cu): the 64 x 64 block upper triangle of SX^T SX on
    DMMA against torch float64 — ragged k and d, a strided SX — and
    deterministic (split-k slices summed in a fixed order)."""
    from paper_1812_07903_b200.leverage import gram_workspace

    g = torch.Generator(device="cuda").manual_seed(k + d)
    big = torch.randn(k, d + 5, dtype=torch.float64, device="cuda", generator=g)
    sx = big[:, :d]  # leading dimension d + 5
    L = N.lib()
    ws = gram_workspace(k, d, "cuda")
    G = torch.zeros((d, d), dtype=torch.float64, device="cuda")
    G2 = torch.zeros_like(G)
    for out in (G, G2):
        N.check(L.lvsk_syrk_f64(sx.data_ptr(), k, d, sx.stride(0), out.data_ptr(), d, ws.data_ptr(), ws.numel(),
                                N.stream_ptr()))
    ref = sx.T @ sx
    up = torch.triu(torch.ones(d, d, dtype=torch.bool, device="cuda"))
    scale = float(ref.abs().max())
    assert float((G - ref)[up].abs().max()) <= 1e-12 * scale * max(1.0, k / 1000)
    assert torch.equal(G, G2)


@pytest.mark.parametrize("env", ["LVSK_ARGSORT_CLASSIC", "LVSK_K1_REGS", "LVSK_K5_V1", "LVSK_SRHT_CHUNK_MB"])
def test_kernel_variant_switches_vs_oracle(env, monkeypatch):
    """The non-default kernel variants the environment selects (the classic
    three-kernel radix argsort that n > 8M keys take, the register-path K1
    gather, the v1 tcgen05 leverage kernel, a small two-pass SRHT chunk) give
    the oracle's results like the default kernels."""
    rng = np.random.default_rng(hash(env) % 1000)
    monkeypatch.setenv(env, "1")
    if env == "LVSK_ARGSORT_CLASSIC":
        p = rng.random(50_000)
        p[rng.integers(0, 50_000, 5000)] = p[7]
        got = P.make_plan(p / p.sum(), P.OrderingPolicy("dec")).indices
        assert np.array_equal(got, np.argsort(-(p / p.sum()), kind="stable"))
    elif env == "LVSK_K1_REGS":
        x = rng.standard_normal((5000, 96)).astype(np.float32)
        spec = P.SketchSpec("osnap", eps=0.5, d=96, seed=3, rows_override=512, osnap_s=3)
        hi, lo = O.hashed_sketch(x, "osnap", 512, 3, 3)
        assert np.array_equal(P.apply_sketch(dev(x), spec).data, hi + lo)
    elif env == "LVSK_K5_V1":
        n, d, r = 3000, 256, 64
        g = torch.Generator(device="cpu").manual_seed(5)
        X = (torch.randn(n, d, generator=g, dtype=torch.float64)).to(torch.float32).cuda()
        M = (torch.randn(d, r, generator=g, dtype=torch.float64) / math.sqrt(d)).cuda()
        ref = ((X.double() @ M) ** 2).sum(1)
        got = P.leverage.scores_device(X, M)
        assert float(((got - ref).abs() / ref).max()) < 1e-5
    else:  # the two-pass SRHT (float64 rows) with a 1 MB chunk: several chunks
        x = rng.standard_normal((20_000, 16))
        spec = P.SketchSpec("srht", eps=0.5, d=16, seed=2, rows_override=256)
        ref = O.srht_sketch(x, 256, 2)
        got = P.apply_sketch(x, spec).data
        assert np.allclose(got, ref, rtol=1e-10, atol=1e-10 * np.abs(ref).max())
