"""CPU oracle for the sketched leverage-score path — TEST INFRASTRUCTURE ONLY.

This module is a plain numpy (float64) restatement of the reference package
``levsketch`` (arXiv 1812.07903, ``/root/reference/pkg/src/levsketch``) for
the hot path ``S·X -> thin SVD + truncation -> fold M -> ||X·M||^2 ->
ordering``.  It exists to CHECK the CUDA product path; nothing in
``paper_1812_07903_b200`` imports it.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may call it.

Pinning: every reference-backed function here is checked bit-exactly against
golden vectors produced by importing the reference itself
(``oracle/gen_golden.py`` -> ``tests/golden/*.npz``, numpy version recorded).
The extensions the reference does not have (Gaussian sketch, JL fold,
fixed-rank truncation, CSR ingestion) are restatements of the published
algorithms and are marked "parity unpinned" where they appear.
"""

from __future__ import annotations

import math

import numpy as np

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
# Stream tags, reference sketch.py:49-50 and order.py:419.
HASH_TAG = {"countsketch": 0x6353, "osnap": 0x6F53, "srht": 0x7253}
SRHT_TAG = 0x5348
ORDER_TAG = 0x4F52
# Extensions (no reference counterpart): JL projection and Gaussian sketch keys.
JL_TAG = 0x4A4C
GAUSS_KEY_XOR = 0x47415553
DEFAULT_C = {"countsketch": 1.0, "osnap": 2.0, "srht": 1.0, "gaussian": 1.0}


# ---------------------------------------------------------------------------
# Sizing (reference sketch.py:89-124)


def osnap_nnz(family: str, d: int, osnap_s: int | None) -> int:
    """Nonzeros per column: 1 except OSNAP (default ceil(log2 d)); sketch.py:93-100."""
    if family != "osnap":
        return 1
    if osnap_s is not None:
        return osnap_s
    return max(1, math.ceil(math.log2(d)))


def sketch_rows(family, eps, d, osnap_s=None, rows_override=None, sizing_c=None) -> int:
    """Row count k; sketch.py:110-124 (gaussian: the CountSketch-free JL rule
    ceil(c*d/eps^2), an extension)."""
    if rows_override is not None:
        return rows_override
    c = DEFAULT_C[family] if sizing_c is None else sizing_c
    if family == "countsketch":
        return max(1, math.ceil(c * (d / eps) ** 2))
    if family == "gaussian":
        return max(1, math.ceil(c * d / eps**2))
    target = c * (d / eps**2) * math.log(d)
    if family == "osnap":
        return max(osnap_nnz(family, d, osnap_s), math.ceil(target))
    p = 1
    while p < max(1, math.ceil(target)):
        p <<= 1
    return p


# ---------------------------------------------------------------------------
# Hash keys and hash functions (reference sketch.py:131-159, 232-239)


def splitmix_keys(seed: int, tag: int, count: int) -> list[int]:
    """``count`` outputs of the seeded splitmix64 stream; sketch.py:131-138."""
    state = (seed ^ (tag * GOLDEN)) & M64
    out = []
    for _ in range(count):
        state = (state + GOLDEN) & M64
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        out.append((z ^ (z >> 31)) & M64)
    return out


class HashParams:
    """Per-block multiply-shift / sign keys; SketchState.__init__ sketch.py:227-239."""

    def __init__(self, family: str, seed: int, k: int, s: int):
        if k < s:
            raise ValueError("k below s")
        base, rem = divmod(k, s)
        self.s = s
        self.k = k
        self.sizes = [base + (1 if j < rem else 0) for j in range(s)]
        offs, acc = [], 0
        for sz in self.sizes:
            offs.append(acc)
            acc += sz
        self.offsets = offs
        keys = splitmix_keys(seed, HASH_TAG[family], 3 * s)
        self.a = [keys[j] | 1 for j in range(s)]
        self.b = [keys[s + j] for j in range(s)]
        self.sign_keys = [keys[2 * s + j] for j in range(s)]
        self.scale = 1.0 / math.sqrt(s)


def mix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on uint64 arrays; sketch.py:141-148."""
    x = np.asarray(x, dtype=np.uint64).copy()
    x ^= x >> np.uint64(30)
    x *= np.uint64(0xBF58476D1CE4E5B9)
    x ^= x >> np.uint64(27)
    x *= np.uint64(0x94D049BB133111EB)
    x ^= x >> np.uint64(31)
    return x


def bucket_of(idx: np.ndarray, a: int, b: int, size: int) -> np.ndarray:
    """Top-32-bit multiply-shift into [0, size); sketch.py:151-154."""
    v = np.uint64(a) * np.asarray(idx, dtype=np.uint64) + np.uint64(b)
    return ((v >> np.uint64(32)) * np.uint64(size)) >> np.uint64(32)


def sign_of(idx: np.ndarray, key: int) -> np.ndarray:
    """+-1.0 from the low bit of mix64(idx ^ key); sketch.py:157-159."""
    bit = mix64(np.asarray(idx, dtype=np.uint64) ^ np.uint64(key)) & np.uint64(1)
    return 1.0 - 2.0 * bit.astype(np.float64)


def block_buckets(hp: HashParams, idx: np.ndarray, j: int) -> np.ndarray:
    return (hp.offsets[j] + bucket_of(idx, hp.a[j], hp.b[j], hp.sizes[j]).astype(np.int64)).astype(np.int64)


# ---------------------------------------------------------------------------
# Compensated hashed sketch (reference sketch.py:166-191, 260-266, 289-312)


def two_sum(a, b):
    """Knuth TwoSum: s + err == a + b exactly; sketch.py:166-170."""
    s = a + b
    bp = s - a
    err = (a - (s - bp)) + (b - bp)
    return s, err


def _compensated_group_add(hi, lo, buckets, contribs):
    """Add contribs[t] to row buckets[t] of (hi, lo), contributions sharing a
    bucket applied in increasing t, each step a TwoSum; sketch.py:173-191."""
    perm = np.argsort(buckets, kind="stable")
    keys = buckets[perm]
    if keys.size == 0:
        return
    first = np.ones(keys.size, dtype=bool)
    first[1:] = keys[1:] != keys[:-1]
    group_start = np.flatnonzero(first)
    # rank of each sorted element inside its bucket group
    start_of = np.repeat(group_start, np.diff(np.append(group_start, keys.size)))
    rank = np.arange(keys.size) - start_of
    for depth in range(int(rank.max()) + 1):
        sel = rank == depth
        rows = perm[sel]
        tgt = keys[sel]
        s, e = two_sum(hi[tgt], contribs[rows])
        hi[tgt] = s
        lo[tgt] += e


def hashed_consume(hi, lo, hp: HashParams, rows: np.ndarray, start_index: int, chunk_rows: int = 1 << 15):
    """Accumulate rows (float64, n_b x d) with global indices start_index.. into
    (hi, lo) in place — equivalent to reference consume_rows for countsketch/osnap."""
    rows = np.asarray(rows, dtype=np.float64)
    for lo_r in range(0, rows.shape[0], chunk_rows):
        blk = rows[lo_r : lo_r + chunk_rows]
        idx = np.arange(start_index + lo_r, start_index + lo_r + blk.shape[0], dtype=np.uint64)
        for j in range(hp.s):
            bk = block_buckets(hp, idx, j)
            sg = sign_of(idx, hp.sign_keys[j])
            _compensated_group_add(hi, lo, bk, (sg * hp.scale)[:, None] * blk)


def hashed_sketch(x, family, k, seed, s=1, start_index=0):
    """(hi, lo) state of a fresh hashed sketch over x; SX = hi + lo."""
    x = np.asarray(x, dtype=np.float64)
    hp = HashParams(family, seed, k, s)
    hi = np.zeros((k, x.shape[1]))
    lo = np.zeros((k, x.shape[1]))
    hashed_consume(hi, lo, hp, x, start_index)
    return hi, lo


def merge_hashed(hi1, lo1, hi2, lo2):
    """Reference merge for hashed states, sketch.py:352-355."""
    s, e = two_sum(hi1, hi2)
    return s, lo1 + lo2 + e


def explicit_hashed_matrix(family, k, seed, s, n):
    """Dense S (k x n) for direct-multiplication checks; sketch.py:392-411."""
    hp = HashParams(family, seed, k, s)
    idx = np.arange(n, dtype=np.uint64)
    S = np.zeros((k, n))
    for j in range(s):
        S[block_buckets(hp, idx, j), np.arange(n)] = sign_of(idx, hp.sign_keys[j]) * hp.scale
    return S


# ---------------------------------------------------------------------------
# SRHT (reference sketch.py:213-226, 248-258, 364-385)


def next_pow2(v: int) -> int:
    p = 1
    while p < v:
        p <<= 1
    return p


def srht_signs_sample(seed: int, m: int, k: int):
    """Signs (m, +-1.0) and sorted sample (k) drawn exactly as sketch.py:220-224."""
    g = np.random.Generator(np.random.Philox(np.random.SeedSequence([SRHT_TAG, seed])))
    signs = (2.0 * g.integers(0, 2, m) - 1.0).astype(np.float64)
    sample = np.sort(g.choice(m, size=k, replace=False))
    return signs, sample


def walsh_hadamard(x) -> np.ndarray:
    """Unnormalised radix-2 WHT along axis 0 (natural/Hadamard order); sketch.py:364-385."""
    y = np.array(x, dtype=np.float64)
    vec = y.ndim == 1
    if vec:
        y = y[:, None]
    m = y.shape[0]
    assert m >= 1 and m & (m - 1) == 0
    h = 1
    while h < m:
        v = y.reshape(m // (2 * h), 2, h, y.shape[1])
        a = v[:, 0].copy()
        b = v[:, 1]
        v[:, 0] = a + b
        v[:, 1] = a - b
        h <<= 1
    return y[:, 0] if vec else y


def srht_sketch(x, k, seed, n_rows=None):
    """SX = (H D X_padded)[sample] / sqrt(k) in float64."""
    x = np.asarray(x, dtype=np.float64)
    n = x.shape[0] if n_rows is None else n_rows
    m = next_pow2(n)
    signs, sample = srht_signs_sample(seed, m, k)
    buf = np.zeros((m, x.shape[1]))
    buf[: x.shape[0]] = x
    return walsh_hadamard(signs[:, None] * buf)[sample] / math.sqrt(k)


def explicit_srht_matrix(k, seed, n):
    """Dense SRHT S (k x n) via popcount parity; sketch.py:398-404."""
    m = next_pow2(n)
    signs, sample = srht_signs_sample(seed, m, k)
    v = sample[:, None].astype(np.uint64) & np.arange(n, dtype=np.uint64)[None, :]
    par = np.zeros_like(v)
    while v.any():
        par ^= v & np.uint64(1)
        v >>= np.uint64(1)
    return (1.0 - 2.0 * par.astype(np.float64)) * signs[None, :n] / math.sqrt(k)


# ---------------------------------------------------------------------------
# Gaussian sketch (extension; parity unpinned by reference tests — the
# reference rejects the family, sketch.py:38-41, 74-75; BASELINE configs 1 and
# 5 define it as i.i.d. N(0, 1/k)).
# S[j, i] = Z[j, i] / sqrt(k); Z[j, i] has bf16 bits MAG[w & 0x7FFF] | (w &
# 0x8000), w = 16-bit field (j & 3) of h = mix64(key + phi * ((i << 24) |
# (j >> 2))) — the reference's splitmix64 finaliser (sketch.py:141-148) run as
# a counter-based stream — and MAG[L] = bf16(Phi^-1(1/2 + (L + 1/2) / 65536)),
# the inverse normal CDF of a 16-bit uniform (definition: csrc/gauss_gen.cuh),
# so CPU and GPU agree bit-for-bit.

_PHI = np.uint64(0x9E3779B97F4A7C15)
GAUSS_LEVELS = 32768


def _inv_normal_cdf(p: float) -> float:
    """Bisection of 0.5 erfc(-x / sqrt 2) = p on [0, 10], 100 halvings
    (the same float64 steps as csrc/gaussian.cu)."""
    lo, hi = 0.0, 10.0
    for _ in range(100):
        mid = 0.5 * (lo + hi)
        if 0.5 * math.erfc(-mid / 1.4142135623730951) < p:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


_GT = None


def gaussian_tables() -> np.ndarray:
    """MAG[32768] as bf16 bit patterns (uint16): bf16_rn(float32(Phi^-1(1/2 +
    (L + 1/2) / 65536)))."""
    global _GT
    if _GT is None:
        raw = np.array([_inv_normal_cdf(0.5 + (L + 0.5) / (2.0 * GAUSS_LEVELS)) for L in range(GAUSS_LEVELS)])
        _GT = (_bf16_rn(raw.astype(np.float32)).view(np.uint32) >> np.uint32(16)).astype(np.uint16)
    return _GT.copy()


def _bf16_rn(x):
    b = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    b = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) & np.uint64(0xFFFF0000)
    return b.astype(np.uint32).view(np.float32)


def _mix64_arr(x):
    x = x ^ (x >> np.uint64(30))
    x = x * np.uint64(0xBF58476D1CE4E5B9)
    x = x ^ (x >> np.uint64(27))
    x = x * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def gaussian_key(seed: int) -> int:
    return ((((seed >> 32) & 0xFFFFFFFF) ^ GAUSS_KEY_XOR) << 32) | (seed & 0xFFFFFFFF)


def gaussian_z(seed: int, k: int, row0: int, n: int) -> np.ndarray:
    """Unscaled Gaussian sketch entries Z (k x n, float32, bf16 values) for
    global rows row0..row0+n-1; S = Z / sqrt(k) (csrc/gauss_gen.cuh)."""
    mag = gaussian_tables().astype(np.uint32)
    i = np.arange(row0, row0 + n, dtype=np.uint64)
    t = np.arange((k + 3) // 4, dtype=np.uint64)
    key = np.uint64(gaussian_key(seed))
    out = np.empty((t.size, 4, n), dtype=np.uint32)
    with np.errstate(over="ignore"):
        h = _mix64_arr(key + _PHI * ((i[None, :] << np.uint64(24)) | t[:, None]))  # (k/4, n)
        for m in range(4):
            w = ((h >> np.uint64(16 * m)) & np.uint64(0xFFFF)).astype(np.uint32)
            out[:, m] = (mag[w & np.uint32(0x7FFF)] | (w & np.uint32(0x8000))) << np.uint32(16)
    return out.reshape(-1, n)[:k].view(np.float32)


def gaussian_bf16_cdf(v) -> np.ndarray:
    """P(bf16_rn(z) <= v) for z ~ N(0, 1) at bf16 values v: Phi at the upper
    rounding boundary of v (the test distribution of the Gaussian family)."""
    from math import erfc

    v = np.asarray(v, dtype=np.float32)
    bits = v.view(np.uint32).astype(np.int64)
    # next bf16 value up (towards +inf); the boundary is the midpoint (ties to even are measure zero)
    up = np.where(v >= 0, bits + 0x10000, bits - 0x10000)
    up = np.where(v.view(np.uint32) == np.uint32(0x80000000), np.int64(0x10000), up)
    nxt = (up & 0xFFFFFFFF).astype(np.uint32).view(np.float32).astype(np.float64)
    mid = 0.5 * (v.astype(np.float64) + nxt)
    return np.array([0.5 * erfc(-m / math.sqrt(2.0)) for m in mid])


def gaussian_sketch(x, k, seed, row0=0):
    """SX = Z @ X / sqrt(k) in float64 (parity unpinned: no reference family)."""
    x = np.asarray(x, dtype=np.float64)
    z = gaussian_z(seed, k, row0, x.shape[0]).astype(np.float64)
    return (z @ x) * (1.0 / math.sqrt(k))


# ---------------------------------------------------------------------------
# Small factorisation, fold, scores (reference svd.py:30-54, leverage.py:75-132)


def thin_svd(a):
    u, s, vt = np.linalg.svd(np.asarray(a, dtype=np.float64), full_matrices=False)
    return u, s, vt


def truncate(s, vt, threshold, rank=None):
    """Keep sigma_j > threshold*sigma_1 (strict, svd.py:40-54); optional fixed
    rank cap (extension, G4)."""
    if not 0 <= threshold < 1:
        raise ValueError("threshold")
    if s.shape[0] == 0 or s[0] <= 0:
        raise ZeroDivisionError("degenerate")
    r = int(np.count_nonzero(s > threshold * s[0]))
    if rank is not None:
        r = min(r, rank)
    return s[:r], vt[:r]


def jl_matrix(seed: int, d: int, r: int) -> np.ndarray:
    """Pi (d x r), N(0, 1/r) entries from Philox(SeedSequence([0x4A4C, seed]))."""
    g = np.random.Generator(np.random.Philox(np.random.SeedSequence([JL_TAG, seed])))
    return g.standard_normal((d, r)) / math.sqrt(r)


def fold(s, vt, pi=None):
    """Basis V'/sigma' (leverage.py:85) or the basis-free JL fold V' S'^-1 V'^T Pi."""
    if np.any(s == 0.0):
        raise ZeroDivisionError("exact zero singular value")
    basis = vt.T / s
    if pi is None:
        return basis
    return basis @ (vt @ pi)


def r_factor(sx):
    """Triangular factor R (positive diagonal) of SX = QR; rows min(k, d)."""
    r = np.linalg.qr(np.asarray(sx, dtype=np.float64), mode="r")
    sg = np.sign(np.diag(r))
    sg[sg == 0] = 1.0
    return r * sg[:, None]


def fold_r(sx, sv_tol, pi, rank=None):
    """JL fold (extension G3, the north star's "R M = Pi"): M = pinv_tau(R) Pi,
    pinv_tau from the SVD of R (same sigma / V as SX) truncated like the
    reference (strict relative threshold, optional rank cap).  With nothing
    truncated this is R^-1 Pi.  When the kept rank r' does not exceed the JL
    width (r' <= Pi's columns) a projection cannot reduce the dimension, so the
    fold is the reference basis V'/sigma' itself (exact scores).
    Returns (M, r')."""
    R = r_factor(sx)
    u, s, vt = np.linalg.svd(R, full_matrices=False)
    s2, vt2 = truncate(s, vt, sv_tol, rank)
    r = s2.shape[0]
    if np.any(s2 == 0.0):
        raise ZeroDivisionError("exact zero singular value")
    if r <= pi.shape[1]:
        return vt2.T / s2, r
    return (vt2.T / s2) @ (u[:, :r].T @ pi), r


def row_scores(x, m):
    """||x_i M||^2 per row; leverage.py:88-95."""
    u = np.asarray(x, dtype=np.float64) @ m
    return np.einsum("ij,ij->i", u, u)


def leverage_from_sketch(x, sx, sv_tol, pi=None, rank=None):
    """Reference path (Pi = None: basis V'/sigma', leverage.py:75-95) or the
    JL fold pinv_tau(R) Pi."""
    if pi is not None:
        m, r = fold_r(sx, sv_tol, pi, rank)
        return row_scores(x, m), r, m
    u, s, vt = thin_svd(sx)
    s, vt = truncate(s, vt, sv_tol, rank)
    m = fold(s, vt, None)
    return row_scores(x, m), s.shape[0], m


# ---------------------------------------------------------------------------
# Ordering (reference order.py:51-108)


def distribution(scores):
    scores = np.asarray(scores, dtype=np.float64)
    return scores / scores.sum()


def epoch_rng(seed, epoch):
    return np.random.Generator(np.random.Philox(np.random.SeedSequence([ORDER_TAG, seed, epoch])))


def order(p, kind="dec", seed=0, epoch=0):
    p = np.asarray(p, dtype=np.float64)
    n = p.size
    if kind == "dec":
        return np.argsort(-p, kind="stable")
    if kind == "shuffle":
        return epoch_rng(seed, epoch).permutation(n)
    if kind == "dec_swr":
        return epoch_rng(seed, epoch).choice(n, size=n, replace=True, p=p)
    with np.errstate(divide="ignore", invalid="ignore"):
        keys = epoch_rng(seed, epoch).exponential(size=n) / p
    return np.argsort(keys, kind="stable")


def partition_rows(n, w):
    """Contiguous ranges, first n mod w one longer; dist.py:66-79."""
    base, rem = divmod(n, w)
    out, lo = [], 0
    for p in range(w):
        hi = lo + base + (1 if p < rem else 0)
        out.append((lo, hi))
        lo = hi
    return out


# ---------------------------------------------------------------------------
# Whole-pipeline drivers used by bench.py's CPU legs and the GPU parity tests


def pipeline_hashed(x, family, k, seed, s, sv_tol, pi=None, rank=None, workers=1):
    """Reference-path leverage scores for countsketch/osnap; ``workers`` > 1
    sketches contiguous partitions in threads and merges in ascending worker
    order exactly as dist.py:104-118."""
    x = np.asarray(x, dtype=np.float64)
    n = x.shape[0]
    hp = HashParams(family, seed, k, s)
    if workers <= 1:
        hi = np.zeros((k, x.shape[1]))
        lo = np.zeros_like(hi)
        hashed_consume(hi, lo, hp, x, 0)
    else:
        from concurrent.futures import ThreadPoolExecutor

        def part(rng):
            a, b = rng
            h = np.zeros((k, x.shape[1]))
            l = np.zeros_like(h)
            hashed_consume(h, l, hp, x[a:b], a)
            return h, l

        with ThreadPoolExecutor(max_workers=workers) as ex:
            states = list(ex.map(part, partition_rows(n, workers)))
        hi, lo = states[0]
        for h2, l2 in states[1:]:
            hi, lo = merge_hashed(hi, lo, h2, l2)
    sx = hi + lo
    scores, r, _ = leverage_from_sketch(x, sx, sv_tol, pi, rank)
    return scores, r, sx
