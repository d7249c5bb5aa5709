"""Seeded synthetic inputs for the five BASELINE.json configs, on the device.

The reference's own generator is ``gen_synthetic`` (``A = G1 G2 + sigma N``,
pkg/src/levsketch/matrix.py:42-72); BASELINE.json defines a different input
per config, and these are them.  The bench and the
config-level parity tests (tests/test_gpu_configs.py) both build their
inputs here, so the oracle checks exactly what is measured.

Row blocks: the row-independent configs (C3, C4, C5) are generated in fixed
chunks of ``CHUNK`` rows, chunk c drawn from ``Generator(seed, c)`` — any
row window [lo, hi) of the n-row matrix can be regenerated alone, bit for
bit, which is how the parity tests check windows of the 4e6 / 8e6-row
configs at their global row offsets.  C1 and C2 have exactly orthonormal
factors over all rows (QR), so they are generated whole.

Configs (BASELINE.json "configs"):
  c1  Gaussian sketch, X = U diag(0.9^i) V^T + 0.01 N, 20000 x 256 fp32,
      k = 1024, r = 64
  c2  CountSketch, X = U diag(linspace(10, 1, 50)) V^T + 0.01 N (rank 50),
      1e6 x 512 fp32, k = 4096, r = 64
  c3  SRHT, X_ij = N(0,1) / sqrt(j + 1), 2^21 x 256 fp32, k = 4096, r = 64
  c4  OSNAP s = 4 on CSR 4e6 x 4096: 80 distinct column ids per row drawn
      Zipf(1.1) over [1, 4096] (the first 80 distinct of 256 draws, in draw
      order), values lognormal(0, 1), rows L2-normalised; k = 16384, r = 128
  c5  Gaussian sketch, X = sigmoid(G1 G2 + 0.05 N) (G1 n x 100 with
      N(0, 1/100) entries, G2 100 x 1024 N(0, 1)), stored bf16,
      8e6 x 1024, k = 2048, rank-100 truncation, r = 128
"""

from __future__ import annotations

import torch

CHUNK = 1 << 16
ZIPF_S = 1.1
C4_NNZ = 80
C4_DRAWS = 256

CONFIGS = {
    "c1": dict(family="gaussian", n=20_000, d=256, k=1024, r=64, s=None, dtype="f32", sv_tol=1e-6, rank=None,
               desc="configs[0]: Gaussian sketch fp32 20000x256, k=1024, r=64"),
    "c2": dict(family="countsketch", n=1_000_000, d=512, k=4096, r=64, s=None, dtype="f32", sv_tol=1e-6, rank=None,
               desc="configs[1]: CountSketch dense fp32 1e6x512, k=4096, r=64"),
    "c3": dict(family="srht", n=2**21, d=256, k=4096, r=64, s=None, dtype="f32", sv_tol=1e-6, rank=None,
               desc="configs[2]: SRHT fp32 2^21x256, k=4096, r=64"),
    "c4": dict(family="osnap", n=4_000_000, d=4096, k=16384, r=128, s=4, dtype="f32", sv_tol=1e-6, rank=None,
               csr=True,
               desc="configs[3]: OSNAP s=4 on CSR 4e6x4096, 80 distinct Zipf(1.1) columns/row, k=16384, r=128"),
    "c5": dict(family="gaussian", n=8_000_000, d=1024, k=2048, r=128, s=None, dtype="bf16", sv_tol=1e-6, rank=100,
               desc="configs[4]: Gaussian sketch on bf16 X 8e6x1024, k=2048, rank-100, r=128"),
}


def _gen(seed: int, stream: int, device) -> torch.Generator:
    return torch.Generator(device=device).manual_seed((seed * 1_000_003 + stream) & ((1 << 63) - 1))


def _orthonormal(rows: int, cols: int, g: torch.Generator, device) -> torch.Tensor:
    q, r = torch.linalg.qr(torch.randn(rows, cols, generator=g, device=device, dtype=torch.float64))
    return q * torch.sign(torch.diagonal(r))  # Haar-distributed


def gen_c1(seed: int = 0, device="cuda") -> torch.Tensor:
    n, d = CONFIGS["c1"]["n"], CONFIGS["c1"]["d"]
    g = _gen(seed, 1, device)
    u = _orthonormal(n, d, g, device)
    v = _orthonormal(d, d, g, device)
    s = 0.9 ** torch.arange(d, device=device, dtype=torch.float64)
    x = (u * s) @ v.T + 0.01 * torch.randn(n, d, generator=g, device=device, dtype=torch.float64)
    return x.to(torch.float32).contiguous()


def gen_c2(seed: int = 0, device="cuda", n: int | None = None) -> torch.Tensor:
    n = CONFIGS["c2"]["n"] if n is None else n
    d = CONFIGS["c2"]["d"]
    g = _gen(seed, 2, device)
    u = _orthonormal(n, 50, g, device)
    v = _orthonormal(d, 50, g, device)
    s = torch.linspace(10.0, 1.0, 50, device=device, dtype=torch.float64)
    x = torch.empty(n, d, device=device, dtype=torch.float32)
    vs = (v * s).T.contiguous()
    for lo in range(0, n, CHUNK * 4):  # bounded float64 temporaries
        hi = min(n, lo + CHUNK * 4)
        noise = torch.randn(hi - lo, d, generator=g, device=device, dtype=torch.float64)
        x[lo:hi] = (u[lo:hi] @ vs + 0.01 * noise).to(torch.float32)
    return x


def _chunks(lo: int, hi: int):
    for c in range(lo // CHUNK, (hi + CHUNK - 1) // CHUNK):
        a, b = c * CHUNK, (c + 1) * CHUNK
        yield c, max(a, lo) - a, min(b, hi) - a


def gen_c3(seed: int = 0, device="cuda", lo: int = 0, hi: int | None = None) -> torch.Tensor:
    hi = CONFIGS["c3"]["n"] if hi is None else hi
    d = CONFIGS["c3"]["d"]
    scale = 1.0 / torch.sqrt(torch.arange(1, d + 1, device=device, dtype=torch.float32))
    out = torch.empty(hi - lo, d, device=device, dtype=torch.float32)
    pos = 0
    for c, a, b in _chunks(lo, hi):
        blk = torch.randn(CHUNK, d, generator=_gen(seed, 3_000_000 + c, device), device=device) * scale
        out[pos : pos + b - a] = blk[a:b]
        pos += b - a
    return out


def _c5_g2(seed: int, device) -> torch.Tensor:
    return torch.randn(100, CONFIGS["c5"]["d"], generator=_gen(seed, 5, device), device=device)


def gen_c5(seed: int = 0, device="cuda", lo: int = 0, hi: int | None = None) -> torch.Tensor:
    hi = CONFIGS["c5"]["n"] if hi is None else hi
    d = CONFIGS["c5"]["d"]
    g2 = _c5_g2(seed, device)
    out = torch.empty(hi - lo, d, device=device, dtype=torch.bfloat16)
    pos = 0
    for c, a, b in _chunks(lo, hi):
        g = _gen(seed, 5_000_000 + c, device)
        g1 = torch.randn(CHUNK, 100, generator=g, device=device) / 10.0
        noise = torch.randn(CHUNK, d, generator=g, device=device)
        out[pos : pos + b - a] = torch.sigmoid((g1 @ g2 + 0.05 * noise)[a:b]).to(torch.bfloat16)
        pos += b - a
    return out


def _zipf_cdf(d: int, device) -> torch.Tensor:
    w = torch.arange(1, d + 1, device=device, dtype=torch.float64).pow(-ZIPF_S)
    return torch.cumsum(w, 0) / w.sum()


def gen_c4(seed: int = 0, device="cuda", lo: int = 0, hi: int | None = None, arrays: bool = False):
    """CSR rows [lo, hi) of the C4 matrix (see module docstring): int64
    indptr, int32 strictly increasing columns, fp32 values — a CSRMatrix, or
    the (indptr, indices, data, shape) tuple with ``arrays=True``."""

    cfg = CONFIGS["c4"]
    hi = cfg["n"] if hi is None else hi
    d = cfg["d"]
    cdf = _zipf_cdf(d, device)
    ptrs, cols, vals = [torch.zeros(1, dtype=torch.int64, device=device)], [], []
    base = 0
    for c, a, b in _chunks(lo, hi):
        g = _gen(seed, 4_000_000 + c, device)
        u = torch.rand(CHUNK, C4_DRAWS, generator=g, device=device, dtype=torch.float64)
        v = torch.exp(torch.randn(CHUNK, C4_NNZ, generator=g, device=device, dtype=torch.float32))
        cand = torch.searchsorted(cdf, u).clamp_(max=d - 1)  # column ids 0..d-1 (Zipf rank - 1)
        # first occurrence of each column in draw order, then the first 80 of them
        key = cand * C4_DRAWS + torch.arange(C4_DRAWS, device=device)
        skey, _ = torch.sort(key, dim=1)
        scol = skey // C4_DRAWS
        first = torch.ones_like(scol, dtype=torch.bool)
        first[:, 1:] = scol[:, 1:] != scol[:, :-1]
        keep = torch.zeros(CHUNK, C4_DRAWS, dtype=torch.bool, device=device)
        keep.scatter_(1, skey % C4_DRAWS, first)
        keep &= torch.cumsum(keep, 1) <= C4_NNZ
        keep = keep[a:b]
        cand = cand[a:b]
        cnt = keep.sum(1)
        # the kept columns of each row, sorted; values assigned in that order
        colm = torch.where(keep, cand, torch.full_like(cand, d))
        colm, _ = torch.sort(colm, dim=1)
        colm = colm[:, :C4_NNZ]
        valid = colm < d
        vm = v[a:b] * valid
        vm = vm / torch.linalg.vector_norm(vm, dim=1, keepdim=True).clamp_min(1e-30)
        cols.append(colm[valid].to(torch.int32))
        vals.append(vm[valid])
        ptrs.append(base + torch.cumsum(cnt, 0))
        base += int(cnt.sum())
    out = (torch.cat(ptrs), torch.cat(cols), torch.cat(vals), (hi - lo, d))
    if arrays:
        return out
    from .csr import CSRMatrix

    return CSRMatrix(*out)


def generate(name: str, seed: int = 0, device="cuda", lo: int = 0, hi: int | None = None, n: int | None = None):
    """The config's X (rows [lo, hi) where the config allows windows)."""
    if name == "c1":
        return gen_c1(seed, device)
    if name == "c2":
        return gen_c2(seed, device, n=n)
    if name == "c3":
        return gen_c3(seed, device, lo, hi if hi is not None else (n if n is not None else None))
    if name == "c4":
        return gen_c4(seed, device, lo, hi if hi is not None else (n if n is not None else None))
    if name == "c5":
        return gen_c5(seed, device, lo, hi if hi is not None else (n if n is not None else None))
    raise KeyError(name)


__all__ = ["CONFIGS", "CHUNK", "generate", "gen_c1", "gen_c2", "gen_c3", "gen_c4", "gen_c5"]
