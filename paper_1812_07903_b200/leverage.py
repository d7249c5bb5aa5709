"""Leverage scores: exact, oracle, and the two sketched variants (+ JL fold).

Drop-in for the reference module (pkg/src/levsketch/leverage.py:33-185).
The sketched methods run entirely on the device:

    X --K1/K3/K4--> SX (k x d, float64) --cuSOLVER fp64--> sigma, V
      --truncate (strict, relative)--> fold M (d x r) --K5--> ||X M||^2

``jl_dim=r`` (extension, BASELINE configs) replaces the d x r' basis V'/sigma'
by the basis-free JL fold M = V' diag(1/sigma') V'^T Pi with
Pi ~ N(0, 1/r) (d x r) drawn from Philox(SeedSequence([0x4A4C, jl_seed]));
with Pi = I it reduces to the reference scores exactly.  ``rank=`` caps the
kept components (fixed-rank truncation, BASELINE config 5).
"""

from __future__ import annotations

import csv
import json
import math
import os
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from . import _native as N
from .config import ensure_capacity
from .errors import CapacityError, DegenerateInputError, DimensionMismatchError, FormatError, SingularInversionError
from .matrix import device_matrix, format_float
from .sketch import SketchSpec, apply_sketch, sketch_rows
from .svd import SvdResult, thin_svd, truncate

MACHINE_RANK_TOL = 1e-12
ORACLE_MAX_ROWS = 5000
_JL_STREAM = 0x4A4C


@dataclass
class LeverageResult:
    scores: np.ndarray
    method: str
    effective_rank: int
    eps: float = 0.0
    spec: SketchSpec | None = None
    sv_tol: float | None = None
    wall_time_s: float | None = None


# ---------------------------------------------------------------------------
# device building blocks shared with pipeline.py and dist.py


def jl_matrix(seed: int, d: int, r: int) -> np.ndarray:
    """Pi (d x r) with N(0, 1/r) entries; host-drawn once, identical to the oracle."""
    g = np.random.Generator(np.random.Philox(np.random.SeedSequence([_JL_STREAM, seed])))
    return g.standard_normal((d, r)) / math.sqrt(r)


_JL_CACHE: dict = {}


def jl_device(seed: int, d: int, r: int) -> torch.Tensor:
    key = (seed, d, r, N.device())
    if key not in _JL_CACHE:
        _JL_CACHE[key] = torch.from_numpy(jl_matrix(seed, d, r)).to(N.device())
    return _JL_CACHE[key]


def factor_device(sx: torch.Tensor, sv_tol: float | None, rank: int | None = None, method: str = "auto"):
    """(sigma, vt) of SX on the device in float64, truncated like svd.truncate
    (strict relative threshold) and optionally capped at ``rank``.

    method "svd": cuSOLVER gesvd of the k x d sketch.  "gram": eigh of the
    d x d Gram SX^T SX (k >= d; its small-sigma accuracy is eps*sigma_1^2/
    sigma_j^2, so "auto" only picks it when the truncation threshold
    discards every component it could misjudge)."""
    k, d = sx.shape
    if method == "auto":
        method = "gram" if (sv_tol is not None and sv_tol >= 1e-6 and k >= d and d >= 256) else "svd"
    if method == "gram":
        g = gram_full(sx)
        lam, v = torch.linalg.eigh(g)
        sigma = torch.sqrt(torch.clamp(lam.flip(0), min=0.0))
        vt = v.flip(1).T
    else:
        _, sigma, vt = torch.linalg.svd(sx, full_matrices=False, driver="gesvd")
    s_host = sigma.cpu().numpy()
    if sv_tol is not None:
        if s_host.shape[0] == 0 or s_host[0] <= 0:
            raise DegenerateInputError("cannot truncate an all-zero matrix (largest singular value is 0)")
        r = int(np.count_nonzero(s_host > sv_tol * s_host[0]))
    else:
        r = s_host.shape[0]
    if rank is not None:
        r = min(r, rank)
    return sigma[:r], vt[:r], s_host[:r]


def fold_device(sigma: torch.Tensor, vt: torch.Tensor, s_host: np.ndarray, pi: torch.Tensor | None) -> torch.Tensor:
    """M = V'/sigma' (d x r', leverage.py:75-85) or the JL fold V' S'^-1 V'^T Pi."""
    if np.any(s_host == 0.0):
        raise SingularInversionError("sketch has an exactly-zero singular value; use the truncated method")
    basis = vt.T / sigma
    if pi is None:
        return basis.contiguous()
    return (basis @ (vt @ pi)).contiguous()


_FOLD_WS: dict = {}
_GRAM_WS: dict = {}
# KG (csrc/gram_i8.cu: the int8-tensor-core Ozaki Gram) from this d up; the
# Grams of d < 2048 (C1-C3, C5: <= 0.14 ms) stay on cuBLAS DGEMM: KG's fixed
# costs (slicing, seven float64 epilogue passes) only amortise on large d
GRAM_KG_MIN_D = int(os.environ.get("LVSK_GRAM_KG_MIN_D", "2048"))
GRAM_KG_MAX_K = 18000


def use_kg(k: int, d: int) -> bool:
    return d >= GRAM_KG_MIN_D and k <= GRAM_KG_MAX_K


def gram_workspace(k: int, d: int, device) -> torch.Tensor:
    L = N.lib()
    nbytes = L.lvsk_gram_workspace_bytes(k, d) if use_kg(k, d) else L.lvsk_syrk_workspace_bytes(k, d)
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def gram_upper(sx: torch.Tensor, ws: torch.Tensor | None = None, flags: torch.Tensor | None = None) -> torch.Tensor:
    """G = SX^T SX with (at least) the block upper triangle computed — KF
    reads the upper triangle.  d >= GRAM_KG_MIN_D: KG on the int8 tensor
    cores (float64-GEMM error class, csrc/gram_i8.cu), 256 x 256 upper
    blocks; below: KD on the float64 tensor cores (csrc/gram_f64.cu), 64 x 64
    upper blocks (half the flops of the full cuBLAS DGEMM it replaces)."""
    k, d = sx.shape
    sx = sx.contiguous()
    if ws is None:  # eager calls: one scratch buffer per (shape, device, stream)
        key = (k, d, sx.device, torch.cuda.current_stream(sx.device).cuda_stream)
        ws = _GRAM_WS.get(key)
        if ws is None:
            ws = _GRAM_WS[key] = gram_workspace(k, d, sx.device)
    G = torch.empty((d, d), dtype=torch.float64, device=sx.device)
    if use_kg(k, d):
        if flags is None:
            flags = torch.zeros(1, dtype=torch.int32, device=sx.device)  # SX was checked by the sketch
        N.check(N.lib().lvsk_gram_f64(sx.data_ptr(), k, d, sx.stride(0), G.data_ptr(), d, ws.data_ptr(), ws.numel(),
                                      flags.data_ptr(), N.stream_ptr()), "gram")
        return G
    N.check(N.lib().lvsk_syrk_f64(sx.data_ptr(), k, d, sx.stride(0), G.data_ptr(), d, ws.data_ptr(), ws.numel(),
                                  N.stream_ptr()), "gram (syrk)")
    return G


def gram_full(sx: torch.Tensor) -> torch.Tensor:
    """Symmetric G = SX^T SX (the eigen routes read all of it)."""
    G = gram_upper(sx)
    return torch.triu(G) + torch.triu(G, 1).T


def cert_limit(sv_tol: float | None) -> float:
    """The certificate's bound on trace(G) * trace(G^-1) (see chol_certified)."""
    lim = _CHOL_KAPPA_GUARD
    if sv_tol is not None and sv_tol > 0:
        lim = min(lim, 1.0 / (sv_tol * sv_tol))
    return lim


def fold_workspace(d: int, r: int, device) -> torch.Tensor:
    return torch.empty(int(N.lib().lvsk_chol_fold_workspace_bytes(d, r)), dtype=torch.uint8, device=device)


def _chol_body(sx: torch.Tensor, pi: torch.Tensor, sv_tol: float | None = None, cert_fail: torch.Tensor | None = None,
               ws: torch.Tensor | None = None, gws: torch.Tensor | None = None, gflags: torch.Tensor | None = None):
    """Shape-static Cholesky fold (CUDA-graph capturable, no host sync):
    G = SX^T SX (cuBLAS DGEMM) = R^T R, then the KF kernel (csrc/factor.cu):
    M = R^-1 Pi and diag = [info, trace(G), trace(G^-1)] with
    trace(G^-1) = ||R^-1||_F^2; the kernel also adds 1 to ``cert_fail`` (a
    device int32) when the certificate of :func:`chol_certified` fails."""
    k, d = sx.shape
    r = pi.shape[1]
    G = gram_upper(sx, gws, gflags)
    if ws is None:  # eager calls: one scratch buffer per (shape, device, stream)
        key = (d, r, sx.device, torch.cuda.current_stream(sx.device).cuda_stream)
        ws = _FOLD_WS.get(key)
        if ws is None:
            ws = _FOLD_WS[key] = fold_workspace(d, r, sx.device)
    pi = pi.contiguous()
    M = torch.empty((d, r), dtype=torch.float64, device=sx.device)
    diag = torch.empty(3, dtype=torch.float64, device=sx.device)
    N.check(N.lib().lvsk_chol_fold(G.data_ptr(), d, G.stride(0), pi.data_ptr(), r, M.data_ptr(), diag.data_ptr(),
                                   cert_limit(sv_tol), N.ptr(cert_fail),
                                   ws.data_ptr(), ws.numel(), N.stream_ptr()), "cholesky fold")
    return M, diag


# kappa(G) <= trace(G) * trace(G^-1); above this the Gram/Cholesky route could
# lose more than ~1e-6 relative accuracy and the QR route runs instead
_CHOL_KAPPA_GUARD = 1e10


def chol_certified(diag, sv_tol: float | None) -> bool:
    """Certificate that the truncation keeps every component:
    lambda_min >= 1/trace(G^-1), lambda_max <= trace(G), so
    trace(G) * trace(G^-1) < 1/sv_tol^2  ==>  every sigma_j > sv_tol * sigma_1."""
    info, tr_g, tr_ginv = (float(v) for v in diag)
    if info != 0 or not (math.isfinite(tr_g) and math.isfinite(tr_ginv)) or tr_ginv <= 0 or tr_g <= 0:
        return False
    prod = tr_g * tr_ginv
    if prod >= _CHOL_KAPPA_GUARD:
        return False
    return not (sv_tol is not None and sv_tol > 0 and prod >= 1.0 / (sv_tol * sv_tol))


def cholesky_fold(sx: torch.Tensor, sv_tol: float | None, pi: torch.Tensor):
    """M = R^-1 Pi when certified (no component truncated), else None."""
    k, d = sx.shape
    if k < d:
        return None
    M, diag = _chol_body(sx, pi)
    return M.contiguous() if chol_certified(diag.tolist(), sv_tol) else None


# the Gram route's sigma / V are accurate to ~eps * kappa^2 relative; above this
# kept-spectrum condition number the QR + Jacobi-SVD route runs instead
_EIGH_KAPPA = 1e4


_EYE: dict = {}


def _chol_inv(G: torch.Tensor) -> torch.Tensor:
    """R^-1 for the positive-diagonal Cholesky factor of the SPD G = R^T R,
    by the KF kernel with Pi = I (csrc/factor.cu: one launch, no host
    synchronisation; replaces cuSOLVER potrf + trsm, ~0.1 ms of launch
    latency per call at b = 136; the C5 fold measured 3.24 ms against 3.61 ms
    with potrf + trsm).  A non-positive pivot yields non-finite
    values, which the caller's residual test rejects."""
    b = G.shape[0]
    key = (b, G.device)
    eye = _EYE.get(key)
    if eye is None:
        eye = _EYE[key] = torch.eye(b, dtype=torch.float64, device=G.device)
    wkey = (b, b, G.device, torch.cuda.current_stream(G.device).cuda_stream)
    ws = _FOLD_WS.get(wkey)
    if ws is None:
        ws = _FOLD_WS[wkey] = fold_workspace(b, b, G.device)
    M = torch.empty((b, b), dtype=torch.float64, device=G.device)
    diag = torch.empty(3, dtype=torch.float64, device=G.device)
    G = G.contiguous()
    N.check(N.lib().lvsk_chol_fold(G.data_ptr(), b, b, eye.data_ptr(), b, M.data_ptr(), diag.data_ptr(),
                                   _CHOL_KAPPA_GUARD, None, ws.data_ptr(), ws.numel(), N.stream_ptr()), "cholesky qr")
    return M


def _cholqr2(Y: torch.Tensor, rounds: int = 2) -> torch.Tensor:
    """Orthonormal basis of range(Y) by two rounds of Cholesky QR (stable for
    cond(Y) up to ~1e7 in float64; one round leaves an orthogonality error of
    ~eps * cond(Y)^2, harmless between power steps, which re-condition the
    block): Y <- Y R^-1 with R^-1 from the KF kernel.  No host
    synchronisation: a failed factorisation yields non-finite values, which
    the caller's residual test rejects."""
    for _ in range(rounds):
        Y = Y @ _chol_inv(Y.T @ Y)
    return Y


def _topk_gram(G: torch.Tensor, want: int, rounds: int = 2, iters: int = 6, tol: float = 1e-12,
               schedule: list[int] | None = None):
    """Top `want` eigenpairs (descending) of the SPD Gram G by block subspace
    iteration: block want + max(16, want / 4) rounded up to 8 (at least 136
    above 96: the eigensolver is faster there), seeded start,
    `iters` power steps with Cholesky-QR re-orthonormalisation per round, then
    one Rayleigh-Ritz (the only small dense eigensolve: ~2 ms on a B200, so it
    is not run per step).  Accepted only when every kept Ritz pair has
    ||G v - theta v|| <= tol * theta_1; else another round, then None (the
    caller falls back to the full eigensolver)."""
    d = G.shape[0]
    b = -(-(want + max(16, want // 4)) // 8) * 8
    if 96 < b < 136:
        # cuSOLVER's float64 eigh takes ~2.1 ms up to n = 131 and ~1.2 ms from
        # n = 132 (a different tridiagonalisation / back-transformation path;
        # tools/eigh_size_probe.py): a slightly wider block is cheaper overall
        b = 136
    b = min(d, b)
    gen = torch.Generator(device=G.device).manual_seed(0x5EED)
    Q = torch.randn(d, b, dtype=G.dtype, device=G.device, generator=gen)
    for _ in range(rounds):
        for it in range(iters):
            # one Cholesky QR per power step (its orthogonality error
            # ~eps * cond^2 is re-conditioned by the next step), CholQR2 on the
            # last (Rayleigh-Ritz needs an orthonormal basis); the residual
            # test below guards the result.  C5: 3.2 -> 2.3 ms against CholQR2
            # on the first two steps as well (tools/c5_rounds_probe.py)
            cq = schedule[it] if schedule is not None else (2 if it == iters - 1 else 1)
            Q = _cholqr2(G @ Q, cq)
        Y = G @ Q
        Bm = Q.T @ Y
        theta, W = torch.linalg.eigh(0.5 * (Bm + Bm.T))
        theta, W = theta.flip(0), W.flip(1)
        V = Q @ W
        res = torch.linalg.vector_norm(Y @ W - V * theta, dim=0)[:want]
        worst = float(res.max())
        if math.isfinite(worst) and worst <= tol * float(theta[0]):
            return theta[:want].contiguous(), V[:, :want].contiguous()
        Q = V
    return None


def _positive_r(sx: torch.Tensor) -> torch.Tensor:
    R = torch.linalg.qr(sx, mode="r")[1]
    sg = torch.sign(torch.diagonal(R))
    sg[sg == 0] = 1.0
    return R * sg[:, None]


def _kept(s_host: np.ndarray, sv_tol: float | None, rank: int | None) -> int:
    if s_host.shape[0] == 0 or s_host[0] <= 0:
        raise DegenerateInputError("cannot truncate an all-zero matrix (largest singular value is 0)")
    r = s_host.shape[0] if sv_tol is None else int(np.count_nonzero(s_host > sv_tol * s_host[0]))
    return min(r, rank) if rank is not None else r


def spectral_fold(sx: torch.Tensor, sv_tol: float | None, rank: int | None, pi: torch.Tensor,
                  force_qr: bool = False):
    """General JL fold M = pinv_tau(R) Pi (oracle fold_r): sigma and V of SX
    from the Gram eigendecomposition when the kept spectrum is well conditioned
    (kappa' <= 1e4), else from a Jacobi SVD of the positive-diagonal QR factor
    R; the reference's strict relative truncation and the optional rank cap.
    When the kept rank r' <= Pi's width the projection cannot reduce the
    dimension and M is the reference basis V'/sigma' (exact scores)."""
    k, d = sx.shape
    jl = pi.shape[1]
    u = None
    ok = False
    if k >= d and not force_qr and rank is not None and rank <= jl and 2 * rank <= d:
        # rank-capped basis fold: only the top `rank` eigenpairs of the Gram are
        # needed — block subspace iteration with a residual certificate
        top = _topk_gram(gram_full(sx), rank)
        if top is not None:
            lam, vcols = top
            sigma = torch.sqrt(torch.clamp(lam, min=0.0))
            s_host = sigma.cpu().numpy()
            r = _kept(s_host, sv_tol, rank)
            if r <= rank and s_host[r - 1] > 0 and s_host[0] / s_host[r - 1] <= _EIGH_KAPPA:
                return (vcols[:, :r] / sigma[:r]).contiguous(), r
    if k >= d and not force_qr:
        lam, v = torch.linalg.eigh(gram_full(sx))
        sigma = torch.sqrt(torch.clamp(lam.flip(0), min=0.0))
        vt = v.flip(1).T
        s_host = sigma.cpu().numpy()
        r = _kept(s_host, sv_tol, rank)
        ok = s_host[r - 1] > 0 and s_host[0] / s_host[r - 1] <= _EIGH_KAPPA
    if not ok:
        R = _positive_r(sx)
        u, sigma, vt = torch.linalg.svd(R, full_matrices=False, driver="gesvdj")
        s_host = sigma.cpu().numpy()
        r = _kept(s_host, sv_tol, rank)
    if np.any(s_host[:r] == 0.0):
        raise SingularInversionError("sketch has an exactly-zero singular value; use the truncated method")
    basis = vt[:r].T / sigma[:r]
    if r <= jl:
        return basis.contiguous(), r
    if k < d:  # R is k x d: "R M = Pi" (Pi: d x r) needs a square factor
        raise DimensionMismatchError(f"a JL fold of width {jl} needs a sketch with at least d = {d} rows "
                                     f"(k = {k}) once the kept rank {r} exceeds the JL width")
    ur = (_positive_r(sx) @ vt[:r].T) / sigma[:r] if u is None else u[:, :r]
    return (basis @ (ur.T @ pi)).contiguous(), r


def qr_fold(sx: torch.Tensor, sv_tol: float | None, rank: int | None, pi: torch.Tensor):
    """:func:`spectral_fold` forced onto the QR + SVD-of-R route."""
    return spectral_fold(sx, sv_tol, rank, pi, force_qr=True)


def sketch_fold(sx: torch.Tensor, sv_tol: float | None, rank: int | None, pi: torch.Tensor | None,
                method: str = "auto"):
    """SX -> (M, effective_rank).

    pi is None (the reference API): M = V'/sigma' from the SVD of SX
    (leverage.py:75-85).  JL (pi given, BASELINE's r): M = pinv_tau(R) Pi —
    the KF Cholesky kernel when :func:`chol_certified` proves nothing is
    truncated (Pi = I when d <= r: the exact scores), else
    :func:`spectral_fold`."""
    k, d = sx.shape
    if pi is None:
        sigma, vt, s_host = factor_device(sx, sv_tol, rank, "svd" if method in ("auto", "chol", "qr") else method)
        return fold_device(sigma, vt, s_host, None), int(s_host.shape[0])
    if method in ("auto", "chol") and rank is None and k >= d:
        M = cholesky_fold(sx, sv_tol, pi if d > pi.shape[1] else torch.eye(d, dtype=sx.dtype, device=sx.device))
        if M is not None:
            return M, d
    return spectral_fold(sx, sv_tol, rank, pi, force_qr=(method == "qr"))


def split_m(M: torch.Tensor, x_dtype: torch.dtype):
    """float64 M -> the SIMT K5 operand(s): float64 for float64 X, else fp32 hi + lo."""
    if x_dtype == torch.float64:
        return M.contiguous(), None
    hi = M.to(torch.float32)
    lo = (M - hi.to(torch.float64)).to(torch.float32)
    return hi.contiguous(), lo.contiguous()


def split_m_tf32(M: torch.Tensor):
    """float64 M -> (Mt_hi, Mt_lo) for the tcgen05 path: M^T with an exactly
    TF32-representable high part (low 13 mantissa bits cleared) and the
    float32 remainder, so hi + lo carries ~22 bits and the tensor core's own
    TF32 reading of each part is exact / harmless."""
    hi = (M.to(torch.float32).view(torch.int32) & ~0x1FFF).view(torch.float32)
    lo = (M - hi.to(torch.float64)).to(torch.float32)
    return hi.T.contiguous(), lo.T.contiguous()


def use_tensor_cores(X: torch.Tensor, r: int) -> bool:
    return (
        X.dtype == torch.float32
        and r <= 128
        and os.environ.get("LVSK_NO_TC", "0") != "1"
        and X.data_ptr() % 16 == 0
        and (X.stride(0) * 4) % 16 == 0
        and (X.shape[1] * 4) % 16 == 0
    )


def use_bf16_tensor_cores(X: torch.Tensor, r: int) -> bool:
    return (
        X.dtype == torch.bfloat16
        and r <= 128
        and os.environ.get("LVSK_NO_TC", "0") != "1"
        and X.data_ptr() % 16 == 0
        and (X.stride(0) * 2) % 16 == 0
        and (X.shape[1] * 2) % 16 == 0
    )


class KernelOperands:
    """K5 operands for a fold M (d x r): TF32 hi/lo transposes (+ bf16 hi) for
    the tcgen05 kernels, fp32 hi/lo or fp64 for the SIMT kernel.  Buffers are
    allocated once; :meth:`set` refills them (CUDA-graph capturable)."""

    def __init__(self, M: torch.Tensor | None, X_like: torch.Tensor, shape: tuple[int, int] | None = None):
        self.d, self.r = M.shape if M is not None else shape
        self.tc = use_tensor_cores(X_like, self.r)
        self.bf16 = use_bf16_tensor_cores(X_like, self.r)
        dev = X_like.device
        self.hb = None
        if self.bf16:
            self.r_pad = 32 if self.r <= 32 else (64 if self.r <= 64 else 128)
            self.a = torch.zeros((2 * self.r_pad, self.d), dtype=torch.bfloat16, device=dev)
            self.b = None
        elif self.tc:
            self.a = torch.empty((self.r, self.d), dtype=torch.float32, device=dev)
            self.b = torch.empty((self.r, self.d), dtype=torch.float32, device=dev)
            if self.r <= 64:
                self.hb = torch.empty((self.r, self.d), dtype=torch.bfloat16, device=dev)
        elif X_like.dtype == torch.float64:
            self.a = torch.empty((self.d, self.r), dtype=torch.float64, device=dev)
            self.b = None
        else:
            self.a = torch.empty((self.d, self.r), dtype=torch.float32, device=dev)
            self.b = torch.empty((self.d, self.r), dtype=torch.float32, device=dev)
        if M is not None:
            self.set(M)

    def set(self, M: torch.Tensor) -> None:
        self.M64 = M
        if self.bf16 or self.tc:  # one split kernel (csrc/leverage.cu)
            Mc = M.contiguous()
            if self.bf16:
                N.check(N.lib().lvsk_split_fold(Mc.data_ptr(), self.d, self.r, 1, self.r_pad, None, None,
                                                self.a.data_ptr(), N.stream_ptr()), "split fold")
            else:
                N.check(N.lib().lvsk_split_fold(Mc.data_ptr(), self.d, self.r, 0, 0, self.a.data_ptr(),
                                                self.b.data_ptr(), N.ptr(self.hb), N.stream_ptr()), "split fold")
        else:
            hi, lo = split_m(M, self.a.dtype)
            self.a.copy_(hi)
            if self.b is not None:
                self.b.copy_(lo)

    def run(self, X: torch.Tensor, out: torch.Tensor, flags_ptr: int) -> None:
        n, d = X.shape
        L = N.lib()
        if self.bf16 and use_bf16_tensor_cores(X, self.r):
            N.check(L.lvsk_leverage_bf16(X.data_ptr(), n, d, X.stride(0), self.a.data_ptr(), self.r, self.r_pad,
                                         out.data_ptr(), flags_ptr, N.stream_ptr()), "leverage pass (tcgen05 bf16)")
            return
        if self.bf16:
            a, b = split_m(self.M64, X.dtype)
            N.check(L.lvsk_rowsumsq_gemm(X.data_ptr(), N.dtype_code(X), n, d, X.stride(0), a.data_ptr(), N.ptr(b),
                                         self.r, out.data_ptr(), flags_ptr, N.stream_ptr()), "leverage pass")
            return
        if self.tc and use_tensor_cores(X, self.r):
            rc = L.lvsk_leverage_tf32x3(X.data_ptr(), n, d, X.stride(0), self.a.data_ptr(), self.b.data_ptr(),
                                        N.ptr(self.hb), self.r, out.data_ptr(), flags_ptr, N.stream_ptr())
            if rc != 5:  # LVSK_ERR_UNSUPPORTED -> SIMT kernel below
                N.check(rc, "leverage pass (tcgen05)")
                return
            a, b = split_m(self.a.T.double() + self.b.T.double(), X.dtype)
        elif self.tc:
            a, b = split_m(self.a.T.double() + self.b.T.double(), X.dtype)
        else:
            a, b = self.a, self.b
        N.check(L.lvsk_rowsumsq_gemm(X.data_ptr(), N.dtype_code(X), n, d, X.stride(0), a.data_ptr(), N.ptr(b),
                                     self.r, out.data_ptr(), flags_ptr, N.stream_ptr()), "leverage pass")


class FoldGraph:
    """The certified Cholesky fold + K5 operand split for a fixed (k, d, r)
    captured once as a CUDA graph; ``run()`` replays it and returns False when
    the certificate fails (caller then takes the eager QR path)."""

    def __init__(self, sx: torch.Tensor, sv_tol: float | None, pi: torch.Tensor, X_like: torch.Tensor):
        k, d = sx.shape
        if d <= pi.shape[1]:  # a JL projection cannot reduce the dimension: exact scores (Pi = I)
            pi = torch.eye(d, dtype=sx.dtype, device=sx.device)
        self.sx, self.sv_tol, self.pi = sx, sv_tol, pi
        self.ops = KernelOperands(None, X_like, (d, pi.shape[1]))
        self.diag = torch.zeros(3, dtype=torch.float64, device=sx.device)
        # device count of replays whose certificate failed (evaluated by the KF kernel)
        self.cert_fail = torch.zeros(1, dtype=torch.int32, device=sx.device)
        self.ws = fold_workspace(d, pi.shape[1], sx.device)  # owned by the graph: replays never share scratch
        self.gws = gram_workspace(k, d, sx.device)
        self.gflags = torch.zeros(1, dtype=torch.int32, device=sx.device)
        self.graph = None
        # warm up cuBLAS handles outside capture
        M, diag = _chol_body(sx, pi, ws=self.ws, gws=self.gws, gflags=self.gflags)
        self.ops.set(M)
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                M, diag = _chol_body(self.sx, self.pi, self.sv_tol, self.cert_fail, self.ws, self.gws, self.gflags)
                self.ops.set(M)
                self.diag.copy_(diag)
        torch.cuda.current_stream().wait_stream(s)
        self.graph = g

    def replay(self) -> None:
        """Enqueue the fold (no host synchronisation); see :meth:`certified`."""
        self.graph.replay()

    def certified(self) -> bool:
        return chol_certified(self.diag.tolist(), self.sv_tol)

    def run(self) -> bool:
        self.replay()
        return self.certified()


def scores_device(X: torch.Tensor, M: torch.Tensor, out: torch.Tensor | None = None, flags=None) -> torch.Tensor:
    """K5: ||X[i] M||^2 for every row (float64 scores on the device)."""
    n, d = X.shape
    if M.shape[0] != d:
        from .errors import DimensionMismatchError

        raise DimensionMismatchError(f"basis has {M.shape[0]} rows, expected {d}")
    if out is None:
        out = torch.empty(n, dtype=torch.float64, device=X.device)
    own = flags is None
    flags = flags or N.Flags()
    KernelOperands(M, X).run(X, out, flags.p)
    if own and flags.read() & N.FLAG_NONFINITE:
        raise FormatError("matrix contains non-finite entries")
    return out


# ---------------------------------------------------------------------------
# reference API


def leverage_exact(a) -> LeverageResult:
    """Exact scores: squared row norms of the thin-SVD left factor restricted
    to the components above the machine-relative rank floor (reference
    leverage.py:44-53).  On the device without forming U (n x d): the
    singular values / right vectors of X come from the small triangular
    factor of a Householder QR (X = Q R, so sigma(R) = sigma(X), V(R) =
    V(X)), and U_r = X V_r / sigma_r, so the scores are the leverage pass
    ||x_i V_r / sigma_r||^2 (float64 rows: the SIMT kernel).  QR keeps
    sigma to float64 relative accuracy where a Gram + eigh route would
    square the condition number at the truncation floor."""
    X = device_matrix(a).to(torch.float64)
    R = torch.linalg.qr(X, mode="r")[1]
    _, s, vt = torch.linalg.svd(R, full_matrices=False)
    s_host = s.cpu().numpy()
    if s_host[0] <= 0:
        raise DegenerateInputError("leverage scores of an all-zero matrix are undefined")
    r = int(np.count_nonzero(s_host > MACHINE_RANK_TOL * s_host[0]))
    M = (vt[:r].T / s[:r]).contiguous()
    scores = scores_device(X.contiguous(), M)
    return LeverageResult(scores=N.host_numpy(scores), method="exact", effective_rank=r)


def leverage_oracle(a) -> LeverageResult:
    """Projector-based scores A (A^T A)^+ A^T (reference leverage.py:56-72)."""
    X = device_matrix(a).to(torch.float64)
    n = X.shape[0]
    if n > ORACLE_MAX_ROWS:
        raise CapacityError(f"oracle forms an n x n projector; n={n} exceeds {ORACLE_MAX_ROWS}")
    ensure_capacity(8 * n * n, "projection matrix")
    if not bool(X.any()):
        raise DegenerateInputError("leverage scores of an all-zero matrix are undefined")
    h = X @ torch.linalg.pinv(X.T @ X) @ X.T
    scores = (h * h).sum(dim=1)
    rank = int(round(float(torch.trace(h))))
    return LeverageResult(scores=N.host_numpy(scores), method="oracle", effective_rank=rank)


def _approx_basis(svd: SvdResult) -> np.ndarray:
    """V / sigma columnwise, refusing an exactly-zero sigma (leverage.py:75-85)."""
    if np.any(svd.sigma == 0.0):
        raise SingularInversionError("sketch has an exactly-zero singular value; use the truncated method")
    return svd.vt.T / svd.sigma


def _block_scores(rows, basis) -> np.ndarray:
    """Squared row norms of rows @ basis through K5 (leverage.py:88-95)."""
    X = device_matrix(rows)
    M = basis if isinstance(basis, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(basis, dtype=np.float64))
    M = M.to(X.device, torch.float64)
    return N.host_numpy(scores_device(X, M))


_STREAM_CHUNK_BYTES = 128 << 20


def _streamed_sketch(a: torch.Tensor, spec: SketchSpec, mem_cap):
    """Pinned host rows -> device in 128 MB chunks on a copy stream, each chunk
    sketched (consume_rows with its global row offset) as soon as it lands, so
    the host->device transfer hides the sketch.  Returns (device X, state)."""
    from .sketch import SketchState, consume_rows

    n, d = a.shape
    X = torch.empty((n, d), dtype=a.dtype, device=N.device())
    state = SketchState(spec, n, mem_cap=mem_cap)
    rows_per = max(1, _STREAM_CHUNK_BYTES // (d * a.element_size()))
    cur = torch.cuda.current_stream()
    cs = torch.cuda.Stream()
    cs.wait_stream(cur)
    events = []
    with torch.cuda.stream(cs):  # every copy is enqueued up front: the copy engine never waits on the host
        for r0 in range(0, n, rows_per):
            r1 = min(n, r0 + rows_per)
            X[r0:r1].copy_(a[r0:r1], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
            events.append((r0, r1, ev))
    for r0, r1, ev in events:
        cur.wait_event(ev)
        consume_rows(state, X[r0:r1], r0)
    return X, state


def _streamable(a, spec) -> bool:
    # opt-in (LVSK_STREAM=1): measured no faster end to end than one whole
    # copy (the 2 GB host->device transfer dominates either way; tools/e2e_ab.py)
    return (os.environ.get("LVSK_STREAM", "0") == "1" and isinstance(a, torch.Tensor) and a.device.type == "cpu" and a.dim() == 2 and a.is_pinned()
            and a.is_contiguous() and a.dtype in (torch.float32, torch.bfloat16, torch.float64)
            and spec.family in ("countsketch", "osnap", "gaussian")
            and a.numel() * a.element_size() >= 2 * _STREAM_CHUNK_BYTES)


def _sketched(a, spec, sv_tol, mem_cap_bytes, jl_dim, jl_seed, rank, method):
    from .csr import CSRMatrix, csr_scores

    m = None if isinstance(a, (np.ndarray, torch.Tensor, list)) else CSRMatrix.from_any(a)
    if m is None and _streamable(a, spec):
        X, state = _streamed_sketch(a, spec, mem_cap_bytes)
        d = X.shape[1]
    else:
        X = m if m is not None else device_matrix(a)
        d = m.d if m is not None else X.shape[1]
        state = apply_sketch(X, spec, mem_cap=mem_cap_bytes)
    sx = state.data_device
    pi = None if jl_dim is None else jl_device(jl_seed, d, jl_dim)
    M, eff = sketch_fold(sx, sv_tol, rank, pi)
    scores = csr_scores(m, M) if m is not None else scores_device(X, M)
    return LeverageResult(
        scores=N.host_numpy(scores),
        method=method,
        effective_rank=eff,
        eps=spec.eps,
        spec=spec,
        sv_tol=sv_tol,
    )


def leverage_sketched(a, spec: SketchSpec, mem_cap_bytes: int | None = None, *, jl_dim: int | None = None,
                      jl_seed: int = 0) -> LeverageResult:
    """Uncorrected sketched scores (reference leverage.py:98-112)."""
    return _sketched(a, spec, None, mem_cap_bytes, jl_dim, jl_seed, None, "sketch")


def leverage_sketched_trunc(a, spec: SketchSpec, sv_tol: float, mem_cap_bytes: int | None = None, *,
                            jl_dim: int | None = None, jl_seed: int = 0, rank: int | None = None) -> LeverageResult:
    """Sketched scores with components sigma_j <= sv_tol * sigma_1 dropped
    (reference leverage.py:115-132)."""
    from .errors import ConfigurationError

    if not 0 <= sv_tol < 1:
        raise ConfigurationError(f"truncation threshold must be in [0, 1), got {sv_tol}")
    return _sketched(a, spec, sv_tol, mem_cap_bytes, jl_dim, jl_seed, rank, "sketch_trunc")


# ---------------------------------------------------------------------------
# scores CSV + JSON sidecar (reference leverage.py:139-185)


def save_scores(result: LeverageResult, csv_path, meta_path=None, extra_meta: dict | None = None) -> None:
    csv_path = Path(csv_path)
    meta_path = Path(meta_path) if meta_path is not None else Path(str(csv_path) + ".json")
    with open(csv_path, "w") as f:
        for i, v in enumerate(np.asarray(result.scores)):
            f.write(f"{i},{format_float(v)}\n")
    meta = {
        "method": result.method,
        "eps": result.eps,
        "sv_tol": result.sv_tol,
        "effective_rank": result.effective_rank,
        "seed": result.spec.seed if result.spec is not None else None,
        "wall_time_s": result.wall_time_s,
        "n": int(np.asarray(result.scores).shape[0]),
    }
    if result.spec is not None:
        meta["sketch"] = {
            "family": result.spec.family,
            "k": sketch_rows(result.spec),
            "osnap_s": result.spec.osnap_s,
            "rows_override": result.spec.rows_override,
            "sizing_c": result.spec.sizing_c,
        }
    if extra_meta:
        meta.update(extra_meta)
    with open(meta_path, "w") as f:
        json.dump(meta, f, indent=2, sort_keys=True)
        f.write("\n")


def load_scores(path) -> np.ndarray:
    path = Path(path)
    scores = []
    with open(path) as f:
        for lineno, row in enumerate(csv.reader(f), start=1):
            if not row:
                continue
            if len(row) != 2:
                raise FormatError(f"{path}: expected index,score at line {lineno}, got {len(row)} fields")
            try:
                scores.append(float(row[1]))
            except ValueError:
                raise FormatError(f"{path}: non-numeric score {row[1]!r} at line {lineno}") from None
    if not scores:
        raise FormatError(f"{path}: no scores found")
    return np.asarray(scores, dtype=np.float64)
