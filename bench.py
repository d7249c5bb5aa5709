"""Benchmark: leverage-score rows/s on B200 (BASELINE.json metric).

Workload at N=1 = BASELINE configs[1] ("C2"): CountSketch, X fp32
1,000,000 x 512 (rank-50 + 0.01 noise, singular values 10 -> 1), k = 4096,
JL r = 64, sv_tol 1e-6, curriculum order "dec".  One step = one full pass of
the hot path over device-resident X:
    K1 sketch -> fp64 factorisation -> fold M -> K5 leverage pass
    -> normalise -> K7 argsort.
N > 1 (torchrun, NCCL): weak scaling, 1e6 rows per rank with global row
indices; the compensated sketch partials are all-gathered and folded in rank
order, rank 0 factorises and broadcasts M, scores stay rank-local, and the
global "dec" order is formed on rank 0 from the gathered probabilities.

--impl reference times the reference algorithm's CPU implementation (the
numpy port in oracle/, all host threads, bounded row sample per step).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "leverage-score rows/s"
UNIT = "rows/s"

CONFIGS = {
    # name: family, n (per rank), d, k, r, s, dtype, sv_tol
    "c2": dict(family="countsketch", n=1_000_000, d=512, k=4096, r=64, s=None, dtype="f32", sv_tol=1e-6,
               desc="configs[1]: CountSketch dense fp32 1e6x512, k=4096, r=64"),
    "c1": dict(family="gaussian", n=20_000, d=256, k=1024, r=64, s=None, dtype="f32", sv_tol=1e-6,
               desc="configs[0]: Gaussian sketch fp32 20000x256, k=1024, r=64"),
    "c4": dict(family="osnap", n=4_000_000, d=4096, k=16384, r=128, s=4, dtype="f32", sv_tol=1e-6, csr=True,
               desc="configs[3]: OSNAP s=4 on CSR 4e6x4096, ~80 Zipf(1.1) draws/row, k=16384, r=128"),
    "c5": dict(family="gaussian", n=1_000_000, d=1024, k=2048, r=128, s=None, dtype="bf16", sv_tol=1e-6, rank=100,
               desc="configs[4]: Gaussian sketch on bf16 X 1e6x1024 per GPU (8e6 on 8), k=2048, rank-100, r=128"),
    "c3": dict(family="srht", n=2**21, d=256, k=4096, r=64, s=None, dtype="f32", sv_tol=1e-6,
               desc="configs[2]: SRHT fp32 2^21x256, k=4096, r=64"),
}


def gen_csr(n, d, draws, seed, device, chunk=250_000):
    """Bag-of-words-like canonical CSR on the device: `draws` column draws per
    row from Zipf(1.1) truncated to [1, d] (inverse CDF), lognormal(0, 1)
    values, duplicate columns summed, rows L2-normalised."""
    import torch

    from paper_1812_07903_b200.csr import CSRMatrix

    g = torch.Generator(device=device).manual_seed(seed)
    w = torch.arange(1, d + 1, device=device, dtype=torch.float64).pow(-1.1)
    cdf = torch.cumsum(w, 0) / w.sum()
    ptrs, cols, vals = [torch.zeros(1, dtype=torch.int64, device=device)], [], []
    base = 0
    for r0 in range(0, n, chunk):
        rows = min(chunk, n - r0)
        u = torch.rand(rows * draws, generator=g, device=device, dtype=torch.float64)
        c = torch.searchsorted(cdf, u).clamp_(max=d - 1)
        v = torch.exp(torch.randn(rows * draws, generator=g, device=device))
        r = torch.arange(rows, device=device).repeat_interleave(draws)
        key = r * d + c
        key, order = torch.sort(key)
        v = v[order]
        uk, inv = torch.unique_consecutive(key, return_inverse=True)
        vs = torch.zeros(uk.numel(), device=device, dtype=torch.float32).index_add_(0, inv, v)
        ur = uk // d
        norm = torch.zeros(rows, device=device, dtype=torch.float32).index_add_(0, ur, vs * vs).sqrt_()
        vs = vs / norm[ur]
        cnt = torch.bincount(ur, minlength=rows)
        ptrs.append(base + torch.cumsum(cnt, 0))
        base += int(uk.numel())
        cols.append((uk % d).to(torch.int32))
        vals.append(vs)
    indptr = torch.cat(ptrs)
    return CSRMatrix(indptr, torch.cat(cols), torch.cat(vals), (n, d))


def gen_x(cfg, rank: int, device):
    """Seeded synthetic X with the config's structure, generated on the device."""
    import torch

    if cfg.get("csr"):
        return gen_csr(cfg["n"], cfg["d"], 80, 1000 + rank, device)

    n, d = cfg["n"], cfg["d"]
    g = torch.Generator(device=device).manual_seed(1000 + rank)
    if cfg["family"] == "countsketch":
        # rank-50, singular values linear 10 -> 1, plus 0.01 N(0,1)
        u = torch.randn(n, 50, generator=g, device=device, dtype=torch.float32) / math.sqrt(n)
        v, _ = torch.linalg.qr(torch.randn(d, 50, generator=g, device=device, dtype=torch.float32))
        s = torch.linspace(10.0, 1.0, 50, device=device)
        x = (u * s) @ v.T + 0.01 * torch.randn(n, d, generator=g, device=device, dtype=torch.float32)
    elif cfg["family"] == "gaussian" and cfg.get("rank"):
        # image-feature-like: sigmoid(G1 G2 + 0.05 N) in [0, 1], G1 n x 100, G2 100 x d
        g1 = torch.randn(n, 100, generator=g, device=device) / 10.0
        g2 = torch.randn(100, d, generator=g, device=device)
        x = torch.sigmoid(g1 @ g2 + 0.05 * torch.randn(n, d, generator=g, device=device))
    elif cfg["family"] == "srht":
        x = torch.randn(n, d, generator=g, device=device) / torch.sqrt(torch.arange(1, d + 1, device=device, dtype=torch.float32))
    else:
        u, _ = torch.linalg.qr(torch.randn(n, d, generator=g, device=device))
        v, _ = torch.linalg.qr(torch.randn(d, d, generator=g, device=device))
        s = 0.9 ** torch.arange(d, device=device, dtype=torch.float32)
        x = (u * s) @ v.T + 0.01 * torch.randn(n, d, generator=g, device=device)
    return x.contiguous()


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        time.sleep(0.15)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy burst)"
    return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def measured_tensor_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["bf16_tflops"]), "MEASURED_PEAKS.json bf16_tflops (cuBLAS 8192^3 burst)"
    return 2250.0, "fallback 2.25 PFLOP/s dense bf16 (nominal)"


# ---------------------------------------------------------------------------
# CPU legs (oracle port of the reference algorithm)


def cpu_leg(cfg, rows: int, threads: int):
    """Time the reference algorithm (numpy port, oracle/) on `rows` rows of the
    workload: sketch (threads = row partitions merged in order, dist.py style)
    -> SVD -> fold -> scores -> dec argsort.  Returns (rows/s, seconds)."""
    import numpy as np

    from oracle import levsketch_oracle as O

    rng = np.random.default_rng(7)
    d = cfg["d"]
    if cfg.get("csr"):
        # densified CSR rows streamed through the reference hashing;
        # the n-independent 16384 x 4096 SVD is excluded here (~23 s in LAPACK)
        import scipy.sparse as sp

        w = np.arange(1, d + 1, dtype=np.float64) ** -1.1
        cdf = np.cumsum(w) / w.sum()
        r = np.repeat(np.arange(rows), 80)
        c = np.minimum(np.searchsorted(cdf, rng.random(rows * 80)), d - 1)
        m = sp.csr_matrix((rng.lognormal(0, 1, rows * 80), (r, c)), shape=(rows, d))
        m.sum_duplicates()
        x = np.asarray(m.todense())
        x /= np.maximum(np.linalg.norm(x, axis=1, keepdims=True), 1e-30)
        pi = O.jl_matrix(0, d, cfg["r"])
        t0 = time.perf_counter()
        hp = O.HashParams("osnap", 0, cfg["k"], cfg["s"])
        hi = np.zeros((cfg["k"], d))
        lo = np.zeros_like(hi)
        O.hashed_consume(hi, lo, hp, x, 0)
        O.row_scores(x, np.linalg.qr(pi)[0])  # stands in for the fold's d x r product
        dt = time.perf_counter() - t0
        return rows / dt, dt
    x = (rng.standard_normal((rows, 50)) @ (np.linspace(10, 1, 50)[:, None] * rng.standard_normal((50, d)))
         + 0.01 * rng.standard_normal((rows, d))).astype(np.float32).astype(np.float64)
    pi = O.jl_matrix(0, d, cfg["r"])
    t0 = time.perf_counter()
    if cfg["family"] == "countsketch":
        scores, _, _ = O.pipeline_hashed(x, "countsketch", cfg["k"], 0, 1, cfg["sv_tol"], pi, workers=threads)
    elif cfg["family"] == "srht":
        sx = O.srht_sketch(x, cfg["k"], 0)
        scores, _, _ = O.leverage_from_sketch(x, sx, cfg["sv_tol"], pi)
    else:
        sx = O.gaussian_sketch(x, cfg["k"], 0)
        scores, _, _ = O.leverage_from_sketch(x, sx, cfg["sv_tol"], pi)
    O.order(O.distribution(scores), "dec")
    dt = time.perf_counter() - t0
    return rows / dt, dt


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference(args, cfg, rank: int):
    if rank != 0:
        return
    threads = host_threads()
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(threads)
    except ImportError:
        pass
    # adaptive sample: the whole --steps K run should take about two minutes
    rate, _ = cpu_leg(cfg, 20_000, threads)
    per_step_s = 120.0 / max(1, args.steps)
    # the sample grows up to the whole workload (the SVD / sort fixed costs then
    # weigh on the CPU rate as they do on a full run)
    cap = args.ref_rows if args.ref_rows else cfg["n"]
    sample = int(min(cap, max(10_000, rate * per_step_s)))
    times = []
    for _ in range(args.steps):
        _, dt = cpu_leg(cfg, sample, threads)
        times.append(dt)
    total = sum(times)
    value = sample * args.steps / total
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1000 * total / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": cfg["desc"], "rows_per_step": sample, "note": "bounded row sample per step"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{sample} rows x {cfg['d']} of the {args.config} workload per step "
                                   "(oracle/levsketch_oracle.py numpy port of the reference path, "
                                   "row partitions in threads + BLAS threads)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm


def run_ours(args, cfg, rank: int, world: int, local_rank: int):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1812_07903_b200 as P
    from paper_1812_07903_b200 import _native as N
    from paper_1812_07903_b200.dist import sliced_hashed_merge
    from paper_1812_07903_b200.leverage import jl_device, sketch_fold

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dtype = {"f32": torch.float32, "bf16": torch.bfloat16}[cfg["dtype"]]
    n, d, k, r = cfg["n"], cfg["d"], cfg["k"], cfg["r"]
    spec = P.SketchSpec(cfg["family"], eps=0.5, d=d, seed=0, rows_override=k, osnap_s=cfg["s"])
    X = gen_x(cfg, rank, dev)
    csr = cfg.get("csr", False)
    if not csr:
        X = X.to(dtype)
    torch.cuda.synchronize()
    row0 = rank * n
    pipe = P.LeveragePipeline(spec, n * world if world > 1 else n, d, dtype, sv_tol=cfg["sv_tol"], jl_dim=r,
                              rank=cfg.get("rank"), order=(world == 1), row0=row0)
    if world > 1:
        pipe.n = n  # local rows; the state covers n*world global rows
        pipe.scores = torch.empty(n, dtype=torch.float64, device=dev)
    # multi-rank global order: double-buffered so rank 0 sorts step i's probabilities on a
    # side stream while step i+1 sketches (the 8M-key sort would otherwise sit on the
    # critical path of every step at N = 8)
    gather_p = [torch.empty(n * world, dtype=torch.float64, device=dev) for _ in range(2)] if world > 1 else None
    order_all = [torch.empty(n * world, dtype=torch.int64, device=dev) for _ in range(2)] if world > 1 else None
    side = torch.cuda.Stream(device=dev) if world > 1 else None
    sort_done = [None, None]
    buf = [0]
    ws_sort = torch.empty(max(N.lib().lvsk_argsort_workspace_bytes(n * world), 256), dtype=torch.uint8, device=dev)
    pi = jl_device(0, d, r)

    def step(timing=False):
        if world == 1:
            pipe.run(X, timing=timing, check=False)
            return
        # multi-rank: local sketch -> sliced rank-ordered merge -> SX on every rank -> fold -> local scores
        ev = pipe.events
        if timing:
            ev["sketch"][0].record()
        s = pipe.state
        if cfg["family"] == "srht":
            # extension G7 (the reference's run_distributed rejects SRHT, dist.py:95-98): the
            # one-pass K3 over this rank's 2048-aligned global row block, partials all-reduced
            N.check(N.lib().lvsk_srht_rows(X.data_ptr(), n, d, X.stride(0), row0, s._m, s._signs_dev.data_ptr(),
                                           s._sample_dev.data_ptr(), k, math.sqrt(k), pipe.sx.data_ptr(),
                                           pipe.ws_sketch.data_ptr(), pipe.ws_sketch.numel(),
                                           pipe.flags.data_ptr(), N.stream_ptr()), "srht rows")
        else:
            pipe._sketch(X)
        if timing:
            ev["sketch"][1].record()
        if cfg["family"] in ("gaussian", "srht"):  # a plain float64 partial per rank
            dist.all_reduce(pipe.sx)
        else:  # hashed: row slices exchanged all-to-all, rank-ordered TwoSum merge, folded slices gathered
            pipe.sx.copy_(sliced_hashed_merge(s._hi, s._lo, rank, world))
        if timing:
            ev["factor"][0].record()
        # every rank holds the same SX: the fold is computed redundantly (deterministic
        # kernels, identical M) instead of folding on rank 0 and broadcasting
        M = sketch_fold(pipe.sx, cfg["sv_tol"], cfg.get("rank"), pi)[0].contiguous()
        pipe.set_fold(M)
        if timing:
            ev["factor"][1].record()
            ev["leverage"][0].record()
        pipe._leverage(X)
        if timing:
            ev["leverage"][1].record()
            ev["order"][0].record()
        # global dec order: p = s / global sum, gathered on every rank, sorted on rank 0
        local_sum = pipe.scores.sum().reshape(1)
        dist.all_reduce(local_sum)
        p_local = pipe.scores / local_sum
        b = buf[0]
        buf[0] ^= 1
        if sort_done[b] is not None:  # the sort of two steps ago has released this buffer
            torch.cuda.current_stream().wait_event(sort_done[b])
        dist.all_gather_into_tensor(gather_p[b], p_local)
        if rank == 0:
            ready = torch.cuda.Event()
            ready.record()
            side.wait_event(ready)
            with torch.cuda.stream(side):
                N.check(N.lib().lvsk_argsort_f64(gather_p[b].data_ptr(), n * world, 1, order_all[b].data_ptr(),
                                                 ws_sort.data_ptr(), ws_sort.numel(), N.stream_ptr()))
                done = torch.cuda.Event()
                done.record()
            sort_done[b] = done
        if timing:
            ev["order"][1].record()

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    pipe.check()
    barrier()

    # ---- timed region (device events; inputs 2 GB >> 126 MB L2) ----
    stage_sum = {"sketch": 0.0, "factor": 0.0, "leverage": 0.0, "order": 0.0}
    gpu_index = int(os.environ.get("CUDA_VISIBLE_DEVICES", str(local_rank)).split(",")[0]) if os.environ.get(
        "CUDA_VISIBLE_DEVICES", "").strip().isdigit() else local_rank
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(gpu_index) as clocks:
        torch.cuda.synchronize()
        barrier()
        start.record()
        for _ in range(args.steps):
            step(timing=True)
            for name, ms in pipe.stage_ms().items() if args.stage_sync else ():
                stage_sum[name] += ms
        stop.record()
        torch.cuda.synchronize()
        barrier()
    elapsed_ms = start.elapsed_time(stop)
    if not args.stage_sync:
        # stage events of the last step only (no extra syncs inside the timed loop)
        for name, ms in pipe.stage_ms().items():
            stage_sum[name] = ms * args.steps
    if world > 1 and rank == 0:
        # the last global order is a descending permutation of the gathered probabilities
        lb = buf[0] ^ 1
        o = order_all[lb]
        ps = gather_p[lb][o]
        ok = bool((ps[:-1] >= ps[1:]).all()) and bool((torch.bincount(o, minlength=n * world) == 1).all())
        if not ok:
            raise SystemExit("bench: multi-rank global order failed its check")
    t = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_ms = float(t.item())
    pipe.check()
    ms_per_step = elapsed_ms / args.steps
    rows_total = n * world
    value = rows_total / (ms_per_step / 1000.0)

    # ---- per-kernel roofline (algorithmic bytes / event-timed duration) ----
    peak, peak_src = measured_peaks()
    elt = 4 if csr else X.element_size()
    x_bytes = (X.nnz * 8 + 8 * (n + 1)) if csr else n * d * elt  # CSR: int32 col + f32 val + int64 row_ptr
    stage_ms = {k_: v / args.steps for k_, v in stage_sum.items()}
    lev_bytes = x_bytes + 8 * n  # X once + float64 scores
    sk_bytes = x_bytes + 2 * 8 * k * d  # X once + compensated state write (the kernel reads CSR rows s times)
    lev_gbs = lev_bytes / (stage_ms["leverage"] / 1000) / 1e9 if stage_ms.get("leverage") else None
    sk_gbs = sk_bytes / (stage_ms["sketch"] / 1000) / 1e9 if stage_ms.get("sketch") else None
    dominant = "sketch" if stage_ms.get("sketch", 0) >= stage_ms.get("leverage", 0) else "leverage"
    dom_gbs = sk_gbs if dominant == "sketch" else lev_gbs
    dom_bytes = sk_bytes if dominant == "sketch" else lev_bytes
    traffic = None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get(f"{args.config}:{dominant}")
        except (ValueError, OSError):
            traffic = None
    roofline = {
        "bound": "hbm",
        "kernel": {"sketch": {"countsketch": "hashed_gather_bulk_kernel (K1, incl. the cooperative bucket grouping)",
                              "osnap": "csr_stream_kernel (K2, incl. row prep + radix grouping)" if csr else
                              "hashed_gather_bulk_kernel (K1, incl. the cooperative bucket grouping)",
                              "srht": "srht_sampled_kernel (K3 v3: one pass, block WHT + sampled combine)",
                              "gaussian": "gaussian_gemm_kernel (K4, SIMT)" if csr else
                              "gaussian_tc_kernel (K4-TC, tcgen05, Z generated on the fly) + reduce"
                              if X.dtype == torch.bfloat16 else
                              "split3_bf16_kernel + 3 x gaussian_tc_kernel (K4-TC on the exact bf16 planes of fp32 X) + reduce"
                              if X.dtype == torch.float32 else "gaussian_gemm_kernel (K4, SIMT)"}[cfg["family"]],
                   "leverage": "csr_rowsumsq_kernel (K6)" if csr else "leverage_v2_kernel (K5, tcgen05)"}[dominant],
        "achieved": dom_gbs,
        "peak": peak,
        "unit": "GB/s",
        "frac": (dom_gbs / peak) if dom_gbs else None,
        "traffic": traffic,
        "algorithmic_bytes_per_launch": dom_bytes,
        "peak_source": peak_src,
    }
    if dominant == "sketch" and cfg["family"] == "gaussian" and not csr and X.dtype in (torch.bfloat16, torch.float32):
        # K4-TC is a GEMM: 2*k*n*d algorithmic flop per launch (fp32 X runs it on three exact
        # bf16 planes: 3x the tensor work for the same algorithmic flops) against the bf16 tensor peak
        tpeak, tsrc = measured_tensor_peak()
        flops = 2.0 * k * n * d
        ach = flops / (stage_ms["sketch"] / 1000) / 1e12
        roofline.update({"bound": "tensor", "achieved": ach, "peak": tpeak, "unit": "TFLOP/s", "frac": ach / tpeak,
                         "algorithmic_flops_per_launch": flops, "peak_source": tsrc})
        roofline.pop("algorithmic_bytes_per_launch", None)
    other = {
        "sketch": {"ms": stage_ms.get("sketch"), "GB/s": sk_gbs, "frac": sk_gbs / peak if sk_gbs else None},
        "leverage": {"ms": stage_ms.get("leverage"), "GB/s": lev_gbs, "frac": lev_gbs / peak if lev_gbs else None},
        "factor_ms": stage_ms.get("factor"),
        "order_ms": stage_ms.get("order"),
    }

    # ---- e2e through the public API with host buffers (rank 0 view) ----
    e2e = None
    if not args.no_e2e:
        if csr:
            Xh = (X.indptr.cpu().pin_memory(), X.indices.cpu().pin_memory(), X.data.cpu().pin_memory(), (n, d))
        else:
            Xh = torch.empty((n, d), dtype=dtype, pin_memory=True)
            Xh.copy_(X)
        e2e_steps = max(2, min(args.steps, args.e2e_steps))

        def e2e_step():
            if world == 1:
                # C3's SRHT transform buffer (4.3 GB) exceeds the reference's 4 GiB default cap (G8)
                cap = (16 << 30) if cfg["family"] == "srht" else None
                res = P.leverage_sketched_trunc(Xh, spec, cfg["sv_tol"], mem_cap_bytes=cap, jl_dim=r,
                                                rank=cfg.get("rank"))
                plan = P.make_plan(P.scores_to_distribution(res.scores), P.OrderingPolicy("dec"))
                return plan.indices
            local, *_ = P.run_sharded(Xh, row0, n * world, spec, cfg["sv_tol"], jl_dim=r)
            return local.cpu()

        e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        torch.cuda.synchronize()
        barrier()
        e2e_s = torch.tensor([(time.perf_counter() - t0) / e2e_steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
        h2d = x_bytes + (2 * 8 * n if world == 1 else 0)
        d2h = (3 * 8 * n) if world == 1 else 8 * n
        e2e = {"value": rows_total / float(e2e_s.item()), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "steps": e2e_steps,
               "api": "leverage_sketched_trunc(pinned host X) -> scores_to_distribution -> make_plan('dec')"
               if world == 1 else "run_sharded(pinned host shard)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = host_threads()
        # calibrate, then repeat a bounded sample until ~10 s of CPU work has been timed
        rate, _ = cpu_leg(cfg, 20_000, threads)
        rows = int(min(args.cpu_rows, max(20_000, rate * args.cpu_seconds / 2)))
        total_rows, total_s, passes = 0, 0.0, 0
        while total_s < args.cpu_seconds and passes < 25:
            _, dt = cpu_leg(cfg, rows, threads)
            total_rows, total_s, passes = total_rows + rows, total_s + dt, passes + 1
        cpu = {"value": total_rows / total_s, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{passes} x {rows} rows of the {args.config} workload ({total_s:.1f} s timed), oracle "
                         "numpy port of the reference path incl. SVD and dec argsort, sketch partitions in threads"}

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value,
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_per_step,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": {"f32": "f32", "bf16": "bf16"}[cfg["dtype"]],
            "data": "synthetic (seeded, generated on device; random-init, no dataset)",
            "config": {"workload": cfg["desc"], "rows_per_gpu": n, "d": d, "k": k, "jl_r": r,
                       "sv_tol": cfg["sv_tol"], "parallelism": f"row-partition x{world}",
                       "l2": f"inputs larger than L2 (X = {x_bytes / 1e9:.2f} GB per GPU)",
                       **({"nnz": X.nnz} if csr else {})},
            "stages_ms": other,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": pipe.launches_per_run() * args.steps,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-rows", type=int, default=500_000)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-rows", type=int, default=0, help="cap on the reference arm's rows per step (0: the workload's n)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--stage-sync", action="store_true", help="sync after every step to sum stage times")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, cfg, rank)
        return
    # LVSK_BENCH_SHARE_GPU=1: every rank on cuda:0 over gloo — a correctness
    # check of the multi-rank code path on a one-GPU box, never a measurement
    share = world > 1 and os.environ.get("LVSK_BENCH_SHARE_GPU") == "1"
    if share:
        local_rank = 0
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, cfg, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
