"""Generate golden vectors by importing the REFERENCE package (this container only).

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden.py

Writes ``tests/golden/reference_golden.npz`` (+ a JSON manifest with the numpy
version).  The GPU box never runs this: it only reads the committed fixtures.
Everything here goes through the reference's public API or its module-level
helpers (sketch.py / leverage.py / dist.py / order.py), so the fixtures pin
both the oracle restatement and the CUDA product path to the reference.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys
from pathlib import Path

import numpy as np

REF = os.environ.get("LEVSKETCH_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

import levsketch as L  # noqa: E402  (the reference)
from levsketch import sketch as LS  # noqa: E402

OUT = Path(__file__).resolve().parents[1] / "tests" / "golden"

LARGE_IDX = np.array(
    [2**32 - 1, 2**32, 999_999, 1_000_000, 2**21 - 1, 2**40 + 12345, 2**63 + 7, 2**64 - 1], dtype=np.uint64
)


def hash_kats(g):
    cases = [
        ("countsketch", 0, 4096, None),
        ("countsketch", 13, 1000, None),
        ("osnap", 0, 16384, 4),
        ("osnap", 5, 1001, 3),
        ("osnap", 7, 178, None),
    ]
    meta = []
    for ci, (fam, seed, k, s) in enumerate(cases):
        d = 16
        spec = L.SketchSpec(fam, eps=0.5, d=d, seed=seed, rows_override=k, osnap_s=s)
        st = L.SketchState(spec, 2**20)
        idx = np.concatenate([np.arange(256, dtype=np.uint64), LARGE_IDX])
        buckets, signs = [], []
        for j in range(spec.s):
            buckets.append(st._block_offsets[j] + LS._bucket_hash(idx, st._hash_a[j], st._hash_b[j], st._block_sizes[j]))
            signs.append(LS._sign_hash(idx, st._sign_keys[j]))
        g[f"hash{ci}_idx"] = idx
        g[f"hash{ci}_buckets"] = np.array(buckets, dtype=np.int64)
        g[f"hash{ci}_signs"] = np.array(signs, dtype=np.float64)
        g[f"hash{ci}_keys"] = np.array([st._hash_a, st._hash_b, st._sign_keys], dtype=np.uint64)
        g[f"hash{ci}_sizes"] = np.array(st._block_sizes, dtype=np.int64)
        g[f"hash{ci}_offsets"] = np.array(st._block_offsets, dtype=np.int64)
        meta.append({"family": fam, "seed": seed, "k": k, "s": spec.s})
    return meta


def sketch_cases(g):
    """Small float64 sketches (hi, lo state + data) incl. partial / merged states."""
    rng = np.random.default_rng(1234)
    cases = [
        ("countsketch", 300, 16, 64, None, 3),
        ("osnap", 300, 16, 96, 3, 5),   # scale 1/sqrt(3) is inexact: pins the fp64 product
        ("osnap", 500, 24, 256, 4, 0),
        ("countsketch", 1500, 40, 333, None, 9),
    ]
    meta = []
    for ci, (fam, n, d, k, s, seed) in enumerate(cases):
        a = rng.standard_normal((n, d)) * np.exp(rng.standard_normal((n, 1)))
        spec = L.SketchSpec(fam, eps=0.5, d=d, seed=seed, rows_override=k, osnap_s=s)
        st = L.apply_sketch(a, spec)
        g[f"sk{ci}_x"] = a
        g[f"sk{ci}_hi"] = st._acc_hi
        g[f"sk{ci}_lo"] = st._acc_lo
        g[f"sk{ci}_data"] = st.data
        # two partial states over [0, n//3) and [n//3, n), then merge
        cut = n // 3
        s1 = L.consume_rows(L.SketchState(spec, n), a[:cut], 0)
        s2 = L.consume_rows(L.SketchState(spec, n), a[cut:], cut)
        mg = L.merge(s1, s2)
        g[f"sk{ci}_part1_hi"] = s1._acc_hi
        g[f"sk{ci}_part1_lo"] = s1._acc_lo
        g[f"sk{ci}_merged"] = mg.data
        meta.append({"family": fam, "n": n, "d": d, "k": k, "s": spec.s, "seed": seed, "cut": cut})
    return meta


def fp32_sketch_cases(g):
    """fp32-valued inputs (upcast), C2/C4-shaped at reduced n: the GPU fp32 path
    must reproduce these float64 sketches bit-exactly."""
    rng = np.random.default_rng(99)
    cases = [("countsketch", 8000, 32, 512, None, 0), ("osnap", 4000, 32, 1024, 4, 0)]
    meta = []
    for ci, (fam, n, d, k, s, seed) in enumerate(cases):
        a = (rng.standard_normal((n, d)) * 3.0).astype(np.float32)
        spec = L.SketchSpec(fam, eps=0.5, d=d, seed=seed, rows_override=k, osnap_s=s)
        st = L.apply_sketch(a.astype(np.float64), spec)
        g[f"f32sk{ci}_x"] = a
        g[f"f32sk{ci}_data"] = st.data
        meta.append({"family": fam, "n": n, "d": d, "k": k, "s": spec.s, "seed": seed})
    return meta


def srht_cases(g):
    rng = np.random.default_rng(77)
    meta = []
    for ci, (n, d, k, seed) in enumerate([(64, 8, 32, 17), (100, 8, 64, 19), (1000, 12, 128, 3), (5000, 16, 256, 0)]):
        a = rng.standard_normal((n, d))
        spec = L.SketchSpec("srht", eps=0.5, d=d, seed=seed, rows_override=k)
        st = L.srht_apply(spec, a)
        g[f"srht{ci}_x"] = a
        g[f"srht{ci}_data"] = st.data
        g[f"srht{ci}_signs"] = st._signs
        g[f"srht{ci}_sample"] = st._sample
        meta.append({"n": n, "d": d, "k": k, "seed": seed})
    # C3-sized signs / sample (seed 0, m = 2^21, k = 4096): full sample + signs digest
    spec = L.SketchSpec("srht", eps=0.5, d=1, seed=0, rows_override=4096)
    st = L.SketchState(spec, 2**21)
    g["srht_c3_sample"] = st._sample
    g["srht_c3_signs_head"] = st._signs[:4096]
    packed = np.packbits(st._signs > 0)
    g["srht_c3_signs_sha256"] = np.frombuffer(hashlib.sha256(packed.tobytes()).digest(), dtype=np.uint8)
    return meta


def fwht_cases(g):
    rng = np.random.default_rng(5)
    x = rng.standard_normal((256, 3))
    g["fwht_x"] = x
    g["fwht_y"] = L.fwht(x)
    g["fwht_imp"] = L.fwht([1.0, 0.0, 0.0, 0.0])


def leverage_cases(g):
    meta = []
    specs = [
        # (synthetic spec, sketch spec kw, sv_tol)  -- mirrors reference test_leverage.py cases
        (dict(n=4096, d=10, rank=10, seed=7), dict(family="countsketch", eps=0.5, d=10, seed=3), None),
        (dict(n=4096, d=10, rank=5, seed=7), dict(family="countsketch", eps=0.5, d=10, seed=3), 1e-3),
        (dict(n=1024, d=100, rank=25, noise_sigma=1e-3, seed=7), dict(family="osnap", eps=0.5, d=100, seed=3), 1e-3),
        (dict(n=1000, d=16, rank=16, seed=3), dict(family="osnap", eps=0.5, d=16, seed=4), 1e-3),
        (dict(n=600, d=12, rank=12, seed=21), dict(family="srht", eps=0.5, d=12, seed=2, rows_override=256), 1e-3),
    ]
    for ci, (syn, skw, tol) in enumerate(specs):
        a = L.gen_synthetic(L.SyntheticSpec(**syn))
        spec = L.SketchSpec(**skw)
        res = L.leverage_sketched(a, spec) if tol is None else L.leverage_sketched_trunc(a, spec, tol)
        g[f"lev{ci}_x"] = a
        g[f"lev{ci}_scores"] = res.scores
        g[f"lev{ci}_exact"] = L.leverage_exact(a).scores
        meta.append({"syn": syn, "spec": skw, "sv_tol": tol, "rank": res.effective_rank, "method": res.method})
    # distributed: w=3 over case 3
    a = g["lev3_x"]
    spec = L.SketchSpec(**specs[3][1])
    res, rep = L.run_distributed(a, spec, 3, 1e-3)
    g["dist_w3_scores"] = res.scores
    g["dist_w3_merged"] = rep.merged.data
    return meta


def order_cases(g):
    rng = np.random.default_rng(11)
    s = rng.random(1000)
    s[::37] = s[5]  # exact ties
    p = L.scores_to_distribution(s)
    g["ord_scores"] = s
    g["ord_p"] = p
    g["ord_dec"] = L.make_plan(p, L.OrderingPolicy("dec", seed=0)).indices
    g["ord_swor_s3_e2"] = L.make_plan(p, L.OrderingPolicy("dec_swor", seed=3), epoch=2).indices
    g["ord_shuffle_s3_e2"] = L.make_plan(p, L.OrderingPolicy("shuffle", seed=3), epoch=2).indices
    g["ord_swr_s3_e2"] = L.make_plan(p, L.OrderingPolicy("dec_swr", seed=3), epoch=2).indices


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    g: dict[str, np.ndarray] = {}
    manifest = {
        "generator": "oracle/gen_golden.py",
        "reference": REF,
        "reference_version": L.__version__,
        "numpy": np.__version__,
        "hash": hash_kats(g),
        "sketch": sketch_cases(g),
        "fp32_sketch": fp32_sketch_cases(g),
        "srht": srht_cases(g),
        "leverage": leverage_cases(g),
        "sizing": {
            "countsketch_eps.5_d16": L.sketch_rows(L.SketchSpec("countsketch", eps=0.5, d=16, sizing_c=1.0)),
            "osnap_eps.5_d16_c1": L.sketch_rows(L.SketchSpec("osnap", eps=0.5, d=16, sizing_c=1.0)),
            "srht_eps.5_d16": L.sketch_rows(L.SketchSpec("srht", eps=0.5, d=16, sizing_c=1.0)),
            "osnap_eps.5_d100": L.sketch_rows(L.SketchSpec("osnap", eps=0.5, d=100)),
        },
    }
    fwht_cases(g)
    order_cases(g)
    np.savez_compressed(OUT / "reference_golden.npz", **g)
    with open(OUT / "reference_golden.json", "w") as f:
        json.dump(manifest, f, indent=1, sort_keys=True, default=str)
        f.write("\n")
    size = (OUT / "reference_golden.npz").stat().st_size
    print(f"wrote {len(g)} arrays, {size / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
