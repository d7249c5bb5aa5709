"""Per-epoch curriculum orderings (drop-in for reference order.py:1-131).

``dec`` and ``dec_swor`` — the policies that sort — run on the device: a
deterministic float64 normalisation kernel and the K7 stable radix argsort
(ties by ascending index, exactly numpy's kind="stable").  ``dec_swor`` keys
Exp(1)/p use the reference's host Philox stream (order.py:66-69) so plans
are bit-identical; ``shuffle`` / ``dec_swr`` are host RNG draws with no hot
loop and stay on the host like the reference.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from . import _native as N
from .errors import ConfigurationError, DegenerateInputError

SHUFFLE = "shuffle"
DEC = "dec"
DEC_SWR = "dec_swr"
DEC_SWOR = "dec_swor"
POLICY_KINDS = (SHUFFLE, DEC, DEC_SWR, DEC_SWOR)

_ORDER_STREAM = 0x4F52


@dataclass(frozen=True)
class OrderingPolicy:
    kind: str
    seed: int = 0

    def __post_init__(self):
        if self.kind not in POLICY_KINDS:
            raise ConfigurationError(f"unknown ordering policy {self.kind!r}; expected one of {POLICY_KINDS}")
        if self.seed < 0:
            raise ConfigurationError(f"seed must be nonnegative, got {self.seed}")


@dataclass
class OrderingPlan:
    epoch: int
    indices: np.ndarray
    policy: OrderingPolicy


def _vector(x, what: str) -> tuple[torch.Tensor, bool]:
    """1-D float64 CUDA tensor and whether the caller handed us a torch tensor."""
    if isinstance(x, torch.Tensor):
        t = x.detach()
        was_torch = True
    else:
        a = np.asarray(x, dtype=np.float64)  # no host copy for a float64 array
        t = torch.from_numpy(a if a.ndim else a.reshape(1))
        was_torch = False
    if t.dim() != 1 or t.numel() == 0:
        raise DegenerateInputError(f"{what}, got shape {tuple(t.shape)}")
    return t.to(N.device(), torch.float64).contiguous(), was_torch


def normalize_device(s: torch.Tensor, out: torch.Tensor | None = None, ws=None, flags=None):
    """p = s / sum(s) on the device; returns (p, total tensor, flags)."""
    n = s.numel()
    out = torch.empty_like(s) if out is None else out
    total = torch.empty(1, dtype=torch.float64, device=s.device)
    flags = flags or N.Flags()
    ws = ws if ws is not None else N.workspace(N.lib().lvsk_normalize_workspace_bytes(n))
    N.check(
        N.lib().lvsk_normalize_scores(s.data_ptr(), n, out.data_ptr(), total.data_ptr(), ws.data_ptr(), ws.numel(), flags.p, N.stream_ptr()),
        "normalize",
    )
    return out, total, flags


def scores_to_distribution(scores):
    """Normalise nonnegative scores into sampling probabilities (order.py:51-63)."""
    s, was_torch = _vector(scores, "scores must be a non-empty 1-D array")
    p, total, flags = normalize_device(s)
    f = flags.read()
    if f & N.FLAG_NONFINITE:
        raise DegenerateInputError("scores contain non-finite values")
    if f & N.FLAG_NEGATIVE:
        raise DegenerateInputError("scores must be nonnegative")
    if float(total.item()) <= 0:
        raise DegenerateInputError("all scores are zero; no sampling distribution exists")
    return p if was_torch else N.host_numpy(p)


def argsort_device(keys: torch.Tensor, descending: bool, out: torch.Tensor | None = None, ws=None) -> torch.Tensor:
    """K7: stable argsort of float64 keys (descending = np.argsort(-keys, stable))."""
    n = keys.numel()
    out = torch.empty(n, dtype=torch.int64, device=keys.device) if out is None else out
    ws = ws if ws is not None else N.workspace(N.lib().lvsk_argsort_workspace_bytes(n))
    N.check(
        N.lib().lvsk_argsort_f64(keys.data_ptr(), n, 1 if descending else 0, out.data_ptr(), ws.data_ptr(), ws.numel(), N.stream_ptr()),
        "argsort",
    )
    return out


def merge_argsort_runs(sorted_keys: torch.Tensor, run_idx: torch.Tensor, counts, descending: bool,
                       out: torch.Tensor | None = None, ws=None, flags=None) -> torch.Tensor:
    """KM: the global stable argsort of R runs of float64 keys in rank order
    (run q has ``counts[q]`` keys) from each run's stable argsort ``run_idx``
    (int32, local to the run) and the run's keys in that order
    (``sorted_keys``), both concatenated run after run — equal to
    :func:`argsort_device` on the concatenated keys, in ceil(log2 R)
    merge-path rounds instead of a full sort (the multi-rank "dec" order:
    every rank sorts its own scores, rank 0 merges)."""
    import ctypes

    n = sorted_keys.numel()
    R = len(counts)
    off = (ctypes.c_int64 * (R + 1))(*([0] + list(np.cumsum(np.asarray(counts, dtype=np.int64)).tolist())))
    out = torch.empty(n, dtype=torch.int64, device=sorted_keys.device) if out is None else out
    ws = ws if ws is not None else N.workspace(N.lib().lvsk_merge_runs_workspace_bytes(n, R))
    fl = flags if flags is not None else N.Flags()
    N.check(N.lib().lvsk_merge_argsort_runs(sorted_keys.data_ptr(), run_idx.data_ptr(), off, R, 1 if descending else 0,
                                            out.data_ptr(), ws.data_ptr(), ws.numel(), fl.p, N.stream_ptr()),
            "merge argsort runs")
    if flags is None and fl.read() & N.FLAG_BADINDEX:  # (callers passing flags check them themselves)
        raise ConfigurationError("a run index lies outside its run")
    return out


def _device_sum(p: torch.Tensor) -> float:
    out = torch.empty(1, dtype=torch.float64, device=p.device)
    ws = N.workspace(N.lib().lvsk_normalize_workspace_bytes(p.numel()))
    N.check(N.lib().lvsk_sum_f64(p.data_ptr(), p.numel(), out.data_ptr(), ws.data_ptr(), ws.numel(), N.stream_ptr()), "sum")
    return float(out.item())


def _epoch_rng(policy: OrderingPolicy, epoch: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(np.random.SeedSequence([_ORDER_STREAM, policy.seed, epoch])))


def make_plan(p, policy: OrderingPolicy, epoch: int = 0) -> OrderingPlan:
    """One epoch's ordering (order.py:72-100)."""
    pt, was_torch = _vector(p, "need a non-empty 1-D distribution")
    total = _device_sum(pt)
    if abs(total - 1.0) > 1e-9:
        raise DegenerateInputError(f"probabilities sum to {total}, not 1")
    if epoch < 0:
        raise ConfigurationError(f"epoch must be nonnegative, got {epoch}")
    n = pt.numel()
    if policy.kind == DEC:
        idx = argsort_device(pt, descending=True)
    elif policy.kind == DEC_SWOR:
        e = torch.from_numpy(_epoch_rng(policy, epoch).exponential(size=n)).to(pt.device)
        idx = argsort_device(e / pt, descending=False)
    elif policy.kind == SHUFFLE:
        idx = torch.from_numpy(_epoch_rng(policy, epoch).permutation(n).astype(np.int64))
    else:  # DEC_SWR: i.i.d. draws, host RNG like the reference
        ph = pt.cpu().numpy()
        idx = torch.from_numpy(_epoch_rng(policy, epoch).choice(n, size=n, replace=True, p=ph).astype(np.int64))
    indices = idx if was_torch else N.host_numpy(idx)
    return OrderingPlan(epoch=epoch, indices=indices, policy=policy)


def emit_batches(plan: OrderingPlan, batch_size: int) -> list:
    if batch_size < 1:
        raise ConfigurationError(f"batch_size must be at least 1, got {batch_size}")
    idx = plan.indices
    n = idx.shape[0]
    return [idx[i : i + batch_size] for i in range(0, n, batch_size)]


def save_plan(plan: OrderingPlan, path) -> None:
    idx = plan.indices.cpu().numpy() if isinstance(plan.indices, torch.Tensor) else plan.indices
    with open(Path(path), "w") as f:
        f.write("\n".join(str(int(i)) for i in idx))
        f.write("\n")


def save_manifest(plans: list[OrderingPlan], files: list[str], batch_size: int, path, extra: dict | None = None) -> None:
    manifest = {
        "policy": plans[0].policy.kind if plans else None,
        "seed": plans[0].policy.seed if plans else None,
        "epochs": len(plans),
        "n": int(plans[0].indices.shape[0]) if plans else 0,
        "batch_size": batch_size,
        "epoch_files": files,
    }
    if extra:
        manifest.update(extra)
    with open(Path(path), "w") as f:
        json.dump(manifest, f, indent=2, sort_keys=True)
        f.write("\n")
