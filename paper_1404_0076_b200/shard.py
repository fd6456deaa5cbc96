"""Multi-GPU plumbing for batches of independent nets.

Nets never share variables, so a batch shards into contiguous slices, one
per rank (one process per GPU); the data path has no collective. The only
communication is control: the max-over-ranks device time and a gather of
per-net outcomes (a few bytes per net) for reporting and verification. These
helpers work with any ``torch.distributed`` backend (``nccl`` on the GPU box,
``gloo`` in the CPU tests).
"""

from __future__ import annotations

from typing import Sequence


def shard_bounds(n_items: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous slice [lo, hi) of ``n_items`` owned by ``rank``; sizes differ by at most one."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    return n_items * rank // world, n_items * (rank + 1) // world


def _tensor(values, device):
    import torch

    return torch.tensor(values, dtype=torch.float64, device=device)


def max_over_ranks(value: float, device="cpu") -> float:
    """Max of a per-rank scalar (device time); identity without a process group."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = _tensor([value], device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(values: Sequence[float], device="cpu") -> list[float]:
    """Element-wise sum of small per-rank vectors (interaction totals)."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return [float(v) for v in values]
    t = _tensor(list(values), device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [float(v) for v in t.tolist()]


def outcome(interactions: int, text: str) -> tuple:
    """A net's gathered outcome: its interaction count and the sha256 prefix of
    its printed normal form (print_configuration, lang.py:371-396) — 24 bytes
    that let rank 0 check every net of every shard."""
    import hashlib

    return int(interactions), hashlib.sha256(text.encode()).hexdigest()[:16]


def gather_outcomes(local: list, world: int) -> list:
    """All ranks' per-net outcome lists concatenated in rank (= input) order."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or world == 1:
        return list(local)
    parts: list = [None] * world
    dist.all_gather_object(parts, local)
    return [x for p in parts for x in p]
