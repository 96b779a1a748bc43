"""Data-parallel plumbing (one process per GPU, torch.distributed).

The DetNet path shards by sample index: every rank owns a
contiguous range of each stream's sample indices, evaluates it with no
data-path exchange, and only the per-batch statistics (and, in training, the
FP64 raw gradient sums) are all-reduced. Works with the NCCL backend on GPUs
and with gloo on CPU (tests/test_multirank_cpu.py)."""
from __future__ import annotations


def shard(per_rank: int, rank: int) -> tuple[int, int]:
    """(first, count) of this rank's sample indices when every rank owns
    `per_rank` consecutive indices of the stream (weak scaling)."""
    return rank * per_rank, per_rank


def split(total: int, rank: int, world: int) -> tuple[int, int]:
    """(first, count) for a fixed global count split as evenly as possible in
    rank order (strong scaling)."""
    lo = total * rank // world
    hi = total * (rank + 1) // world
    return lo, hi - lo


def reduce_stats(dist, stats):
    """Sum per-rank [loss_sum, symbol_errors, symbols, flagged] in place
    (FP64 tensor); returns the BatchEval fields of the global batch."""
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(stats)
    loss_sum, errors, symbols, flagged = (float(v) for v in stats.tolist())
    n = symbols
    return {"loss_sum": loss_sum, "symbol_errors": int(errors), "symbols": int(symbols),
            "flagged": int(flagged)}


def allreduce_grad(dist, raw):
    """Sum the raw per-rank gradient sums (record layout, FP64) in place."""
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(raw)
    return raw
