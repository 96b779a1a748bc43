"""Data-parallel plumbing (one process per GPU, torch.distributed).

The DetNet path shards by sample index: every rank owns a
contiguous, 8,192-sample-chunk-aligned range of each stream's sample
indices, evaluates it with no data-path exchange, and only the per-batch
statistics (and, in training, the raw gradient sums) are reduced.

Loss sums are reduced in the engine's canonical order: each rank contributes
its per-chunk sums (``Context.chunk_sums()``, k_reduce's first level), the
ranks all-gather them and every rank folds the global chunk sequence in
order -- the single-device fold, so the result does not depend on the rank
count (the reference's thread-count invariance, kernels.cpp:93-103). Integer
counts are all-reduced (exact in any order). Works with the NCCL backend on
GPUs and with gloo on CPU (tests/test_multirank_cpu.py)."""
from __future__ import annotations

CHUNK = 8192  # samples per canonical reduction chunk (engine: RED_CHUNK_TILES * TILE)


def shard(per_rank: int, rank: int) -> tuple[int, int]:
    """(first, count) of this rank's sample indices when every rank owns
    `per_rank` consecutive indices of the stream (weak scaling). Chunk-aligned
    when per_rank is a multiple of CHUNK, as the canonical fold requires."""
    return rank * per_rank, per_rank


def fold_chunks(dist, chunk_sums):
    """Global loss sum: all-gather every rank's chunk sums (rank order = global
    sample order) and fold them sequentially from 0.0."""
    import torch
    local = torch.as_tensor(chunk_sums, dtype=torch.float64).flatten()
    parts = [local]
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        world = dist.get_world_size()
        cnt = torch.tensor([local.numel()], dtype=torch.int64, device=local.device)
        counts = [torch.zeros_like(cnt) for _ in range(world)]
        dist.all_gather(counts, cnt)
        width = int(max(int(c.item()) for c in counts))
        pad = torch.zeros(width, dtype=torch.float64, device=local.device)
        pad[:local.numel()] = local
        gathered = [torch.zeros_like(pad) for _ in range(world)]
        dist.all_gather(gathered, pad)
        parts = [g[:int(c.item())] for g, c in zip(gathered, counts)]
    acc = 0.0
    for p in parts:
        for v in p.tolist():
            acc += v
    return acc


def reduce_stats(dist, chunk_sums, counts):
    """BatchEval fields of the global batch: `chunk_sums` this rank's
    canonical loss chunk sums, `counts` an int64 tensor [symbol_errors,
    symbols, flagged] (all-reduced in place)."""
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(counts)
    errors, symbols, flagged = (int(v) for v in counts.tolist())
    loss_sum = fold_chunks(dist, chunk_sums)
    n = symbols
    return {"loss_sum": loss_sum, "symbol_errors": errors, "symbols": symbols, "flagged": flagged,
            "samples": n}


def allreduce_grad(dist, raw):
    """Sum the raw per-rank gradient sums (+ loss-sum slot; record layout,
    FP64) in place."""
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(raw)
    return raw
