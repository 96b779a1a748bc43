"""World-size-2 (gloo, CPU) check of the data-parallel plumbing: sharded
evaluation statistics (loss folded from the ranks' chunk sums in global chunk
order -- bit-identical to one process) and sharded raw-gradient sums,
all-reduced, equal the single-process results of the same global batch
(computed here with the oracle, since this container has no GPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


CH = 8  # stand-in for the engine's 8,192-sample chunk (per-rank shards are chunk-aligned)


def _chunk_sums(loss):
    out = []
    for i in range(0, len(loss), CH):
        acc = 0.0
        for v in loss[i:i + CH]:
            acc += float(v)
        out.append(acc)
    return out


def _worker(rank, world, port, out):
    import torch.distributed as dist

    from oracle.oracle import Oracle, xavier_model
    from paper_2003_09446_b200.parallel import allreduce_grad, reduce_stats, shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle()
    m = xavier_model(orc, n_tx=4, n_rx=8, depth=3, seed=9)
    per_rank = 40
    first, count = shard(per_rank, rank)
    base = orc.lib.or_split(__import__("ctypes").byref(orc.rng(1, 2)))
    H, x, y, _ = orc.generate_range(base, 8, 4, first, count, 7.0, 14.0)
    ev = orc.evaluate(m, H, y, x)
    counts = torch.tensor([int(ev["errors"].sum()), count * 4, int(ev["flagged"].sum())],
                          dtype=torch.int64)
    red = reduce_stats(dist, _chunk_sums(ev["loss"]), counts)
    g = orc.batch_gradient(m, H, y, x)
    raw = torch.from_numpy(g["grads"] * count)  # undo the per-rank mean -> raw sums
    allreduce_grad(dist, raw)
    if rank == 0:
        out.put((red, raw.numpy() / (per_rank * world)))
    dist.destroy_process_group()


def test_two_rank_reduction_matches_single_process(oracle):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    red, grad = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle.oracle import xavier_model
    import ctypes as C
    m = xavier_model(oracle, n_tx=4, n_rx=8, depth=3, seed=9)
    base = oracle.lib.or_split(C.byref(oracle.rng(1, 2)))
    H, x, y, _ = oracle.generate_range(base, 8, 4, 0, 80, 7.0, 14.0)
    ev = oracle.evaluate(m, H, y, x)
    assert red["symbol_errors"] == int(ev["errors"].sum())
    assert red["symbols"] == 80 * 4 and red["flagged"] == int(ev["flagged"].sum())
    # the canonical fold over the global chunk sequence: bit-identical
    acc = 0.0
    for v in _chunk_sums(ev["loss"]):
        acc += v
    assert red["loss_sum"] == acc
    full = oracle.batch_gradient(m, H, y, x)["grads"]
    assert np.max(np.abs(grad - full)) <= 1e-12 * np.max(np.abs(full))
