"""Scenario sharding across GPUs (one process per GPU, torch.distributed).

Scenarios are independent, so the sweep partitions into contiguous shards
with no collective on the data path; every rank freezes the
same graph, simulates its shard, and the per-scenario results (makespan,
lane busy) are gathered once at the end -- NCCL over NVLink on GPUs, gloo in
the CPU tests.  Per-task start matrices stay sharded where they were produced.
"""

from __future__ import annotations

import numpy as np


def shard_range(n_scenarios: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced [s0, s1) of rank ``rank`` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n_scenarios, world)
    s0 = rank * base + min(rank, extra)
    return s0, s0 + base + (1 if rank < extra else 0)


def gather_results(local: np.ndarray, n_scenarios: int, group=None, device=None) -> np.ndarray:
    """All-gather per-scenario rows of every rank's shard into the full
    [n_scenarios, ...] array (one collective; shards padded to equal size)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    s0, s1 = shard_range(n_scenarios, world, rank)
    if local.shape[0] != s1 - s0:
        raise ValueError("local rows do not match this rank's shard")
    width = -(-n_scenarios // world)
    tail = local.shape[1:]
    pad = np.zeros((width,) + tail, dtype=local.dtype)
    pad[: s1 - s0] = local
    t = torch.from_numpy(pad)
    if device is not None:
        t = t.to(device)
    bufs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(bufs, t, group=group)
    out = np.empty((n_scenarios,) + tail, dtype=local.dtype)
    for r, b in enumerate(bufs):
        a0, a1 = shard_range(n_scenarios, world, r)
        out[a0:a1] = b.cpu().numpy()[: a1 - a0]
    return out


def table_rows(table, s0: int, s1: int):
    """Slice a batch.ScenarioTable to scenarios [s0, s1)."""
    from .batch import ScenarioTable

    sub = ScenarioTable(n_scenarios=s1 - s0)
    if table.dense is not None:
        sub.dense = table.dense[:, s0:s1]
    if table.overrides:
        sub.overrides = {r: np.asarray(v)[s0:s1] for r, v in table.overrides.items()}
    if table.scale_ptr is not None:
        ptr = np.asarray(table.scale_ptr)
        sub.scale_ptr = (ptr[s0:s1 + 1] - ptr[s0]).astype(np.int32)
        sub.scale = np.asarray(table.scale)[ptr[s0]:ptr[s1]]
    if table.chain_perm is not None:
        sub.chain_perm = np.asarray(table.chain_perm)[s0:s1]
    if table.chain_present is not None:
        sub.chain_present = np.asarray(table.chain_present)[s0:s1]
    sub.vdnn_rank = table.vdnn_rank
    return sub
