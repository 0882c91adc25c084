"""N>1 host-side logic with world_size 2 over gloo on CPU: scenario
partitioning, table slicing and the single result gather."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2006_03318_b200.shard import shard_range, table_rows


def test_shard_range_partitions():
    for S in (0, 1, 7, 64, 65536, 65537):
        for world in (1, 2, 3, 8):
            got = [shard_range(S, world, r) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == S
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            sizes = [b - a for a, b in got]
            assert max(sizes) - min(sizes) <= 1


def test_table_rows_slices_every_field():
    from paper_2006_03318_b200 import _native as N
    from paper_2006_03318_b200.batch import ScenarioTable
    S = 10
    steps = np.zeros(S * 2, N.SCALE_STEP_DTYPE)
    steps["num"] = np.arange(S * 2) + 1
    steps["den"] = 1
    t = ScenarioTable(n_scenarios=S, dense=np.arange(3 * S).reshape(3, S).astype(np.int32),
                      overrides={2: np.arange(S)}, scale_ptr=np.arange(0, 2 * S + 1, 2),
                      scale=steps, chain_perm=np.zeros((S, 4), np.int16),
                      chain_present=np.ones((S, 1), np.uint8))
    sub = table_rows(t, 3, 7)
    assert sub.n_scenarios == 4
    assert sub.dense.tolist() == t.dense[:, 3:7].tolist()
    assert sub.overrides[2].tolist() == [3, 4, 5, 6]
    assert sub.scale_ptr.tolist() == [0, 2, 4, 6, 8]
    assert sub.scale["num"].tolist() == list(range(7, 15))
    assert sub.chain_perm.shape == (4, 4)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, S, q):
    import torch.distributed as dist
    from paper_2006_03318_b200.shard import gather_results, shard_range
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s0, s1 = shard_range(S, world, rank)
    # each rank "simulates" its shard: makespan = 1000 * global scenario id
    local = (np.arange(s0, s1, dtype=np.int64) * 1000)[:, None].repeat(3, 1)
    full = gather_results(local, S)
    q.put((rank, full.tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("S", [9, 16])
def test_gather_results_world2_gloo(S):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, S, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = (np.arange(S, dtype=np.int64) * 1000)[:, None].repeat(3, 1).tolist()
    for _rank, full in out:
        assert full == want


def _sim_worker(rank, world, port, q):
    """One rank of a sharded sweep: both ranks on device 0 (a one-GPU box),
    a real simulate_batch of this rank's contiguous scenario shard, results
    gathered once over gloo."""
    import torch.distributed as dist
    from paper_2006_03318_b200.batch import ScenarioTable, simulate_batch
    from paper_2006_03318_b200.frozen import FrozenGraph
    from paper_2006_03318_b200.shard import gather_results, shard_range, table_rows
    from paper_2006_03318_b200.workloads import resnet_like_graph
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = resnet_like_graph(n_pairs=300, seed=3)
    fz = FrozenGraph.from_graph(g, device=0)
    S = 203
    rng = np.random.default_rng(7)
    base = fz.duration[fz.order]
    dense = ((2 * base[:, None] * rng.integers(900, 1101, (fz.n, S)) + 1000) // 2000)
    table = ScenarioTable(n_scenarios=S, dense=dense.astype(np.int64))
    s0, s1 = shard_range(S, world, rank)
    sub = table_rows(table, s0, s1)
    sub.dense = np.ascontiguousarray(sub.dense)
    res = simulate_batch(fz, sub)
    local = np.concatenate([res.makespan[:, None], res.lane_busy], axis=1)
    full = gather_results(local, S)
    if rank == 0:
        whole = simulate_batch(fz, table)
        q.put(("ok", full.tolist(),
               np.concatenate([whole.makespan[:, None], whole.lane_busy], axis=1).tolist()))
    dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_simulate_world2_gloo_matches_single_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sim_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    tag, sharded, single = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert tag == "ok" and sharded == single
