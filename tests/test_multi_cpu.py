"""Multi-process (world_size 2, gloo, CPU) coverage of the request-sharded path:
shards are disjoint and complete, the job time is the max over ranks, and compressing shards
separately gives per-request results identical to compressing the whole batch."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import oracle as O  # noqa: E402
from zpc_inputs import CONFIGS, make_host_workload, scaled  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rids = bench.shard_rids(rank, world, 3, 6)
    gathered = [torch.zeros(3, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(rids.astype(np.int64)))
    t = bench.max_over_ranks(10.0 + rank, dist)
    if rank == 0:
        out.put((torch.cat(gathered).tolist(), t))
    dist.barrier()
    dist.destroy_process_group()


def test_sharding_and_max_over_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ids, t = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert sorted(ids) == list(range(6)) and len(set(ids)) == 6
    assert t == 11.0


def _kept_of(cfg, rids, seed=17):
    hw = make_host_workload(cfg, seed, rids=rids)
    lay = hw.layout
    geo = O.Geometry(L=cfg.L, h_kv=cfg.h_kv, h_q=cfg.h_q, d=cfg.d, b=cfg.b, N_total=lay.N_total, M=lay.M,
                     w=cfg.w, dtype=cfg.dtype)
    out = O.compress(geo, O.Params(n_max=cfg.n_max, pool_kernel=cfg.pool_kernel), hw.k_cache, hw.v_cache,
                     hw.q_cache, lay.q_slots, lay.seq_lens, lay.tables, hw.budgets, None, lay.free_stack,
                     lay.free_top)
    assert out.status == O.OK
    res = {}
    for i, rid in enumerate(rids):
        for l in range(cfg.L):
            for h in range(cfg.h_kv):
                kept = out.kept[(i, l, h)]
                tbl = out.fin.tables[i]
                rows = np.stack([out.k_cache[l, tbl[k // cfg.b], k % cfg.b, h] for k in range(len(kept))])
                res[(int(rid), l, h)] = (kept.tolist(), rows.tobytes())
    return res


def test_sharded_results_equal_unsharded():
    """Per-request results do not depend on how requests are split across GPUs (data are keyed by
    global request id; requests own disjoint blocks)."""
    cfg = scaled(CONFIGS["qwen7b"], L=1, h_kv=2, h_q=4, d=64, n_max=5, seq_lens=[90, 80, 100, 70], budget=64,
                 free_slack=4)
    whole = _kept_of(cfg, np.arange(4))
    part = {}
    for shard in (np.array([0, 1]), np.array([2, 3])):
        part.update(_kept_of(cfg, shard))
    assert whole.keys() == part.keys()
    for k in whole:
        assert whole[k] == part[k], k


@pytest.mark.parametrize("R", [1, 2, 7, 12, 64])
def test_query_slots_distinct(R):
    from zpc_inputs.workloads import make_layout
    cfg = scaled(CONFIGS["qwen7b"], L=1, seq_lens=[300] * R)
    lay = make_layout(cfg, 0, np.arange(R))
    assert len(set(lay.q_slots.tolist())) == R and (lay.q_slots < lay.M).all()


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_strong_shards_are_contiguous_and_complete(world):
    """--scaling strong (contiguous ranges): the 64-request qwen7b batch split over P ranks."""
    ids = [bench.shard_rids(r, world, 64, 64, "strong") for r in range(world)]
    flat = np.concatenate(ids)
    assert flat.tolist() == list(range(64))
    assert all(np.all(np.diff(x) == 1) for x in ids if len(x) > 1)
    assert max(len(x) for x in ids) - min(len(x) for x in ids) <= 1
