"""Request sharding through the library: two processes on one GPU (gloo for the
gather), each calling zpc_compress on its strong-scaling shard, reproduce a single-process run of the
same request ids byte for byte -- per request: new lengths, kept lists and the compacted K/V rows in
logical order (block ids differ between the two pool layouts, the bytes may not) -- and the bench's
sharding-invariant output checksum adds up to the single run's."""
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
from paper_2603_08743_b200 import zipc  # noqa: E402
from paper_2603_08743_b200.batch import batch_of, desc_params  # noqa: E402
from zpc_inputs import CONFIGS, scaled  # noqa: E402
from zpc_inputs.device import generate  # noqa: E402

pytestmark = pytest.mark.gpu

CFG = scaled(CONFIGS["qwen7b"], L=2, h_kv=2, h_q=14, n_max=9, seq_lens=[300, 257, 416, 257, 333, 290],
             budget=(32, 128), free_slack=5)
SEED = 29
R = len(CFG.seq_lens)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(rids):
    """Compress the given global request ids on cuda:0; per request id: (new_lens, kept lists, K rows,
    V rows) in logical order, plus the bench's output checksum."""
    w = generate(CFG, SEED, np.asarray(rids), device="cuda")
    desc, params = desc_params(w)
    zipc.zpc_compress(desc, params, batch_of(w, desc, params))
    torch.cuda.synchronize()
    assert int(w.status.item()) == 0
    lay = zipc.zpc_workspace_layout_get(desc, params, len(rids))
    units = len(rids) * CFG.L * CFG.h_kv
    kept = w.workspace[lay.kept:lay.kept + 4 * units * lay.kept_stride].view(torch.int32)
    kept = kept.view(len(rids), CFG.L, CFG.h_kv, lay.kept_stride).cpu().numpy()
    nl = w.new_lens.cpu().numpy()
    tables = w.tables.cpu().numpy()
    out = {}
    for i, rid in enumerate(rids):
        rows_k, rows_v, ks = [], [], []
        for l in range(CFG.L):
            for h in range(CFG.h_kv):
                ell = int(nl[i, l, h])
                t = torch.arange(ell, device="cuda")
                tb = torch.from_numpy(tables[i, :CFG.n_max].astype(np.int64)).cuda()[t // CFG.b]
                rows_k.append(w.k[l, tb, t % CFG.b, h].cpu().numpy())
                rows_v.append(w.v[l, tb, t % CFG.b, h].cpu().numpy())
                ks.append(kept[i, l, h, :ell].copy())
        out[int(rid)] = (nl[i].copy(), ks, rows_k, rows_v)
    return out, bench.output_checksum(w, desc, params, np.asarray(rids))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    rids = bench.shard_rids(rank, world, R, R, "strong")
    res = _run(rids)
    objs = [None] * world
    dist.all_gather_object(objs, res)
    if rank == 0:
        q.put(objs)
    dist.barrier()
    dist.destroy_process_group()


def test_two_processes_equal_single_process(cuda_ok):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    shards = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    single, ck_single = _run(list(range(R)))
    merged = {}
    for res, _ in shards:
        assert not set(res) & set(merged)           # disjoint shards
        merged.update(res)
    assert sorted(merged) == list(range(R))         # complete
    for rid in range(R):
        a, b = merged[rid], single[rid]
        np.testing.assert_array_equal(a[0], b[0])
        for x, y in zip(a[1] + a[2] + a[3], b[1] + b[2] + b[3]):
            np.testing.assert_array_equal(x, y)
    assert sum(ck for _, ck in shards) % bench.CHECK_MOD == ck_single
