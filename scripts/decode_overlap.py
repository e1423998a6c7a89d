#!/usr/bin/env python
"""NEXT-3: asynchronous compression against a decode load.

The paper runs compression on the requests that hit N_max while the other running requests keep
decoding ("Requests ready for decoding proceed without waiting for compression to finish",
PAPER.md:157), and reports a compression step at ~40-70 % of a decode step when the two run
sequentially. This script measures that on one B200 at the paper's operating point
(Qwen3-8B shape, b = 256, w = 16, N_max = 9; the `paper_op` config):

  decode load  = one synthetic decode step of R_run running requests: per layer the QKV / O / gate-up
                 / down projections of the Qwen3-8B shape (hidden 4096, intermediate 12288, cuBLAS
                 bf16) and paged decode attention over a [N][b][h_kv][d] bf16 pool (flash_attn's
                 paged kvcache kernel, page = b = 256). Random weights, Philox-free torch randn data:
                 this is a load generator, not the product, and nothing here is checked for values.
  compression  = zpc_compress over the config's wave of requests (the product path, libzipc).

Reported (CUDA events, medians over --steps): decode alone, compression alone, the two sequential on
one stream, and the two launched together on two streams (decode step time under the concurrent
compression, and the joined time). Writes one JSON line to stdout.

    python scripts/decode_overlap.py [--running 128] [--wave 4] [--steps 20]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

HIDDEN, INTER = 4096, 12288   # Qwen3-8B public config (not given by the paper)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--running", type=int, default=128, help="decoding requests per step")
    ap.add_argument("--dec-len", type=int, default=2304, help="tokens per decoding request (N_max * b)")
    ap.add_argument("--wave", type=int, default=0, help="requests per compression call (default: config's)")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--seed", type=int, default=2603)
    args = ap.parse_args()

    import torch
    from flash_attn import flash_attn_with_kvcache

    from bench import ClockSampler
    from paper_2603_08743_b200 import zipc
    from paper_2603_08743_b200.batch import batch_of, desc_params
    from zpc_inputs import CONFIGS
    from zpc_inputs.device import generate

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    cfg = CONFIGS["paper_op"]
    wave = args.wave or cfg.wave

    # ---- compression workload (product path)
    w = generate(cfg, args.seed, np.arange(wave), device=dev)
    desc, params = desc_params(w, flags=0)
    batch = batch_of(w, desc, params)
    lay = w.layout
    touched = np.unique(np.concatenate([lay.tables[:, :cfg.n_max].ravel(), lay.free_stack[:lay.free_top]]))
    touched_d = torch.from_numpy(touched[touched >= 0].astype(np.int64)).to(dev)
    k0, v0 = w.k.index_select(1, touched_d), w.v.index_select(1, touched_d)
    state0 = {n: getattr(w, n).clone() for n in ("tables", "free_stack", "free_top")}

    def restore(s):
        with torch.cuda.stream(s):
            w.k.index_copy_(1, touched_d, k0)
            w.v.index_copy_(1, touched_d, v0)
            for n, t in state0.items():
                getattr(w, n).copy_(t)

    # ---- decode load
    g = torch.Generator(device=dev).manual_seed(args.seed)
    R, L, b, hk, hq, d = args.running, cfg.L, cfg.b, cfg.h_kv, cfg.h_q, cfg.d
    nb = (args.dec_len + b - 1) // b
    dk = torch.randn(L, R * nb, b, hk, d, device=dev, dtype=torch.bfloat16, generator=g)
    dv = torch.randn(L, R * nb, b, hk, d, device=dev, dtype=torch.bfloat16, generator=g)
    table = torch.randperm(R * nb, device=dev, generator=g).view(R, nb).to(torch.int32)
    lens = torch.full((R,), args.dec_len, device=dev, dtype=torch.int32)
    sc = 0.02
    Wqkv = [torch.randn(HIDDEN, (hq + 2 * hk) * d, device=dev, dtype=torch.bfloat16, generator=g) * sc for _ in range(L)]
    Wo = [torch.randn(hq * d, HIDDEN, device=dev, dtype=torch.bfloat16, generator=g) * sc for _ in range(L)]
    Wgu = [torch.randn(HIDDEN, 2 * INTER, device=dev, dtype=torch.bfloat16, generator=g) * sc for _ in range(L)]
    Wd = [torch.randn(INTER, HIDDEN, device=dev, dtype=torch.bfloat16, generator=g) * sc for _ in range(L)]
    x0 = torch.randn(R, HIDDEN, device=dev, dtype=torch.bfloat16, generator=g)
    weight_bytes = sum(t.numel() * 2 for ws in (Wqkv, Wo, Wgu, Wd) for t in ws)
    kv_bytes = 2 * L * R * args.dec_len * hk * d * 2

    def decode_step():
        x = x0
        for l in range(L):
            qkv = x @ Wqkv[l]
            q = qkv[:, :hq * d].reshape(R, 1, hq, d)
            o = flash_attn_with_kvcache(q, dk[l], dv[l], cache_seqlens=lens, block_table=table, causal=True)
            x = o.reshape(R, hq * d) @ Wo[l]
            gu = x @ Wgu[l]
            x = (torch.nn.functional.silu(gu[:, :INTER]) * gu[:, INTER:]) @ Wd[l]
        return x

    def compress(s):
        zipc.zpc_compress(desc, params, batch, s)

    s_dec = torch.cuda.current_stream()
    s_cmp = torch.cuda.Stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def run(mode):
        restore(s_dec)
        torch.cuda.synchronize()
        a, b_, c0, c1 = ev(), ev(), ev(), ev()
        if mode == "decode":
            a.record(s_dec); decode_step(); b_.record(s_dec)
            torch.cuda.synchronize()
            return dict(decode=a.elapsed_time(b_))
        if mode == "compress":
            a.record(s_dec); compress(s_dec); b_.record(s_dec)
            torch.cuda.synchronize()
            return dict(compress=a.elapsed_time(b_))
        if mode == "serial":
            a.record(s_dec); c0.record(s_dec); compress(s_dec); c1.record(s_dec); decode_step(); b_.record(s_dec)
            torch.cuda.synchronize()
            return dict(total=a.elapsed_time(b_), compress=c0.elapsed_time(c1), decode=c1.elapsed_time(b_))
        # async: both streams start after the same event
        start = ev()
        start.record(s_dec)
        s_cmp.wait_event(start)
        with torch.cuda.stream(s_cmp):
            c0.record(s_cmp); compress(s_cmp); c1.record(s_cmp)
        a.record(s_dec); decode_step(); b_.record(s_dec)
        s_dec.wait_event(c1)
        end = ev(); end.record(s_dec)
        torch.cuda.synchronize()
        return dict(total=start.elapsed_time(end), compress=c0.elapsed_time(c1), decode=a.elapsed_time(b_))

    modes = ["decode", "compress", "serial", "async"]
    for _ in range(args.warmup):
        for m in modes:
            run(m)
    assert int(w.status.item()) == 0, zipc.status_string(int(w.status.item()))
    sampler = ClockSampler(0)
    sampler.start()
    res = {m: [] for m in modes}
    for _ in range(args.steps):
        for m in modes:
            res[m].append(run(m))
    clocks = sampler.stop()
    assert int(w.status.item()) == 0, zipc.status_string(int(w.status.item()))
    med = {m: {k: statistics.median(r[k] for r in res[m]) for k in res[m][0]} for m in modes}
    dec, cmp_ = med["decode"]["decode"], med["compress"]["compress"]
    line = {
        "experiment": "async compression vs decode (NEXT-3, PAPER.md:142-157)",
        "config": {"workload": f"paper_op: Qwen3-8B shape L={L} h_kv={hk} h_q={hq} d={d} b={b} w={cfg.w} "
                               f"N_max={cfg.n_max}; compression wave {wave} x T={cfg.seq_lens[0]}; decode load "
                               f"{R} running requests x {args.dec_len} tokens",
                   "decode_load": "per layer: cuBLAS bf16 QKV/O/gate-up/down projections (hidden 4096, "
                                  "intermediate 12288) + flash_attn paged decode attention (page 256)",
                   "decode_weight_bytes": weight_bytes, "decode_kv_bytes": kv_bytes},
        "ms": med,
        "compress_over_decode": cmp_ / dec,
        "decode_slowdown_async": med["async"]["decode"] / dec,
        "serial_ms": med["serial"]["total"], "async_ms": med["async"]["total"],
        "async_saving_frac": 1.0 - med["async"]["total"] / med["serial"]["total"],
        "steps": args.steps, "clocks": clocks,
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
