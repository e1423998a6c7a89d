#!/usr/bin/env python
"""Benchmark of the Zipage compression step (BASELINE.json metric: requests compressed/s and
fraction of HBM peak), one process per GPU, requests sharded by rank (weak scaling).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config qwen7b] [--impl zipc|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

A step = one zpc_compress call over the per-GPU batch (configs[1]: 64 requests x 8192 tokens,
Qwen2.5-7B shape) — all stages a0..a6. Between steps the modified part of the pool is restored
from a pristine copy (untimed, on the same stream; it also writes > L2 so L2 is flushed); each
step is timed with CUDA events on the launching stream; the job time is the max over ranks.
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0
NOMINAL_HBM_GBS = 8000.0   # B200 data-sheet HBM3e bandwidth (report the measured and the nominal peak)
FALLBACK_BF16_TFLOPS = 1590.0


def load_peaks():
    try:
        p = json.load(open(PEAKS_PATH))
        return dict(hbm=float(p["hbm_gbs"]), bf16=float(p["bf16_tflops"]),
                    bf16_sust=float(p.get("bf16_tflops_sustained", p["bf16_tflops"])), src="measured")
    except Exception:
        return dict(hbm=FALLBACK_HBM_GBS, bf16=FALLBACK_BF16_TFLOPS, bf16_sust=1400.0, src="fallback")


# ---------------------------------------------------------------- clocks sampler
THROTTLE_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
                 0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
                 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


class ClockSampler:
    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
        except Exception:
            self.proc = None
            return

        def read():
            for line in self.proc.stdout:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) == 3:
                    try:
                        self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                    except ValueError:
                        pass
        self.thread = threading.Thread(target=read, daemon=True)
        self.thread.start()

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        if not self.samples:
            return None
        busy = [s for s in self.samples if not (s[2] & 0x1)] or self.samples
        reasons = set()
        for s in busy:
            for bit, name in THROTTLE_BITS.items():
                if s[2] & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(s[0] for s in busy), "sm_max_mhz": max(s[1] for s in busy),
                "reasons": sorted(reasons), "samples": len(busy)}


# ---------------------------------------------------------------- oracle (CPU baseline / reference arm)
def oracle_sample(cfg, seed, rids, n_req):
    """Host inputs for n_req sampled requests, as a compact sub-pool (untimed preparation)."""
    from zpc_inputs import make_host_workload, scaled
    sub = scaled(cfg, seq_lens=[cfg.seq_lens[int(r)] for r in rids[:n_req]], free_slack=8)
    return make_host_workload(sub, seed, rids=np.arange(n_req))


_ORACLE_CACHE = {}


RED_PARAMS = (0.2, 0.4, 0.8)   # lambda, tau, p (NEXT-1)


def time_oracle(cfg, seed, n_req, budget_s=20.0, redundancy=False):
    """Time the oracle (as it stands) on a bounded sample: whole requests restricted to a layer
    subset (the oracle's cost is per (layer, head) unit; req/s is scaled by units per request)."""
    import oracle as O
    import torch
    from zpc_inputs import scaled
    # threads the oracle actually runs on: its Python loop is single-threaded; its matmuls (logits, cosines) run
    # in numpy's BLAS pool
    try:
        import threadpoolctl
        threads = max([1] + [p["num_threads"] for p in threadpoolctl.threadpool_info() if p.get("user_api") == "blas"])
    except Exception:
        threads = 1
    key = (cfg.name, seed, n_req)
    if key not in _ORACLE_CACHE:
        sub = scaled(cfg, L=min(cfg.L, 2))
        hw = oracle_sample(sub, seed, np.arange(max(1, n_req)), max(1, n_req))
        _ORACLE_CACHE[key] = (sub, hw)
    sub, hw = _ORACLE_CACHE[key]
    lay = hw.layout
    geo = O.Geometry(L=sub.L, h_kv=sub.h_kv, h_q=sub.h_q, d=sub.d, b=sub.b, N_total=lay.N_total, M=lay.M,
                     w=sub.w, dtype=sub.dtype)
    prm = O.Params(n_max=sub.n_max, pool_kernel=sub.pool_kernel,
                   flags=(O.F_PREFIX if lay.ref_counts is not None else 0) | (O.F_REDUNDANCY if redundancy else 0),
                   lam=RED_PARAMS[0], tau=RED_PARAMS[1], sim_p=RED_PARAMS[2])
    units_done = 0
    t0 = time.perf_counter()
    while True:
        out = O.compress(geo, prm, hw.k_cache, hw.v_cache, hw.q_cache, lay.q_slots, lay.seq_lens, lay.tables,
                         hw.budgets, lay.ref_counts, lay.free_stack, lay.free_top)
        assert out.status == O.OK
        units_done += len(lay.seq_lens) * sub.L * sub.h_kv
        el = time.perf_counter() - t0
        if el >= budget_s:
            break
    units_per_req = cfg.L * cfg.h_kv
    req_per_s = units_done / units_per_req / el
    return req_per_s, dict(units=units_done, seconds=el, threads=threads,
                           sample=f"{len(lay.seq_lens)} request(s) x {sub.L} of {cfg.L} layers x {cfg.h_kv} heads, "
                                  f"T={int(lay.seq_lens[0])}, repeated {units_done // (sub.L * sub.h_kv)}x; "
                                  f"req/s = units/s / {units_per_req} units per request")


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ---------------------------------------------------------------- sharding (multi-GPU, weak scaling)
def shard_rids(rank, world, per_gpu, R_total, scaling="weak"):
    """Global request ids compressed by `rank` (data are keyed by global request id, so a request's
    bytes and results do not depend on the GPU count; contiguous ranges).
    weak:   a contiguous block of per_gpu ids per rank (wrapping over the config's R_total), so every
            rank's workload has the same shape;
    strong: the per_gpu-request batch of one GPU split into contiguous ranges over the ranks (the
            total work is fixed; P = 8 on qwen7b leaves 8 requests = 896 units per GPU)."""
    if scaling == "strong":
        lo, hi = rank * per_gpu // world, (rank + 1) * per_gpu // world
        return np.arange(lo, hi) % R_total
    return np.arange(rank * per_gpu, (rank + 1) * per_gpu) % R_total


CHECK_MOD = (1 << 61) - 1
CHECK_P = 1_000_003


def output_checksum(w, desc, params, rids):
    """Sharding-invariant checksum of a call's selection (the kept lists determine every byte the
    compaction moves): per unit a polynomial hash of its kept positions, weighted by the unit's GLOBAL
    identity (request id, layer, head), summed mod 2^61-1. The sum over ranks equals a single-GPU run of
    the same request ids."""
    import torch
    from paper_2603_08743_b200 import zipc
    cfg = w.cfg
    R = len(rids)
    lay = zipc.zpc_workspace_layout_get(desc, params, R)
    units = R * cfg.L * cfg.h_kv
    ks = lay.kept_stride
    kept = w.workspace[lay.kept:lay.kept + 4 * units * ks].view(torch.int32).view(units, ks).to(torch.int64)
    ell = w.new_lens.reshape(units).to(torch.int64)
    pw = torch.from_numpy(np.array([pow(CHECK_P, i, (1 << 31) - 1) for i in range(ks)], np.int64)).to(kept.device)
    mask = torch.arange(ks, device=kept.device)[None, :] < ell[:, None]
    hu = (((kept + 1) * pw[None, :]) * mask).sum(1) % ((1 << 31) - 1)          # per unit, < 2^31
    gid = (torch.from_numpy(np.asarray(rids, np.int64)).to(kept.device)[:, None] * (cfg.L * cfg.h_kv)
           + torch.arange(cfg.L * cfg.h_kv, device=kept.device)[None, :]).reshape(units) + 1
    prod = (hu * (gid % ((1 << 29) - 3))).cpu().numpy()                         # < 2^60 each
    return int(sum(int(x) for x in prod) % CHECK_MOD)                             # exact (Python ints)


def max_over_ranks(value, dist=None, device=None):
    """Job time = max over ranks (the contract's timing rule); NCCL on GPUs, gloo in CPU tests."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------- measured DRAM traffic
PROFILES = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles")
# committed `ncu --set full` captures of the bench's exact launches (scripts/ncu_capture.sh)
TRAFFIC_FILES = {("qwen7b", False): "r02_traffic.json", ("qwen7b", True): "r02_traffic_lse.json",
                 ("paper_op", False): "r02_traffic_paper_op.json"}


def measured_traffic(cfg, per_gpu, lse_input=False):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the score, compaction and redundancy kernels
    from the committed capture of this exact workload (the config's default wave), else {}."""
    f = TRAFFIC_FILES.get((cfg.name, bool(lse_input)))
    if f is None or per_gpu != (cfg.wave or cfg.R):
        return {}
    try:
        kern = json.load(open(os.path.join(PROFILES, f)))["kernels"]
    except (OSError, ValueError, KeyError):
        return {}
    out = {}
    for name, rec in kern.items():
        tot = rec["dram_bytes_read"] + rec["dram_bytes_write"]
        if "k_score" in name and f"<{cfg.h_q // cfg.h_kv}, {cfg.w}, {cfg.d}" in name:
            out["score"] = tot
        elif "k_compact" in name:
            out["compact"] = tot
        elif "k_red_" in name:
            out["redundancy"] = tot
    return out


def redundancy_roofline(cfg, seq_lens, world, red_ms, peaks, traffic=None):
    """NEXT-1 stage: reads K once (T*d*e per unit) and writes r (4T per unit): HBM-bound."""
    e = 2 if cfg.dtype == "bf16" else 4
    T = np.asarray(seq_lens, np.int64)
    byts = int((T * cfg.d * e + 4 * T).sum() * cfg.L * cfg.h_kv)
    ach = byts / (red_ms / 1e3) / 1e9 if red_ms else None
    if cfg.dtype == "bf16" and cfg.b == 16:
        kern = "k_red_mma"
    elif cfg.dtype == "bf16" and cfg.b % 16 == 0 and 16 < cfg.b <= 256:
        kern = "k_red_umma"
    else:
        kern = "k_red_generic"
    # the within-block Gram matrices: b x b x d multiply-adds per block
    flops = int(2 * cfg.b * cfg.d * (-(-T // cfg.b) * cfg.b).sum() * cfg.L * cfg.h_kv)
    return {"kernel": kern, "bound": "hbm",
            "achieved": ach, "peak": peaks["hbm"], "unit": "GB/s", "frac": ach / peaks["hbm"] if ach else None,
            "algorithmic_bytes_per_launch": byts, "ms": red_ms, "traffic": traffic,
            "gram_tflops": flops / (red_ms / 1e3) / 1e12 if red_ms else None}


def score_roofline(ab, passes, score_ms, peaks, traffic):
    """Roofline of the score kernel (a1+a2), SURVEY §8(d). Its arithmetic intensity is passes x G*w flop per
    K byte (2*G*w*d flops per token per pass over T*d*e bytes); above the measured ridge (bf16 TF/s / HBM
    GB/s, ~254 flop/B) the kernel is tensor-bound: the default two-pass call at G*w = 224 (qwen7b) is at
    448 flop/B. Then `achieved` is the algorithmic two-pass contraction (no M padding, no normaliser
    K-step) in TFLOP/s against the measured bf16 peak; the north star's HBM fraction is kept beside it."""
    secs = score_ms / 1e3
    flops = ab["flops_score"] * passes
    hbm_gbs = ab["score"] / secs / 1e9
    hbm = {"achieved": hbm_gbs, "peak": peaks["hbm"], "unit": "GB/s", "frac": hbm_gbs / peaks["hbm"],
           "frac_of_nominal_8TBs": hbm_gbs / NOMINAL_HBM_GBS, "algorithmic_bytes_per_launch": ab["score"]}
    ridge = peaks["bf16"] * 1e12 / (peaks["hbm"] * 1e9)
    intensity = flops / ab["score"]
    base = {"kernel": "score (a1+a2)", "passes": passes, "intensity_flop_per_byte": intensity,
            "ridge_flop_per_byte": ridge, "peak_src": peaks["src"], "traffic": traffic,
            "traffic_unit": "bytes/launch (dram read+write, ncu --set full)"}
    if intensity > ridge:
        tf = flops / secs / 1e12
        return {**base, "bound": "tensor", "achieved": tf, "peak": peaks["bf16"], "unit": "TFLOP/s",
                "frac": tf / peaks["bf16"], "algorithmic_flops_per_launch": flops,
                "frac_of_sustained": tf / peaks["bf16_sust"],
                "hbm": hbm}
    return {**base, "bound": "hbm", **hbm}


# ---------------------------------------------------------------- GPU arm
def algorithmic_bytes(cfg, seq_lens, budgets, moves, lse_input=False):
    """SURVEY §8(d) per-unit algorithmic bytes summed over the batch (+ the 4*G*w normaliser bytes a
    unit reads with ZPC_F_LSE_INPUT)."""
    e = 2 if cfg.dtype == "bf16" else 4
    T = np.asarray(seq_lens, np.int64)
    units_per_req = cfg.L * cfg.h_kv
    score = int((T * cfg.d * e + cfg.G * cfg.w * cfg.d * e + 4 * T + (4 * cfg.G * cfg.w if lse_input else 0)).sum()
                * units_per_req)
    ell = np.minimum(np.asarray(budgets, np.int64), T[:, None, None])
    select = int((4 * T).sum() * units_per_req + 4 * ell.sum())
    compact = int(4 * moves * cfg.d * e)
    flops_score = int(2 * cfg.G * cfg.w * cfg.d * T.sum() * units_per_req)
    return dict(score=score, select=select, compact=compact, flops_score=flops_score)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="qwen7b")
    ap.add_argument("--impl", default="zipc", choices=["zipc", "reference"])
    ap.add_argument("--seed", type=int, default=2603)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cudacore", action="store_true", help="force the CUDA-core scoring kernel")
    ap.add_argument("--redundancy", action="store_true",
                    help="NEXT-1: lightning redundancy + temperature softmax in the selection score "
                         "(lambda 0.2, tau 0.4 as PAPER.md:718 recommends; p 0.8, the paper gives none)")
    ap.add_argument("--lse-input", action="store_true",
                    help="NEXT-4: single-pass scoring with the window normalisers supplied (ZPC_F_LSE_INPUT); "
                         "the normalisers a decode engine would hold are produced untimed by one two-pass "
                         "zpc_score call before the timed steps")
    ap.add_argument("--wave", type=int, default=0, help="requests per call per GPU (default: the config's)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: per_gpu requests on every rank; strong: the one-GPU batch split over the ranks")
    ap.add_argument("--select-kernel", default="auto", choices=["auto", "smem", "reg"],
                    help="A/B: params.variant select override (k_select / k_select_reg)")
    ap.add_argument("--compact-nt", type=int, default=0, choices=[0, 128, 256, 512, 1024],
                    help="A/B: params.variant compaction CTA width override (0 = by unit count)")
    ap.add_argument("--graph", action="store_true",
                    help="NEXT-3: replay the whole step as one captured CUDA graph (launch-bound small batches); "
                         "value/ms_per_step then come from the graph replays, stage_ms from the eager steps")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    from zpc_inputs import CONFIGS
    cfg = CONFIGS[args.config]
    per_gpu = args.wave or cfg.wave or cfg.R
    workload = (f"{cfg.name}: {per_gpu} req/GPU x {cfg.seq_lens[0]} tok, L={cfg.L} h_kv={cfg.h_kv} h_q={cfg.h_q} "
                f"d={cfg.d} b={cfg.b} w={cfg.w} N_max={cfg.n_max} budget={cfg.budget} pool={cfg.pool_kernel}"
                + (f" prefix={cfg.prefix_tokens}" if cfg.prefix_tokens else "")
                + (" + NEXT-1 lightning redundancy (lambda=0.2 tau=0.4 p=0.8)" if args.redundancy else "")
                + (" + NEXT-4 window LSE input (single-pass score)" if args.lse_input else "")
                + (" [CUDA graph]" if args.graph else ""))

    if args.impl == "reference":
        if rank != 0:
            return 0
        # a reference step = one bounded sample of the workload (whole sampled requests on a layer subset, ~3 s);
        # ms_per_step is that step's measured wall time, value = requests' worth of units per second over them
        units_done, secs = 0, 0.0
        info = None
        for _ in range(args.warmup):
            time_oracle(cfg, args.seed, 1, budget_s=0.5, redundancy=args.redundancy)
        for _ in range(args.steps):
            _, info = time_oracle(cfg, args.seed, 1, budget_s=3.0, redundancy=args.redundancy)
            units_done += info["units"]
            secs += info["seconds"]
        value = units_done / (cfg.L * cfg.h_kv) / secs
        line = {"impl": "reference", "metric": "requests_compressed_per_s", "value": value, "unit": "req/s",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1000.0 * secs / args.steps, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (zpc_inputs Philox recipe)",
                "config": {"workload": workload},
                "cpu_baseline": {"value": value, "unit": "req/s", "cores": info["threads"], "kind": "oracle",
                                 "sample": info["sample"], "cpu": cpu_model()},
                "e2e": {"value": value, "unit": "req/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return 0

    import torch
    import torch.distributed as dist
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())

    from paper_2603_08743_b200 import zipc
    from paper_2603_08743_b200.batch import batch_of, desc_params
    from zpc_harness import window_lse_from_two_pass
    if args.select_kernel != "auto" or args.compact_nt:
        zipc.DEFAULT_VARIANT = zipc.variant(select={"auto": 0, "smem": 1, "reg": 2}[args.select_kernel],
                                            compact_nt=args.compact_nt)
    from zpc_inputs.device import generate

    rids = shard_rids(rank, world, per_gpu, cfg.R, args.scaling)
    w = generate(cfg, args.seed, rids, device=dev)
    flags = zipc.ZPC_F_COUNT_MOVES | (zipc.ZPC_F_SCORE_CUDACORE if args.cudacore else 0)
    if args.lse_input:
        w.window_lse = window_lse_from_two_pass(w, flags)
    desc, params = desc_params(w, flags=flags, redundancy=RED_PARAMS if args.redundancy else None,
                               lse_input=args.lse_input)
    batch = batch_of(w, desc, params)
    stream = torch.cuda.current_stream()
    lay = w.layout
    nm = cfg.n_max
    # pristine copies of everything a step mutates
    touched = np.unique(np.concatenate([lay.tables[:, :nm].ravel(), lay.free_stack[:lay.free_top]]))
    touched = touched[touched >= 0]
    touched_d = torch.from_numpy(touched.astype(np.int64)).to(dev)
    k0 = w.k.index_select(1, touched_d)
    v0 = w.v.index_select(1, touched_d)
    state0 = {n: getattr(w, n).clone() for n in ("tables", "free_stack", "free_top")}
    refs0 = None if w.ref_counts is None else w.ref_counts.clone()

    def restore():
        w.k.index_copy_(1, touched_d, k0)
        w.v.index_copy_(1, touched_d, v0)
        for n, t in state0.items():
            getattr(w, n).copy_(t)
        if refs0 is not None:
            w.ref_counts.copy_(refs0)

    stages = [zipc.zpc_plan, zipc.zpc_score, zipc.zpc_select, zipc.zpc_compact, zipc.zpc_finalize]
    stage_names = ["plan", "score", "select", "compact", "finalize"]
    if args.redundancy:   # NEXT-1 stage between score and select (zpc_compress runs it in that order)
        stages.insert(2, zipc.zpc_redundancy)
        stage_names.insert(2, "redundancy")

    def step(evs):          # the same work stage by stage: the per-stage breakdown behind the rooflines
        evs[0].record(stream)
        for i, fn in enumerate(stages):
            fn(desc, params, batch, stream)
            evs[i + 1].record(stream)

    def step_call(evs):     # the timed step: ONE zpc_compress call (the public API)
        evs[0].record(stream)
        zipc.zpc_compress(desc, params, batch, stream)
        evs[1].record(stream)

    mk = lambda: [torch.cuda.Event(enable_timing=True) for _ in range(len(stages) + 1)]  # noqa: E731
    for _ in range(max(3, args.warmup)):
        restore()
        step(mk())
        restore()
        step_call(mk())
    torch.cuda.synchronize()
    assert int(w.status.item()) == 0, zipc.status_string(int(w.status.item()))
    moves = int(w.workspace[zipc.zpc_workspace_layout_get(desc, params, len(rids)).moves:][:8].view(torch.int64).item())

    sampler = ClockSampler(local if world > 1 else torch.cuda.current_device())
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    time.sleep(0.3)
    call_evs = []
    wall0 = time.perf_counter()
    for _ in range(args.steps):
        restore()
        evs = mk()
        step_call(evs)
        call_evs.append(evs)
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    step_ms_total = float(sum(evs[0].elapsed_time(evs[1]) for evs in call_evs))
    eager_ms = step_ms_total
    # per-stage breakdown (after the timed region, same inputs): stage-by-stage calls
    all_evs = []
    for _ in range(args.steps):
        restore()
        evs = mk()
        step(evs)
        all_evs.append(evs)
    torch.cuda.synchronize()
    stage_ms = np.zeros(len(stages))
    for evs in all_evs:
        for i in range(len(stages)):
            stage_ms[i] += evs[i].elapsed_time(evs[i + 1])
    graph_info = None
    if args.graph:
        # the same stage sequence captured once; restores stay outside the graph (untimed)
        g = torch.cuda.CUDAGraph()
        restore()
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            cap = torch.cuda.current_stream()
            zipc.zpc_compress(desc, params, batch, cap)
        g_ms = 0.0
        for i in range(max(3, args.warmup) + args.steps):
            restore()
            a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            g.replay()
            b_.record(stream)
            b_.synchronize()
            if i >= max(3, args.warmup):
                g_ms += a.elapsed_time(b_)
        assert int(w.status.item()) == 0, zipc.status_string(int(w.status.item()))
        step_ms_total = g_ms
        graph_info = {"graph_ms_per_step": g_ms / args.steps, "eager_ms_per_step": eager_ms / args.steps}
    max_ms = max_over_ranks(step_ms_total, dist, dev)
    ms_per_step = max_ms / args.steps
    T_sum = int(lay.seq_lens.sum())
    checksum = output_checksum(w, desc, params, rids)
    peaks = load_peaks()
    ab = algorithmic_bytes(cfg, lay.seq_lens, w.budgets_host, moves, args.lse_input)
    # per-rank record, all-gathered over NCCL (SURVEY.md §8(d) timing protocol): time, requests, sum T,
    # moved rows, algorithmic bytes, output checksum
    rec = [step_ms_total / args.steps, len(rids), T_sum, moves, ab["score"] + ab["select"] + ab["compact"],
           checksum]
    if world > 1:
        t = torch.tensor(rec, dtype=torch.float64, device=dev)
        ck = torch.tensor([checksum], dtype=torch.int64, device=dev)
        g_rec = [torch.zeros_like(t) for _ in range(world)]
        g_ck = [torch.zeros_like(ck) for _ in range(world)]
        dist.all_gather(g_rec, t)
        dist.all_gather(g_ck, ck)
        ranks = [dict(ms_per_step=float(x[0]), requests=int(x[1]), sum_T=int(x[2]), moved_rows=int(x[3]),
                      algorithmic_bytes=int(x[4]), checksum=int(c.item())) for x, c in zip(g_rec, g_ck)]
    else:
        ranks = [dict(ms_per_step=rec[0], requests=rec[1], sum_T=rec[2], moved_rows=rec[3], algorithmic_bytes=rec[4],
                      checksum=checksum)]
    R_all = sum(r["requests"] for r in ranks)
    T_all = sum(r["sum_T"] for r in ranks)
    value = R_all / (ms_per_step / 1000.0)
    job_checksum = sum(r["checksum"] for r in ranks) % CHECK_MOD

    score_ms = stage_ms[stage_names.index("score")] / args.steps
    compact_ms = stage_ms[stage_names.index("compact")] / args.steps
    step_bytes = ab["score"] + ab["select"] + ab["compact"]
    traffic = measured_traffic(cfg, per_gpu, args.lse_input)
    passes = 1 if args.lse_input else 2
    tensor_tf = ab["flops_score"] * passes / (score_ms / 1e3) / 1e12   # passes x 2*G*w*d per token
    roofline = score_roofline(ab, passes, score_ms, peaks, traffic.get("score"))
    extra = {
        "stage_ms": {n: round(float(x) / args.steps, 4) for n, x in zip(stage_names, stage_ms)},
        "stage_ms_source": "stage-by-stage calls after the timed region (the timed step is one zpc_compress call)",
        "score_tensor_tflops": tensor_tf, "score_passes": passes,
        "compact_roofline": {"achieved": ab["compact"] / (compact_ms / 1e3) / 1e9 if compact_ms else None,
                             "peak": peaks["hbm"], "unit": "GB/s", "moved_rows": moves,
                             "frac": (ab["compact"] / (compact_ms / 1e3) / 1e9) / peaks["hbm"] if compact_ms else None,
                             "traffic": traffic.get("compact"), "algorithmic_bytes_per_launch": ab["compact"]},
        "step_hbm_frac": step_bytes / (ms_per_step / 1e3) / 1e9 / peaks["hbm"],
        "step_hbm_frac_of_nominal_8TBs": step_bytes / (ms_per_step / 1e3) / 1e9 / NOMINAL_HBM_GBS,
        **({"redundancy_roofline": redundancy_roofline(cfg, lay.seq_lens, world,
                                                        stage_ms[stage_names.index("redundancy")] / args.steps,
                                                        peaks, traffic.get("redundancy"))} if args.redundancy else {}),
        "kv_tokens_per_s": T_all / (ms_per_step / 1e3),
        "ranks": ranks, "output_checksum": job_checksum,
        **({"cuda_graph": graph_info} if graph_info else {}),
        "wall_s_incl_restores": wall,
    }

    # ---- e2e: host bookkeeping through zpc_compress_host (H2D + step + D2H every step)
    e2e = None
    if not args.no_e2e:
        host = {n: getattr(w, n).cpu().pin_memory() for n in ("q_slots", "seq_lens", "budgets", "new_lens",
                                                            "new_num_blocks", "freed", "num_freed", "status")}
        host_t0 = {n: state0[n].cpu().pin_memory() for n in ("tables", "free_stack", "free_top")}
        host_live = {n: t.clone().pin_memory() for n, t in host_t0.items()}
        href = None if refs0 is None else refs0.cpu().pin_memory()
        href_live = None if href is None else href.clone().pin_memory()
        need = zipc.zpc_workspace_bytes_host(desc, params, len(rids), lay.table_stride, lay.N_total,
                                             int(w.freed.numel()))
        ws_h = torch.empty(need, dtype=torch.uint8, device=dev)
        hb = zipc.make_batch(k_cache=w.k, v_cache=w.v, q_cache=w.q, q_slots=host["q_slots"],
                             seq_lens=host["seq_lens"], block_tables=host_live["tables"], budgets=host["budgets"],
                             new_lens=host["new_lens"], new_num_blocks=host["new_num_blocks"], ref_counts=href_live,
                             free_stack=host_live["free_stack"], free_top=host_live["free_top"],
                             freed_blocks=host["freed"], num_freed=host["num_freed"], workspace=ws_h,
                             status=host["status"], window_lse=w.window_lse)
        R = len(rids)
        h2d = 4 * (R * 2 + R * lay.table_stride + host["budgets"].numel() + lay.N_total + 1) + \
            (4 * lay.N_total if href is not None else 0)
        d2h = 4 * (R * lay.table_stride + host["new_lens"].numel() + R + lay.N_total + int(w.freed.numel()) + 3) + \
            (4 * lay.N_total if href is not None else 0)
        e2e_ms = 0.0
        # the pinned host arrays are device-accessible: one gather and one scatter kernel instead of ~17 copies
        params_h = zipc.zpc_params.from_buffer_copy(params)
        params_h.flags |= zipc.ZPC_F_HOST_MAPPED
        ge = None
        if args.graph:
            # --graph: the same public call captured once (its host<->device copies become memcpy nodes that read
            # and write the pinned host arrays at every replay), as a serving loop with fixed staging buffers would
            restore()
            torch.cuda.synchronize()
            ge = torch.cuda.CUDAGraph()
            with torch.cuda.graph(ge):
                zipc.zpc_compress_host(desc, params_h, hb, torch.cuda.current_stream())
        for i in range(max(3, args.warmup) + args.steps):
            restore()
            for n in host_live:
                host_live[n].copy_(host_t0[n])
            if href_live is not None:
                href_live.copy_(href)
            torch.cuda.synchronize()
            a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            if ge is not None:
                ge.replay()
            else:
                zipc.zpc_compress_host(desc, params_h, hb, stream)
            b_.record(stream)
            b_.synchronize()
            assert int(host["status"][0]) == 0
            if i >= max(3, args.warmup):
                e2e_ms += a.elapsed_time(b_)
        e2e_max = max_over_ranks(e2e_ms, dist, dev)
        e2e = {"value": R_all / (e2e_max / args.steps / 1e3), "unit": "req/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "path": ("zpc_compress_host" + (" captured as one CUDA graph (memcpy nodes + kernels, replayed per "
                                                 "step)" if args.graph else "") +
                        ": block tables, budgets, free stack, ref counts host-resident (pinned, read and written in "
                        "place by one gather and one scatter kernel: ZPC_F_HOST_MAPPED); "
                        "K/V/Q caches device-resident (the paged pool lives in HBM)")}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v_cpu, info = time_oracle(cfg, args.seed, 1, budget_s=15.0, redundancy=args.redundancy)
        cpu = {"value": v_cpu, "unit": "req/s", "cores": info["threads"], "kind": "oracle",
               "sample": info["sample"], "cpu": cpu_model(), "seconds": info["seconds"]}

    # kernels one zpc_compress call launches: plan (2), the scoring family (k_coop_plan + k_score_coop: 2; k_score_res
    # or k_score_tc/ovl: 1; k_lse_cc + k_final_cc: 2), redundancy (1), select (1), compact (1), finalize (2)
    path = zipc.zpc_score_path(desc, params)
    score_kernels = {zipc.ZPC_PATH_COOP: 2, zipc.ZPC_PATH_RESIDENT: 1, zipc.ZPC_PATH_TC: 1}.get(path, 2)
    launches_per_step = 2 + score_kernels + 2 + 2
    if args.redundancy:
        launches_per_step += 1
    if rank == 0:
        line = {"metric": "requests_compressed_per_s", "value": value, "unit": "req/s", "n_gpus": world,
                "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": cfg.dtype,
                "data": "synthetic (zpc_inputs Philox recipe, generated in HBM)",
                "config": {"workload": workload, "requests_per_gpu": per_gpu if args.scaling == "weak" else len(rids),
                           "requests_total": R_all,
                           "l2": "pool > L2 (15 GB K for qwen7b); modified blocks restored from a pristine copy "
                                 "between steps (untimed, writes > L2)",
                           "parallelism": f"request-sharded x{world} ({args.scaling} scaling), no data-path "
                                          f"collective; NCCL all-gathers the per-rank stats"},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches_per_step * args.steps, "clocks": clocks, **extra}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
