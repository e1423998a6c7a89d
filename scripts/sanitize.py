"""compute-sanitizer driver: one small zpc_compress per kernel family (no oracle, execution only).

    compute-sanitizer --tool memcheck python scripts/sanitize.py [case ...]
Cases (default all): toy (fp32, CUDA-core score, k_select, k_red_generic), 7b (k_score_coop, k_select_reg,
k_compact), 7b_serial (k_score_tc two-pass), 8b (k_score_ovl, G*w = 128), 32b_d64 (coop G = 5, d = 64),
paper_op (k_score_tc w = 16, b = 256), lse (single-pass), red16 (k_red_mma), red256 (k_red_tile),
global_prefix (NEXT-2 with shared prefix), cudacore (k_lse_cc / k_final_cc), validate (k_validate).
Every call must leave status 0.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_08743_b200 import zipc  # noqa: E402
from paper_2603_08743_b200.batch import batch_of, desc_params  # noqa: E402
from zpc_inputs import CONFIGS, global_history, make_host_workload, scaled  # noqa: E402
from zpc_inputs.device import from_host  # noqa: E402

S7 = dict(L=2, h_kv=2, h_q=14, n_max=9, seq_lens=[300, 257, 416, 1100], budget=128, free_slack=5)
CASES = {
    "toy": (CONFIGS["toy"], {}),
    "7b": (scaled(CONFIGS["qwen7b"], **S7), {}),
    "7b_serial": (scaled(CONFIGS["qwen7b"], **S7), dict(variant=zipc.ZPC_V_SCORE_SERIAL)),
    "8b": (scaled(CONFIGS["llama8b"], L=2, h_kv=2, h_q=8, n_max=9, seq_lens=[513, 700, 1030], budget=(32, 128),
                  wave=0), {}),
    "32b_d64": (scaled(CONFIGS["qwen32b"], L=2, h_kv=2, h_q=10, d=64, n_max=6, seq_lens=[200, 333], budget=80,
                       wave=0), {}),
    "paper_op": (scaled(CONFIGS["paper_op"], L=2, h_kv=2, h_q=8, seq_lens=[2304, 2100, 2500], wave=0,
                        free_slack=3), {}),
    "lse": (scaled(CONFIGS["qwen7b"], **S7), dict(lse=True)),
    "red16": (scaled(CONFIGS["qwen7b"], **S7), dict(redundancy=(0.2, 0.4, 0.35))),
    "red256": (scaled(CONFIGS["paper_op"], L=2, h_kv=2, h_q=8, seq_lens=[2304, 2149], budget=2048, wave=0,
                      free_slack=3), dict(redundancy=(0.2, 0.4, 0.35))),
    "global_prefix": (scaled(CONFIGS["prefix"], L=2, h_kv=2, h_q=14, n_max=9, seq_lens=[400] * 3, prefix_tokens=160,
                             budget=128, wave=0, free_slack=4), dict(global_alpha=0.8)),
    "cudacore": (scaled(CONFIGS["qwen7b"], **S7), dict(flags=zipc.ZPC_F_SCORE_CUDACORE)),
    "validate": (scaled(CONFIGS["qwen7b"], **S7), dict(flags=zipc.ZPC_F_VALIDATE)),
}


def run(name):
    cfg, o = CASES[name]
    hw = make_host_workload(cfg, 7)
    if o.get("global_alpha") is not None:
        hw.f_cache, hw.is_compressed = global_history(cfg, 7, hw.layout.N_total, hw.layout.rids)
    w = from_host(hw)
    if o.get("lse"):
        from zpc_harness import window_lse_from_two_pass
        w.window_lse = window_lse_from_two_pass(w, 0)
    desc, params = desc_params(w, flags=o.get("flags", 0), redundancy=o.get("redundancy"),
                               global_alpha=o.get("global_alpha"), lse_input=bool(o.get("lse")))
    if "variant" in o:
        params.variant = o["variant"]
    b = batch_of(w, desc, params)
    zipc.zpc_compress(desc, params, b)
    torch.cuda.synchronize()
    st = int(w.status.item())
    print(f"{name}: status {st}", flush=True)
    assert st == 0, name


if __name__ == "__main__":
    for n in (sys.argv[1:] or list(CASES)):
        run(n)
    print("sanitize cases: ok")
