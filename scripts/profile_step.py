"""One zpc_compress step on a reduced batch of a BASELINE config, for ncu captures.

    ncu --set full -k regex:k_score_tc -c 1 python scripts/profile_step.py --config qwen7b --requests 8
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_08743_b200 import zipc  # noqa: E402
from paper_2603_08743_b200.batch import batch_of, desc_params  # noqa: E402
from zpc_inputs import CONFIGS  # noqa: E402
from zpc_inputs.device import generate  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="qwen7b")
ap.add_argument("--requests", type=int, default=8)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--cudacore", action="store_true")
ap.add_argument("--redundancy", action="store_true")
ap.add_argument("--lse-input", action="store_true", help="NEXT-4 single-pass scoring")
a = ap.parse_args()
cfg = CONFIGS[a.config]
w = generate(cfg, 2603, np.arange(a.requests))
flags = zipc.ZPC_F_SCORE_CUDACORE if a.cudacore else 0
if a.lse_input:
    from zpc_harness import window_lse_from_two_pass
    w.window_lse = window_lse_from_two_pass(w, flags)
desc, params = desc_params(w, flags=flags, redundancy=(0.2, 0.4, 0.8) if a.redundancy else None,
                           lse_input=a.lse_input)
b = batch_of(w, desc, params)
for _ in range(a.steps):
    zipc.zpc_compress(desc, params, b)
torch.cuda.synchronize()
print("status", int(w.status.item()))
