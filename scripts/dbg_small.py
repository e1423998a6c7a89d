"""Run one small 7B-shaped zpc_compress call and report the CUDA error string (debugging aid)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

from helpers import run_gpu  # noqa: E402
from zpc_inputs import CONFIGS, make_host_workload, scaled  # noqa: E402
from zpc_inputs.device import from_host  # noqa: E402

cfg = scaled(CONFIGS["qwen7b"], L=2, h_kv=2, h_q=14, n_max=9, seq_lens=[300, 257, 416, 257], budget=128, free_slack=5)
w = from_host(make_host_workload(cfg, 3))
try:
    run_gpu(w)
    torch.cuda.synchronize()
    print("ok status", int(w.status.item()))
except Exception as e:  # noqa: BLE001
    print("error:", e)
rt = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
if rt:
    rt.cudaGetLastError.restype = ctypes.c_int
    rt.cudaGetErrorString.restype = ctypes.c_char_p
    e = rt.cudaGetLastError()
    print("cudaGetLastError", e, rt.cudaGetErrorString(e))
