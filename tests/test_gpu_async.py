"""NEXT-3 asynchronous compression: zpc_compress on a side stream while another
stream keeps the GPU busy (a stand-in for the decode step) must give the same bytes as a call on an
idle GPU, and both must pass the oracle parity rules (tests/helpers.py). The ABI's concurrency rule
(include/zipc.h): the library keeps no global state, so only the caller's stream orders the stages."""
import pytest
import torch

from zpc_inputs import CONFIGS, make_host_workload, scaled
from zpc_inputs.device import from_host
from paper_2603_08743_b200 import zipc
from paper_2603_08743_b200.batch import batch_of, desc_params

from helpers import full_check, gpu_results, snapshot_inputs

pytestmark = pytest.mark.gpu

CFG = scaled(CONFIGS["paper_op"], L=3, seq_lens=[2304, 2100, 2560, 2304], wave=0, free_slack=6)


def _compress(busy):
    w = from_host(make_host_workload(CFG, 41))
    inp = snapshot_inputs(w)
    desc, params = desc_params(w)
    b = batch_of(w, desc, params)
    side = torch.cuda.Stream()
    torch.cuda.synchronize()
    if busy:
        a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
        start = torch.cuda.Event()
        start.record()
        side.wait_event(start)
        with torch.cuda.stream(side):
            zipc.zpc_compress(desc, params, b, side)
        for _ in range(8):   # the "decode" load on the main stream, overlapping the call
            a = (a @ a).clamp_(-1, 1)
    else:
        zipc.zpc_compress(desc, params, b, side)
    torch.cuda.synchronize()
    res = gpu_results(w, desc, params)
    full_check(w, inp, res)
    return res


def test_async_equals_idle(cuda_ok):
    idle = _compress(False)
    busy = _compress(True)
    for k in ("S", "kept", "k", "v", "tables", "new_lens", "freed", "stack"):
        assert (idle[k] == busy[k]).all(), k
    assert idle["top"] == busy["top"]
