"""CPU-only checks of the C ABI: the library loads, exports every function include/zipc.h
declares, and the host-side argument checks behave (no kernels are launched)."""
import ctypes
import os
import re

import pytest

from paper_2603_08743_b200 import zipc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "zipc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(zpc_[a-z_]+)\s*\(", src)))


def test_header_declares_expected_entry_points():
    assert set(header_functions()) == set(zipc.EXPORTS)


def test_library_exports_every_declared_symbol():
    L = zipc.lib()
    for name in header_functions():
        assert hasattr(L, name), name
    assert zipc.zpc_abi_version() == zipc.ABI_VERSION == 6


def _desc(**kw):
    d = dict(L=28, h_kv=4, h_q=28, d=128, b=16, N_total=33000, M=70, w=32, dtype="bf16")
    d.update(kw)
    return zipc.make_desc(d["L"], d["h_kv"], d["h_q"], d["d"], d["b"], d["N_total"], d["M"], d["w"], d["dtype"])


def test_workspace_bytes_and_layout():
    p = zipc.make_params(129, 7, 8192, 0)
    n = zipc.zpc_workspace_bytes(_desc(), p, 64)
    lay = zipc.zpc_workspace_layout_get(_desc(), p, 64)
    assert n == lay.total_bytes > 64 * 28 * 4 * 8192 * 4
    assert lay.kept_stride == 128 * 16
    offs = [lay.scores, lay.kept, lay.targets, lay.reserved, lay.n_prefix, lay.lse, lay.moves, lay.redundancy,
            lay.internal]
    assert offs == sorted(offs) and all(o % 256 == 0 for o in offs)
    assert lay.internal == lay.redundancy            # zero-size region without ZPC_F_REDUNDANCY


def test_redundancy_region_and_params():
    """ZPC_F_REDUNDANCY adds an fp32 [R][L][h_kv][max_seq_len] region and validates lambda/tau/p."""
    p0 = zipc.make_params(129, 7, 8192, 0)
    p1 = zipc.make_params(129, 7, 8192, zipc.ZPC_F_REDUNDANCY)
    lay0 = zipc.zpc_workspace_layout_get(_desc(), p0, 64)
    lay1 = zipc.zpc_workspace_layout_get(_desc(), p1, 64)
    assert lay1.internal - lay1.redundancy >= 64 * 28 * 4 * 8192 * 4
    assert lay1.total_bytes - lay0.total_bytes >= 64 * 28 * 4 * 8192 * 4
    for bad in (dict(redundancy_lambda=-0.1), dict(redundancy_tau=0.0), dict(redundancy_tau=-1.0),
                dict(redundancy_p=1.5), dict(redundancy_p=-0.1), dict(redundancy_lambda=float("nan"))):
        pb = zipc.make_params(129, 7, 8192, zipc.ZPC_F_REDUNDANCY, **bad)
        assert zipc.zpc_workspace_bytes(_desc(), pb, 4) == 0, bad
        # without the flag the same values are ignored
        pn = zipc.make_params(129, 7, 8192, 0, **bad)
        assert zipc.zpc_workspace_bytes(_desc(), pn, 4) > 0, bad
    assert zipc.zpc_workspace_bytes(_desc(b=64, dtype="fp32"), p1, 4) == 0   # fp32: one warp per block, b <= 32
    assert zipc.zpc_workspace_bytes(_desc(b=40), p1, 4) == 0                   # bf16 tile kernel: multiples of 16
    assert zipc.zpc_workspace_bytes(_desc(b=512), p1, 4) == 0                  # ... up to 256
    assert zipc.zpc_workspace_bytes(_desc(b=256, N_total=2000), p1, 4) > 0     # the paper's b = 256


def test_per_layer_offset_overflow_rejected():
    """Kernels address a layer's K/V plane with 32-bit element offsets: a per-layer pool of >= 2^32
    elements (N_total * b * h_kv * d) is ZPC_ERR_INVALID_ARG (workspace size 0), one block fewer is fine."""
    p = zipc.make_params(129, 7, 8192)
    limit = (1 << 32) // (16 * 4 * 128)   # 524288 blocks of b = 16, h_kv = 4, d = 128
    assert zipc.zpc_workspace_bytes(_desc(N_total=limit), p, 4) == 0
    assert zipc.zpc_workspace_bytes(_desc(N_total=limit - 1), p, 4) > 0


def test_variant_bits_validated():
    d = _desc()
    assert zipc.zpc_workspace_bytes(d, zipc.make_params(129, 7, 8192, variant=zipc.variant(select=2, compact_nt=512)), 4) > 0
    assert zipc.zpc_workspace_bytes(d, zipc.make_params(129, 7, 8192, variant=3 << zipc.ZPC_V_SELECT_SHIFT), 4) == 0
    assert zipc.zpc_workspace_bytes(d, zipc.make_params(129, 7, 8192, variant=5 << zipc.ZPC_V_COMPACT_SHIFT), 4) == 0
    assert zipc.zpc_workspace_bytes(d, zipc.make_params(129, 7, 8192, variant=1 << 20), 4) == 0


@pytest.mark.parametrize("bad", [dict(h_q=30), dict(d=96), dict(w=0), dict(dtype=7), dict(h_q=4 * 9, w=32)])
def test_invalid_descriptors(bad):
    assert zipc.zpc_workspace_bytes(_desc(**bad), zipc.make_params(129, 7, 8192), 4) == 0


@pytest.mark.parametrize("pk,nmax,msl", [(2, 129, 8192), (7, 1, 8192), (7, 129, 0), (7, 129, 262145)])
def test_invalid_params(pk, nmax, msl):
    assert zipc.zpc_workspace_bytes(_desc(), zipc.make_params(nmax, pk, msl), 4) == 0


def test_compress_rejects_bad_args_before_enqueueing():
    d, p = _desc(), zipc.make_params(129, 7, 8192)
    b = zipc.zpc_batch()
    assert zipc.zpc_compress(d, p, b, stream=0, check=False) == zipc.ZPC_ERR_INVALID_ARG
    # workspace too small (fake, never dereferenced: the check happens first)
    buf = (ctypes.c_int32 * 8)()
    addr = (ctypes.addressof(buf) + 255) & ~255
    b = zipc.zpc_batch(workspace=addr + 256, workspace_bytes=16, status=addr, num_requests=0,
                       free_stack=addr, free_top=addr, freed_blocks=addr, num_freed=addr)
    assert zipc.zpc_compress(d, p, b, stream=0, check=False) == zipc.ZPC_ERR_WORKSPACE
    assert zipc.status_string(zipc.ZPC_ERR_NO_FREE_BLOCKS).startswith("free stack")


def test_global_score_params():
    """ZPC_F_GLOBAL_SCORE validates alpha in [0, 1]; without the flag alpha is ignored."""
    for bad in (-0.1, 1.5, float("inf")):
        assert zipc.zpc_workspace_bytes(_desc(), zipc.make_params(129, 7, 8192, zipc.ZPC_F_GLOBAL_SCORE,
                                                                  global_alpha=bad), 4) == 0
        assert zipc.zpc_workspace_bytes(_desc(), zipc.make_params(129, 7, 8192, 0, global_alpha=bad), 4) > 0
    assert zipc.zpc_workspace_bytes(_desc(), zipc.make_params(129, 7, 8192, zipc.ZPC_F_GLOBAL_SCORE,
                                                              global_alpha=0.8), 4) > 0


def test_score_path_query():
    """zpc_score_path reports the scoring kernel family a call takes, with no launch (include/zipc.h)."""
    p = zipc.make_params(129, 7, 8192, 0)
    assert zipc.zpc_score_path(_desc(), p) == zipc.ZPC_PATH_COOP                       # qwen7b: G = 7, w = 32
    assert zipc.zpc_score_path(_desc(h_kv=8, h_q=32), p) == zipc.ZPC_PATH_TC           # llama8b: G = 4
    assert zipc.zpc_score_path(_desc(h_q=4), p) == zipc.ZPC_PATH_TC                    # MHA, G = 1
    assert zipc.zpc_score_path(_desc(h_q=24), p) == zipc.ZPC_PATH_TC                   # G = 6
    po = zipc.make_params(9, 7, 2304, 0)
    assert zipc.zpc_score_path(_desc(h_kv=8, h_q=32, b=256, w=16, N_total=1000), po) == zipc.ZPC_PATH_RESIDENT   # paper_op
    assert zipc.zpc_score_path(_desc(h_kv=8, h_q=32, b=256, w=16, N_total=1000), zipc.make_params(9, 7, 8192, 0)) == zipc.ZPC_PATH_TC
    assert zipc.zpc_score_path(_desc(h_kv=8, h_q=64, b=256, w=16, N_total=1000), po) == zipc.ZPC_PATH_TC   # G = 8
    assert zipc.zpc_score_path(_desc(w=8), p) == zipc.ZPC_PATH_CUDACORE
    assert zipc.zpc_score_path(_desc(dtype="fp32"), p) == zipc.ZPC_PATH_CUDACORE
    assert zipc.zpc_score_path(_desc(), zipc.make_params(129, 7, 8192, zipc.ZPC_F_SCORE_CUDACORE)) == zipc.ZPC_PATH_CUDACORE
    assert zipc.zpc_score_path(_desc(), zipc.make_params(129, 7, 8192, zipc.ZPC_F_LSE_INPUT)) == zipc.ZPC_PATH_TC
    assert zipc.zpc_score_path(_desc(), zipc.make_params(129, 7, 8192, 0, variant=zipc.ZPC_V_SCORE_SERIAL)) == zipc.ZPC_PATH_TC
    assert zipc.zpc_score_path(_desc(d=96), p) == zipc.ZPC_ERR_INVALID_ARG
