"""GPU: the KV-head split without an all-gather (vsp_vs_prefill_mirrored).

The attention epilogue stores every O tile and LSE row into the caller's output and, at the
same offsets, into up to 7 mirror buffers (the other ranks' full-layer outputs mapped over
NVLink with CUDA IPC). Checked here on one B200: mirrors are bit-identical copies in both O
layouts, argument errors carry the C ABI's messages, and two processes sharing the GPU
assemble the layer through IPC-mapped buffers exactly as the one-process call computes it.
"""
import os
import socket
import subprocess
import sys

import pytest
import torch

from helpers import qkv

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def vsp():
    import paper_2603_04460_b200 as m
    m.load_library()
    return m


def _layer(vsp, n=1280, hq=8, hkv=4):
    q, k, v = qkv(n, hq, hkv, seed=31)
    p = vsp.make_indexer_params(hkv, 128, 256, torch.Generator().manual_seed(4), head_sigma=0.5)
    return q, k, v, p, vsp.BudgetConfig(0.6, 0.7, 1, None)


@pytest.mark.parametrize("head_major", [True, False])
def test_mirrors_receive_identical_outputs(vsp, head_major):
    q, k, v, p, b = _layer(vsp)
    o0, l0, _ = vsp.vs_prefill(q, k, v, p, b, head_major=head_major)
    ms = [(torch.full_like(o0, 3.0), torch.full_like(l0, 7.0)) for _ in range(3)]
    before = vsp.kernel_launches()
    o1, l1, _ = vsp.vs_prefill(q, k, v, p, b, head_major=head_major, mirrors=ms)
    torch.cuda.synchronize()
    assert vsp.kernel_launches() - before == 4  # K1, K2, planning, K3: the copies are in K3
    assert torch.equal(o1, o0) and torch.equal(l1, l0)
    for mo, ml in ms:
        assert torch.equal(mo, o0) and torch.equal(ml, l0)


def test_mirror_argument_errors(vsp):
    q, k, v, p, b = _layer(vsp, n=512)
    o = torch.empty(q.shape[1], 512, 128, dtype=q.dtype, device=q.device)
    with pytest.raises(vsp.VspError, match="at most 7 mirrors"):
        vsp.vs_prefill(q, k, v, p, b, head_major=True, mirrors=[(o, None)] * 8)
    with pytest.raises(vsp.VspError, match="LSE mirrors must match lse"):
        vsp.vs_prefill(q, k, v, p, b, head_major=True, mirrors=[(o, None)])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_two_ranks_assemble_the_layer_through_ipc_mirrors():
    port = _free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "mirror_worker.py")], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    outs = [p.communicate(timeout=300)[0] for p in procs]
    for p, out in zip(procs, outs):
        assert p.returncode == 0, out[-3000:]
        assert "assembled == one-process layer: True" in out
