"""Exchange + update kernels (csrc/stz_peer.cuh): the fused SGD + split-plane
repack against the separate SGD and pack kernels (bit-exact), the
single-member stz_allreduce_sgd, and the multi-member peer-memory exchange
(tools/peer_check.py) as separate processes -- all on one GPU (IPC mapping and
barrier between processes sharing cuda:0) and, where the box has them, one
process per GPU over NVLink.  The exchange replaces stanza_runtime.py:309-350
(allreduce_sum, collectives.py:117-157, then sgd_step, tensor_core.py:366-388)."""

import os
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ptr(t):
    import ctypes
    return ctypes.c_void_p(t.data_ptr())


def _stream():
    import ctypes
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


@pytest.mark.parametrize("D,D8", [(1000, 1000), (37, 40)])
def test_sgd_pack_matches_sgd_then_pack(lib, D, D8):
    """stz_sgd_momentum_pack == stz_sgd_momentum + stzx_pack_rows, bit for bit,
    for a vector of [gap | W rows x D | gap | W2 | tail]."""
    from paper_1812_10624_b200 import _lib
    g = torch.Generator().manual_seed(3)
    rows = 64
    n = 8 + rows * D + 12 + rows * D + 7
    n = (n + 3) // 4 * 4 + 3          # ragged tail
    off1 = 8
    off2 = (off1 + rows * D + 12 + 3) // 4 * 4
    assert off2 + rows * D <= n
    w = torch.randn(n, generator=g).cuda()
    v = (0.1 * torch.randn(n, generator=g)).cuda()
    gr = (5 * torch.randn(n, generator=g)).cuda()
    w2, v2 = w.clone(), v.clone()
    pa = torch.zeros((3, rows, D8), dtype=torch.bfloat16, device="cuda")
    pb = torch.zeros_like(pa)
    ranges = [(off1, rows * D, pa.data_ptr(), pa[0].numel(), D, D8),
              (off2, rows * D, pb.data_ptr(), pb[0].numel(), D, D8)]
    ra = _lib.range_array(ranges)
    _lib.call("stz_sgd_momentum_pack", _ptr(w), _ptr(v), _ptr(gr), n, 0.05, 0.9,
              1.0 / 384, ra, 2, _stream())
    _lib.call("stz_sgd_momentum", _ptr(w2), _ptr(v2), _ptr(gr), n, 0.05, 0.9, 1.0 / 384,
              _stream())
    qa, qb = torch.zeros_like(pa), torch.zeros_like(pb)
    for q, off in ((qa, off1), (qb, off2)):
        _lib.call("stzx_pack_rows", _ptr(w2[off:]), _ptr(q), q[0].numel(), rows, D, D8,
                  _stream())
    torch.cuda.synchronize()
    assert torch.equal(w, w2) and torch.equal(v, v2)
    assert torch.equal(pa.view(torch.int16), qa.view(torch.int16))
    assert torch.equal(pb.view(torch.int16), qb.view(torch.int16))


def test_sgd_pack_rejects_bad_ranges(lib):
    from paper_1812_10624_b200 import _lib
    from paper_1812_10624_b200.tensor_core import ShapeMismatch
    w = torch.zeros(1024, device="cuda")
    p = torch.zeros((3, 10, 8), dtype=torch.bfloat16, device="cuda")
    for bad in [(2, 80, p.data_ptr(), 80, 8, 8),        # offset not 16-byte aligned
                (0, 84, p.data_ptr(), 80, 8, 8),        # not whole rows
                (1000, 80, p.data_ptr(), 80, 8, 8)]:    # past the end
        with pytest.raises(ShapeMismatch):
            _lib.call("stz_sgd_momentum_pack", _ptr(w), _ptr(w), _ptr(w), 1024, 0.1, 0.9, 1.0,
                      _lib.range_array([bad]), 1, _stream())


def test_allreduce_sgd_single_member(lib):
    """nranks == 1: the update of the member's own gradient, no barrier."""
    from paper_1812_10624_b200 import _lib
    g = torch.Generator().manual_seed(5)
    n = 4099
    w = torch.randn(n, generator=g).cuda()
    v = torch.randn(n, generator=g).cuda()
    gr = torch.randn(n, generator=g).cuda()
    w2, v2 = w.clone(), v.clone()
    flags = torch.zeros(_lib.PEER_FLAG_WORDS, dtype=torch.int32, device="cuda")
    ra = _lib.range_array([])
    _lib.call("stz_allreduce_sgd", _lib.ptr_array([gr.data_ptr()]),
              _lib.ptr_array([gr.data_ptr()]), _lib.ptr_array([flags.data_ptr()]), 1, 0,
              _ptr(w), _ptr(v), n, 0.05, 0.9, 0.25, ra, 0, _stream())
    _lib.call("stz_sgd_momentum", _ptr(w2), _ptr(v2), _ptr(gr), n, 0.05, 0.9, 0.25, _stream())
    torch.cuda.synchronize()
    assert torch.equal(w, w2) and torch.equal(v, v2)


def test_ipc_handle_offset(lib):
    """The handle names the allocation; the offset locates the tensor in it."""
    import ctypes
    from paper_1812_10624_b200 import _lib
    base = torch.zeros(1 << 20, device="cuda")
    view = base[4096:]
    h = ctypes.create_string_buffer(_lib.IPC_HANDLE_BYTES)
    off0, off1 = ctypes.c_size_t(), ctypes.c_size_t()
    _lib.call("stz_ipc_handle", _ptr(base), h, ctypes.byref(off0))
    h0 = bytes(h.raw)
    _lib.call("stz_ipc_handle", _ptr(view), h, ctypes.byref(off1))
    assert bytes(h.raw) == h0
    assert off1.value - off0.value == 4096 * 4


def _torchrun(nproc, *args, timeout=600):
    env = dict(os.environ, PYTHONPATH=ROOT)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1",
           f"--master-port={29600 + nproc + 7 * len(args)}",
           os.path.join(ROOT, "tools", "peer_check.py"), *args]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env)
    text = out.stdout + out.stderr
    assert out.returncode == 0, text[-3000:]
    assert "PASS" in text, text[-3000:]


@pytest.mark.parametrize("members", [2, 3])
def test_peer_exchange_processes_on_one_gpu(lib, members):
    """R processes on cuda:0: IPC-mapped buffers, the flag barrier and the
    reduce-push across process boundaries; bit-exact vs numpy."""
    _torchrun(members, "--same-gpu", "--numel", "300007", "--iters", "3")


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs 2 GPUs")
def test_peer_exchange_over_nvlink(lib):
    n = torch.cuda.device_count()
    _torchrun(min(n, 8), "--numel", "2000003", "--iters", "4")
