"""The one-process-per-GPU deployment against the oracle (tools/dist_parity.py).

Every rank is a separate process.  On a 1-GPU box they all share cuda:0
(gloo carries the one-time handle exchange; the CONV<->FC link and the
gradient exchange run between the processes as peer-memory kernels through
CUDA IPC -- the same kernels as between GPUs); with >= N GPUs each rank gets
its own GPU over NCCL + NVLink.  Bars: the reference's
(tests/test_stanza_runtime.py:53-83, test_acceptance.py:76-102):
max_param_dev <= 1e-5 for parameters and velocities after N iterations,
losses within 1e-5, every CONV / FC replica bit-identical, the reference's
phase sequence on the ledger.  Covered: 1:1, 3:1, 2:2, 7:1, 6:2 (BASELINE's
splits) with 1, 2 and 4 micro-batches, AlexNet at parity K = 2 with 2
micro-batches, the checkpoint -> FC-replica restore round trip, and
MissingSource when a peer never delivers."""

import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LOG = os.path.join(ROOT, "gpurun_out", "dist_parity.log")
_PORT = [29700]


def _run(nproc, *args, same_gpu=True, timeout=900):
    _PORT[0] += 1
    env = dict(os.environ, PYTHONPATH=ROOT, OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1", f"--master-port={_PORT[0]}",
           os.path.join(ROOT, "tools", "dist_parity.py"), *args]
    if same_gpu:
        cmd.append("--same-gpu")
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env)
    text = out.stdout + out.stderr
    os.makedirs(os.path.dirname(LOG), exist_ok=True)
    with open(LOG, "a") as fh:
        fh.write(f"$ {' '.join(cmd[2:])}\n")
        fh.write("".join(l + "\n" for l in out.stdout.splitlines()
                         if l.startswith(("{", "PASS", "FAIL"))))
    assert out.returncode == 0, text[-4000:]
    assert "PASS" in text and "FAIL" not in text, text[-4000:]
    return text


@pytest.mark.parametrize("nc,nf", [(1, 1), (3, 1), (2, 2)])
def test_tiny_micro_batches(lib, nc, nf):
    """tiny_cnn (K=4), 8 iterations, micro-batches 1, 2 and 4."""
    _run(nc + nf, "--n-conv", str(nc), "--n-fc", str(nf), "--iters", "8", "--micro", "1,2,4")


@pytest.mark.parametrize("nc,nf", [(7, 1), (6, 2)])
def test_eight_process_role_maps(lib, nc, nf):
    """The 8-GPU splits (7 CONV : 1 FC, 6 : 2 with the FC-group exchange)
    as 8 processes: R = 7 and R = 6 peer exchanges, fan-in 7 / 3 gathers."""
    _run(nc + nf, "--n-conv", str(nc), "--n-fc", str(nf), "--iters", "6", "--micro", "2")


def test_tiny32_fifty_iterations(lib):
    """BASELINE config 1 (tiny_cnn32, 2 CONV : 1 FC) for 50 iterations."""
    _run(3, "--n-conv", "2", "--n-fc", "1", "--model", "tiny_cnn32", "--iters", "50",
         "--seed", "3", "--data-seed", "7", "--micro", "1,2")


@pytest.mark.parametrize("nc,nf", [(1, 1), (3, 1)])
def test_alexnet_parity_batch(lib, nc, nf):
    """AlexNet layer shapes at parity K = 2 with 2 micro-batches (the
    benchmarked pipelined path), 3 iterations."""
    _run(nc + nf, "--n-conv", str(nc), "--n-fc", str(nf), "--model", "alexnet_exec",
         "--batch-k", "2", "--iters", "3", "--micro", "2", "--seed", "3", "--data-seed", "7")


@pytest.mark.parametrize("nc,nf", [(3, 1), (2, 2)])
def test_checkpoint_replica_round_trip(lib, nc, nf):
    """checkpoint() replicates FC worker 0's (w, v) to a CONV worker's GPU;
    the FC state is lost and restore_fc_replica() brings it back; the run
    ends with the uninterrupted run's param_digest (stanza_runtime.py
    :182-211, checkpointing.py:44-65)."""
    _run(nc + nf, "--n-conv", str(nc), "--n-fc", str(nf), "--iters", "6", "--micro", "2",
         "--checkpoint")


@pytest.mark.parametrize("absent", ["conv", "fc"])
def test_missing_source(lib, absent):
    """A peer that never delivers: the waiting side's train() raises
    MissingSource after net.default_timeout (stanza_runtime.py:37-38, :77-82,
    :295-299) instead of hanging."""
    _run(2, "--n-conv", "1", "--n-fc", "1", "--missing", absent)


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs 2 GPUs")
def test_over_nvlink_two_gpus(lib):
    _run(2, "--n-conv", "1", "--n-fc", "1", "--iters", "6", "--micro", "1,2", same_gpu=False)
    _run(2, "--n-conv", "1", "--n-fc", "1", "--iters", "6", "--micro", "2",
         "--exchange", "nccl", same_gpu=False)


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 4,
                    reason="needs 4 GPUs")
@pytest.mark.parametrize("nc,nf", [(3, 1), (2, 2)])
def test_over_nvlink_four_gpus(lib, nc, nf):
    _run(4, "--n-conv", str(nc), "--n-fc", str(nf), "--iters", "6", "--micro", "1,2,4",
         same_gpu=False)
    _run(4, "--n-conv", str(nc), "--n-fc", str(nf), "--model", "alexnet_exec", "--batch-k", "2",
         "--iters", "3", "--micro", "2", "--seed", "3", "--data-seed", "7", same_gpu=False)
