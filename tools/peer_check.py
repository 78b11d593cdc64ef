"""Fused exchange + update over peer memory (stz_allreduce_sgd) vs its CPU
restatement, one process per member.

    python -m torch.distributed.run --nproc-per-node R --master-addr 127.0.0.1 \
        tools/peer_check.py [--same-gpu] [--numel N] [--iters I]

Each member draws a seeded gradient vector per iteration; the group runs
PeerExchange.run (barrier -> reduce-push -> barrier -> SGD + split-plane
repack).  Rank 0 checks, bit-exactly, every member's (w, v) against numpy:
the gradient sum in group-rank order (fp32 RN left fold), then the
reference's momentum step (tensor_core.py:366-388), and the repacked planes
against the split of w.  --same-gpu puts every member on cuda:0 (gloo for the
host plumbing), so the IPC mapping and the barrier are exercised on a 1-GPU
box; otherwise member r uses cuda:r over NCCL.  Prints PASS/FAIL."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1812_10624_b200 import _lib  # noqa: E402
from paper_1812_10624_b200.comm import PeerExchange  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--same-gpu", action="store_true")
ap.add_argument("--numel", type=int, default=1_000_003)
ap.add_argument("--iters", type=int, default=3)
args = ap.parse_args()

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = 0 if args.same_gpu else int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("gloo" if args.same_gpu else "nccl",
                        **({} if args.same_gpu else {"device_id": dev}))
_lib.load()
_lib.call("stz_set_peer_timeout_ms", 120000)

D = 1000                     # FC-like row-major slice [rows][D], D % 8 == 0
rows = 300
N = max(args.numel, rows * D + 4096)
OFF = 1024                   # the packed slice starts 4 KB in (16-byte aligned)
LR, MU, NB = 0.05, 0.9, 384


class FlatBlock:
    """The BlockEngine surface PeerExchange uses: flat (w, v, g) + one
    row-major plane slice."""

    def __init__(self):
        g = torch.Generator().manual_seed(1234)
        self.device, self.total = dev, N
        self.params_flat = torch.randn(N, generator=g).to(dev)
        self.vel_flat = (0.1 * torch.randn(N, generator=g)).to(dev)
        self.grad_flat = torch.zeros(N, device=dev)
        self.planes = torch.zeros((3, rows, D), dtype=torch.bfloat16, device=dev)
        self._r = _lib.range_array([(OFF, rows * D, self.planes.data_ptr(),
                                     self.planes[0].numel(), D, D)])

    tag = ""

    def fused_pack_ranges(self):
        return self._r, 1, frozenset()

    def fused_param_count(self):
        return rows * D

    def pack_weights(self, skip=frozenset()):
        pass


def grads_of(it, r):
    return np.random.default_rng([77, it, r]).standard_normal(N).astype(np.float32)


def split3(x):
    """The split-plane format: P0 = rn_bf16(x), P1 = rn_bf16(x-P0), P2 = rest."""
    t = torch.from_numpy(x)
    p0 = t.to(torch.bfloat16)
    r0 = t - p0.float()
    p1 = r0.to(torch.bfloat16)
    p2 = (r0 - p1.float()).to(torch.bfloat16)
    return [p.view(torch.int16).numpy() for p in (p0, p1, p2)]


blk = FlatBlock()
w0 = blk.params_flat.cpu().numpy().copy()
v0 = blk.vel_flat.cpu().numpy().copy()
px = PeerExchange(blk, None, rank, world)
for it in range(args.iters):
    blk.grad_flat.copy_(torch.from_numpy(grads_of(it, rank)))
    px.run(NB, LR, MU)
torch.cuda.synchronize(dev)
w = blk.params_flat.cpu().numpy()
v = blk.vel_flat.cpu().numpy()
pl = blk.planes.view(torch.int16).cpu().numpy()
mine = [w, v, pl]
objs = [None] * world
dist.all_gather_object(objs, mine)
if rank == 0:
    f32 = np.float32
    lr, mu, inv = f32(LR), f32(MU), f32(1.0) / f32(NB)
    we, ve = w0.copy(), v0.copy()
    for it in range(args.iters):
        g = grads_of(it, 0)
        for r in range(1, world):
            g = (g + grads_of(it, r)).astype(f32)
        ve = (ve * mu).astype(f32) + (g * inv).astype(f32)
        we = (we - (lr * ve).astype(f32)).astype(f32)
    exp_pl = np.stack([p.reshape(rows, D) for p in split3(we[OFF:OFF + rows * D])])
    bad = []
    for r, (wr, vr, plr) in enumerate(objs):
        if not np.array_equal(wr, we):
            bad.append(f"w[{r}] maxdiff {np.abs(wr - we).max():.3e}")
        if not np.array_equal(vr, ve):
            bad.append(f"v[{r}] maxdiff {np.abs(vr - ve).max():.3e}")
        if not np.array_equal(plr, exp_pl):
            bad.append(f"planes[{r}] {int((plr != exp_pl).sum())} differ")
    print(("PASS" if not bad else "FAIL " + "; ".join(bad)) +
          f" peer exchange R={world} n={N} iters={args.iters} same_gpu={args.same_gpu}",
          flush=True)
dist.barrier()
px.close()
dist.destroy_process_group()
