"""One process per role: StanzaCluster across processes vs the oracle.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        tools/dist_parity.py --n-conv C --n-fc F [--model tiny_cnn] [--iters 8]
        [--micro M] [--exchange peer|nccl] [--same-gpu] [--checkpoint]
        [--missing conv|fc] [--batch-k K]

Each rank is one CONV or FC worker (rank < C: CONV).  ``--same-gpu`` puts
every rank on cuda:0 with gloo for the host plumbing (the peer-memory link
and exchange still run between the processes through CUDA IPC), so the
multi-process step is exercised on a 1-GPU box; otherwise rank r uses
cuda:r over NCCL.  Rank 0 checks against oracle/stanza_oracle.py's
layer_separated_train (the reference's StanzaCluster restated, pinned to the
reference's own outputs) with the reference's bars
(tests/test_stanza_runtime.py:53-83, test_acceptance.py:76-102):
max_param_dev <= 1e-5 on parameters, velocities within 1e-5 of the largest
velocity (per-tensor deviations are reported), losses within 1e-5
relative, every CONV (and FC) replica bit-identical, and the ledger phase
sequence.  ``--checkpoint``: train half, checkpoint() (FC replica to a
CONV worker's GPU), lose the FC state, restore_fc_replica(), train the rest
-- the final state must have the uninterrupted run's param_digest.
``--missing conv|fc``: that role never runs its step; the other side's
train() must raise MissingSource within net.default_timeout.
Prints one JSON line and PASS/FAIL."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import stanza_oracle as orc  # noqa: E402
from paper_1812_10624_b200 import _lib, model_partition as mp  # noqa: E402
from paper_1812_10624_b200.checkpointing import param_digest  # noqa: E402
from paper_1812_10624_b200.comm import RoleComm  # noqa: E402
from paper_1812_10624_b200.stanza_runtime import MissingSource, StanzaCluster  # noqa: E402
from paper_1812_10624_b200.tensor_core import as_tuple  # noqa: E402
from paper_1812_10624_b200.transport import NetConfig  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n-conv", type=int, required=True)
ap.add_argument("--n-fc", type=int, required=True)
ap.add_argument("--model", default="tiny_cnn")
ap.add_argument("--batch-k", type=int, default=None)
ap.add_argument("--iters", type=int, default=8)
ap.add_argument("--micro", default=None, help="micro-batch counts, comma-separated")
ap.add_argument("--exchange", default=None)
ap.add_argument("--same-gpu", action="store_true")
ap.add_argument("--checkpoint", action="store_true")
ap.add_argument("--missing", choices=["conv", "fc"], default=None)
ap.add_argument("--seed", type=int, default=5)
ap.add_argument("--data-seed", type=int, default=11)
ap.add_argument("--tol", type=float, default=1e-5)
args = ap.parse_args()

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = 0 if args.same_gpu else int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
if args.same_gpu:
    dist.init_process_group("gloo")
else:
    dist.init_process_group("cpu:gloo,cuda:nccl", device_id=dev)
_lib.load()
spec = mp.builtin_model(args.model, args.batch_k)
classes = spec.layers[-2].out_dim
comm = RoleComm(args.n_conv, args.n_fc)
mk = orc.batch_fn(spec.input_shape, spec.batch_k, args.data_seed, classes=classes)
net = NetConfig(default_timeout=3.0 if args.missing else 60.0)


MICROS = [None] if args.micro is None else [int(m) for m in args.micro.split(",")]
MICRO = MICROS[0]


def cluster(**kw):
    return StanzaCluster(spec, n_conv=args.n_conv, n_fc=args.n_fc, batch_fn=mk, lr=0.05,
                         momentum=0.9, seed=args.seed, device=dev, comm=comm,
                         micro_batches=MICRO, exchange=args.exchange, net=net, **kw)


def replicas_identical(cl) -> bool:
    """Every CONV replica equals CONV 0's and every FC replica FC 0's, bit for bit."""
    ok = torch.ones(1)
    for eng, ranks in ((cl.conv, comm.conv_ranks), (cl.fcs[0] if cl.fcs else None, comm.fc_ranks)):
        for flat in ((eng.params_flat, eng.vel_flat) if eng is not None else ()):
            mine = flat.cpu()
            objs = [None] * len(ranks)
            grp = comm.conv_group if eng is cl.conv else comm.fc_group
            if grp is None:
                continue
            dist.all_gather_object(objs, mine.numpy().tobytes(), group=grp)
            ok[0] = min(float(ok[0]), float(all(o == objs[0] for o in objs)))
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    return bool(ok.item() == 1.0)


t0 = time.time()
if args.missing:
    cl = cluster()
    absent = (comm.is_conv and args.missing == "conv") or (not comm.is_conv and args.missing == "fc")
    raised = None
    if not absent:
        try:
            cl.train(1)
        except MissingSource as e:
            raised = str(e)
    flag = torch.tensor([1.0 if (absent or raised) else 0.0])
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    msgs = [None] * world
    dist.all_gather_object(msgs, raised)
    if rank == 0:
        ok = flag.item() == 1.0
        print(json.dumps({"check": "missing_source", "absent": args.missing,
                          "n_conv": args.n_conv, "n_fc": args.n_fc, "raised": msgs,
                          "seconds": round(time.time() - t0, 1)}), flush=True)
        print(f"{'PASS' if ok else 'FAIL'} missing-source {args.missing} absent at "
              f"{args.n_conv}:{args.n_fc}", flush=True)
    dist.barrier()
    sys.exit(0)

reference = None
all_ok = True
for MICRO in MICROS:
    whole_digest = None
    if args.checkpoint:                              # the uninterrupted run first
        ref_cl = cluster()
        w = ref_cl.train(args.iters)
        whole_digest = param_digest(w.state.params) if w.state is not None else None
        ref_cl.close()
    cl = cluster()
    if args.checkpoint:
        half = args.iters // 2
        r1 = cl.train(half)
        cl.checkpoint()
        if cl.fcs:                                   # the FC workers lose their state
            cl.fcs[0].params_flat.zero_()
            cl.fcs[0].vel_flat.fill_(1.0)
            cl.fcs[0].pack_weights()
        it = cl.restore_fc_replica()
        res = cl.train(args.iters - half)
        losses = r1.losses + res.losses
        blob_ok = None
        if cl.replica_snapshots:
            from paper_1812_10624_b200.checkpointing import state_from_bytes
            rep = state_from_bytes(next(iter(cl.replica_snapshots.values())))
            blob_ok = rep.iteration == it == half
        blobs = [None] * world
        dist.all_gather_object(blobs, blob_ok)
    else:
        res = cl.train(args.iters)
        losses = res.losses
    rep_ok = replicas_identical(cl)
    labels = [p.label for p in cl.transport.ledger.phases]
    if rank == 0:
        if reference is None:
            layers = [as_tuple(l) for l in spec.layers]
            reference = orc.layer_separated_train(layers, spec.batch_k, args.n_conv, args.n_fc,
                                                  args.iters, args.seed, mk)
        rp, rv, rl = reference
        dev_p = orc.max_param_dev(res.state.params, rp)
        dev_v = orc.max_param_dev(res.state.velocities, rv)
        vmax = max(float(np.abs(t).max()) for row in rv for t in row)
        worst_v = sorted(((orc.rel_err(a, b), li, ti, float(np.abs(b).max()),
                           float(np.abs(np.asarray(a, np.float64) - b).max()))
                          for li, (ra, rb) in enumerate(zip(res.state.velocities, rv))
                          for ti, (a, b) in enumerate(zip(ra, rb))), reverse=True)[:3]
        dl = max(abs(a - b) / abs(b) for a, b in zip(losses, rl))
        want = ["conv_compute", "activations", "fc_compute", "boundary", "exchange", "update"]
        if args.checkpoint:
            half = args.iters // 2
            want_labels = want * half + ["checkpoint"] + want * (args.iters - half)
        else:
            want_labels = want * args.iters
        # velocities against the largest one (per-tensor ratios of small
        # velocities compare rounding noise with noise; reported below)
        vdev_abs = max(float(np.abs(np.asarray(a, np.float64) - b).max())
                       for ra, rb in zip(res.state.velocities, rv) for a, b in zip(ra, rb))
        ok = dev_p <= args.tol and vdev_abs <= args.tol * vmax and dl <= args.tol and rep_ok \
            and labels == want_labels
        line = {"check": "dist_parity", "n_conv": args.n_conv, "n_fc": args.n_fc,
                "model": args.model, "batch_k": spec.batch_k, "iters": args.iters,
                "micro": cl.micro, "exchange": cl.exchange,
                "transport": "gloo+peer (one GPU)" if args.same_gpu else
                f"{dist.get_backend()} ({world} GPUs)",
                "max_param_dev": dev_p, "max_velocity_dev": dev_v,
                "velocity_dev_global": vdev_abs / vmax if vmax else None, "loss_rel": dl,
                "replicas_identical": rep_ok, "ledger_phases_ok": labels == want_labels,
                "worst_velocity_tensors": [[round(w[0], 9), w[1], w[2], w[3], w[4]]
                                           for w in worst_v], "max_velocity": vmax,
                "seconds": round(time.time() - t0, 1)}
        if args.checkpoint:
            line["replica_blob_ok"] = any(b for b in blobs if b is not None)
            line["digest_equals_uninterrupted"] = param_digest(res.state.params) == whole_digest
            ok = ok and line["replica_blob_ok"] and line["digest_equals_uninterrupted"]
        all_ok = all_ok and ok
        print(json.dumps(line), flush=True)
        print(f"{'PASS' if ok else 'FAIL'} dist {args.n_conv}:{args.n_fc} {args.model} "
              f"K={spec.batch_k} iters={args.iters} micro={cl.micro} exchange={cl.exchange} "
              f"max_param_dev={dev_p:.2e} max_vel_dev={dev_v:.2e} loss_rel={dl:.2e} "
              f"replicas_identical={rep_ok}", flush=True)
    cl.close()
dist.barrier()
dist.destroy_process_group()
sys.exit(0 if all_ok else 1)
