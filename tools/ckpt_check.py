"""One process per GPU: the FC checkpoint replica over NVLink and FC
recovery (StanzaCluster.checkpoint / restore_fc_replica) vs an uninterrupted
run.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        tools/ckpt_check.py <n_conv> <n_fc> [model] [iters_before] [iters_after]

Run A trains before+after iterations.  Run B trains `before`, checkpoints
(FC worker 0's w, v land on a seeded-random CONV worker's GPU), loses every
FC worker's state (zeroed), restores it from the replica, and trains `after`
more.  Rank 0 prints PASS when both runs end with the same param_digest and
the holder's STZC blob matches the snapshot's FC block."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import torch, torch.distributed as dist
import stanza_oracle as orc
from paper_1812_10624_b200 import _lib, model_partition as mp
from paper_1812_10624_b200.checkpointing import param_digest, state_from_bytes
from paper_1812_10624_b200.comm import RoleComm
from paper_1812_10624_b200.stanza_runtime import StanzaCluster

n_conv, n_fc = int(sys.argv[1]), int(sys.argv[2])
model = sys.argv[3] if len(sys.argv) > 3 else "tiny_cnn"
before = int(sys.argv[4]) if len(sys.argv) > 4 else 3
after = int(sys.argv[5]) if len(sys.argv) > 5 else 3
local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
_lib.load()
spec = mp.builtin_model(model)
comm = RoleComm(n_conv, n_fc)
mk = orc.batch_fn(spec.input_shape, spec.batch_k, 11)
mkc = lambda: StanzaCluster(spec, n_conv=n_conv, n_fc=n_fc, batch_fn=mk, lr=0.05,  # noqa: E731
                            momentum=0.9, seed=5, device=dev, comm=comm)
whole = mkc().train(before + after)
cl = mkc()
cl.train(before)
snap = cl.checkpoint()
blob_ok = torch.ones(1, device=dev)
cut = cl.partition.split_index
blobs = [None] * dist.get_world_size()
dist.all_gather_object(blobs, cl.replica_snapshots.get(cl.conv_ids[cl._replica_holder]))
if cl.fcs:
    cl.fcs[0].params_flat.zero_()
    cl.fcs[0].vel_flat.zero_()
    cl.fcs[0].pack_weights()
it = cl.restore_fc_replica()
res = cl.train(after)
if dist.get_rank() == 0:
    held = [b for b in blobs if b is not None]
    rep = state_from_bytes(held[0]) if len(held) == 1 else None
    ok_blob = rep is not None and rep.iteration == before and \
        param_digest(rep.params) == param_digest(snap.params[cut:])
    ok = ok_blob and it == before and \
        param_digest(res.state.params) == param_digest(whole.state.params)
    print(f"{'PASS' if ok else 'FAIL'} ckpt {n_conv}:{n_fc} {model} holder=conv{cl._replica_holder} "
          f"blob_ok={ok_blob} resumed_equal="
          f"{param_digest(res.state.params) == param_digest(whole.state.params)}", flush=True)
dist.barrier()
dist.destroy_process_group()
