"""One process per GPU: StanzaCluster over NCCL vs the oracle.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        tools/dist_parity.py <n_conv> <n_fc> [model] [iters] [micro_batches]
Rank 0 prints PASS/FAIL with max_param_dev against the reference algorithm
and checks that every CONV replica is bit-identical."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np, torch, torch.distributed as dist
import stanza_oracle as orc
from paper_1812_10624_b200 import _lib, model_partition as mp
from paper_1812_10624_b200.comm import RoleComm
from paper_1812_10624_b200.stanza_runtime import StanzaCluster
from paper_1812_10624_b200.tensor_core import as_tuple

n_conv, n_fc = int(sys.argv[1]), int(sys.argv[2])
model = sys.argv[3] if len(sys.argv) > 3 else "tiny_cnn"
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 8
micro = int(sys.argv[5]) if len(sys.argv) > 5 else None
exchange = sys.argv[6] if len(sys.argv) > 6 else None   # "peer" (default on NCCL) | "nccl"
local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
_lib.load()
spec = mp.builtin_model(model)
comm = RoleComm(n_conv, n_fc)
mk = orc.batch_fn(spec.input_shape, spec.batch_k, 11)
cl = StanzaCluster(spec, n_conv=n_conv, n_fc=n_fc, batch_fn=mk, lr=0.05, momentum=0.9,
                   seed=5, device=dev, comm=comm, micro_batches=micro,
                   exchange=exchange)
res = cl.train(iters)
# replica identity across CONV ranks (reference test_stanza_runtime.py:70-83)
ok_rep = torch.ones(1, device=dev)
if cl.conv is not None:
    mine = cl.conv.params_flat.clone()
    ref = mine.clone()
    if comm.conv_group is not None:
        dist.broadcast(ref, src=0, group=comm.conv_group)
    ok_rep[0] = float(torch.equal(mine, ref))
if cl.fcs and comm.fc_group is not None:     # FC replicas too when n_fc > 1
    mine = cl.fcs[0].params_flat.clone()
    ref = mine.clone()
    dist.broadcast(ref, src=n_conv, group=comm.fc_group)
    ok_rep[0] = min(float(ok_rep[0]), float(torch.equal(mine, ref)))
dist.all_reduce(ok_rep, op=dist.ReduceOp.MIN)
if dist.get_rank() == 0:
    layers = [as_tuple(l) for l in spec.layers]
    rp, rv, rl = orc.layer_separated_train(layers, spec.batch_k, n_conv, n_fc, iters, 5, mk)
    dev_p = orc.max_param_dev(res.state.params, rp)
    dl = max(abs(a - b) / abs(b) for a, b in zip(res.losses, rl))
    ok = dev_p <= 1e-5 and dl <= 1e-5 and ok_rep.item() == 1.0
    print(f"{'PASS' if ok else 'FAIL'} dist {n_conv}:{n_fc} {model} iters={iters} micro={cl.micro} "
          f"exchange={cl.exchange} "
          f"max_param_dev={dev_p:.2e} loss_rel={dl:.2e} replicas_identical={bool(ok_rep.item())}",
          flush=True)
dist.barrier()
dist.destroy_process_group()
