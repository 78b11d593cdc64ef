"""Debug: which gradient tensors of ResNet-50 @64x64 K=2 go non-finite."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import torch, numpy as np
import stanza_oracle as orc
from paper_1812_10624_b200.model_partition import resnet
from paper_1812_10624_b200.stanza_runtime import StanzaCluster
side = int(sys.argv[1]) if len(sys.argv) > 1 else 64
k = int(sys.argv[2]) if len(sys.argv) > 2 else 2
spec = resnet(batch_k=k, side=side)
mk = orc.batch_fn(spec.input_shape, k, 7, classes=1000)
cl = StanzaCluster(spec, n_conv=1, n_fc=1, batch_fn=mk, lr=0.005, seed=3, device="cuda:0")
for it in range(1):
    cl.load_batch(it)
    cl.step()
    torch.cuda.synchronize()
    eng = cl.conv
    bad = []
    def walk(e, pre):
        for li, row in enumerate(e.grads):
            for ti, t in enumerate(row):
                if not torch.isfinite(t).all():
                    bad.append(f"{pre}{li}.{ti}")
        for i, op in enumerate(e.ops):
            if e.acts[i] is not None and not torch.isfinite(e.acts[i].to_float()).all():
                bad.append(f"{pre}act{i}:{op.kind}")
            if e.gin[i] is not None and not torch.isfinite(e.gin[i].to_float()).all():
                bad.append(f"{pre}gin{i}:{op.kind}")
            if i in e.bnstats and not torch.isfinite(e.bnstats[i]).all():
                bad.append(f"{pre}stats{i}")
        for i, kids in e.children.items():
            for kk, nm in zip(kids, "bs"):
                if kk is not None:
                    walk(kk, f"{pre}r{i}{nm}.")
    walk(eng, "")
    print("iter", it, "nonfinite acts/gin/stats:", [b for b in bad if ":" in b or "stats" in b][:60], flush=True)
    print("gboundary finite", bool(torch.isfinite(cl.gboundary.to_float()).all()),
          "fc grads finite", bool(torch.isfinite(cl.fcs[0].grad_flat).all()))
    print("stem stats", cl.conv.bnstats[1][0, :4].tolist())
