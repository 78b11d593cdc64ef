"""One AlexNet (K=128) co-located layer-separated step for ncu: 2 warm-up
steps, then exactly one more step (the one to profile), inside the NVTX
range "step"."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1812_10624_b200 import _lib
from paper_1812_10624_b200.model_partition import builtin_model
from paper_1812_10624_b200.stanza_runtime import StanzaCluster
model = sys.argv[1] if len(sys.argv) > 1 else "alexnet_exec"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 128
_lib.load()
spec = builtin_model(model, k)
cl = StanzaCluster(spec, n_conv=1, n_fc=1, batch_fn=None, lr=0.01, seed=3, device="cuda:0")
x = torch.randn(cl.x.shape, device="cuda:0")
y = torch.randint(0, 1000, cl.labels.shape, device="cuda:0", dtype=torch.int32)
# the bench's measured tile overrides (off with STZ_AUTOTUNE=0)
if os.environ.get("STZ_AUTOTUNE", "1") != "0":
    print("tile overrides:", _lib.autotune_tiles(lambda: cl.step(x=x, labels=y)))
for _ in range(2):
    cl.step(x=x, labels=y)
torch.cuda.synchronize()
n0 = _lib.load().stz_launch_count()
torch.cuda.nvtx.range_push("step")   # ncu --nvtx --nvtx-include "step/" isolates it
cl.step(x=x, labels=y)
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("launches per step:", _lib.load().stz_launch_count() - n0)
