"""Per-tensor deviation of the tiny Inception (BN-free) step vs the oracle:
prints the worst parameter / velocity tensors with their layer and shape
(debugging aid for tests/test_gpu_inception.py)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

import stanza_oracle as orc  # noqa: E402
from paper_1812_10624_b200.model_partition import tiny_inception  # noqa: E402
from paper_1812_10624_b200.stanza_runtime import StanzaCluster  # noqa: E402
from paper_1812_10624_b200.tensor_core import as_tuple, param_shapes  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 1
nc = int(sys.argv[2]) if len(sys.argv) > 2 else 1
spec = tiny_inception(batch_k=4, bn=False)
mk = orc.batch_fn(spec.input_shape, 4, 7, classes=10)
res = StanzaCluster(spec, n_conv=nc, n_fc=1, batch_fn=mk, lr=0.05, momentum=0.9, seed=3,
                    device="cuda:0").train(iters)
torch.cuda.synchronize()
rp, rv, rl = orc.layer_separated_train([as_tuple(l) for l in spec.layers], 4, nc, 1, iters, 3, mk,
                                       lr=0.05)
print("losses", res.losses, rl)
for what, got, ref in (("param", res.state.params, rp), ("velocity", res.state.velocities, rv)):
    rows = []
    for li, (ra, rb) in enumerate(zip(got, ref)):
        shapes = param_shapes(spec.layers[li])
        for ti, (a, b) in enumerate(zip(ra, rb)):
            rows.append((orc.rel_err(a, b), li, ti, shapes[ti], float(np.abs(b).max()),
                         float(np.abs(np.asarray(a, np.float64) - b).max())))
    rows.sort(reverse=True)
    print(what, "worst:")
    for r in rows[:12]:
        print("  rel %.3e layer %d tensor %d shape %s max|ref| %.3e max|diff| %.3e" % r)
