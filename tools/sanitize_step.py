"""Small steps for compute-sanitizer (tools/sanitize.sh): every kernel family
of the layer-separated step once, at tiny shapes, co-located on cuda:0.

    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_step.py [model]

model: tiny_cnn (conv / pool / FC / softmax / SGD), tiny_resnet (BatchNorm,
residual, global pool), tiny_inception (rectangular convs, average pool,
concat) or alexnet (AlexNet layer shapes at K=2: space-to-depth conv1, band
conv, TMA im2col and CTA-pair GEMMs, split-K reduces).  Two iterations,
checked against the oracle so a sanitizer-clean run is also a correct one."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import torch  # noqa: E402

import stanza_oracle as orc  # noqa: E402
from paper_1812_10624_b200 import model_partition as mp  # noqa: E402
from paper_1812_10624_b200.stanza_runtime import StanzaCluster  # noqa: E402
from paper_1812_10624_b200.tensor_core import as_tuple  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "tiny_cnn"
spec = {"tiny_cnn": mp.tiny_cnn(), "tiny_resnet": mp.tiny_resnet(),
        "tiny_inception": mp.tiny_inception(batch_k=2), "alexnet": mp.alexnet(batch_k=2)}[name]
classes = spec.layers[-2].out_dim
mk = orc.batch_fn(spec.input_shape, spec.batch_k, 7, classes=classes)
nc, nf = (1, 1) if name == "alexnet" else (2, 1)
res = StanzaCluster(spec, n_conv=nc, n_fc=nf, batch_fn=mk, lr=0.01, momentum=0.9, seed=3,
                    device="cuda:0", graphs=False).train(2)
torch.cuda.synchronize()
ref_p, _, ref_l = orc.layer_separated_train([as_tuple(l) for l in spec.layers], spec.batch_k,
                                            nc, nf, 2, 3, mk, lr=0.01)
dev = orc.max_param_dev(res.state.params, ref_p)
print(f"sanitize_step {name} {nc}:{nf}: max_param_dev {dev:.2e} losses {res.losses}", flush=True)
