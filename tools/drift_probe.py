"""Parameter drift vs the oracle over training iterations, per GEMM core."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np, torch
import stanza_oracle as orc
from paper_1812_10624_b200 import _lib, tiny_cnn
from paper_1812_10624_b200.stanza_runtime import StanzaCluster
from paper_1812_10624_b200.tensor_core import as_tuple
lib = _lib.load()
spec = tiny_cnn()
layers = [as_tuple(l) for l in spec.layers]
for nc in (4, 8):
    mk = orc.batch_fn(spec.input_shape, spec.batch_k, 7)
    # oracle trajectory checkpoints
    refs, st = [], None
    for c in range(5):
        p, v, _ = orc.layer_separated_train(layers, spec.batch_k, nc, 1, 10, 3, mk, state=st,
                                            start_iteration=10 * c) if False else (None, None, None)
    ref_states = []
    params = orc.seeded_init(layers, 3); vel = [[np.zeros_like(t) for t in l] for l in params]
    for c in range(5):
        params, vel, _ = orc.layer_separated_train(layers, spec.batch_k, nc, 1, 10, 3, mk,
                                                   state=(params, vel), start_iteration=10 * c)
        ref_states.append(params)
    for impl in (0, 2, 1):
        lib.stz_set_gemm_impl(impl)
        cl = StanzaCluster(spec, n_conv=nc, n_fc=1, batch_fn=mk, lr=0.05, seed=3, device="cuda:0")
        devs = []
        for c in range(5):
            r = cl.train(10)
            devs.append(orc.max_param_dev(r.state.params, ref_states[c]))
        print(f"n_conv={nc} impl={impl}: " + " ".join(f"{d:.2e}" for d in devs), flush=True)
lib.stz_set_gemm_impl(0)
