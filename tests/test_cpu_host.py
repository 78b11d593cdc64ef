"""Host-side logic on CPU: role map, model cut and grammar, init digests,
engine fusion plan, checkpoint formats -- against the reference's pins."""

import hashlib

import numpy as np
import pytest
import torch

import golden_io
from paper_1812_10624_b200 import model_partition as mp
from paper_1812_10624_b200.checkpointing import (TrainState, deserialize_params,
                                                 param_digest, serialize_params,
                                                 state_from_bytes, state_to_bytes)
from paper_1812_10624_b200.roles import equal_split, gpu_roles, group_rows, plan_groups
from paper_1812_10624_b200.tensor_core import (CorruptCheckpoint, FullyConnected,
                                               ShapeMismatch, seeded_init)


def test_plan_groups_reference_pins():
    """stanza_runtime.py:41-56; test_stanza_runtime.py:26-30."""
    assert plan_groups(4, 2) == [0, 0, 1, 1]
    assert plan_groups(5, 2) == [0, 0, 0, 1, 1]
    assert plan_groups(6, 1) == [0] * 6
    assert plan_groups(3, 3) == [0, 1, 2]
    with pytest.raises(mp.ConfigError):
        plan_groups(2, 3)
    with pytest.raises(mp.ConfigError):
        plan_groups(0, 1)


def test_plan_groups_bit_exact_vs_reference_table():
    for key, expected in golden_io.meta()["plan_groups"].items():
        nc, nf = map(int, key.split("x"))
        assert plan_groups(nc, nf) == expected
        for j in range(nf):
            lo, hi = group_rows(expected, j)
            assert expected[lo:hi] == [j] * (hi - lo)


def test_equal_split_and_roles():
    assert equal_split(7, 3) == [3, 2, 2]
    assert gpu_roles(1) == (1, 1) and gpu_roles(2) == (1, 1)
    assert gpu_roles(4) == (3, 1) and gpu_roles(8) == (7, 1)
    assert gpu_roles(8, fc_workers=2) == (6, 2)


@pytest.mark.parametrize("name,factory", [("alexnet", mp.alexnet), ("vgg16", mp.vgg16),
                                          ("tiny_cnn", mp.tiny_cnn)])
def test_split_counts_match_reference(name, factory):
    ref = golden_io.meta()["specs"][name]
    part = mp.split(factory(1))
    assert part.split_index == ref["split_index"]
    assert part.conv_params == ref["conv_params"]
    assert part.fc_params == ref["fc_params"]
    assert part.boundary_activations == ref["boundary_activations"]


def test_mlp_split_and_errors():
    ref = golden_io.meta()["specs"]["tiny_mlp_b4"]
    part = mp.mlp_split(mp.tiny_mlp(), 4)
    assert (part.conv_params, part.fc_params, part.boundary_activations) == \
        (ref["conv_params"], ref["fc_params"], ref["boundary_activations"])
    with pytest.raises(mp.BadBoundary):
        mp.mlp_split(mp.tiny_mlp(), 7)   # back block has no FC
    with pytest.raises(mp.NoConvBlock):
        mp.split(mp.tiny_mlp())
    prof = mp.split(mp.PROFILES["alexnet"])
    assert prof.split_index is None and prof.conv_params == 2_469_696
    with pytest.raises(mp.NotExecutable):
        _ = prof.conv_block


def test_model_grammar_round_trip():
    text = """name alexnet_exec
    batch_k 128
    input 3 224 224
    layer conv 3 64 11 4 2
    layer relu
    layer maxpool 3 2
    layer conv 64 192 5 1 2
    layer relu
    layer maxpool 3 2
    layer conv 192 384 3 1 1
    layer relu
    layer conv 384 256 3 1 1
    layer relu
    layer conv 256 256 3 1 1
    layer relu
    layer maxpool 3 2
    layer flatten
    layer fc 9216 4096
    layer relu
    layer fc 4096 4096
    layer relu
    layer fc 4096 1000
    layer softmax_ce  # loss head
    """
    spec = mp.parse_model_text(text)
    assert spec.layers == mp.alexnet().layers
    total, _ = mp.count_params(spec)
    assert total == 61_100_840
    for bad in ("name x\nbatch_k 1\nlayer conv 1 2\ninput 1 4 4",
                "batch_k 1\ninput 3\nlayer relu", "name x\nbatch_k 1\nparams_total 10\nlayer relu"):
        with pytest.raises(mp.ConfigError):
            mp.parse_model_text(bad)
    with pytest.raises(ShapeMismatch):
        mp.executable_spec("bad", [FullyConnected(3, 2)], (4,), 1)


@pytest.mark.parametrize("name,factory", [("alexnet", mp.alexnet), ("vgg16", mp.vgg16)])
def test_seeded_init_digest_matches_reference(name, factory):
    params = seeded_init(factory(1).layers, 3)
    h = hashlib.sha256()
    for layer in params:
        for t in layer:
            h.update(np.ascontiguousarray(t, dtype=np.float32).tobytes())
    assert h.hexdigest() == golden_io.meta()["specs"][name]["init_seed3_sha256"]


def test_checkpoint_formats_round_trip():
    g = golden_io.train()["train_tiny_1x1"]
    p, v = golden_io.nested_state(g)
    blob = serialize_params(p)
    back = deserialize_params(blob)
    assert param_digest(back) == param_digest(p)
    st = TrainState(10, p, v)
    again = state_from_bytes(state_to_bytes(st))
    assert again.iteration == 10 and param_digest(again.velocities) == param_digest(v)
    with pytest.raises(CorruptCheckpoint):
        state_from_bytes(state_to_bytes(st)[:-8])
    with pytest.raises(CorruptCheckpoint):
        deserialize_params(b"XXXX" + blob[4:])


def test_engine_fusion_plan_alexnet():
    """The fused plan (CPU tensors: no kernel runs): conv+ReLU fused, ReLU
    backward folded into the consumer's input-gradient kernel, first conv's
    input gradient skipped, FC block boundary gradient unmasked."""
    from paper_1812_10624_b200.engine import BlockEngine
    spec = mp.alexnet(1)
    part = mp.split(spec)
    conv = BlockEngine(part.conv_block, spec.input_shape, 1, "cpu", need_input_grad=False)
    kinds = [(o.kind, o.fused_relu, o.mask_from, o.relu_bwd_fused, o.skip_dgrad)
             for o in conv.ops]
    assert kinds[0] == ("conv", True, -1, False, True)
    assert kinds[2][0] == "maxpool" and kinds[2][2] == 1      # pool1 bwd masked by relu1
    assert kinds[3][0] == "conv" and kinds[3][2] == -1       # conv2 input is a pool output
    assert kinds[8][0] == "conv" and kinds[8][2] == 7        # conv4 bwd masked by relu3
    assert all(o.relu_bwd_fused for o in conv.ops if o.kind == "relu")
    assert conv.param_count == part.conv_params
    fc = BlockEngine(part.fc_block, (part.boundary_activations,), 1, "cpu")
    assert fc.ops[0].mask_from == -1 and fc.ops[2].mask_from == 1
    assert fc.param_count == part.fc_params
    # every per-tensor view 16-byte aligned inside the flat buffer
    for row in fc.slots:
        for off, _, _ in row:
            assert off % 4 == 0


def test_runtime_and_bench_import():
    """The public runtime, the communicator and bench.py import without a GPU."""
    import importlib
    rt = importlib.import_module("paper_1812_10624_b200.stanza_runtime")
    for name in ("StanzaCluster", "StanzaResult", "MissingSource", "NodeId", "Role", "Tag",
                 "NetConfig"):
        assert hasattr(rt, name), name
    comm = importlib.import_module("paper_1812_10624_b200.comm")
    for name in ("RoleComm", "PeerLink", "PeerExchange"):
        assert hasattr(comm, name), name
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    bench = importlib.import_module("bench")
    assert callable(bench.main) and callable(bench.reference_arm)
