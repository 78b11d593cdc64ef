"""Planner (paper_1812_10624_b200/planner.py) against the reference perf model's
own outputs (tests/golden/planner.json, made by oracle/make_planner_golden.py
from /root/reference/pkg/src/stanza/perf_model.py), the reference tests'
hand-checked values (tests/test_perf_model.py:22-60), and -- on a GPU -- the
measured-constants path."""

import json
import os

import pytest

from paper_1812_10624_b200 import planner as pl
from paper_1812_10624_b200.model_partition import ConfigError, builtin_model, split

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "planner.json")))


def _consts(name):
    g = GOLD["constants"][name]
    return pl.PerfConstants(bandwidth=g["bandwidth"], conv_time=g["conv_time"],
                            fc_unit_time=g["fc_unit_time"], ps_compute_time=g["ps_compute_time"])


def test_window_matches_reference():
    for n, w in GOLD["window"].items():
        assert pl.window(int(n)) == w
    with pytest.raises(ValueError):
        pl.window(0)


def test_hand_checked_values():
    """reference tests/test_perf_model.py:44-60 (AlexNet profile, 10 Gb/s, no compute)."""
    alex = split(builtin_model("alexnet"))
    zero = pl.PerfConstants(bandwidth=10e9)
    for (nc, nf), t in (((4, 1), 0.0460050432), ((8, 1), 0.0841070592), ((4, 4), 0.3827890688)):
        assert abs(pl.stanza_iter_time(alex, nc, nf, zero) - t) <= 1e-12 * t


@pytest.mark.parametrize("model", sorted(GOLD["models"]))
def test_iter_time_and_assignment_match_reference(model):
    rec = GOLD["models"][model]
    part = split(builtin_model(model))
    assert (part.conv_params, part.fc_params, part.boundary_activations, part.spec.batch_k) == \
        (rec["conv_params"], rec["fc_params"], rec["boundary"], rec["batch_k"])
    held = part.spec.batch_k * part.boundary_activations * 4
    mems = {"none": None, "2x": 2.5 * held, "tiny": 0.5 * held}
    for cname in GOLD["constants"]:
        c = _consts(cname)
        for key, t in rec["iter_time"][cname].items():
            nc, nf = map(int, key.split(","))
            assert pl.stanza_iter_time(part, nc, nf, c) == t
            assert pl.stanza_throughput(part, nc, nf, c) == rec["throughput"][cname][key]
        for key, want in rec["assign"][cname].items():
            total, mem = key.split(",")
            if want is None:
                with pytest.raises(pl.Infeasible):
                    pl.assign_nodes(part, int(total), c, fc_memory_bytes=mems[mem])
            else:
                a = pl.assign_nodes(part, int(total), c, fc_memory_bytes=mems[mem])
                assert [a.n_conv, a.n_fc, a.throughput] == want


def test_constants_text_round_trip():
    for name, g in GOLD["constants"].items():
        c = _consts(name)
        assert pl.format_constants_text(c, name) == g["text"]
        assert pl.parse_constants_text(g["text"]) == c
    with pytest.raises(ConfigError):
        pl.parse_constants_text("latency 3\n")
    with pytest.raises(ConfigError):
        pl.PerfConstants(bandwidth=0)


def test_bad_pairs_rejected():
    part = split(builtin_model("alexnet"))
    c = pl.PerfConstants()
    for nc, nf in ((0, 1), (1, 0), (2, 3)):
        with pytest.raises(ConfigError):
            pl.stanza_iter_time(part, nc, nf, c)


def test_pipelined_model_overlaps_fc():
    part = split(builtin_model("alexnet"))
    c = pl.PerfConstants(bandwidth=7.2e12, conv_time=4e-3, fc_unit_time=1e-3)
    bsp = pl.stanza_iter_time(part, 3, 1, c)
    pip = pl.pipelined_iter_time(part, 3, 1, c, micro=2)
    assert pip < bsp
    assert pip >= c.conv_time
    # FC-bound split: the FC worker's g*T_f sets the pace
    c2 = pl.PerfConstants(bandwidth=7.2e12, conv_time=1e-3, fc_unit_time=1e-3)
    assert pl.pipelined_iter_time(part, 7, 1, c2) >= 7e-3


@pytest.mark.gpu
def test_measured_constants_on_gpu(lib):
    c, info = pl.measure_constants(builtin_model("tiny_cnn32"), reps=3)
    assert c.conv_time > 0 and c.fc_unit_time > 0 and c.ps_compute_time >= c.conv_time
    assert c.bandwidth > 0 and info["hbm_free_bytes"] > 0
    a = pl.assign_nodes(split(builtin_model("tiny_cnn32")), 8, c,
                        fc_memory_bytes=info["hbm_free_bytes"])
    assert a.n_conv + a.n_fc == 8
