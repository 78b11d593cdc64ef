"""Loaders for the committed golden fixtures (made by oracle/make_golden.py
from the reference itself)."""

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _group(path):
    data = np.load(path)
    out = {}
    for key in data.files:
        case, field = key.split("__", 1)
        out.setdefault(case, {})[field] = data[key]
    return out


def ops():
    return _group(os.path.join(GOLDEN, "ops.npz"))


def train():
    return _group(os.path.join(GOLDEN, "train.npz"))


def meta():
    with open(os.path.join(GOLDEN, "meta.json")) as fh:
        return json.load(fh)


def nested_state(case):
    """(params, velocities) nested lists from a train fixture (p{layer}_{slot})."""
    slots = {}
    for key in case:
        if key[0] == "p" and key[1].isdigit():
            li, ti = map(int, key[1:].split("_"))
            slots.setdefault(li, []).append(ti)
    n_layers = max(slots) + 1
    params = [[case[f"p{li}_{ti}"] for ti in sorted(slots.get(li, []))] for li in range(n_layers)]
    vels = [[case[f"v{li}_{ti}"] for ti in sorted(slots.get(li, []))] for li in range(n_layers)]
    return params, vels
