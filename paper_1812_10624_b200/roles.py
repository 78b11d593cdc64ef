"""CONV-worker / FC-worker role assignment (bit-exact with the reference).

``plan_groups`` restates stanza_runtime.py:41-56 over ``equal_split``
(ps_runtime.py:27-32): contiguous, near-equal groups, the remainder going
to the first FC workers.  ``gpu_roles`` maps a GPU count of one 8xB200 box
to the (n_conv, n_fc) split the bench uses.
"""

from __future__ import annotations

from .model_partition import ConfigError


def equal_split(total: int, parts: int) -> list[int]:
    """Near-equal shard sizes; the first ``total % parts`` get one more."""
    if parts < 1:
        raise ConfigError(f"cannot split into {parts} shards")
    base, extra = divmod(total, parts)
    return [base + (i < extra) for i in range(parts)]


def plan_groups(n_conv: int, n_fc: int) -> list[int]:
    """conv_to_fc: the FC worker serving each CONV worker."""
    if n_conv < 1 or n_fc < 1:
        raise ConfigError("need at least one CONV and one FC worker, got "
                          f"n_conv={n_conv} n_fc={n_fc}")
    if n_fc > n_conv:
        raise ConfigError(f"more FC workers ({n_fc}) than CONV workers ({n_conv}) "
                          "leaves some idle")
    out: list[int] = []
    for j, size in enumerate(equal_split(n_conv, n_fc)):
        out += [j] * size
    return out


def group_rows(conv_to_fc: list[int], fc_index: int) -> tuple[int, int]:
    """[first, last+1) CONV indices of an FC group (groups are contiguous)."""
    members = [i for i, j in enumerate(conv_to_fc) if j == fc_index]
    return members[0], members[-1] + 1


# GPUs on one box -> (n_conv, n_fc); 1 GPU co-locates both roles
GPU_ROLES = {1: (1, 1), 2: (1, 1), 4: (3, 1), 8: (7, 1)}


def gpu_roles(n_gpus: int, fc_workers: int | None = None) -> tuple[int, int]:
    if fc_workers is not None:
        if n_gpus == 1:
            return (1, 1)
        return (n_gpus - fc_workers, fc_workers)
    if n_gpus in GPU_ROLES:
        return GPU_ROLES[n_gpus]
    return (n_gpus - 1, 1)
