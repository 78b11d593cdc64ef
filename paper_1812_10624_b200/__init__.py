"""B200-native Stanza (arXiv 1812.10624) layer-separated training step.

Drop-in for the reference package's hot path (``stanza.stanza_runtime``):
``split`` / ``plan_groups`` / ``StanzaCluster(...).train`` keep the reference
API, while every layer op runs as hand-written sm_100a CUDA behind the C ABI
in include/stanza_b200.h (built in-tree as libstz_b200.so).
"""

from .model_partition import (ConfigError, ModelSpec, Partition, alexnet, builtin_model,
                              mlp_split, parse_model_text, split, tiny_cnn, tiny_cnn32,
                              tiny_mlp, vgg16)
from .roles import equal_split, gpu_roles, plan_groups

__all__ = ["ConfigError", "ModelSpec", "Partition", "alexnet", "builtin_model", "equal_split",
           "gpu_roles", "mlp_split", "parse_model_text", "plan_groups", "split", "tiny_cnn",
           "tiny_cnn32", "tiny_mlp", "vgg16", "StanzaCluster", "StanzaResult"]


def __getattr__(name):
    if name in ("StanzaCluster", "StanzaResult", "MissingSource"):
        from . import stanza_runtime
        return getattr(stanza_runtime, name)
    raise AttributeError(name)
