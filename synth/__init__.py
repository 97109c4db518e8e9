"""Seeded input generators shared by the oracle and the CUDA path.

Holds none of the method's arithmetic: model hyper-parameters, deterministic
random-init weights and synthetic workloads only.
"""
from .config import ModelConfig, PRESETS, PAD_ID, UNK_ID, BOS_ID, EOS_ID  # noqa: F401
from .weights import generate_weights, canonical_shapes, param_count, WEIGHT_SEED  # noqa: F401
from .workload import Workload, newstest_like, tiny_workload, random_tokens, DATA_SEED  # noqa: F401
