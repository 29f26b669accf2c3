"""Deterministic synthetic traces: the reference's ``SynthConfig`` /
``generate_synthetic`` (traceio.py:165-296) restated draw for draw, so the
same config gives the same bytes (pinned against the reference's
conformance fixture and generator hashes in tests/test_synth.py).

Keys are correlated across layers (K_l = rho K_base + sqrt(1 - rho^2) noise,
optionally kv-head-permuted per layer); queries concentrate along per-group
directions so the softmax is heavy-tailed; optional X/Y hidden states carry a
depth profile for the importance weights.  Host-side data generation for
tests, benches and calibration -- not part of the attention hot path.
"""

from dataclasses import dataclass
from typing import List, Optional

import numpy as np

from .exceptions import InvalidArgumentError
from .host_types import AttentionTrace


@dataclass
class SynthConfig:
    """traceio.py:165-215 (same fields, defaults and validation)."""

    num_layers: int
    num_query_heads: int
    num_kv_heads: int
    head_dim: int
    seq_len: int
    seed: int = 0
    layer_correlation: float = 1.0
    head_permutations: Optional[List[List[int]]] = None
    heavy_tail_temperature: float = 4.0
    query_correlation: float = 0.85
    layer0_temperature_scale: float = 1.0
    include_xy: bool = False
    prompt_id: str = ""

    def validate(self):
        if not (0.0 <= self.layer_correlation <= 1.0):
            raise InvalidArgumentError("layer_correlation must be in [0, 1]")
        if not (0.0 <= self.query_correlation <= 1.0):
            raise InvalidArgumentError("query_correlation must be in [0, 1]")
        if self.heavy_tail_temperature <= 0 or self.layer0_temperature_scale <= 0:
            raise InvalidArgumentError("temperatures must be > 0")
        if self.num_query_heads % self.num_kv_heads != 0:
            raise InvalidArgumentError("num_query_heads must be divisible by num_kv_heads")
        if self.head_permutations is not None:
            if len(self.head_permutations) != self.num_layers:
                raise InvalidArgumentError("head_permutations must list one permutation per layer")
            for i, perm in enumerate(self.head_permutations):
                if sorted(perm) != list(range(self.num_kv_heads)):
                    raise InvalidArgumentError(f"layer {i} permutation is not a permutation of kv heads")


def _unit_rows(a: np.ndarray) -> np.ndarray:
    return a / np.linalg.norm(a, axis=-1, keepdims=True)


def generate_synthetic(config: SynthConfig) -> AttentionTrace:
    """traceio.py:218-296: identical configs give identical bytes."""
    config.validate()
    L, Hq, Hkv, d, N = (config.num_layers, config.num_query_heads, config.num_kv_heads, config.head_dim,
                        config.seq_len)
    G = Hq // Hkv
    rho = config.layer_correlation
    rng = np.random.default_rng(config.seed)
    k_base = rng.standard_normal((Hkv, N, d))
    v_base = rng.standard_normal((Hkv, N, d))
    group_dirs = _unit_rows(rng.standard_normal((Hkv, d)))
    jitter = _unit_rows(rng.standard_normal((Hq, N, d)))
    c = config.query_correlation
    heads = np.arange(Hq) // G
    dirs = _unit_rows(np.sqrt(c) * group_dirs[heads][:, None, :] + np.sqrt(1.0 - c) * jitter)
    perms = config.head_permutations or [list(range(Hkv))] * L
    mix = np.sqrt(1.0 - rho * rho)
    Q = np.empty((L, Hq, N, d), dtype=np.float32)
    K = np.empty((L, Hkv, N, d), dtype=np.float32)
    V = np.empty((L, Hkv, N, d), dtype=np.float32)
    for layer in range(L):
        perm = perms[layer]
        k_noise = rng.standard_normal((Hkv, N, d))
        v_noise = rng.standard_normal((Hkv, N, d))
        tau = config.heavy_tail_temperature * (config.layer0_temperature_scale if layer == 0 else 1.0)
        for g in range(Hkv):
            K[layer, g] = (rho * k_base[perm[g]] + mix * k_noise[g]).astype(np.float32)
            V[layer, g] = (rho * v_base[perm[g]] + mix * v_noise[g]).astype(np.float32)
            src = perm[g] * G + np.arange(G)
            Q[layer, g * G:(g + 1) * G] = (tau * np.sqrt(d) * dirs[src]).astype(np.float32)
    X = Y = None
    if config.include_xy:
        model_dim = Hq * d
        x_base = rng.standard_normal((N, model_dim)) / np.sqrt(model_dim)
        X = np.repeat(x_base[None, :, :], L, axis=0).astype(np.float32)
        Y = np.empty((L, N, model_dim), dtype=np.float32)
        aligns = np.linspace(0.1, 0.95, L)     # early attention rewrites the representation
        for layer in range(L):
            noise = rng.standard_normal((N, model_dim)) / np.sqrt(model_dim)
            a = aligns[layer]
            Y[layer] = (a * x_base + np.sqrt(1.0 - a * a) * noise).astype(np.float32)
    return AttentionTrace(L, Hq, Hkv, d, N, Q, K, V, X, Y, prompt_id=config.prompt_id or f"synth-seed{config.seed}")
