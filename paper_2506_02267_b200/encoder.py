"""Encoder configuration/parameters and the GPU encode / SKUT forward.

Public names follow ``seqrank.encoder`` (encoder.py:24-462).  Parameter
initialisation reproduces the reference draw order so the same seed gives
bit-identical weights; ``encode_batch`` / ``forward_fused`` / ``pool`` run
on the B200 through the native library.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .core import ValidationError

LN_EPS = 1e-5
_LAYER_TENSOR_NAMES = ("wq", "wk", "wv", "wo", "w1", "w2",
                       "ln1_scale", "ln1_shift", "ln2_scale", "ln2_shift")


@dataclass(frozen=True)
class EncoderConfig:
    """encoder.py:24-44."""

    embed_dim: int = 32
    seq_len: int = 192
    ffn_dim: int = 32
    num_layers: int = 2
    action_rows: int = 16
    surface_rows: int = 256

    @property
    def d_model(self) -> int:
        return 2 * self.embed_dim

    def validate(self) -> None:
        if min(self.embed_dim, self.seq_len, self.ffn_dim, self.num_layers) < 1:
            raise ValidationError("encoder dimensions must be positive")


@dataclass
class LayerParams:
    wq: np.ndarray
    wk: np.ndarray
    wv: np.ndarray
    wo: np.ndarray
    w1: np.ndarray
    w2: np.ndarray
    ln1_scale: np.ndarray
    ln1_shift: np.ndarray
    ln2_scale: np.ndarray
    ln2_shift: np.ndarray


@dataclass
class EncoderParams:
    config: EncoderConfig
    action_table: np.ndarray
    surface_table: np.ndarray
    position_table: np.ndarray
    layers: list[LayerParams] = field(default_factory=list)
    out_linear: np.ndarray = None

    @classmethod
    def init(cls, cfg: EncoderConfig, rng: np.random.Generator, dtype=np.float32) -> "EncoderParams":
        """Draw order of encoder.py:75-108: per layer wq, wk, wv, wo, w1, w2;
        then the action, surface, position tables; then out_linear."""
        cfg.validate()
        d, f = cfg.d_model, cfg.ffn_dim

        def w(*shape, scale=1.0 / np.sqrt(d)):
            return rng.normal(0.0, scale, shape).astype(dtype)

        layers = []
        for _ in range(cfg.num_layers):
            wq, wk, wv, wo, w1 = w(d, d), w(d, d), w(d, d), w(d, d), w(d, f)
            w2 = w(f, d, scale=1.0 / np.sqrt(f))
            layers.append(LayerParams(wq, wk, wv, wo, w1, w2, np.ones(d, dtype), np.zeros(d, dtype),
                                      np.ones(d, dtype), np.zeros(d, dtype)))
        action = w(cfg.action_rows, d, scale=0.1)
        surface = w(cfg.surface_rows, d, scale=0.1)
        position = w(cfg.seq_len, d, scale=0.1)
        return cls(cfg, action, surface, position, layers, w(d, d))

    def named_tensors(self) -> dict[str, np.ndarray]:
        t = {"encoder.action_table": self.action_table,
             "encoder.surface_table": self.surface_table,
             "encoder.position_table": self.position_table,
             "encoder.out_linear": self.out_linear}
        for i, layer in enumerate(self.layers):
            for name in _LAYER_TENSOR_NAMES:
                t[f"encoder.layer{i}.{name}"] = getattr(layer, name)
        return t

    @classmethod
    def from_tensors(cls, cfg: EncoderConfig, tensors: dict[str, np.ndarray]) -> "EncoderParams":
        layers = [LayerParams(**{n: tensors[f"encoder.layer{i}.{n}"] for n in _LAYER_TENSOR_NAMES})
                  for i in range(cfg.num_layers)]
        return cls(cfg, tensors["encoder.action_table"], tensors["encoder.surface_table"],
                   tensors["encoder.position_table"], layers, tensors["encoder.out_linear"])


def forward_fused(features, mask, params_or_engine, extra_mask=None, arena=None, tile: int = 64,
                  mode: str = "fp32"):
    """GPU SKUT forward (encoder.py:314-462) over (B, L, 64) features.

    ``params_or_engine`` is an :class:`~paper_2506_02267_b200.runtime.Engine`
    holding the model.  Padded query rows are not computed (never read: keys
    mask them and pooling skips them) and come back as zeros.  ``extra_mask``
    (NAL training masks, encoder.py:366-377) is not on the serving path.
    """
    if extra_mask is not None:
        raise ValidationError("extra_mask is a training-only feature and not on the serving path")
    from .runtime import Engine

    if not isinstance(params_or_engine, Engine):
        raise ValidationError("forward_fused needs an Engine with the model loaded")
    f = np.asarray(features)
    if f.ndim != 3:
        raise ValidationError("expected a (batch, length, d_model) feature tensor")
    return params_or_engine.forward(f, np.asarray(mask, bool), mode=mode)
