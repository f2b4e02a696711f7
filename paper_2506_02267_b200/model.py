"""Ranking model configuration and parameters (construction / load / save).

Follows ``seqrank.trainer`` (trainer.py:42-161): ``ModelConfig``,
``HeadParams``, ``RankingModel.init/load/save`` with the same RNG draw order
and SRCK tensor names, so checkpoints and seeds are interchangeable with the
reference.  Training (backward, optimisers, NAL) is not on the serving path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import checkpoint
from .core import ValidationError
from .dataset import HEAD_NAMES, NUM_HEADS
from .encoder import EncoderConfig, EncoderParams
from .nnsearch import NNConfig


@dataclass(frozen=True)
class HeadConfig:
    """Head order and utility weights of the final score (losses.py:22-39)."""

    names: tuple[str, ...] = HEAD_NAMES
    ce_weights: tuple[float, ...] = (1.0, 1.0, 1.0, 1.0)
    utility_weights: tuple[float, ...] = (1.0, 0.5, 0.25, -2.0)

    def validate(self) -> None:
        if not (len(self.names) == len(self.ce_weights) == len(self.utility_weights)):
            raise ValidationError("head weight lengths must match head names")
        if not all(np.isfinite(w) for w in self.ce_weights + self.utility_weights):
            raise ValidationError("head weights must be finite")


@dataclass(frozen=True)
class ModelConfig:
    """trainer.py:42-70."""

    encoder: EncoderConfig = EncoderConfig()
    nn: NNConfig = NNConfig()
    ctx_dim: int = 8
    hidden_dim: int = 64
    heads: HeadConfig = HeadConfig()

    def validate(self) -> None:
        self.encoder.validate()
        self.nn.validate()
        self.heads.validate()
        if self.encoder.seq_len != self.nn.seq_len:
            raise ValidationError("encoder seq_len must equal the assembly length")
        if min(self.ctx_dim, self.hidden_dim) < 1:
            raise ValidationError("model dimensions must be positive")

    @classmethod
    def for_nn(cls, nn: NNConfig) -> "ModelConfig":
        return cls(encoder=EncoderConfig(seq_len=nn.seq_len), nn=nn)


@dataclass
class HeadParams:
    w1: np.ndarray
    b1: np.ndarray
    w2: np.ndarray
    b2: np.ndarray


@dataclass
class RankingModel:
    config: ModelConfig
    encoder: EncoderParams
    head: HeadParams
    nal_proj: np.ndarray

    @classmethod
    def init(cls, cfg: ModelConfig, seed: int = 0, dtype=np.float32) -> "RankingModel":
        """trainer.py:88-102: rng([seed, 0]); encoder; head w1, w2; nal proj."""
        cfg.validate()
        rng = np.random.default_rng([seed, 0])
        enc = EncoderParams.init(cfg.encoder, rng, dtype)
        d = cfg.encoder.d_model
        in_dim = d + cfg.encoder.embed_dim + cfg.ctx_dim
        w1 = rng.normal(0, 1 / np.sqrt(in_dim), (in_dim, cfg.hidden_dim)).astype(dtype)
        w2 = rng.normal(0, 1 / np.sqrt(cfg.hidden_dim), (cfg.hidden_dim, NUM_HEADS)).astype(dtype)
        head = HeadParams(w1, np.zeros(cfg.hidden_dim, dtype), w2, np.zeros(NUM_HEADS, dtype))
        nal = rng.normal(0, 1 / np.sqrt(d), (d, cfg.encoder.embed_dim)).astype(dtype)
        return cls(cfg, enc, head, nal)

    def named_tensors(self) -> dict[str, np.ndarray]:
        t = self.encoder.named_tensors()
        t.update({"head.w1": self.head.w1, "head.b1": self.head.b1, "head.w2": self.head.w2,
                  "head.b2": self.head.b2, "nal.proj": self.nal_proj})
        return t

    def save(self, path) -> None:
        """trainer.py:131-143: tensors + 12-int ``meta.config``."""
        t = dict(self.named_tensors())
        c, nn = self.config, self.config.nn
        e = c.encoder
        t["meta.config"] = np.array([e.embed_dim, e.seq_len, e.ffn_dim, e.num_layers, e.action_rows,
                                     e.surface_rows, c.ctx_dim, c.hidden_dim, nn.recent,
                                     nn.k_lifelong, nn.k_realtime, nn.k_impression], np.float32)
        checkpoint.save_tensors(path, t)

    @classmethod
    def load(cls, path) -> "RankingModel":
        """trainer.py:145-161."""
        t = checkpoint.load_tensors(path)
        meta = t.pop("meta.config").astype(int)
        cfg = ModelConfig(encoder=EncoderConfig(*[int(v) for v in meta[:6]]),
                          nn=NNConfig(*[int(v) for v in meta[8:12]]),
                          ctx_dim=int(meta[6]), hidden_dim=int(meta[7]))
        return cls(cfg, EncoderParams.from_tensors(cfg.encoder, t),
                   HeadParams(t["head.w1"], t["head.b1"], t["head.w2"], t["head.b2"]), t["nal.proj"])
