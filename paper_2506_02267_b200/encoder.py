"""Encoder configuration/parameters and the GPU encode / SKUT forward.

Public names follow ``seqrank.encoder`` (encoder.py:24-462).  Parameter
initialisation reproduces the reference draw order so the same seed gives
bit-identical weights; ``encode`` / ``encode_batch`` / ``forward_fused`` /
``forward_reference`` / ``pool`` take the reference's ``EncoderParams`` (or
an Engine) and run on the B200 through the native library.
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


@dataclass
class EncodedSequence:
    """Per-token feature rows (seq_len, d_model); masked rows are zero (encoder.py:140-145)."""

    features: np.ndarray
    mask: np.ndarray


def _nn_of(seqs) -> "NNConfig":
    """The NNConfig whose segment layout the assembled sequences carry."""
    from .nnsearch import NNConfig

    lens = {g.name: g.stop - g.start for g in seqs[0].segments}
    return NNConfig(recent=lens["recent_realtime"], k_lifelong=lens["nn_lifelong"],
                    k_realtime=lens["nn_realtime_tail"], k_impression=lens["nn_impression"])


def _layout_nn(S: int) -> "NNConfig":
    """Any segment split of length S within the per-segment k budget (the
    caller-feature kernels only use S)."""
    from .nnsearch import NNConfig

    k = min(S, 256)
    return NNConfig(recent=S - k, k_lifelong=k, k_realtime=0, k_impression=0)


def _engine(params_or_engine, nn, requests=1, items=1, tokens=1):
    """The Engine for an API call: the caller's Engine, or the calling
    thread's implicit engine holding these EncoderParams (built once per
    (params object, layout), never per call; params are immutable after load,
    SPEC.md:297)."""
    from .model import HeadParams, ModelConfig, RankingModel
    from .runtime import Engine, implicit_engine

    if isinstance(params_or_engine, Engine):
        return params_or_engine
    params = params_or_engine
    if not isinstance(params, EncoderParams):
        raise ValidationError("expected EncoderParams or an Engine")
    models = params.__dict__.setdefault("_tav2_models", {})
    model = models.get(nn)
    if model is None:  # encoder-only model: the head is not read by these calls
        cfg = ModelConfig(encoder=params.config, nn=nn)
        d, e, h = params.config.d_model, params.config.embed_dim, cfg.hidden_dim
        z = np.zeros
        head = HeadParams(z((d + e + cfg.ctx_dim, h), np.float32), z(h, np.float32), z((h, 4), np.float32),
                          z(4, np.float32))
        model = models[nn] = RankingModel(cfg, params, head, z((d, e), np.float32))
    return implicit_engine(nn, requests=requests, items=items, tokens=tokens, model=model)


def encode_batch(seqs, candidates: np.ndarray, params) -> tuple[np.ndarray, np.ndarray]:
    """Eq. 4 features of assembled sequences (encoder.py:161-188) on the GPU
    (tav2_encode) -> (features [B, L, 64] f32, mask [B, L] bool)."""
    if len(seqs) == 0:
        S = params.config.seq_len if isinstance(params, EncoderParams) else params.config.nn.seq_len
        return np.zeros((0, S, 64), np.float32), np.zeros((0, S), bool)
    toks = int(sum(np.count_nonzero(s.mask) for s in seqs))
    eng = _engine(params, _nn_of(seqs), requests=len(seqs), items=len(seqs), tokens=max(toks, 1))
    return eng.encode(list(seqs), np.asarray(candidates, np.float32))


def encode(seq, candidate: np.ndarray, params) -> EncodedSequence:
    """One assembled sequence against its candidate (encoder.py:148-158)."""
    f, mask = encode_batch([seq], np.asarray(candidate, np.float32)[None, :], params)
    return EncodedSequence(f[0], mask[0])


def forward_fused(features, mask, params_or_engine, extra_mask=None, arena=None, tile: int = 64,
                  mode: str = "fp32"):
    """GPU SKUT forward (encoder.py:314-462) over (B, L, 64) features.

    ``params_or_engine``: the reference's ``EncoderParams`` (served by the
    calling thread's implicit engine) or an
    :class:`~paper_2506_02267_b200.runtime.Engine` holding the model.
    Padded query rows are not computed (never read: keys mask them and
    pooling skips them) and come back as zeros.  ``extra_mask`` ([L, L] or
    [B, L, L] bool; the NAL training masks, encoder.py:366-377) is ANDed into
    causal & key-valid; a row with no allowed key gets a zero attention
    output (tav2_forward_masked: the f32 running-max kernel).
    """
    f = np.asarray(features)
    if f.ndim != 3:
        raise ValidationError("expected a (batch, length, d_model) feature tensor")
    eng = _engine(params_or_engine, _layout_nn(f.shape[1]))
    return eng.forward(f, np.asarray(mask, bool), mode=mode, extra_mask=extra_mask)


def forward_reference(enc: EncodedSequence, params, extra_mask=None, mode: str = "fp32") -> np.ndarray:
    """One encoded sequence through the transformer (encoder.py:221-246; the
    reference's layered and fused forwards agree to ~3e-6)."""
    return forward_fused(enc.features[None], enc.mask[None], params, extra_mask, mode=mode)[0]


def pool(u: np.ndarray, mask: np.ndarray, params_or_engine) -> np.ndarray:
    """Linear projection then elementwise max over valid positions, zeros
    when every position is masked (encoder.py:265-273), on the GPU
    (tav2_pool).  ``u`` is (L, d) as in the reference, or a (B, L, d) batch."""
    u = np.asarray(u, np.float32)
    single = u.ndim == 2
    ub, mb = (u[None], np.asarray(mask, bool)[None]) if single else (u, np.asarray(mask, bool))
    eng = _engine(params_or_engine, _layout_nn(ub.shape[1]))
    out = eng.pool(ub, mb)
    return out[0] if single else out
