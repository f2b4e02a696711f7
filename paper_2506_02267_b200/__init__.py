"""B200-native TransAct V2 serving-time ranking path (drop-in for the
``seqrank`` 0.1.0 serving path).

Host API mirrors the reference module names; compute runs in the sm_100a
library ``_lib/libtav2.so`` (C ABI in ``include/tav2.h``).
"""

from .core import (  # noqa: F401
    EMBED_DIM, LIFELONG_CAP, REALTIME_CAP, IMPRESSION_CAP, TokenBlock, UserSequences,
    ValidationError, dequantize, l2_normalize_rows, quantize, unit_embeddings,
)
from .dataset import (  # noqa: F401
    HEAD_NAMES, NUM_HEADS, SyntheticConfig, context_features, generate_requests, generate_synthetic,
    synthetic_requests,
)
from .encoder import (  # noqa: F401
    EncodedSequence, EncoderConfig, EncoderParams, LayerParams, encode, encode_batch, forward_fused,
    forward_reference, pool,
)
from .model import HeadConfig, HeadParams, ModelConfig, RankingModel  # noqa: F401
from .nnsearch import (  # noqa: F401
    AssembledSequence, DedupBatch, NNConfig, Segment, assemble, build_dedup_batch, fused_assemble,
    similarity_scores, top_k_nn,
)

__version__ = "0.1.0"


def __getattr__(name):  # lazy: torch + the native library load on first use
    if name in ("Engine", "Capacity"):
        from . import runtime

        return getattr(runtime, name)
    if name in ("rank", "rank_many", "RankResponse"):
        from . import serving

        return getattr(serving, name)
    if name in ("model_forward", "ForwardState", "TrainBatch"):
        from . import trainer

        return getattr(trainer, name)
    raise AttributeError(name)
