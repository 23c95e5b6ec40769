"""paper_2601_03067_b200: B200-native (sm_100a) joint encoding of KV-cache blocks.

Drop-in for the reference kvfuse fusion path (BFF / CFF tree fusion, block
tables, refold, paged attention) with every hot op in hand-written CUDA
behind a C ABI (include/kvfuse_b200.h, libkvfuse_b200.so). See DESIGN.md.
"""

from .attention import (
    AttentionQuery,
    SoftmaxDistribution,
    DecodeSchedule,
    attention_drift,
    chunk_prefill,
    decode_schedule,
    state_decode_schedule,
    paged_attention,
    paged_decode,
    softmax,
)
from .core import (
    BlockTable,
    CacheDims,
    FusedCache,
    FusedLayer,
    LayerView,
    PagedKvCache,
    UnfoldedLayer,
    cff_chunk_count,
    cosine_similarity,
    refold,
    unfold_bff,
    unfold_cff,
)
from .engine import FusionEngine, FusionState, Geometry
from .errors import (
    AlignmentError,
    ConfigError,
    CorruptionError,
    DivergenceError,
    DomainError,
    FormatError,
    InsufficientDataError,
    InvalidCacheError,
    KvFuseError,
    ZeroVectorError,
)
from .fusion import (
    CSV_HEADER,
    AdaptPolicy,
    FusionConfig,
    FusionEvent,
    FusionOutcome,
    FusionReport,
    MergeRecord,
    adapt_threshold,
    fast_fusion,
    fuse_batch,
    fuse_chunks,
    reports_to_csv,
    tune_threshold,
)

__version__ = "0.1.0"

__all__ = [
    "AdaptPolicy", "AlignmentError", "AttentionQuery", "BlockTable", "CSV_HEADER", "CacheDims",
    "ConfigError", "CorruptionError", "DivergenceError", "DomainError", "FormatError",
    "FusedCache", "FusedLayer", "FusionConfig", "FusionEngine", "FusionEvent", "FusionOutcome",
    "FusionReport", "FusionState", "Geometry", "InsufficientDataError", "InvalidCacheError",
    "KvFuseError", "LayerView", "MergeRecord", "PagedKvCache", "SoftmaxDistribution",
    "UnfoldedLayer", "ZeroVectorError", "adapt_threshold", "attention_drift", "cff_chunk_count", "chunk_prefill",
    "DecodeSchedule", "cosine_similarity", "decode_schedule", "fast_fusion", "fuse_batch", "fuse_chunks", "paged_attention",
    "paged_decode", "refold", "reports_to_csv", "softmax", "state_decode_schedule", "tune_threshold", "unfold_bff",
    "unfold_cff",
]
