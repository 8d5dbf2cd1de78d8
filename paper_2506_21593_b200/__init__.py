"""B200-native PentaRAG fast-routing hot path (arxiv 2506.21593).

Drop-in, device-resident replacements for the reference ``ragcascade``
stores on the per-query-batch hot path — ``FlatIndex`` (index.py),
``FixedKVCache`` / ``SemanticCache`` (caches.py), ``MainKnowledgeBase`` /
``AdaptiveKnowledgeMemory`` (knowledge.py) and ``CascadeRouter``
(router.py) — backed by libpentarag.so (hand-written sm_100a kernels behind
the C ABI in include/pentarag.h).
"""
from .errors import (
    AllLayersMissed,
    BackendUnavailable,
    CascadeError,
    CorruptSnapshot,
    DeviceError,
    DeviceUnavailable,
    DimensionMismatch,
    EmptyContext,
    EmptyInput,
    EmptyKnowledgeBase,
    EmptyQuery,
    InvalidVector,
    NativeLibraryMissing,
)
from .caches import CacheEntry, FixedKVCache, SemanticCache, writeback
from .errors import MalformedJsonl
from .generation import (DeviceKnowledgeTable, StubBackend, StubKnowledgeTable, generate_with_context,
                         memory_recall)
from .index import MODE_AUTO, MODE_EXACT, MODE_TENSOR, MODE_TENSOR_I8, BatchResult, FlatIndex, SearchHit
from .knowledge import AdaptiveKnowledgeMemory, MainKnowledgeBase, ingest_corpus
from .router import CascadeRouter, LayerProbe, RouterConfig, RouteTraceEvent, TraceLog, export_triples
from .service import MicroBatcher
from .sharded import ShardedFlatIndex, ShardedRowIndex, shard_range
from .records import CASCADE_ORDER, AnswerRecord, LayerTag, Passage, Query, TrainingTriple, validate_query
from .vectors import DIMENSION, HASH_SEED, EmbeddingVector, HashEmbedder, cosine, tokenize

__version__ = "0.1.0"
