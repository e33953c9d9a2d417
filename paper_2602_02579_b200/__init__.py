"""B200-native ProphetKV selective-recompute prefill -- drop-in for the ``pikv`` hot path.

Public names follow the reference package (``pikv/__init__.py:10-33``) for the
path in scope: assemble -> score_prophet -> fuse_layers / select_top_p ->
recompute_selected (with replace_entries) -> finalize_query, plus the types they
exchange.  Everything runs on hand-written sm_100a kernels behind the C ABI in
``include/pkv.h``; there is no CPU fallback.
"""

from .chunkfile import load_chunk, load_chunk_pinned, store_chunk
from .chunkstore import AssembledCache, ChunkKV, assemble, chunk_content_id, mark_finalized, replace_entries
from .errors import (ArgumentError, ConfigError, EngineError, FormatError, IncompatibleError, InputError,
                     NumericsError, ShapeError, StateError, TruncatedError)
from .model import (DeviceModel, FlopCounter, FlopTally, KVCache, LayerWeights, ModelConfig, ModelWeights,
                    random_weights)
from .decode import GenerationResult, decode_step, greedy_generate
from .prefill import PrefillTrace, full_prefill, precompute_chunk
from .querypass import QueryPassResult, query_pass
from .recompute import (AnswerRecord, FinalizeResult, RecomputePlan, StrategyRun, finalize_query,
                        recompute_selected, run_strategy, selection_digest)
from .selection import (STRATEGIES, SelectionResult, ValueScores, fuse_layers, score_cacheblend_l1, score_epic,
                        score_kvshare_l1, score_prophet, score_random, select_top_p)
from .tensor import ratio_budget, top_k_indices

__version__ = "0.1.0"

__all__ = [name for name in dir() if not name.startswith("_")]
