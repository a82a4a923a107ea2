"""paper_2605_08568_b200 -- B200-native (sm_100a) PARSE rank-expert hot path.

Router (mean_pool -> score -> select_topk), pattern-cache retrieval, expert
gather/aggregation and the two-stage rank-expert contraction, behind the
reference's own API names (see api.py) over the C-ABI in include/parse_gpu.h.
"""
from ._lib import CudaError, launch_count  # noqa: F401
from .api import *  # noqa: F401,F403
from .api import (AccessTrace, AggregatedLayer, CacheEntry, ColRange, ExecEngine, ExecPlan,  # noqa: F401
                  ExecProvider, ExecVariant, FactorizedLayer, FactorizedModel, FactorizedProvider,
                  LaunchDesc, LaunchKind, PatternCache, ProjectionProvider, PromptEmbedding,
                  RankSelection, RetrieveResult, RouterParams, RoutingProvider, aggregate_layout,
                  aggregated_forward, aggregated_forward_batched, build_plan, cache_insert,
                  check_selection, cosine, embed_pool, make_patterns, make_router, masked_forward,
                  maximal_runs, mean_pool, retrieve, retrieve_device, rng_gaussian, route_select, route_select_pooled,
                  scattered_forward, score, silu_mul, PatternServer, PromptSelection, PackedExperts, pack_selected, prefill_packed, copy_io, prefill_batched, SelectionBatch, masked_forward_union, module_forward_union, UnionProgram, module_forward, mlp_forward, mlp_forward_chain, select_topk, single_layer_k, store_rank, tensor_id,
                  variant_aggregated, variant_fused)
from . import dist, embed, loaders, train  # noqa: F401,E402
from .loaders import load_cache, load_factorized  # noqa: F401,E402
