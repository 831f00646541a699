"""B200-native BLEST pull BFS (arXiv 2512.21967): GPU BVSS builder + fused persistent
sm_100a BFS kernel behind the reference's API (see include/blest_b200.h for the C-ABI and
include/blest_b200.hpp for the C++ drop-in façade)."""
from .api import (  # noqa: F401
    KUNREACHED, RMAT_ABC, AutoConfig, AutoResult, BfsResult, Bvss, BvssStats, EngineConfig,
    EngineCounters, EngineMode, FrontierState, Graph, LevelTrace, OrderingPlan,
    OrderingStrategy, Permutation, PrePass, SelectDefaults, SocialLikeReport, apply_permutation,
    build_bvss, bvss_stats, choose_mode, classify_social_like, compression_ratio, device_info,
    engine_mode_from_string, init_state, jaccard_with_windows, make_permutation,
    ordering_strategy_from_string, prepare, random_order, rcm, relabel_permutation, run_auto,
    run_auto_prebuilt, run_batch, run_eager, run_lazy, select_plan, update_divergence,
    RoundtripReport, load_bvss, load_graph, load_permutation, reference_bfs, save_bvss,
    save_permutation, tile_pull, validate_roundtrip)
from ._lib import BlestCudaError, BlestLogicError, LIB_PATH, ParseError  # noqa: F401
