"""ctypes binding of libktune_cuda.so (include/ktune_cuda.h).

The library is built in-tree (paper_2001_08743_b200/libktune_cuda.so, see
csrc/Makefile). There is no fallback: if the shared object is missing or
cannot be loaded, importing the product API raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

from .errors import BackendError, ConfigError, CudaError, LogicError, SpaceExhaustedError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KTUNE_LIB_PATH") or os.path.join(HERE, "libktune_cuda.so")  # override: A/B builds

KTUNE_OK, ERR_CONFIG, ERR_BACKEND, ERR_EXHAUSTED, ERR_LOGIC, ERR_CUDA, ERR_NOMEM = range(7)
F_DEVICE = 1
F_EXACT_ROLLOUT = 2
F_STEP_MAJOR = 4
F_STEP_MAJOR_GROUPED = 8
OPT_FORCE_EXACT, OPT_KMEANS_MODE, OPT_PROFILE, OPT_ROLLOUT_DELTA, OPT_ROLLOUT_CHECK, OPT_ROLLOUT_FUSE_GBT, \
    OPT_ROLLOUT_SEGMENTS, OPT_FORCE_SHARDED, OPT_KMEANS_BOUND_LOG2, OPT_ROLLOUT_STREAMED = 1, 2, 3, 4, 5, 6, 7, 8, 9, 10
STAT_LAUNCHES, STAT_KPP_FALLBACKS, STAT_DECISION_FALLBACKS, STAT_ASSIGN_FALLBACKS, \
    STAT_SNAP_CHAINS, STAT_LLOYD_ITERS, STAT_KPP_PICKS, STAT_ROLLOUT_NS, STAT_ROLLOUT_CALLS, \
    STAT_GBT_NS, STAT_GBT_CALLS, STAT_ASSIGN_NS, STAT_ASSIGN_CALLS, STAT_XS_SEQUENTIAL, \
    STAT_XS_SEGMENTS, STAT_ROLLOUT_FALLBACKS, STAT_ROLLOUT_CHECKED, STAT_ROLLOUT_MISMATCH, \
    STAT_ROLLOUT_MAXERR, STAT_ROLLOUT_TC, STAT_KMEANS_ABORTS = range(1, 22)

P = C.c_void_p
i32 = C.c_int32
i64 = C.c_int64
u64 = C.c_uint64
dbl = C.c_double


class RuleOp(C.Structure):
    _fields_ = [("code", C.c_int32), ("pad", C.c_int32), ("arg", C.c_int64)]


class TreeNode(C.Structure):
    _fields_ = [("feature", C.c_int32), ("left", C.c_int32), ("right", C.c_int32),
                ("pad", C.c_int32), ("threshold", C.c_double), ("value", C.c_double)]


class GbtModelC(C.Structure):
    _fields_ = [("num_trees", C.c_int32), ("num_features", C.c_int32),
                ("base_prediction", C.c_double), ("learning_rate", C.c_double),
                ("tree_offsets", C.POINTER(C.c_int32)), ("nodes", C.POINTER(TreeNode)),
                ("training_sse", C.POINTER(C.c_double))]


class RolloutTaskC(C.Structure):
    _fields_ = [("space", P), ("ac", P), ("gbt", P), ("num_episodes", i64),
                ("episode_offset", i64), ("explore_seed", u64), ("init_idx", P), ("idx", P),
                ("score", P), ("actions", P), ("logp", P), ("value", P), ("logp_f32", P), ("value_f32", P),
                ("idx_u8", P), ("actions_u2", P), ("score_f32", P), ("ids_u32", P)]


class SaParamsC(C.Structure):
    _fields_ = [("initial_temperature", C.c_double), ("cooling_rate", C.c_double)]


class SaTaskC(C.Structure):
    _fields_ = [("space", P), ("gbt", P), ("num_chains", i64), ("chain_offset", i64), ("sa_seed", u64),
                ("init_idx", P), ("idx", P), ("score", P), ("accepted", P)]


class KmeansOutC(C.Structure):
    _fields_ = [("centroids", P), ("assignments", P), ("l2_loss", P), ("iteration_losses", P),
                ("num_losses", P)]


class SamplingParamsC(C.Structure):
    _fields_ = [("threshold", C.c_double), ("k_min", C.c_int32), ("k_max_exclusive", C.c_int32),
                ("max_iters", C.c_int32), ("restarts", C.c_int32)]


class PpoParamsC(C.Structure):
    _fields_ = [("clip_epsilon", C.c_double), ("value_coef", C.c_double), ("entropy_coef", C.c_double),
                ("num_epochs", C.c_int32), ("pad", C.c_int32), ("minibatch_size", C.c_int64)]


class SweepOutC(C.Structure):
    _fields_ = [("k", P), ("centroids", P), ("assignments", P), ("l2_loss", P), ("k_losses", P),
                ("num_k", P), ("snapped", P)]


# name -> (restype, argtypes); every symbol include/ktune_cuda.h declares.
SIGNATURES = {
    "ktune_abi_version": (C.c_int, []),
    "ktune_last_error": (C.c_char_p, [P]),
    "ktune_ctx_create": (C.c_int, [C.c_int, C.POINTER(P)]),
    "ktune_ctx_create_dist": (C.c_int, [C.c_int, C.c_int, C.c_int, P, C.POINTER(P)]),
    "ktune_nccl_get_unique_id": (C.c_int, [P]),
    "ktune_ctx_destroy": (C.c_int, [P]),
    "ktune_ctx_set_stream": (C.c_int, [P, P]),
    "ktune_ctx_stream": (P, [P]),
    "ktune_ctx_synchronize": (C.c_int, [P]),
    "ktune_ctx_set_option": (C.c_int, [P, C.c_int, i64]),
    "ktune_ctx_stat": (C.c_int, [P, C.c_int, C.POINTER(i64)]),
    "ktune_ctx_reset_stats": (C.c_int, [P]),
    "ktune_rule_compile": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(C.c_char_p), C.POINTER(RuleOp),
                                     C.POINTER(C.c_int), C.c_char_p, C.c_int]),
    "ktune_rule_eval": (C.c_int, [C.POINTER(RuleOp), C.c_int, P]),
    "ktune_space_create": (C.c_int, [P, C.c_int, P, P, C.POINTER(RuleOp), C.c_int, C.POINTER(P)]),
    "ktune_space_destroy": (C.c_int, [P]),
    "ktune_space_id_of": (C.c_int, [P, P, i64, P]),
    "ktune_space_config_at": (C.c_int, [P, P, i64, P]),
    "ktune_space_validate": (C.c_int, [P, P, i64, P]),
    "ktune_gbt_fit": (C.c_int, [P, P, i64, C.c_int, C.c_int, C.c_int, dbl, C.c_int, u64,
                                C.POINTER(GbtModelC)]),
    "ktune_gbt_model_free": (None, [C.POINTER(GbtModelC)]),
    "ktune_gbt_create": (C.c_int, [P, P, C.c_int, dbl, dbl, C.c_int, P, P, C.POINTER(P)]),
    "ktune_gbt_destroy": (C.c_int, [P]),
    "ktune_gbt_predict_idx": (C.c_int, [P, P, P, C.c_int, i64, P, C.c_int]),
    "ktune_gbt_predict_features": (C.c_int, [P, P, P, i64, P, C.c_int]),
    "ktune_ac_num_params": (i64, [C.c_int, C.c_int, C.c_int]),
    "ktune_ac_init_params": (C.c_int, [C.c_int, C.c_int, C.c_int, u64, P]),
    "ktune_ac_create": (C.c_int, [P, C.c_int, C.c_int, C.c_int, P, C.POINTER(P)]),
    "ktune_ac_destroy": (C.c_int, [P]),
    "ktune_ac_forward": (C.c_int, [P, P, P, i64, P, P, P, C.c_int]),
    "ktune_ac_forward_cache": (C.c_int, [P, P, P, i64, P, P, P, P, P, P, P, C.c_int]),
    "ktune_ac_backward": (C.c_int, [P, P, P, P, P, P, i64, P, P, P, C.c_int]),
    "ktune_ac_get_params": (C.c_int, [P, P, P]),
    "ktune_adam_create": (C.c_int, [P, i64, dbl, dbl, dbl, dbl, C.POINTER(P)]),
    "ktune_adam_destroy": (C.c_int, [P]),
    "ktune_adam_step": (C.c_int, [P, P, P, P, C.c_int]),
    "ktune_adam_state": (C.c_int, [P, P, P, P, C.POINTER(i64)]),
    "ktune_compute_gae": (C.c_int, [P, i64, C.c_int32, P, P, P, dbl, dbl, P, P, C.c_int]),
    "ktune_ppo_update": (C.c_int, [P, P, P, C.POINTER(PpoParamsC), i64, P, P, P, P, P, u64, P, C.c_int]),
    "ktune_rollout": (C.c_int, [P, C.c_int, C.POINTER(RolloutTaskC), C.c_int32, C.c_int]),
    "ktune_sa_search": (C.c_int, [P, C.c_int, C.POINTER(SaTaskC), C.c_int32, C.POINTER(SaParamsC), C.c_int]),
    "ktune_make_candidate_set": (C.c_int, [P, P, P, i64, P, C.POINTER(i64)]),
    "ktune_candidates_from_rows": (C.c_int, [P, P, P, P, i64, P, P, C.POINTER(i64), C.c_int]),
    "ktune_candidates_gather": (C.c_int, [P, P, P, P, i64, C.POINTER(i64), C.c_int]),
    "ktune_candidates_gather_copy": (C.c_int, [P, P, P, P, P, C.c_int]),
    "ktune_ctx_create_hostcomm": (C.c_int, [C.c_int, C.c_int, C.c_int, P, P, P, C.POINTER(P)]),
    "ktune_knob_histogram": (C.c_int, [P, P, P, C.c_int, i64, P, C.c_int]),
    "ktune_kmeans_run": (C.c_int, [P, P, P, C.c_int, i64, C.c_int, u64, C.c_int, C.c_int,
                                   C.POINTER(KmeansOutC), C.c_int]),
    "ktune_adaptive_sweep": (C.c_int, [P, P, P, C.c_int, P, i64, C.POINTER(SamplingParamsC), u64,
                                       C.POINTER(SweepOutC), C.c_int]),
    "ktune_snap": (C.c_int, [P, P, P, C.c_int, P, C.c_int, P, i64, P, C.c_int]),
    "ktune_adaptive_sample": (C.c_int, [P, P, P, P, i64, P, i64, C.POINTER(SamplingParamsC), u64,
                                        P, C.POINTER(C.c_int32)]),
    "ktune_synthesize_sample": (C.c_int, [P, P, i64, P, i64, C.POINTER(u64), P]),
    "ktune_debug_math": (C.c_int, [P, C.c_int, P, i64, P]),
    "ktune_debug_trace": (C.c_int, [P, P]),
}

_lib = None


def lib():
    """Load libktune_cuda.so (fails loudly: there is no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(make -f paper_2001_08743_b200/csrc/Makefile). The product has no CPU fallback.")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


_EXC = {ERR_CONFIG: ConfigError, ERR_BACKEND: BackendError, ERR_EXHAUSTED: SpaceExhaustedError,
        ERR_LOGIC: LogicError, ERR_CUDA: CudaError, ERR_NOMEM: BackendError}


def check(rc: int, ctx=None) -> None:
    if rc == KTUNE_OK:
        return
    msg = lib().ktune_last_error(ctx).decode(errors="replace")
    raise _EXC.get(rc, BackendError)(msg or f"ktune error {rc}")
