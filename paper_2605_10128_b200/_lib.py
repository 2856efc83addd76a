"""ctypes binding of libtopopt_b200.so (include/topopt_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2605_10128_b200/csrc``). There is no Python or CPU fallback
for the engine: if the library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# TGB_LIB_PATH: an alternative build of the same library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("TGB_LIB_PATH") or os.path.join(_HERE, "_lib", "libtopopt_b200.so")

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
u8p = C.POINTER(C.c_uint8)
u64p = C.POINTER(C.c_uint64)
f64p = C.POINTER(C.c_double)


class GridDesc(C.Structure):
    _fields_ = [
        ("n_nodes", C.c_int32), ("n_branches", C.c_int32), ("n_injections", C.c_int32), ("slack", C.c_int32),
        ("branch_from", i32p), ("branch_to", i32p), ("branch_x", f64p), ("branch_limit", f64p),
        ("branch_in_service", u8p), ("injection_node", i32p), ("injection_net_mw", f64p),
        ("n_contingencies", C.c_int32), ("cont_branch_ptr", i32p), ("cont_branch", i32p),
        ("cont_inj_ptr", i32p), ("cont_inj", i32p),
        ("n_substations", C.c_int32), ("sub_node", i32p), ("sub_term_ptr", i32p), ("term_kind", i32p),
        ("term_element", i32p),
        ("n_busbar_outages", C.c_int32), ("bo_substation", i32p), ("bo_busbar", i32p),
        ("bo_implied_ptr", i32p), ("bo_implied", i32p),
        ("n_timesteps", C.c_int32), ("injection_net_mw_t", f64p),
    ]


class ActionSetDesc(C.Structure):
    _fields_ = [
        ("n_actions", C.c_int32), ("action_substation", i32p), ("action_lambda_r", i32p),
        ("action_group_ptr", i32p), ("action_group", u8p), ("action_busbar_ptr", i32p),
        ("action_implied_ptr", i32p), ("action_implied", i32p),
        ("n_disconnectables", C.c_int32), ("disconnectables", i32p),
    ]


class DcConfigC(C.Structure):
    _fields_ = [("islanding_penalty_mw", C.c_double), ("worst_k", C.c_int32), ("weight_c0", C.c_double),
                ("weight_c", C.c_double), ("fitness_variant", C.c_int32), ("threads", C.c_int32)]


class ScoresC(C.Structure):
    _fields_ = [("lambda_o", f64p), ("lambda_c", i32p), ("lambda_c0", i32p), ("lambda_b", f64p),
                ("lambda_d", i32p), ("lambda_s", i32p), ("lambda_r", i32p), ("fitness", f64p),
                ("islanded", u8p), ("worst_idx", i32p), ("worst_energy", f64p), ("worst_n", i32p),
                ("islanded_outages", i32p), ("islanded_busbar_outages", i32p)]


class QdConfigC(C.Structure):
    _fields_ = [("n_a", C.c_int32), ("n_d", C.c_int32), ("batch_size", C.c_int32),
                ("iters_per_epoch", C.c_int32), ("cell_capacity", C.c_int32), ("mutation_mean", C.c_double),
                ("p_action", C.c_double * 4), ("p_disc", C.c_double * 4), ("p_crossover_parent1", C.c_double),
                ("d_max", C.c_int32), ("s_max", C.c_int32), ("r_max", C.c_int32), ("seed", C.c_uint64),
                ("max_evaluations", C.c_int64), ("max_seconds", C.c_double), ("rng", C.c_int32)]


class SnapshotView(C.Structure):
    _fields_ = [("epoch", C.c_int32), ("evaluations", C.c_int64), ("best_fitness", C.c_double),
                ("final_snapshot", C.c_int32), ("n_entries", C.c_int32), ("n_slots", C.c_int32),
                ("cell", i32p), ("genome", i32p), ("fitness", f64p), ("lambda_o", f64p),
                ("lambda_c", i32p), ("lambda_c0", i32p), ("lambda_b", f64p), ("lambda_d", i32p),
                ("lambda_s", i32p), ("lambda_r", i32p), ("worst_idx", i32p), ("worst_energy", f64p),
                ("worst_n", i32p), ("worst_k", C.c_int32)]


class OptStats(C.Structure):
    _fields_ = [("evaluations", C.c_int64), ("epochs", C.c_int32), ("n_trace", C.c_int32)]


class AcConfigC(C.Structure):
    _fields_ = [("tolerance_pu", C.c_double), ("max_iterations", C.c_int32), ("worst_k_nonconverged", C.c_int32),
                ("nonconverged_fraction", C.c_double), ("similarity_distance", C.c_int32),
                ("dominance_fitness_frac", C.c_double), ("improvement_threshold_frac", C.c_double)]


class AcBaselineC(C.Structure):
    _fields_ = [("lambda_o", C.c_double), ("critical_count", C.c_int32), ("base_converged", C.c_uint8),
                ("base_energy", C.c_double), ("pre_fitness", C.c_double)]


class AcCaseOutC(C.Structure):
    _fields_ = [("converged", u8p), ("iterations", i32p), ("overload_energy", f64p), ("critical_count", i32p),
                ("loading_mva", f64p), ("vm_pu", f64p), ("va_rad", f64p)]


SNAPSHOT_CB = C.CFUNCTYPE(None, C.POINTER(SnapshotView), C.c_void_p)

# (name, restype, argtypes) for every entry point of include/topopt_b200.h
SIGNATURES = [
    ("tg_last_error", C.c_char_p, []),
    ("tg_version", C.c_char_p, []),
    ("tg_free", None, [C.c_void_p]),
    ("tg_grid_from_json", C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(C.c_void_p)]),
    ("tg_grid_destroy", None, [C.c_void_p]),
    ("tg_grid_describe", C.c_int, [C.c_void_p, C.POINTER(GridDesc)]),
    ("tg_grid_to_json", C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    ("tg_grid_content_hash", C.c_int, [C.c_void_p, C.POINTER(C.c_uint64)]),
    ("tg_grid_branch_id", C.c_char_p, [C.c_void_p, C.c_int32]),
    ("tg_build_ptdf", C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_double)]),
    ("tg_actionset_build", C.c_int, [C.c_void_p, C.c_uint64, C.c_int64, C.POINTER(C.c_void_p)]),
    ("tg_actionset_build_device", C.c_int, [C.c_void_p, C.c_uint64, C.c_int64, C.c_int, C.POINTER(C.c_void_p)]),
    ("tg_actionset_from_json", C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_void_p)]),
    ("tg_actionset_to_json", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]),
    ("tg_actionset_destroy", None, [C.c_void_p]),
    ("tg_actionset_describe", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(ActionSetDesc)]),
    ("tg_context_create", C.c_int, [C.POINTER(GridDesc), C.POINTER(ActionSetDesc), C.POINTER(DcConfigC), C.c_int,
                                    C.POINTER(C.c_void_p)]),
    ("tg_context_destroy", None, [C.c_void_p]),
    ("tg_evaluate_batch", C.c_int, [C.c_void_p, i32p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                    C.POINTER(ScoresC), f64p, f64p, f64p, f64p]),
    ("tg_evaluate_batch_device", C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                           C.POINTER(ScoresC)]),
    ("tg_pre_score", C.c_int, [C.c_void_p, C.POINTER(ScoresC), f64p]),
    ("tg_optimizer_run", C.c_int, [C.c_void_p, C.POINTER(QdConfigC), SNAPSHOT_CB, C.c_void_p, i32p,
                                   C.POINTER(OptStats), i64p, f64p, C.c_int32]),
    ("tg_archive_export", C.c_int, [C.c_void_p, C.POINTER(SnapshotView)]),
    ("tg_archive_replay", C.c_int, [C.c_void_p, C.POINTER(QdConfigC), i32p, C.c_int32, C.POINTER(ScoresC), u8p]),
    ("tg_descriptor_to_cell", C.c_int32, [C.c_int32, C.c_int32, C.c_int32, C.POINTER(QdConfigC)]),
    ("tg_mutate_lanes", C.c_int, [C.c_void_p, C.POINTER(QdConfigC), i32p, u64p, C.c_int32, i32p]),
    ("tg_crossover_lanes", C.c_int, [C.c_void_p, C.POINTER(QdConfigC), i32p, i32p, u64p, C.c_int32, i32p]),
    ("tg_context_info", C.c_int, [C.c_void_p, i64p, C.c_int32]),
    ("tg_kernel_launches", C.c_int64, [C.c_void_p]),
    ("tg_qd_begin", C.c_int, [C.c_void_p, C.POINTER(QdConfigC)]),
    ("tg_qd_step", C.c_int, [C.c_void_p, C.c_int32]),
    ("tg_qd_fetch", C.c_int, [C.c_void_p, C.c_int32, C.POINTER(SnapshotView)]),
    ("tg_qd_offspring", C.c_int, [C.c_void_p, i32p]),
    ("tg_qd_insert", C.c_int, [C.c_void_p, i32p, C.POINTER(ScoresC)]),
    ("tg_context_stream", C.c_void_p, [C.c_void_p]),
    ("tg_sweep_timing", C.c_int, [C.c_void_p, C.c_int32, f64p, i64p]),
    ("tg_batch_ranks", C.c_int, [C.c_void_p, C.c_int32, i32p]),
    ("tg_sweep_rows", C.c_int, [C.c_void_p, i64p, i64p, i64p, i64p]),
    ("tg_sweep_chunks", C.c_int, [C.c_void_p, i64p, i64p]),
    ("tg_fp64_peak", C.c_int, [C.c_int, f64p]),
    ("tg_channel_create", C.c_void_p, [C.c_int64]),
    ("tg_channel_destroy", None, [C.c_void_p]),
    ("tg_channel_push", None, [C.c_void_p, C.POINTER(SnapshotView)]),
    ("tg_channel_sink", None, [C.POINTER(SnapshotView), C.c_void_p]),
    ("tg_channel_close", None, [C.c_void_p]),
    ("tg_channel_pop", C.c_int32, [C.c_void_p, C.c_int32, C.POINTER(SnapshotView)]),
    ("tg_channel_pending", C.c_int64, [C.c_void_p]),
    ("tg_channel_dropped", C.c_int64, [C.c_void_p]),
    ("tg_qd_generation_begin", C.c_int, [C.c_void_p]),
    ("tg_qd_evaluate_lanes", C.c_int, [C.c_void_p, C.c_int32, C.c_int32]),
    ("tg_qd_scores_blob_bytes", C.c_int, [C.c_void_p, C.c_int32, i64p]),
    ("tg_qd_scores_pack", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
    ("tg_qd_scores_unpack", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
    ("tg_qd_generation_end", C.c_int, [C.c_void_p]),
    ("tg_archive_blob_bytes", C.c_int, [C.c_void_p, i64p]),
    ("tg_archive_pack", C.c_int, [C.c_void_p, C.c_void_p]),
    ("tg_archive_merge", C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
    ("tg_islands_unique_id", C.c_int, [C.c_void_p]),
    ("tg_islands_create", C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
    ("tg_islands_destroy", None, [C.c_void_p]),
    ("tg_islands_exchange", C.c_int, [C.c_void_p]),
    ("tg_islands_step", C.c_int, [C.c_void_p, C.c_int32, C.c_int32]),
    ("tg_islands_shard_step", C.c_int, [C.c_void_p, C.c_int32, C.c_int32]),
    ("tg_ac_context_create", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(AcConfigC), C.c_int,
                                       C.POINTER(C.c_void_p)]),
    ("tg_ac_context_destroy", None, [C.c_void_p]),
    ("tg_ac_baseline_get", C.c_int, [C.c_void_p, C.POINTER(AcBaselineC), u8p, f64p]),
    ("tg_ac_run_cases", C.c_int, [C.c_void_p, i32p, C.c_int32, C.c_int32, C.c_int32, i32p, i32p, C.c_int32,
                                  C.POINTER(AcCaseOutC)]),
    ("tg_ac_worst_k_check", C.c_int, [C.c_void_p, i32p, C.c_int32, C.c_int32, C.c_int32, i32p, i32p, C.c_int32,
                                      i32p]),
    ("tg_ac_full_validation", C.c_int, [C.c_void_p, i32p, C.c_int32, C.c_int32, C.c_int32, i32p, u8p, f64p]),
    ("tg_ac_kernel_launches", C.c_int64, [C.c_void_p]),
]


def load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
            "(the engine has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


LIB = load()
