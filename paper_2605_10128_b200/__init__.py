"""B200-native DC N-1 MapElites engine (drop-in for the reference's hot path).

Host API mirroring /root/reference/proj/include/topopt over the C ABI of
libtopopt_b200.so (include/topopt_b200.h); see api.py.
"""
from .api import (ActionSet, CapacityError, ConfigError, CudaError, DcConfig, DcContext, FlowResult, Genome,
                  GridModel, IoError, IslandedContingency, OptimizerResult, OptimizerStats, ParseError, QdConfig,
                  RepertoireSnapshot, ScoreArrays, ScoreVector, SingularSystem, SnapshotChannel, SnapshotEntry,
                  TopoptError,
                  ValidationError, build_action_set, cell_count, descriptor_to_cell, grid_from_json_text,
                  kIslandedFitness, load_action_set, load_grid, run_optimizer, save_action_set, build_ptdf)
from . import ac  # noqa: E402,F401  (AC validation stage, ac_validator.hpp)
from .api import (QdSession, archive_replay, batch_ranks, context_stream, crossover_lanes,  # noqa: E402,F401
                  evaluate_raw, fp64_peak_tflops, mutate_lanes, sweep_chunks, sweep_rows, sweep_timing)

__all__ = [name for name in dir() if not name.startswith("_")]
