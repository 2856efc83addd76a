"""Python mirror of the reference's C++ API for the DC N-1 MapElites path.

Names, argument meaning and error kinds follow /root/reference/proj/include/topopt:
  grid_model.hpp:130-139  -> load_grid, grid_from_json_text, GridModel
  importer.hpp:80-94      -> build_action_set, load_action_set, save_action_set, ActionSet
  genome.hpp:13-47        -> Genome (canonical_key, counts)
  dc_engine.hpp:16-150    -> DcConfig, ScoreVector, FlowResult, DcContext
  qd_optimizer.hpp:15-118 -> QdConfig, descriptor_to_cell, cell_count, run_optimizer,
                             RepertoireSnapshot, OptimizerResult
Every call goes through the C ABI of libtopopt_b200.so (include/topopt_b200.h);
the evaluation runs on the GPU and there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import threading
import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib as L

LIB = L.LIB


# ---------------------------------------------------------------- errors (errors.hpp:9-34)
class TopoptError(RuntimeError):
    pass


class ParseError(TopoptError):
    pass


class ValidationError(TopoptError):
    pass


class IslandedContingency(TopoptError):
    pass


class SingularSystem(TopoptError):
    pass


class ConfigError(TopoptError):
    pass


class IoError(TopoptError):
    pass


class CudaError(TopoptError):
    pass


class CapacityError(TopoptError):
    pass


_ERRORS = {1: ParseError, 2: ValidationError, 3: IslandedContingency, 4: SingularSystem, 5: ConfigError,
           6: IoError, 7: CudaError, 8: CapacityError}


def _check(status: int) -> None:
    if status != 0:
        msg = LIB.tg_last_error().decode(errors="replace")
        raise _ERRORS.get(status, TopoptError)(msg)


def _ptr(arr: np.ndarray, ctype):
    return arr.ctypes.data_as(C.POINTER(ctype))


# ---------------------------------------------------------------- grid / actions
class GridModel:
    """Host network model (grid_model.hpp:80-127), owned by the C library."""

    def __init__(self, handle: C.c_void_p, text: str):
        self._h = handle
        self._text = text
        d = L.GridDesc()
        _check(LIB.tg_grid_describe(self._h, C.byref(d)))
        self.desc = d
        self.n_nodes = d.n_nodes
        self.n_branches = d.n_branches
        self.n_injections = d.n_injections
        self.n_contingencies = d.n_contingencies
        self.n_busbar_outages = d.n_busbar_outages
        self.n_substations = d.n_substations
        self.slack = d.slack
        E = d.n_branches
        self.branch_limit = np.ctypeslib.as_array(d.branch_limit, shape=(E,)).copy() if E else np.zeros(0)
        self.branch_from = np.ctypeslib.as_array(d.branch_from, shape=(E,)).copy() if E else np.zeros(0, np.int32)
        self.branch_to = np.ctypeslib.as_array(d.branch_to, shape=(E,)).copy() if E else np.zeros(0, np.int32)

    def to_json_text(self) -> str:
        """grid_to_json_text (grid_model.cpp:423-485): the canonical dump."""
        p = C.c_void_p()
        _check(LIB.tg_grid_to_json(self._h, C.byref(p)))
        try:
            return C.string_at(p).decode()
        finally:
            LIB.tg_free(p)

    def content_hash(self) -> int:
        """grid_content_hash (grid_model.cpp:494-503), the action-cache key."""
        h = C.c_uint64()
        _check(LIB.tg_grid_content_hash(self._h, C.byref(h)))
        return int(h.value)

    def __del__(self):
        if getattr(self, "_h", None):
            LIB.tg_grid_destroy(self._h)
            self._h = None


def grid_from_json_text(text: str) -> GridModel:
    raw = text.encode()
    h = C.c_void_p()
    _check(LIB.tg_grid_from_json(raw, len(raw), C.byref(h)))
    return GridModel(h, text)


def load_grid(path: str) -> GridModel:
    try:
        with open(path, "r", encoding="utf-8") as f:
            text = f.read()
    except OSError as exc:
        raise IoError(f"cannot open grid file '{path}'") from exc
    return grid_from_json_text(text)


class ActionSet:
    """Action encoding (importer.hpp:28-35): ids contiguous per substation."""

    def __init__(self, handle: C.c_void_p, grid: GridModel):
        self._h = handle
        self._grid = grid
        d = L.ActionSetDesc()
        _check(LIB.tg_actionset_describe(self._h, grid._h, C.byref(d)))
        self.desc = d
        A, D = d.n_actions, d.n_disconnectables
        self.substation = np.ctypeslib.as_array(d.action_substation, shape=(A,)).copy() if A else np.zeros(0, np.int32)
        self.lambda_r = np.ctypeslib.as_array(d.action_lambda_r, shape=(A,)).copy() if A else np.zeros(0, np.int32)
        gptr = np.ctypeslib.as_array(d.action_group_ptr, shape=(A + 1,)).copy()
        ng = int(gptr[-1])
        grp = np.ctypeslib.as_array(d.action_group, shape=(ng,)).copy() if ng else np.zeros(0, np.uint8)
        self.groups = [grp[gptr[a]:gptr[a + 1]].tolist() for a in range(A)]
        self.disconnectables = (np.ctypeslib.as_array(d.disconnectables, shape=(D,)).copy()
                                if D else np.zeros(0, np.int32))
        self.station_ranges = {}
        for a, s in enumerate(self.substation.tolist()):
            lo, hi = self.station_ranges.get(s, (a, a))
            self.station_ranges[s] = (lo, a + 1)

    @property
    def n_actions(self) -> int:
        return len(self.substation)

    def substation_of(self, action_id: int) -> int:
        return int(self.substation[action_id])

    def to_json_text(self) -> str:
        p = C.c_void_p()
        _check(LIB.tg_actionset_to_json(self._h, self._grid._h, C.byref(p)))
        try:
            return C.string_at(p).decode()
        finally:
            LIB.tg_free(p)

    def __del__(self):
        if getattr(self, "_h", None):
            LIB.tg_actionset_destroy(self._h)
            self._h = None


def build_action_set(grid: GridModel, seed: int = 0, cap: int = 1 << 23, device: Optional[int] = None) -> ActionSet:
    """build_action_set (importer.cpp:341-356). device=None: islanding validation on the
    host threads; device=k: on GPU k (tg_actionset_build_device). Same ids either way."""
    h = C.c_void_p()
    if device is None:
        _check(LIB.tg_actionset_build(grid._h, seed, cap, C.byref(h)))
    else:
        _check(LIB.tg_actionset_build_device(grid._h, seed, cap, device, C.byref(h)))
    return ActionSet(h, grid)


def build_ptdf(grid: GridModel, device: int = 0) -> np.ndarray:
    """build_ptdf (importer.cpp:358-401): PTDFMatrix::sensitivities [E, N]
    computed on the GPU (slack column and out-of-service rows zero)."""
    out = np.zeros((grid.n_branches, grid.n_nodes))
    _check(LIB.tg_build_ptdf(grid._h, device, _ptr(out, C.c_double)))
    return out


def save_action_set(actions: ActionSet, grid: GridModel, path: str) -> None:
    try:
        with open(path, "w", encoding="utf-8") as f:
            f.write(actions.to_json_text() + "\n")
    except OSError as exc:
        raise IoError(f"cannot write action cache '{path}'") from exc


def load_action_set(grid: GridModel, path: str) -> Optional[ActionSet]:
    try:
        with open(path, "r", encoding="utf-8") as f:
            raw = f.read().encode()
    except OSError:
        return None
    h = C.c_void_p()
    if LIB.tg_actionset_from_json(grid._h, raw, len(raw), C.byref(h)) != 0:
        return None
    return ActionSet(h, grid)


# ---------------------------------------------------------------- genome (genome.hpp:13-35)
@dataclass
class Genome:
    action_slots: List[int]
    disconnection_slots: List[int]

    @staticmethod
    def empty(n_a: int, n_d: int) -> "Genome":
        return Genome([-1] * n_a, [-1] * n_d)

    def split_count(self) -> int:
        return sum(1 for a in self.action_slots if a >= 0)

    def disconnection_count(self) -> int:
        return sum(1 for d in self.disconnection_slots if d >= 0)

    def is_empty(self) -> bool:
        return self.split_count() == 0 and self.disconnection_count() == 0

    def action_ids(self) -> List[int]:
        return sorted(a for a in self.action_slots if a >= 0)

    def disconnection_ids(self) -> List[int]:
        return sorted(d for d in self.disconnection_slots if d >= 0)

    def canonical_key(self) -> str:
        return ("a:" + "".join(f"{a}," for a in self.action_ids()) + "d:" +
                "".join(f"{d}," for d in self.disconnection_ids()))


# ---------------------------------------------------------------- DC engine
@dataclass
class DcConfig:
    islanding_penalty_mw: float = 10000.0
    worst_k: int = 20
    weight_c0: float = 200.0
    weight_c: float = 50.0
    fitness_variant: int = 1
    threads: int = 0

    def to_c(self) -> L.DcConfigC:
        return L.DcConfigC(self.islanding_penalty_mw, self.worst_k, self.weight_c0, self.weight_c,
                           self.fitness_variant, self.threads)


@dataclass
class ScoreVector:
    lambda_o: float = 0.0
    lambda_c: int = 0
    lambda_c0: int = 0
    lambda_b: float = 0.0
    lambda_d: int = 0
    lambda_s: int = 0
    lambda_r: int = 0
    fitness: float = 0.0
    islanded: bool = False
    worst_contingencies: List[Tuple[int, float]] = field(default_factory=list)


kIslandedFitness = -math.inf


class ScoreArrays:
    """Batch scores as numpy arrays (the SoA tg_scores of the C ABI)."""

    def __init__(self, n: int, worst_k: int):
        self.lambda_o = np.zeros(n)
        self.lambda_c = np.zeros(n, np.int32)
        self.lambda_c0 = np.zeros(n, np.int32)
        self.lambda_b = np.zeros(n)
        self.lambda_d = np.zeros(n, np.int32)
        self.lambda_s = np.zeros(n, np.int32)
        self.lambda_r = np.zeros(n, np.int32)
        self.fitness = np.zeros(n)
        self.islanded = np.zeros(n, np.uint8)
        self.worst_idx = np.full((n, max(worst_k, 1)), -1, np.int32)
        self.worst_energy = np.zeros((n, max(worst_k, 1)))
        self.worst_n = np.zeros(n, np.int32)
        self.islanded_outages = np.zeros(n, np.int32)
        self.islanded_busbar_outages = np.zeros(n, np.int32)

    def to_c(self) -> L.ScoresC:
        return L.ScoresC(_ptr(self.lambda_o, C.c_double), _ptr(self.lambda_c, C.c_int32),
                         _ptr(self.lambda_c0, C.c_int32), _ptr(self.lambda_b, C.c_double),
                         _ptr(self.lambda_d, C.c_int32), _ptr(self.lambda_s, C.c_int32),
                         _ptr(self.lambda_r, C.c_int32), _ptr(self.fitness, C.c_double),
                         _ptr(self.islanded, C.c_uint8), _ptr(self.worst_idx, C.c_int32),
                         _ptr(self.worst_energy, C.c_double), _ptr(self.worst_n, C.c_int32),
                         _ptr(self.islanded_outages, C.c_int32), _ptr(self.islanded_busbar_outages, C.c_int32))

    def score(self, i: int) -> ScoreVector:
        n = int(self.worst_n[i])
        return ScoreVector(float(self.lambda_o[i]), int(self.lambda_c[i]), int(self.lambda_c0[i]),
                           float(self.lambda_b[i]), int(self.lambda_d[i]), int(self.lambda_s[i]),
                           int(self.lambda_r[i]), float(self.fitness[i]), bool(self.islanded[i]),
                           [(int(self.worst_idx[i, k]), float(self.worst_energy[i, k])) for k in range(n)])


@dataclass
class FlowResult:
    base: np.ndarray
    max_contingency: np.ndarray
    max_busbar: np.ndarray
    outage_energy: np.ndarray
    islanded_outages: int
    islanded_busbar_outages: int


def _genome_array(genomes, n_a: Optional[int] = None, n_d: Optional[int] = None) -> Tuple[np.ndarray, int, int]:
    if isinstance(genomes, np.ndarray):
        if n_a is None or n_d is None:
            raise ConfigError("n_a and n_d are required with a genome array")
        return np.ascontiguousarray(genomes, dtype=np.int32).reshape(-1, n_a + n_d), n_a, n_d
    genomes = list(genomes)
    if not genomes:
        return np.zeros((0, 0), np.int32), n_a or 0, n_d or 0
    na = max(len(g.action_slots) for g in genomes)
    nd = max(len(g.disconnection_slots) for g in genomes)
    arr = np.full((len(genomes), na + nd), -1, np.int32)
    for i, g in enumerate(genomes):
        arr[i, :len(g.action_slots)] = g.action_slots
        arr[i, na:na + len(g.disconnection_slots)] = g.disconnection_slots
    return arr, na, nd


class DcContext:
    """Device-resident DcContext (dc_engine.hpp:95-150). Keeps the grid and
    action set alive like the reference's non-owning pointers require."""

    def __init__(self, grid: GridModel, actions: ActionSet, config: Optional[DcConfig] = None, device: int = 0):
        self.grid = grid
        self.actions = actions
        self.config = config or DcConfig()
        self._cfg_c = self.config.to_c()
        h = C.c_void_p()
        _check(LIB.tg_context_create(C.byref(grid.desc), C.byref(actions.desc), C.byref(self._cfg_c), device,
                                     C.byref(h)))
        self._h = h
        pre = ScoreArrays(1, 0)
        lbp = C.c_double()
        _check(LIB.tg_pre_score(self._h, C.byref(pre.to_c()), C.byref(lbp)))
        self._pre = pre.score(0)
        self._lambda_b_pre = lbp.value

    def close(self) -> None:
        if getattr(self, "_h", None):
            LIB.tg_context_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    # dc_engine.hpp:112-113
    def pre_optimization_score(self) -> ScoreVector:
        return self._pre

    def lambda_b_pre(self) -> float:
        return self._lambda_b_pre

    def evaluate_arrays(self, genomes, n_a: Optional[int] = None, n_d: Optional[int] = None,
                        batch_size: int = 0, flows: bool = False):
        """Scores (ScoreArrays) and optionally FlowResult arrays for a genome batch."""
        arr, na, nd = _genome_array(genomes, n_a, n_d)
        n = arr.shape[0]
        k = self.config.worst_k
        sc = ScoreArrays(n, k)
        if n == 0:
            return (sc, None) if flows else sc
        base = fmax = fbus = energy = None
        nullp = C.POINTER(C.c_double)()
        if flows:
            E, K = self.grid.n_branches, self.grid.n_contingencies
            base = np.zeros((n, E))
            fmax = np.zeros((n, E))
            fbus = np.zeros((n, E))
            energy = np.zeros((n, max(K, 1)))
        _check(LIB.tg_evaluate_batch(self._h, _ptr(arr, C.c_int32), n, na, nd, batch_size, C.byref(sc.to_c()),
                                     _ptr(base, C.c_double) if flows else nullp,
                                     _ptr(fmax, C.c_double) if flows else nullp,
                                     _ptr(fbus, C.c_double) if flows else nullp,
                                     _ptr(energy, C.c_double) if flows and self.grid.n_contingencies else nullp))
        if flows:
            return sc, FlowResult(base, fmax, fbus, energy[:, :self.grid.n_contingencies],
                                  sc.islanded_outages.copy(), sc.islanded_busbar_outages.copy())
        return sc

    # dc_engine.cpp:439-468
    def evaluate_batch(self, genomes: Sequence[Genome], batch_size: int = 0) -> List[ScoreVector]:
        sc = self.evaluate_arrays(genomes, batch_size=batch_size)
        return [sc.score(i) for i in range(len(sc.fitness))]

    # dc_engine.cpp:424-437
    def evaluate(self, genome: Genome) -> ScoreVector:
        return self.evaluate_batch([genome])[0]

    def screen(self, genome: Genome) -> FlowResult:
        _, fr = self.evaluate_arrays([genome], flows=True)
        return fr

    def kernel_launches(self) -> int:
        return int(LIB.tg_kernel_launches(self._h))

    def info(self) -> dict:
        v = np.zeros(10, np.int64)
        _check(LIB.tg_context_info(self._h, _ptr(v, C.c_int64), 10))
        keys = ["n_nodes", "n_branches", "n_contingencies", "n_single", "n_special", "n_busbar_outages",
                "n_actions", "n_disconnectables", "k_padded", "device_bytes"]
        return dict(zip(keys, v.tolist()))


# ---------------------------------------------------------------- QD (qd_optimizer.hpp)
@dataclass
class QdConfig:
    n_a: int = 3
    n_d: int = 2
    batch_size: int = 64
    iters_per_epoch: int = 500
    cell_capacity: int = 4
    mutation_mean: float = 2.0
    p_action: Tuple[float, float, float, float] = (0.2, 0.2, 0.5, 0.1)
    p_disc: Tuple[float, float, float, float] = (0.25, 0.25, 0.5, 0.0)
    p_crossover_parent1: float = 0.75
    d_max: int = 2
    s_max: int = 3
    r_max: int = 45
    seed: int = 1
    max_evaluations: int = -1
    max_seconds: float = -1.0
    # lane RNG: "replay" = the reference's per-lane std::mt19937_64 stream bit
    # for bit; "philox" = counter-based Philox4x32-10 (extension, same distributions)
    rng: str = "replay"

    def to_c(self) -> L.QdConfigC:
        c = L.QdConfigC()
        c.n_a, c.n_d, c.batch_size, c.iters_per_epoch = self.n_a, self.n_d, self.batch_size, self.iters_per_epoch
        c.cell_capacity, c.mutation_mean = self.cell_capacity, self.mutation_mean
        for i in range(4):
            c.p_action[i] = self.p_action[i]
            c.p_disc[i] = self.p_disc[i]
        c.p_crossover_parent1 = self.p_crossover_parent1
        c.d_max, c.s_max, c.r_max = self.d_max, self.s_max, self.r_max
        c.seed, c.max_evaluations, c.max_seconds = self.seed, self.max_evaluations, self.max_seconds
        if self.rng not in ("replay", "philox"):
            raise ConfigError(f"rng must be 'replay' or 'philox', not {self.rng!r}")
        c.rng = 1 if self.rng == "philox" else 0
        return c


def cell_count(cfg: QdConfig) -> int:
    return (cfg.d_max + 1) * (cfg.s_max + 1) * (cfg.r_max + 1)


def descriptor_to_cell(lambda_d: int, lambda_s: int, lambda_r: int, cfg: QdConfig) -> int:
    return int(LIB.tg_descriptor_to_cell(lambda_d, lambda_s, lambda_r, C.byref(cfg.to_c())))


@dataclass
class SnapshotEntry:
    cell: int
    genome: Genome
    score: ScoreVector


@dataclass
class RepertoireSnapshot:
    epoch: int
    evaluations: int
    best_fitness: float
    final: bool
    entries: List[SnapshotEntry]


def _snapshot_from_view(v: L.SnapshotView, n_a: int) -> RepertoireSnapshot:
    n, ns, k = v.n_entries, v.n_slots, v.worst_k
    entries = []
    for i in range(n):
        g = [v.genome[i * ns + j] for j in range(ns)]
        wn = v.worst_n[i]
        sc = ScoreVector(v.lambda_o[i], v.lambda_c[i], v.lambda_c0[i], v.lambda_b[i], v.lambda_d[i],
                         v.lambda_s[i], v.lambda_r[i], v.fitness[i], False,
                         [(v.worst_idx[i * k + j], v.worst_energy[i * k + j]) for j in range(wn)])
        entries.append(SnapshotEntry(v.cell[i], Genome(g[:n_a], g[n_a:]), sc))
    return RepertoireSnapshot(v.epoch, v.evaluations, v.best_fitness, bool(v.final_snapshot), entries)


@dataclass
class OptimizerStats:
    evaluations: int
    epochs: int
    fitness_trace: List[Tuple[int, float]]


@dataclass
class OptimizerResult:
    repertoire: RepertoireSnapshot
    stats: OptimizerStats


class SnapshotChannel:
    """SnapshotChannel (channel.hpp:15-79) in native code: single-producer
    single-consumer queue; a bounded channel never blocks the producer, when
    full the oldest non-final snapshot is dropped; capacity 0 = unbounded.
    Passed to run_optimizer(channel=...), the device loop feeds it from C++
    (tg_channel_sink) while a consumer thread pops (the AC stage,
    pipeline.cpp:354-425)."""

    def __init__(self, capacity: int = 0, n_a: int = 3):
        self._h = LIB.tg_channel_create(int(capacity))
        if not self._h:
            raise TopoptError("channel allocation failed")
        self.n_a = n_a

    def push(self, snap: RepertoireSnapshot) -> None:
        n = len(snap.entries)
        ns = len(snap.entries[0].genome.action_slots) + len(snap.entries[0].genome.disconnection_slots) if n else 0
        wk = max([len(e.score.worst_contingencies) for e in snap.entries] + [0])
        arr = {
            "cell": np.array([e.cell for e in snap.entries], np.int32),
            "genome": np.array([e.genome.action_slots + e.genome.disconnection_slots for e in snap.entries],
                               np.int32).reshape(-1),
            "fitness": np.array([e.score.fitness for e in snap.entries]),
            "lambda_o": np.array([e.score.lambda_o for e in snap.entries]),
            "lambda_c": np.array([e.score.lambda_c for e in snap.entries], np.int32),
            "lambda_c0": np.array([e.score.lambda_c0 for e in snap.entries], np.int32),
            "lambda_b": np.array([e.score.lambda_b for e in snap.entries]),
            "lambda_d": np.array([e.score.lambda_d for e in snap.entries], np.int32),
            "lambda_s": np.array([e.score.lambda_s for e in snap.entries], np.int32),
            "lambda_r": np.array([e.score.lambda_r for e in snap.entries], np.int32),
            "worst_n": np.array([len(e.score.worst_contingencies) for e in snap.entries], np.int32),
            "worst_idx": np.zeros(n * wk, np.int32), "worst_energy": np.zeros(n * wk),
        }
        for i, e in enumerate(snap.entries):
            for j, (k, v) in enumerate(e.score.worst_contingencies):
                arr["worst_idx"][i * wk + j] = k
                arr["worst_energy"][i * wk + j] = v
        v = L.SnapshotView()
        v.epoch, v.evaluations, v.best_fitness = snap.epoch, snap.evaluations, snap.best_fitness
        v.final_snapshot, v.n_entries, v.n_slots, v.worst_k = int(snap.final), n, ns, wk
        for name, a in arr.items():
            setattr(v, name, _ptr(a, C.c_double if a.dtype == np.float64 else C.c_int32))
        LIB.tg_channel_push(self._h, C.byref(v))

    def close(self) -> None:
        LIB.tg_channel_close(self._h)

    def _pop(self, blocking: bool) -> Optional[RepertoireSnapshot]:
        v = L.SnapshotView()
        if not LIB.tg_channel_pop(self._h, int(blocking), C.byref(v)):
            return None
        return _snapshot_from_view(v, self.n_a)

    def pop(self) -> Optional[RepertoireSnapshot]:
        """Blocks until a snapshot arrives or the channel is closed and drained."""
        return self._pop(True)

    def try_pop(self) -> Optional[RepertoireSnapshot]:
        return self._pop(False)

    def has_pending(self) -> bool:
        return LIB.tg_channel_pending(self._h) > 0

    def dropped(self) -> int:
        return int(LIB.tg_channel_dropped(self._h))

    def __del__(self):
        if getattr(self, "_h", None):
            LIB.tg_channel_destroy(self._h)
            self._h = None


def run_optimizer(ctx: DcContext, cfg: QdConfig, sink: Optional[Callable[[RepertoireSnapshot], None]] = None,
                  stop=None, channel: Optional[SnapshotChannel] = None) -> OptimizerResult:
    """run_optimizer (qd_optimizer.cpp:344-417) on the device-resident loop.
    Snapshots go to `sink` (Python callable, called on this thread) or, with
    `channel`, straight into a native SnapshotChannel."""
    ccfg = cfg.to_c()
    errors: List[BaseException] = []

    def _cb(view_p, _user):
        if sink is None:
            return
        try:
            sink(_snapshot_from_view(view_p.contents, cfg.n_a))
        except BaseException as exc:  # surfaced after the run
            errors.append(exc)

    if channel is not None:
        if sink is not None:
            raise ConfigError("pass either sink or channel")
        cb = C.cast(LIB.tg_channel_sink, L.SNAPSHOT_CB)
        user = C.c_void_p(channel._h)
    else:
        cb = L.SNAPSHOT_CB(_cb)
        user = None
    stats = L.OptStats()
    cap = 1 << 16
    tev = np.zeros(cap, np.int64)
    tbest = np.zeros(cap)
    # `stop` (the reference's std::atomic<bool>*, qd_optimizer.hpp:116-118) is
    # polled by the native loop: a threading.Event is mirrored into a private
    # int32 flag; an array must already be a contiguous int32 buffer (a copy
    # would never see the caller's store)
    watcher = None
    done = None
    if stop is None:
        stop_arr = None
    elif isinstance(stop, threading.Event):
        stop_arr = np.zeros(1, np.int32)
        done = threading.Event()

        def _mirror():
            while not done.is_set():
                if stop.wait(0.005):
                    stop_arr[0] = 1
                    return
        watcher = threading.Thread(target=_mirror, daemon=True)
        watcher.start()
    else:
        if not (isinstance(stop, np.ndarray) and stop.dtype == np.int32 and stop.size >= 1
                and stop.flags["C_CONTIGUOUS"]):
            raise ConfigError("stop must be a threading.Event or a contiguous numpy int32 array")
        stop_arr = stop
    stop_p = _ptr(stop_arr, C.c_int32) if stop_arr is not None else C.POINTER(C.c_int32)()
    try:
        _check(LIB.tg_optimizer_run(ctx._h, C.byref(ccfg), cb, user, stop_p, C.byref(stats), _ptr(tev, C.c_int64),
                                    _ptr(tbest, C.c_double), cap))
    finally:
        if watcher is not None:
            done.set()
            watcher.join()
    if errors:
        raise errors[0]
    view = L.SnapshotView()
    _check(LIB.tg_archive_export(ctx._h, C.byref(view)))
    rep = _snapshot_from_view(view, cfg.n_a)
    trace = [(int(tev[i]), float(tbest[i])) for i in range(stats.n_trace)]
    return OptimizerResult(rep, OptimizerStats(int(stats.evaluations), int(stats.epochs), trace))


# ---------------------------------------------------------------- device operator access (parity tests)
def mutate_lanes(ctx: DcContext, cfg: QdConfig, parents: np.ndarray, seeds: np.ndarray) -> np.ndarray:
    """mutate() (qd_optimizer.cpp:202-210) on the device, one lane per (parent, seed)."""
    par = np.ascontiguousarray(parents, np.int32).reshape(-1, cfg.n_a + cfg.n_d)
    sd = np.ascontiguousarray(seeds, np.uint64)
    out = np.zeros_like(par)
    c = cfg.to_c()
    _check(LIB.tg_mutate_lanes(ctx._h, C.byref(c), _ptr(par, C.c_int32), _ptr(sd, C.c_uint64), par.shape[0],
                               _ptr(out, C.c_int32)))
    return out


def crossover_lanes(ctx: DcContext, cfg: QdConfig, p1: np.ndarray, p2: np.ndarray, seeds: np.ndarray) -> np.ndarray:
    """crossover() (qd_optimizer.cpp:235-277) on the device, one lane per entry."""
    a = np.ascontiguousarray(p1, np.int32).reshape(-1, cfg.n_a + cfg.n_d)
    b = np.ascontiguousarray(p2, np.int32).reshape(-1, cfg.n_a + cfg.n_d)
    sd = np.ascontiguousarray(seeds, np.uint64)
    out = np.zeros_like(a)
    c = cfg.to_c()
    _check(LIB.tg_crossover_lanes(ctx._h, C.byref(c), _ptr(a, C.c_int32), _ptr(b, C.c_int32),
                                  _ptr(sd, C.c_uint64), a.shape[0], _ptr(out, C.c_int32)))
    return out


def archive_replay(ctx: DcContext, cfg: QdConfig, genomes: np.ndarray, scores: ScoreArrays):
    """Repertoire::insert (qd_optimizer.cpp:281-303) replayed on the device archive;
    returns (per-insert results, snapshot of the archive)."""
    g = np.ascontiguousarray(genomes, np.int32).reshape(-1, cfg.n_a + cfg.n_d)
    n = g.shape[0]
    ins = np.zeros(n, np.uint8)
    c = cfg.to_c()
    _check(LIB.tg_archive_replay(ctx._h, C.byref(c), _ptr(g, C.c_int32), n, C.byref(scores.to_c()),
                                 _ptr(ins, C.c_uint8)))
    view = L.SnapshotView()
    _check(LIB.tg_archive_export(ctx._h, C.byref(view)))
    return ins.astype(bool), _snapshot_from_view(view, cfg.n_a)


class QdSession:
    """Step-wise run_optimizer (tg_qd_begin / tg_qd_step / tg_qd_fetch): the
    loop the reference runs between two snapshots, with generations enqueued on
    the device without host synchronization."""

    def __init__(self, ctx: DcContext, cfg: QdConfig):
        self.ctx = ctx
        self.cfg = cfg
        self._c = cfg.to_c()
        _check(LIB.tg_qd_begin(ctx._h, C.byref(self._c)))

    def step(self, n_iters: int = 1) -> None:
        _check(LIB.tg_qd_step(self.ctx._h, n_iters))

    def offspring(self) -> np.ndarray:
        """This generation's lanes (device mutation / crossover), without evaluating them."""
        out = np.zeros((self.cfg.batch_size, self.cfg.n_a + self.cfg.n_d), np.int32)
        _check(LIB.tg_qd_offspring(self.ctx._h, _ptr(out, C.c_int32)))
        return out

    def insert(self, genomes: np.ndarray, scores: ScoreArrays) -> None:
        """Insert externally scored lanes in lane order and advance the generation."""
        g = np.ascontiguousarray(genomes, np.int32)
        _check(LIB.tg_qd_insert(self.ctx._h, _ptr(g, C.c_int32), C.byref(scores.to_c())))

    def fetch(self, final: bool = False) -> RepertoireSnapshot:
        view = L.SnapshotView()
        _check(LIB.tg_qd_fetch(self.ctx._h, int(final), C.byref(view)))
        return _snapshot_from_view(view, self.cfg.n_a)

    # ---- batch-sharded generation (islands.py: BatchShard drives these)
    def generation_begin(self) -> None:
        _check(LIB.tg_qd_generation_begin(self.ctx._h))

    def evaluate_lanes(self, lo: int, hi: int) -> None:
        _check(LIB.tg_qd_evaluate_lanes(self.ctx._h, lo, hi))

    def scores_blob_bytes(self, n: int) -> int:
        v = C.c_int64()
        _check(LIB.tg_qd_scores_blob_bytes(self.ctx._h, n, C.byref(v)))
        return v.value

    def scores_pack(self, lo: int, hi: int, d_blob: int) -> None:
        _check(LIB.tg_qd_scores_pack(self.ctx._h, lo, hi, C.c_void_p(d_blob)))

    def scores_unpack(self, lo: int, hi: int, d_blob: int) -> None:
        _check(LIB.tg_qd_scores_unpack(self.ctx._h, lo, hi, C.c_void_p(d_blob)))

    def generation_end(self) -> None:
        _check(LIB.tg_qd_generation_end(self.ctx._h))

    # ---- island exchange (islands.py drives these over torch.distributed)
    def blob_bytes(self) -> int:
        v = C.c_int64()
        _check(LIB.tg_archive_blob_bytes(self.ctx._h, C.byref(v)))
        return v.value

    def pack(self, d_blob: int) -> None:
        """Enqueue the archive -> island blob copy into device memory at d_blob."""
        _check(LIB.tg_archive_pack(self.ctx._h, C.c_void_p(d_blob)))

    def merge(self, d_blobs: int, n_islands: int) -> None:
        """Enqueue the merge of n_islands consecutive device blobs into the archive."""
        _check(LIB.tg_archive_merge(self.ctx._h, C.c_void_p(d_blobs), n_islands))


def context_stream(ctx: DcContext) -> int:
    """cudaStream_t of the context (for caller-side CUDA events)."""
    return int(LIB.tg_context_stream(ctx._h) or 0)


def sweep_timing(ctx: DcContext, enable: bool) -> Tuple[float, int]:
    """Toggle live event timing of the fused sweep; returns (ms, launches) so far."""
    ms = C.c_double()
    n = C.c_int64()
    _check(LIB.tg_sweep_timing(ctx._h, int(enable), C.byref(ms), C.byref(n)))
    return ms.value, n.value


def batch_ranks(ctx: DcContext, n: int) -> np.ndarray:
    out = np.zeros(n, np.int32)
    _check(LIB.tg_batch_ranks(ctx._h, n, _ptr(out, C.c_int32)))
    return out


def fp64_peak_tflops(device: int = 0) -> float:
    v = C.c_double()
    _check(LIB.tg_fp64_peak(device, C.byref(v)))
    return v.value


def evaluate_raw(ctx: DcContext, genomes_ptr: int, n: int, n_a: int, n_d: int, scores: "L.ScoresC") -> None:
    """tg_evaluate_batch on caller-owned host buffers given as raw pointers
    (e.g. pinned memory): H2D genomes, evaluate, D2H scores."""
    nullp = C.POINTER(C.c_double)()
    _check(LIB.tg_evaluate_batch(ctx._h, C.cast(C.c_void_p(genomes_ptr), C.POINTER(C.c_int32)), n, n_a, n_d, n,
                                 C.byref(scores), nullp, nullp, nullp, nullp))


def sweep_rows(ctx: DcContext) -> Tuple[int, int, int, int]:
    """(computed, offered, overloaded, partial) (branch row x candidate-warp x tile)
    blocks of the sweep since the last call: `partial` passed the per-row bound
    (first FMA computed), `computed` also passed the per-element bound (all
    FMAs), `overloaded` took the exact (overload) path."""
    a = C.c_int64()
    b = C.c_int64()
    o = C.c_int64()
    p = C.c_int64()
    _check(LIB.tg_sweep_rows(ctx._h, C.byref(a), C.byref(b), C.byref(o), C.byref(p)))
    return a.value, b.value, o.value, p.value


def sweep_chunks(ctx: DcContext) -> Tuple[int, int]:
    """(chunk tests, hot chunks) of the chunked scores-only sweep since the last call (resets)."""
    a, h = C.c_int64(), C.c_int64()
    _check(LIB.tg_sweep_chunks(ctx._h, C.byref(a), C.byref(h)))
    return a.value, h.value
