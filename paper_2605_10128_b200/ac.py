"""Python mirror of the reference's AC validation stage (ac_validator.hpp:18-140).

  AcConfig, AcCaseResult, AcNetwork, ac_power_flow   ac_validator.hpp:18-56
  RejectionReason, ValidationStage, ValidationRecord,
  Candidate, EliminationOutcome, AcValidator,
  record_to_json                                      ac_validator.hpp:58-140

Every power flow runs on the GPU behind the C ABI (tg_ac_*, include/topopt_b200.h):
the cases of a call are solved together, one CTA per (genome, contingency)
case. The host keeps the reference's decision logic that is not numeric work:
eliminate() (similarity, dominance, improvement threshold) and the validation
history. AcValidator.validate_queue() validates a whole elimination queue
with two device batches (worst-k stage for every candidate, then full N-1 for
the survivors) and records exactly what a loop of validate() calls records
(validate() does not depend on earlier validations, ac_validator.cpp:475-495).
"""
from __future__ import annotations

import ctypes as C
import enum
import json
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _lib as L
from .api import (ActionSet, ConfigError, DcContext, Genome, GridModel, ScoreVector, _check, _genome_array, _ptr)

LIB = L.LIB


@dataclass
class AcConfig:
    tolerance_pu: float = 1e-6
    max_iterations: int = 30
    worst_k_nonconverged: int = 2
    nonconverged_fraction: float = 0.05
    similarity_distance: int = 1
    dominance_fitness_frac: float = 0.01
    improvement_threshold_frac: float = 0.05

    def to_c(self) -> L.AcConfigC:
        return L.AcConfigC(self.tolerance_pu, self.max_iterations, self.worst_k_nonconverged,
                           self.nonconverged_fraction, self.similarity_distance, self.dominance_fitness_frac,
                           self.improvement_threshold_frac)


@dataclass
class AcCaseResult:
    converged: bool
    iterations: int
    loading_mva: np.ndarray
    vm_pu: np.ndarray
    va_rad: np.ndarray


class RejectionReason(enum.IntEnum):
    None_ = 0
    Nonconvergence = 1
    OverloadNotImproved = 2
    CriticalCountIncreased = 3
    EliminatedSimilar = 4
    EliminatedDominated = 5
    EliminatedBelowThreshold = 6


_REASON_NAMES = ["none", "nonconvergence", "overload_not_improved", "critical_count_increased",
                 "eliminated_similar", "eliminated_dominated", "eliminated_below_threshold"]


def to_string(reason: RejectionReason) -> str:
    """ac_validator.cpp:295-311"""
    return _REASON_NAMES[int(reason)]


class ValidationStage(enum.IntEnum):
    None_ = 0
    WorstK = 1
    FullN1 = 2


@dataclass
class ValidationRecord:
    genome: Genome
    dc_score: ScoreVector
    stage: ValidationStage = ValidationStage.None_
    accepted: bool = False
    reason: RejectionReason = RejectionReason.None_
    ac_lambda_o: float = 0.0


@dataclass
class Candidate:
    genome: Genome
    dc_score: ScoreVector


@dataclass
class EliminationOutcome:
    queue: List[int] = field(default_factory=list)
    pruned: List[Tuple[int, RejectionReason]] = field(default_factory=list)


def genome_distance(a: Genome, b: Genome) -> int:
    """genome.cpp:64-73: symmetric differences of the action and disconnection id sets."""
    return (len(set(a.action_ids()) ^ set(b.action_ids())) +
            len(set(a.disconnection_ids()) ^ set(b.disconnection_ids())))


class AcContext:
    """Device tables of the AC stage plus the baseline of the unchanged grid
    (AcValidator constructor, ac_validator.cpp:313-343)."""

    def __init__(self, grid: GridModel, actions: ActionSet, dc: Optional[DcContext] = None,
                 config: Optional[AcConfig] = None, device: int = 0):
        self.grid, self.actions, self.dc = grid, actions, dc
        self.config = config or AcConfig()
        self._cfg_c = self.config.to_c()
        h = C.c_void_p()
        _check(LIB.tg_ac_context_create(grid._h, actions._h, dc._h if dc is not None else None,
                                        C.byref(self._cfg_c), device, C.byref(h)))
        self._h = h
        b = L.AcBaselineC()
        K = grid.n_contingencies
        self.case_converged = np.zeros(max(K, 1), np.uint8)
        self.case_energy = np.zeros(max(K, 1))
        _check(LIB.tg_ac_baseline_get(self._h, C.byref(b), _ptr(self.case_converged, C.c_uint8),
                                      _ptr(self.case_energy, C.c_double)))
        self.case_converged = self.case_converged[:K].astype(bool)
        self.case_energy = self.case_energy[:K]
        self.baseline_lambda_o = b.lambda_o
        self.baseline_critical_count = b.critical_count
        self.baseline_base_converged = bool(b.base_converged)
        self.baseline_base_energy = b.base_energy
        self.pre_fitness = b.pre_fitness

    def close(self) -> None:
        if getattr(self, "_h", None):
            LIB.tg_ac_context_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def kernel_launches(self) -> int:
        return int(LIB.tg_ac_kernel_launches(self._h))

    def run_cases(self, genomes, case_genome, case_contingency, n_a: Optional[int] = None,
                  n_d: Optional[int] = None, loading: bool = True, voltages: bool = True) -> dict:
        """AcNetwork(grid, apply_genome(genomes[case_genome[i]])).run_case(case_contingency[i])
        for every i (ac_validator.cpp:26-272), overload_energy / critical_count included."""
        arr, na, nd = _genome_array(genomes, n_a, n_d)
        cg = np.ascontiguousarray(case_genome, np.int32)
        ck = np.ascontiguousarray(case_contingency, np.int32)
        n = len(cg)
        if len(ck) != n:
            raise ConfigError("case_genome and case_contingency differ in length")
        E, V = self.grid.n_branches, self.grid.n_nodes + na
        out = {"converged": np.zeros(n, np.uint8), "iterations": np.zeros(n, np.int32),
               "overload_energy": np.zeros(n), "critical_count": np.zeros(n, np.int32)}
        if loading:
            out["loading_mva"] = np.zeros((n, E))
        if voltages:
            out["vm_pu"] = np.zeros((n, V))
            out["va_rad"] = np.zeros((n, V))
        nullp = C.POINTER(C.c_double)()
        o = L.AcCaseOutC(_ptr(out["converged"], C.c_uint8), _ptr(out["iterations"], C.c_int32),
                         _ptr(out["overload_energy"], C.c_double), _ptr(out["critical_count"], C.c_int32),
                         _ptr(out["loading_mva"], C.c_double) if loading else nullp,
                         _ptr(out["vm_pu"], C.c_double) if voltages else nullp,
                         _ptr(out["va_rad"], C.c_double) if voltages else nullp)
        if n:
            _check(LIB.tg_ac_run_cases(self._h, _ptr(arr, C.c_int32), arr.shape[0], na, nd, _ptr(cg, C.c_int32),
                                       _ptr(ck, C.c_int32), n, C.byref(o)))
        out["converged"] = out["converged"].astype(bool)
        return out

    def worst_k_check_arrays(self, genomes, worst_idx: np.ndarray, worst_n: np.ndarray, n_a=None, n_d=None):
        arr, na, nd = _genome_array(genomes, n_a, n_d)
        n = arr.shape[0]
        wi = np.ascontiguousarray(worst_idx, np.int32).reshape(n, -1)
        wn = np.ascontiguousarray(worst_n, np.int32)
        reason = np.zeros(n, np.int32)
        if n:
            _check(LIB.tg_ac_worst_k_check(self._h, _ptr(arr, C.c_int32), n, na, nd, _ptr(wi, C.c_int32),
                                           _ptr(wn, C.c_int32), wi.shape[1], _ptr(reason, C.c_int32)))
        return reason

    def full_validation_arrays(self, genomes, n_a=None, n_d=None):
        arr, na, nd = _genome_array(genomes, n_a, n_d)
        n = arr.shape[0]
        reason = np.zeros(n, np.int32)
        acc = np.zeros(n, np.uint8)
        lo = np.zeros(n)
        if n:
            _check(LIB.tg_ac_full_validation(self._h, _ptr(arr, C.c_int32), n, na, nd, _ptr(reason, C.c_int32),
                                             _ptr(acc, C.c_uint8), _ptr(lo, C.c_double)))
        return reason, acc.astype(bool), lo


class AcNetwork:
    """AcNetwork(grid, apply_genome(genome)) (ac_validator.hpp:38-56); cases solve on the GPU."""

    def __init__(self, ctx: AcContext, genome: Genome):
        self.ctx, self.genome = ctx, genome

    def run_cases(self, contingencies: Sequence[int]) -> List[AcCaseResult]:
        ks = list(contingencies)
        r = self.ctx.run_cases([self.genome], [0] * len(ks), ks)
        return [AcCaseResult(bool(r["converged"][i]), int(r["iterations"][i]), r["loading_mva"][i],
                             r["vm_pu"][i], r["va_rad"][i]) for i in range(len(ks))]

    def run_case(self, contingency: int) -> AcCaseResult:
        return self.run_cases([contingency])[0]

    def overload_energy(self, r: AcCaseResult) -> float:
        lim = self.ctx.grid.branch_limit
        return float(np.sum(np.maximum(r.loading_mva - lim, 0.0)))

    def critical_count(self, r: AcCaseResult) -> int:
        return int(np.sum(r.loading_mva > self.ctx.grid.branch_limit))


def ac_power_flow(ctx: AcContext, genome: Genome) -> AcCaseResult:
    return AcNetwork(ctx, genome).run_case(-1)


def _swd(s: ScoreVector) -> int:
    return s.lambda_d + s.lambda_s + s.lambda_r


class AcValidator:
    """AcValidator (ac_validator.hpp:93-140): baseline on construction, the
    power-flow stages on the GPU, elimination and history on the host."""

    def __init__(self, grid: GridModel, actions: ActionSet, dc: DcContext, config: Optional[AcConfig] = None,
                 device: int = 0):
        self.ctx = AcContext(grid, actions, dc, config, device)
        self.grid, self.actions, self.dc = grid, actions, dc
        self._config = self.ctx.config
        self._pre = dc.pre_optimization_score().fitness
        self._validated: List[Tuple[Genome, int, float]] = []
        self._records: List[ValidationRecord] = []

    def config(self) -> AcConfig:
        return self._config

    def baseline_lambda_o(self) -> float:
        return self.ctx.baseline_lambda_o

    def baseline_critical_count(self) -> int:
        return self.ctx.baseline_critical_count

    def records(self) -> List[ValidationRecord]:
        return self._records

    # ac_validator.cpp:345-397
    def eliminate(self, candidates: Sequence[Candidate]) -> EliminationOutcome:
        eps = self._config.dominance_fitness_frac * abs(self._pre)
        theta = self._config.improvement_threshold_frac * abs(self._pre)
        out = EliminationOutcome()
        for i, c in enumerate(candidates):
            mine = _swd(c.dc_score)

            def dominated_by(other_swd, other_fit):
                return other_swd < mine and other_fit >= c.dc_score.fitness - eps

            why = RejectionReason.None_
            if any(genome_distance(c.genome, g) <= self._config.similarity_distance for g, _, _ in self._validated):
                why = RejectionReason.EliminatedSimilar
            elif any(dominated_by(_swd(o.dc_score), o.dc_score.fitness) for o in candidates):
                why = RejectionReason.EliminatedDominated
            elif any(dominated_by(s, f) for _, s, f in self._validated):
                why = RejectionReason.EliminatedDominated
            elif not np.isfinite(c.dc_score.fitness) or c.dc_score.fitness - self._pre < theta:
                why = RejectionReason.EliminatedBelowThreshold
            if why == RejectionReason.None_:
                out.queue.append(i)
            else:
                out.pruned.append((i, why))
        out.queue.sort(key=lambda i: (-candidates[i].dc_score.fitness, candidates[i].genome.canonical_key()))
        return out

    @staticmethod
    def _worst_arrays(scores: Sequence[ScoreVector]):
        k = max([len(s.worst_contingencies) for s in scores] + [1])
        wi = np.full((len(scores), k), -1, np.int32)
        wn = np.zeros(len(scores), np.int32)
        for i, s in enumerate(scores):
            wn[i] = len(s.worst_contingencies)
            for j, (c, _) in enumerate(s.worst_contingencies):
                wi[i, j] = c
        return wi, wn

    def worst_k_check_batch(self, genomes: Sequence[Genome], scores: Sequence[ScoreVector]) -> List[RejectionReason]:
        if not genomes:
            return []
        wi, wn = self._worst_arrays(scores)
        return [RejectionReason(int(r)) for r in self.ctx.worst_k_check_arrays(genomes, wi, wn)]

    # ac_validator.cpp:399-425
    def worst_k_check(self, genome: Genome, dc_score: ScoreVector) -> RejectionReason:
        return self.worst_k_check_batch([genome], [dc_score])[0]

    def full_validation_batch(self, genomes: Sequence[Genome], scores: Sequence[ScoreVector]) -> List[ValidationRecord]:
        if not genomes:
            return []
        reason, acc, lo = self.ctx.full_validation_arrays(genomes)
        return [ValidationRecord(g, s, ValidationStage.FullN1, bool(acc[i]), RejectionReason(int(reason[i])),
                                 float(lo[i])) for i, (g, s) in enumerate(zip(genomes, scores))]

    # ac_validator.cpp:427-473
    def full_validation(self, genome: Genome, dc_score: ScoreVector) -> ValidationRecord:
        return self.full_validation_batch([genome], [dc_score])[0]

    # ac_validator.cpp:475-495
    def validate(self, candidate: Candidate) -> ValidationRecord:
        return self.validate_queue([candidate])[0]

    def validate_queue(self, candidates: Sequence[Candidate]) -> List[ValidationRecord]:
        """validate() for every candidate in order, as two device batches."""
        cands = list(candidates)
        for c in cands:
            self._validated.append((c.genome, _swd(c.dc_score), c.dc_score.fitness))
        early = self.worst_k_check_batch([c.genome for c in cands], [c.dc_score for c in cands])
        go = [i for i, r in enumerate(early) if r == RejectionReason.None_]
        full = dict(zip(go, self.full_validation_batch([cands[i].genome for i in go], [cands[i].dc_score for i in go])))
        recs = []
        for i, c in enumerate(cands):
            rec = full[i] if i in full else ValidationRecord(c.genome, c.dc_score, ValidationStage.WorstK, False,
                                                             early[i])
            self._records.append(rec)
            recs.append(rec)
        return recs

    def record_elimination(self, candidate: Candidate, reason: RejectionReason) -> None:
        self._records.append(ValidationRecord(candidate.genome, candidate.dc_score, ValidationStage.None_, False,
                                              reason))


def record_to_json(record: ValidationRecord, grid: GridModel, actions: ActionSet) -> str:
    """ac_validator.cpp:497-534 (nlohmann ordered_json dump: compact, key order kept)."""
    ids = [b["id"] for b in json.loads(grid._text)["branches"]]
    stage = {ValidationStage.None_: "eliminated", ValidationStage.WorstK: "worst_k",
             ValidationStage.FullN1: "full_n1"}[record.stage]
    fit = record.dc_score.fitness
    d = {"actions": record.genome.action_ids(),
         "disconnections": [ids[int(actions.disconnectables[x])] for x in record.genome.disconnection_ids()],
         "lambda_d": record.dc_score.lambda_d, "lambda_s": record.dc_score.lambda_s,
         "lambda_r": record.dc_score.lambda_r, "dc_fitness": fit if np.isfinite(fit) else -1e30,
         "dc_lambda_o": record.dc_score.lambda_o, "stage": stage,
         "verdict": "accepted" if record.accepted else "rejected",
         "reason": "" if record.accepted else to_string(record.reason), "ac_lambda_o": record.ac_lambda_o}
    return json.dumps(d, separators=(",", ":"))
