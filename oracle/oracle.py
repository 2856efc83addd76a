"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes wrapper of oracle/_build/liboracle.so, the C++ restatement of the
reference's DC N-1 MapElites path (see oracle/src/oracle.hpp). Imported only by
tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference).
The product package never imports this module.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle.so")
KATS_PATH = os.path.join(HERE, "_build", "oracle_kats")


def build() -> None:
    subprocess.run(["make", "-C", HERE, "-j8"], check=True, stdout=subprocess.DEVNULL)


class QdConfigC(C.Structure):
    _fields_ = [("n_a", C.c_int32), ("n_d", C.c_int32), ("batch_size", C.c_int32),
                ("iters_per_epoch", C.c_int32), ("cell_capacity", C.c_int32), ("mutation_mean", C.c_double),
                ("p_action", C.c_double * 4), ("p_disc", C.c_double * 4), ("p_crossover_parent1", C.c_double),
                ("d_max", C.c_int32), ("s_max", C.c_int32), ("r_max", C.c_int32), ("seed", C.c_uint64),
                ("max_evaluations", C.c_int64), ("max_seconds", C.c_double)]


def qd_config(**kw) -> QdConfigC:
    d = dict(n_a=3, n_d=2, batch_size=64, iters_per_epoch=500, cell_capacity=4, mutation_mean=2.0,
             p_action=(0.2, 0.2, 0.5, 0.1), p_disc=(0.25, 0.25, 0.5, 0.0), p_crossover_parent1=0.75,
             d_max=2, s_max=3, r_max=45, seed=1, max_evaluations=-1, max_seconds=-1.0)
    d.update(kw)
    c = QdConfigC()
    for k, v in d.items():
        if k in ("p_action", "p_disc"):
            arr = getattr(c, k)
            for i in range(4):
                arr[i] = v[i]
        else:
            setattr(c, k, v)
    return c


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        vp, i32p, f64p, u8p = C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_double), C.POINTER(C.c_uint8)
        L.oc_last_error.restype = C.c_char_p
        L.oc_free.argtypes = [vp]
        L.oc_context_create.argtypes = [C.c_char_p, C.c_uint64, C.c_int64, C.c_double, C.c_int, C.c_double,
                                        C.c_double, C.c_int, C.c_int, C.POINTER(vp)]
        L.oc_context_destroy.argtypes = [vp]
        L.oc_context_info.argtypes = [vp]
        L.oc_context_info.restype = vp
        L.oc_evaluate.argtypes = [vp, i32p, C.c_int, C.c_int, C.c_int, f64p, i32p, i32p, f64p, i32p, i32p, i32p,
                                  f64p, u8p, i32p, f64p, i32p, f64p, f64p, f64p, f64p, i32p, i32p]
        L.oc_time_evaluate_batch.argtypes = [vp, i32p, C.c_int, C.c_int, C.c_int, C.c_int]
        L.oc_time_evaluate_batch.restype = C.c_double
        L.oc_mutate.argtypes = [vp, C.POINTER(QdConfigC), i32p, C.c_uint64, i32p, i32p, i32p]
        L.oc_crossover.argtypes = [vp, C.POINTER(QdConfigC), i32p, i32p, C.c_uint64, i32p]
        L.oc_run_optimizer.argtypes = [vp, C.POINTER(QdConfigC), C.c_int]
        L.oc_run_optimizer.restype = vp
        L.oc_run_optimizer_trace.argtypes = [vp, C.POINTER(QdConfigC)]
        L.oc_run_optimizer_trace.restype = vp
        L.oc_run_optimizer_timed.argtypes = [vp, C.POINTER(QdConfigC), f64p, C.c_int, C.POINTER(C.c_int64)]
        L.oc_run_optimizer_timed.restype = C.c_int
        L.oc_random_grid_json.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]
        L.oc_random_grid_json.restype = vp
        L.oc_random_genomes.argtypes = [vp, C.c_int, C.c_int, C.c_uint64, C.c_int, i32p]
        L.oc_rebuild_flows.argtypes = [vp, i32p, C.c_int, C.c_int, f64p, i32p]
        L.oc_grid_json.argtypes = [vp]
        L.oc_grid_json.restype = vp
        L.oc_grid_hash.argtypes = [vp]
        L.oc_grid_hash.restype = C.c_uint64
        L.oc_action_cache.argtypes = [vp]
        L.oc_action_cache.restype = vp
        L.oc_action_cache_load.argtypes = [vp, C.c_char_p]
        L.oc_action_cache_load.restype = C.c_int64
        L.oc_build_ptdf.argtypes = [vp, f64p]
        L.oc_ac_cases.argtypes = [vp, C.c_double, C.c_int, i32p, C.c_int, C.c_int, i32p, i32p, C.c_int, C.c_int,
                                  u8p, i32p, f64p, i32p, f64p, f64p, f64p]
        L.oc_ac_validator_create.argtypes = [vp, C.c_double, C.c_int, C.c_int, C.c_double, C.c_int, C.c_double,
                                             C.c_double, C.POINTER(vp)]
        L.oc_ac_validator_destroy.argtypes = [vp]
        L.oc_ac_baseline.argtypes = [vp, f64p, i32p, u8p, f64p, u8p, f64p]
        L.oc_ac_worst_k.argtypes = [vp, i32p, C.c_int, C.c_int, C.c_int, i32p, i32p, C.c_int, i32p]
        L.oc_mini_congestion_json.restype = vp
        L.oc_ac_full.argtypes = [vp, i32p, C.c_int, C.c_int, C.c_int, i32p, u8p, f64p]
        _lib = L
    return _lib


def _take_string(p) -> str:
    if not p:
        raise RuntimeError(lib().oc_last_error().decode())
    try:
        return C.string_at(p).decode()
    finally:
        lib().oc_free(p)


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def random_grid_json(seed, n_nodes=20, extra_edges=10, n_outages=5, n_stations=2, multi=False, injection=False,
                     busbar=False) -> str:
    """tests/helpers.hpp:435-553 random_grid, serialized."""
    return _take_string(lib().oc_random_grid_json(seed, n_nodes, extra_edges, n_outages, n_stations, int(multi),
                                                  int(injection), int(busbar)))


def mini_congestion_json() -> str:
    """tests/helpers.hpp:83-103 mini_congestion_grid as grid JSON."""
    return _take_string(lib().oc_mini_congestion_json())


class OracleContext:
    """Grid + ActionSet + DcContext of the restated reference."""

    def __init__(self, grid_json: str, penalty=10000.0, worst_k=20, weight_c0=200.0, weight_c=50.0, variant=1,
                 threads=0, enum_seed=0, enum_cap=0):
        self.h = C.c_void_p()
        rc = lib().oc_context_create(grid_json.encode(), enum_seed, enum_cap, penalty, worst_k, weight_c0, weight_c,
                                     variant, threads, C.byref(self.h))
        if rc != 0:
            raise RuntimeError(f"oracle error {rc}: {lib().oc_last_error().decode()}")
        self.worst_k = worst_k
        self.info = json.loads(_take_string(lib().oc_context_info(self.h)))

    def grid_json(self) -> str:
        """grid_to_json_text (grid_model.cpp:423-485)."""
        return _take_string(lib().oc_grid_json(self.h))

    def build_ptdf(self) -> np.ndarray:
        """build_ptdf (importer.cpp:358-401): [E, N]."""
        E, N = self.info["n_branches"], self.info["n_nodes"]
        out = np.zeros((E, N))
        if lib().oc_build_ptdf(self.h, _p(out, C.c_double)) != 0:
            raise RuntimeError(lib().oc_last_error().decode())
        return out

    def grid_hash(self) -> int:
        """grid_content_hash (grid_model.cpp:494-503)."""
        return int(lib().oc_grid_hash(self.h))

    def action_cache(self) -> str:
        """save_action_set's text (importer.cpp:407-430)."""
        return _take_string(lib().oc_action_cache(self.h))

    def load_action_cache(self, text: str) -> int:
        """load_action_set (importer.cpp:432-479): action count, -1 if rejected."""
        return int(lib().oc_action_cache_load(self.h, text.encode()))

    def __del__(self):
        if getattr(self, "h", None):
            lib().oc_context_destroy(self.h)
            self.h = None

    def evaluate(self, genomes: np.ndarray, n_a: int, n_d: int, flows: bool = False) -> dict:
        g = np.ascontiguousarray(genomes, np.int32).reshape(-1, n_a + n_d)
        n = g.shape[0]
        E, K, wk = self.info["n_branches"], self.info["n_contingencies"], self.worst_k
        out = dict(lambda_o=np.zeros(n), lambda_c=np.zeros(n, np.int32), lambda_c0=np.zeros(n, np.int32),
                   lambda_b=np.zeros(n), lambda_d=np.zeros(n, np.int32), lambda_s=np.zeros(n, np.int32),
                   lambda_r=np.zeros(n, np.int32), fitness=np.zeros(n), islanded=np.zeros(n, np.uint8),
                   worst_idx=np.zeros((n, max(wk, 1)), np.int32), worst_val=np.zeros((n, max(wk, 1))),
                   worst_n=np.zeros(n, np.int32), islanded_outages=np.zeros(n, np.int32),
                   islanded_busbar=np.zeros(n, np.int32))
        nul = C.POINTER(C.c_double)()
        if flows:
            out.update(base=np.zeros((n, E)), fmax=np.zeros((n, E)), fbus=np.zeros((n, E)),
                       energy=np.zeros((n, max(K, 1))))
        i32, f64 = C.c_int32, C.c_double
        rc = lib().oc_evaluate(self.h, _p(g, i32), n_a, n_d, n, _p(out["lambda_o"], f64), _p(out["lambda_c"], i32),
                               _p(out["lambda_c0"], i32), _p(out["lambda_b"], f64), _p(out["lambda_d"], i32),
                               _p(out["lambda_s"], i32), _p(out["lambda_r"], i32), _p(out["fitness"], f64),
                               _p(out["islanded"], C.c_uint8), _p(out["worst_idx"], i32), _p(out["worst_val"], f64),
                               _p(out["worst_n"], i32),
                               _p(out["base"], f64) if flows else nul, _p(out["fmax"], f64) if flows else nul,
                               _p(out["fbus"], f64) if flows else nul, _p(out["energy"], f64) if flows else nul,
                               _p(out["islanded_outages"], i32), _p(out["islanded_busbar"], i32))
        if rc != 0:
            raise RuntimeError(lib().oc_last_error().decode())
        if flows:
            out["energy"] = out["energy"][:, :K]
        return out

    def time_evaluate_batch(self, genomes: np.ndarray, n_a: int, n_d: int, reps: int = 1) -> float:
        g = np.ascontiguousarray(genomes, np.int32).reshape(-1, n_a + n_d)
        return lib().oc_time_evaluate_batch(self.h, _p(g, C.c_int32), n_a, n_d, g.shape[0], reps)

    def random_genomes(self, n: int, n_a: int = 3, n_d: int = 2, seed: int = 1) -> np.ndarray:
        out = np.zeros((n, n_a + n_d), np.int32)
        rc = lib().oc_random_genomes(self.h, n_a, n_d, seed, n, _p(out, C.c_int32))
        if rc != 0:
            raise RuntimeError(lib().oc_last_error().decode())
        return out

    def mutate(self, cfg: QdConfigC, parent, seed: int):
        ns = cfg.n_a + cfg.n_d
        par = np.ascontiguousarray(parent, np.int32)
        child = np.zeros(ns, np.int32)
        ops = np.zeros(64, np.int32)
        nops = C.c_int32()
        rc = lib().oc_mutate(self.h, C.byref(cfg), _p(par, C.c_int32), seed, _p(child, C.c_int32),
                             _p(ops, C.c_int32), C.byref(nops))
        if rc != 0:
            raise RuntimeError(lib().oc_last_error().decode())
        return child, ops[:nops.value]

    def crossover(self, cfg: QdConfigC, p1, p2, seed: int):
        ns = cfg.n_a + cfg.n_d
        a = np.ascontiguousarray(p1, np.int32)
        b = np.ascontiguousarray(p2, np.int32)
        child = np.zeros(ns, np.int32)
        rc = lib().oc_crossover(self.h, C.byref(cfg), _p(a, C.c_int32), _p(b, C.c_int32), seed, _p(child, C.c_int32))
        if rc != 0:
            raise RuntimeError(lib().oc_last_error().decode())
        return child

    def run_optimizer(self, cfg: QdConfigC, all_snapshots: bool = False) -> dict:
        return json.loads(_take_string(lib().oc_run_optimizer(self.h, C.byref(cfg), int(all_snapshots))))

    def run_optimizer_trace(self, cfg: QdConfigC) -> dict:
        """run_optimizer with each iteration's offspring and scores (lockstep parity)."""
        return json.loads(_take_string(lib().oc_run_optimizer_trace(self.h, C.byref(cfg))))

    def run_optimizer_timed(self, cfg: QdConfigC):
        """run_optimizer; returns (per-iteration end stamps in seconds, evaluations)."""
        cap = 1 << 16
        st = np.zeros(cap)
        ev = C.c_int64()
        n = lib().oc_run_optimizer_timed(self.h, C.byref(cfg), _p(st, C.c_double), cap, C.byref(ev))
        if n < 0:
            raise RuntimeError(lib().oc_last_error().decode())
        return st[:n], int(ev.value)

    def rebuild_flows(self, genome, n_a: int, n_d: int):
        g = np.ascontiguousarray(genome, np.int32)
        f = np.zeros(self.info["n_branches"])
        sing = C.c_int32()
        rc = lib().oc_rebuild_flows(self.h, _p(g, C.c_int32), n_a, n_d, _p(f, C.c_double), C.byref(sing))
        if rc != 0:
            raise RuntimeError(lib().oc_last_error().decode())
        return None if sing.value else f


class OracleAc:
    """AcNetwork / AcValidator of the restated reference (oracle/src/ac.cpp) on an OracleContext."""

    def __init__(self, orc: "OracleContext", tol=1e-6, max_iter=30, q=2, frac=0.05, sim=1, dom=0.01, thr=0.05):
        self.orc, self.tol, self.max_iter = orc, tol, max_iter
        self.h = C.c_void_p()
        if lib().oc_ac_validator_create(orc.h, tol, max_iter, q, frac, sim, dom, thr, C.byref(self.h)) != 0:
            raise RuntimeError(lib().oc_last_error().decode())
        K = orc.info["n_contingencies"]
        lo, cr, bc, be = C.c_double(), C.c_int32(), C.c_uint8(), C.c_double()
        cc, ce = np.zeros(max(K, 1), np.uint8), np.zeros(max(K, 1))
        lib().oc_ac_baseline(self.h, C.byref(lo), C.byref(cr), C.byref(bc), C.byref(be), _p(cc, C.c_uint8),
                             _p(ce, C.c_double))
        self.baseline = dict(lambda_o=lo.value, critical=cr.value, base_converged=bool(bc.value),
                             base_energy=be.value, case_converged=cc[:K].astype(bool), case_energy=ce[:K])

    def __del__(self):
        if getattr(self, "h", None):
            lib().oc_ac_validator_destroy(self.h)
            self.h = None

    def cases(self, genomes, n_a, n_d, case_genome, case_cont, threads=0, loading=True) -> dict:
        g = np.ascontiguousarray(genomes, np.int32).reshape(-1, n_a + n_d)
        cg = np.ascontiguousarray(case_genome, np.int32)
        ck = np.ascontiguousarray(case_cont, np.int32)
        n = len(cg)
        E, V = self.orc.info["n_branches"], self.orc.info["n_nodes"] + n_a
        out = dict(converged=np.zeros(n, np.uint8), iterations=np.zeros(n, np.int32), overload_energy=np.zeros(n),
                   critical_count=np.zeros(n, np.int32))
        nul = C.POINTER(C.c_double)()
        if loading:
            out.update(loading_mva=np.zeros((n, E)), vm_pu=np.zeros((n, V)), va_rad=np.zeros((n, V)))
        f64 = C.c_double
        rc = lib().oc_ac_cases(self.orc.h, self.tol, self.max_iter, _p(g, C.c_int32), n_a, n_d, _p(cg, C.c_int32),
                               _p(ck, C.c_int32), n, threads or (os.cpu_count() or 1), _p(out["converged"], C.c_uint8),
                               _p(out["iterations"], C.c_int32), _p(out["overload_energy"], f64),
                               _p(out["critical_count"], C.c_int32),
                               _p(out["loading_mva"], f64) if loading else nul,
                               _p(out["vm_pu"], f64) if loading else nul, _p(out["va_rad"], f64) if loading else nul)
        if rc != 0:
            raise RuntimeError(lib().oc_last_error().decode())
        out["converged"] = out["converged"].astype(bool)
        return out

    def worst_k_check(self, genomes, n_a, n_d, worst_idx, worst_n) -> np.ndarray:
        g = np.ascontiguousarray(genomes, np.int32).reshape(-1, n_a + n_d)
        n = g.shape[0]
        wi = np.ascontiguousarray(worst_idx, np.int32).reshape(n, -1)
        wn = np.ascontiguousarray(worst_n, np.int32)
        reason = np.zeros(n, np.int32)
        if lib().oc_ac_worst_k(self.h, _p(g, C.c_int32), n_a, n_d, n, _p(wi, C.c_int32), _p(wn, C.c_int32),
                               wi.shape[1], _p(reason, C.c_int32)) != 0:
            raise RuntimeError(lib().oc_last_error().decode())
        return reason

    def full_validation(self, genomes, n_a, n_d):
        g = np.ascontiguousarray(genomes, np.int32).reshape(-1, n_a + n_d)
        n = g.shape[0]
        reason, acc, lo = np.zeros(n, np.int32), np.zeros(n, np.uint8), np.zeros(n)
        if lib().oc_ac_full(self.h, _p(g, C.c_int32), n_a, n_d, n, _p(reason, C.c_int32), _p(acc, C.c_uint8),
                            _p(lo, C.c_double)) != 0:
            raise RuntimeError(lib().oc_last_error().decode())
        return reason, acc.astype(bool), lo
