"""GPU parity of the batched AC Newton-Raphson stage (tg_ac_*)
against the oracle restatement of ac_validator.cpp, plus the reference's own AC
tests (test_ac_validator.cpp:15-395) run on the device.

Tolerances: the device and the oracle run the same Newton iteration from the
same flat start; they differ only in rounding (FMA contraction, summation order
of the block reductions), so converged flags and iteration counts are exact,
loadings / voltages / energies agree to 1e-8 relative (scale max(1, |x|)),
far inside the 1e-6 p.u. mismatch tolerance that stops the iteration."""
import json
import os

import numpy as np
import pytest

from oracle.oracle import OracleAc, OracleContext, mini_congestion_json, random_grid_json

pytestmark = pytest.mark.gpu

TOL = 1e-8


def _rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b)))) if a.size else 0.0


def _pair(text, **cfg):
    import paper_2605_10128_b200 as P
    from paper_2605_10128_b200.ac import AcConfig, AcValidator

    g = P.grid_from_json_text(text)
    a = P.build_action_set(g)
    dc = P.DcContext(g, a)
    val = AcValidator(g, a, dc, AcConfig(**cfg))
    orc = OracleContext(text)
    oac = OracleAc(orc, **{k: v for k, v in {"tol": cfg.get("tolerance_pu", 1e-6),
                                             "max_iter": cfg.get("max_iterations", 30)}.items()})
    return val, dc, orc, oac


def _ac_json(text, scale=0.5, r_ratio=0.1):
    """A solvable AC operating point for a random test grid (tests/helpers.hpp
    random_grid): generation rescaled to the load, all injections scaled by
    `scale`, r = r_ratio x (at scale 1 most of these grids have no AC solution)."""
    d = json.loads(text)
    gen = sum(i["p_mw"] for i in d["injections"] if i["kind"] == "generator")
    load = sum(i["p_mw"] for i in d["injections"] if i["kind"] == "load")
    for inj in d["injections"]:
        inj["p_mw"] *= scale * (1.0 if inj["kind"] == "load" else load / gen)
        inj["q_mvar"] = inj.get("q_mvar", 0.0) * scale
    for b in d["branches"]:
        b["r_pu"] = r_ratio * b["x_pu"]
    return json.dumps(d)


def _compare_cases(val, oac, genomes, n_a=3, n_d=2, ks=None):
    n = len(genomes)
    K = val.grid.n_contingencies
    ks = list(range(-1, K)) if ks is None else ks
    cg = np.repeat(np.arange(n), len(ks)).astype(np.int32)
    ck = np.tile(np.array(ks, np.int32), n)
    got = val.ctx.run_cases(genomes, cg, ck, n_a, n_d)
    ref = oac.cases(genomes, n_a, n_d, cg, ck)
    assert np.array_equal(got["converged"], ref["converged"]), "converged flags"
    ok = ref["converged"]
    # a converging Newton run takes the same steps up to rounding; a diverging
    # one (no solution) is chaotic, so where it crosses 1e8 / non-finite
    # depends on rounding: counts are exact only for converged cases
    bad = np.nonzero(ok & (got["iterations"] != ref["iterations"]))[0]
    assert bad.size == 0, f"iteration counts of converged cases {bad[:10]}: {got['iterations'][bad[:10]]} vs {ref['iterations'][bad[:10]]}"
    assert _rel(got["loading_mva"][ok], ref["loading_mva"][ok]) <= TOL
    assert _rel(got["vm_pu"][ok], ref["vm_pu"][ok]) <= TOL
    assert _rel(got["va_rad"][ok], ref["va_rad"][ok]) <= TOL
    assert _rel(got["overload_energy"], ref["overload_energy"]) <= TOL
    lim = val.grid.branch_limit
    edge = np.abs(ref["loading_mva"] - lim[None, :]) <= TOL * np.maximum(1.0, lim[None, :])
    diff = got["critical_count"] != ref["critical_count"]
    assert not np.any(diff & ~edge.any(axis=1)), "critical counts off the knife edge"
    return got, ref


# ---------------------------------------------------------------- reference KATs
def _two_bus(x, r, p, q):
    return json.dumps({"nodes": [{"id": "s"}, {"id": "b"}],
                       "branches": [{"id": "sb", "from": "s", "to": "b", "x_pu": x, "r_pu": r, "limit_mw": 100.0}],
                       "injections": [{"id": "l", "node": "b", "p_mw": p, "q_mvar": q, "kind": "load"}],
                       "slack": "s"})


def test_two_bus_cases():
    """test_ac_validator.cpp:31-75, 170-184"""
    from paper_2605_10128_b200.ac import ac_power_flow
    import paper_2605_10128_b200 as P

    val, *_ = _pair(_two_bus(0.1, 0.01, 0.0, 0.0))
    r = ac_power_flow(val.ctx, P.Genome.empty(0, 0))
    assert r.converged and r.iterations == 1 and r.loading_mva.max() < 1e-9 and abs(r.vm_pu[1] - 1.0) < 1e-12

    val, *_ = _pair(_two_bus(0.1, 0.01, 50.0, 10.0))
    r = ac_power_flow(val.ctx, P.Genome.empty(0, 0))
    assert r.converged
    v1, z, s = 1.0 + 0j, 0.01 + 0.1j, 0.5 + 0.1j
    v2 = v1
    for _ in range(500):
        v2 = v1 - z * np.conj(s / v2)
    got = r.vm_pu[1] * np.exp(1j * r.va_rad[1])
    assert abs(got - v2) < 1e-6
    sf = v1 * np.conj((v1 - v2) / z) * 100.0
    assert sf.real > 50.0 and abs(r.loading_mva[0] - abs(sf)) <= 1e-6 * abs(sf)

    val, *_ = _pair(_two_bus(0.5, 0.05, 400.0, 100.0))
    assert not ac_power_flow(val.ctx, P.Genome.empty(0, 0)).converged


def test_grid14_published_and_balance(data_dir):
    """test_ac_validator.cpp:77-134: published magnitudes within 1e-3, bus power balance within 1e-6"""
    from paper_2605_10128_b200.ac import ac_power_flow
    import paper_2605_10128_b200 as P

    text = open(os.path.join(data_dir, "grid14.json")).read()
    val, dc, orc, oac = _pair(text)
    r = ac_power_flow(val.ctx, P.Genome.empty(0, 0))
    assert r.converged and r.iterations <= 10
    pub = [1.060, 1.045, 1.010, 1.018, 1.020, 1.070, 1.062, 1.090, 1.056, 1.051, 1.057, 1.055, 1.050, 1.036]
    d = json.loads(text)
    idx = {n["id"]: i for i, n in enumerate(d["nodes"])}
    for bus, vm in zip([str(i) for i in range(1, 15)], pub):
        assert abs(r.vm_pu[idx[bus]] - vm) < 1e-3
    n = len(d["nodes"])
    V = r.vm_pu[:n] * np.exp(1j * r.va_rad[:n])
    S = np.zeros(n, complex)
    for b in d["branches"]:
        f, t = idx[b["from"]], idx[b["to"]]
        y = 1.0 / complex(b.get("r_pu", 0.0), b["x_pu"])
        ysh = 1j * b.get("b_pu", 0.0) / 2
        tap = b.get("tap", 1.0)
        S[f] += V[f] * np.conj((y + ysh) / tap ** 2 * V[f] - y / tap * V[t])
        S[t] += V[t] * np.conj(-y / tap * V[f] + (y + ysh) * V[t])
    for i, nd in enumerate(d["nodes"]):
        S[i] += V[i] * np.conj(1j * nd.get("shunt_b_pu", 0.0) * V[i])
    for i, nd in enumerate(d["nodes"]):
        if i == idx[d["slack"]]:
            continue
        p = q = 0.0
        pv = False
        for inj in d["injections"]:
            if inj["node"] != nd["id"]:
                continue
            if inj["kind"] == "generator":
                p += inj["p_mw"] / 100
                pv = pv or "v_setpoint_pu" in inj
            else:
                p -= inj["p_mw"] / 100
                q -= inj.get("q_mvar", 0.0) / 100
        assert abs(S[i].real - p) < 1e-6
        if not pv:
            assert abs(S[i].imag - q) < 1e-6


def test_validator_congestion_fixture():
    """test_ac_validator.cpp:136-168, 186-233, 374-395 on the device"""
    import paper_2605_10128_b200 as P
    from paper_2605_10128_b200.ac import (AcNetwork, Candidate, RejectionReason, ValidationStage, record_to_json)

    text = mini_congestion_json()
    val, dc, orc, oac = _pair(text)
    assert val.baseline_lambda_o() > 0.0
    assert abs(val.baseline_lambda_o() - oac.baseline["lambda_o"]) <= TOL * max(1, oac.baseline["lambda_o"])
    assert val.baseline_critical_count() == oac.baseline["critical"]
    d = json.loads(text)
    ids = [b["id"] for b in d["branches"]]
    mf = [i for i, e in enumerate(val.actions.disconnectables.tolist()) if ids[e] == "mf"][0]
    clear = P.Genome.empty(3, 2)
    clear.disconnection_slots[0] = mf
    cs = dc.evaluate(clear)
    assert abs(cs.fitness) < 1e-9
    none = P.Genome.empty(3, 2)
    assert val.worst_k_check(none, dc.evaluate(none)) == RejectionReason.OverloadNotImproved
    assert val.worst_k_check(clear, cs) == RejectionReason.None_
    rec = val.full_validation(clear, cs)
    assert rec.accepted and rec.ac_lambda_o < val.baseline_lambda_o() and rec.stage == ValidationStage.FullN1
    parsed = json.loads(record_to_json(rec, val.grid, val.actions))
    assert parsed["stage"] == "full_n1" and parsed["lambda_d"] == 1 and parsed["verdict"] == "accepted"
    assert parsed["disconnections"] == ["mf"]
    assert val.validate(Candidate(clear, cs)).accepted
    out = val.eliminate([Candidate(clear, cs)])
    assert out.queue == [] and out.pruned == [(0, RejectionReason.EliminatedSimilar)]
    # split f so that o-af strands the load (136-168)
    names = [t for t in next(s for s in d["substations"] if s["node"] == "f")["terminals"]]
    elems = [t["element"] for t in names]
    st_f = [s["node"] for s in d["substations"]].index("f")
    for aid in range(val.actions.n_actions):
        if val.actions.substation[aid] != st_f:
            continue
        grp = val.actions.groups[aid]
        load_stays = not grp[elems.index("load")]
        mf_moves = all(grp[i] for i, e in enumerate(elems) if e in ("mf", "mf2"))
        if load_stays and mf_moves:
            g = P.Genome.empty(3, 2)
            g.action_slots[0] = aid
            net = AcNetwork(val.ctx, g)
            af = [c["id"] for c in d["contingencies"]].index("o-af")
            assert net.run_case(-1).converged and not net.run_case(af).converged


def test_critical_count_rejection():
    """test_ac_validator.cpp:264-298"""
    import paper_2605_10128_b200 as P
    from paper_2605_10128_b200.ac import RejectionReason

    text = json.dumps({
        "nodes": [{"id": "a"}, {"id": "m"}, {"id": "f"}],
        "branches": [{"id": "af", "from": "a", "to": "f", "x_pu": 0.3, "limit_mw": 200.0},
                     {"id": "am", "from": "a", "to": "m", "x_pu": 0.05, "limit_mw": 107.0},
                     {"id": "mf", "from": "m", "to": "f", "x_pu": 0.05, "limit_mw": 45.0},
                     {"id": "mf2", "from": "m", "to": "f", "x_pu": 0.2, "limit_mw": 100.0}],
        "injections": [{"id": "g", "node": "a", "p_mw": 100.0, "kind": "generator", "v_setpoint_pu": 1.02},
                       {"id": "load", "node": "f", "p_mw": 100.0, "q_mvar": 20.0, "kind": "load"}],
        "contingencies": [{"id": "o-af", "branches": ["af"]}, {"id": "o-am", "branches": ["am"]}],
        "slack": "a"})
    val, dc, orc, oac = _pair(text)
    assert val.baseline_critical_count() == 1
    mf = [i for i, e in enumerate(val.actions.disconnectables.tolist()) if e == 2][0]
    g = P.Genome.empty(3, 2)
    g.disconnection_slots[0] = mf
    rec = val.full_validation(g, dc.evaluate(g))
    assert not rec.accepted and rec.reason == RejectionReason.CriticalCountIncreased
    assert rec.ac_lambda_o < val.baseline_lambda_o()


def test_elimination_heuristics():
    """test_ac_validator.cpp:300-372 (host logic over a device-built validator)"""
    import paper_2605_10128_b200 as P
    from paper_2605_10128_b200.ac import Candidate, RejectionReason

    val, dc, orc, oac = _pair(mini_congestion_json())
    pre = dc.pre_optimization_score().fitness
    assert pre < 0

    def make(fit, d, s, r):
        g = P.Genome.empty(3, 2)
        g.disconnection_slots[0] = d % 2
        return Candidate(g, P.ScoreVector(fitness=fit, lambda_d=d, lambda_s=s, lambda_r=r))

    simple, twin = make(-10.0, 1, 0, 0), make(-10.0, 1, 1, 3)
    twin.genome.disconnection_slots[0] = 1
    out = val.eliminate([simple, twin])
    assert out.pruned == [(1, RejectionReason.EliminatedDominated)] and out.queue == [0]
    out = val.eliminate([make(pre + 0.01 * abs(pre), 1, 0, 0)])
    assert out.pruned[0][1] == RejectionReason.EliminatedBelowThreshold
    good, better = make(-5.0, 1, 0, 0), make(-1.0, 1, 0, 0)
    better.genome.disconnection_slots[0] = 1
    assert val.eliminate([good, better]).queue == [1, 0]
    rng = np.random.default_rng(42)
    gen = orc.random_genomes(60, 3, 2, seed=42)
    pool = []
    for row in gen:
        g = P.Genome(row[:3].tolist(), row[3:].tolist())
        pool.append(Candidate(g, P.ScoreVector(fitness=float(rng.uniform(pre, 0.0)), lambda_d=g.disconnection_count(),
                                               lambda_s=g.split_count(), lambda_r=int(rng.integers(0, 4)))))
    out = val.eliminate(pool)
    eps, theta = 0.01 * abs(pre), 0.05 * abs(pre)
    swd = lambda s: s.lambda_d + s.lambda_s + s.lambda_r  # noqa: E731
    assert len(out.queue) + len(out.pruned) == len(pool)
    for i in out.queue:
        assert pool[i].dc_score.fitness - pre >= theta
        for o in pool:
            assert not (swd(o.dc_score) < swd(pool[i].dc_score) and o.dc_score.fitness >= pool[i].dc_score.fitness - eps)


# ---------------------------------------------------------------- parity vs the oracle
def test_grid14_congested_cases_vs_oracle(data_dir):
    text = open(os.path.join(data_dir, "grid14_congested.json")).read()
    val, dc, orc, oac = _pair(text)
    bl = oac.baseline
    assert abs(val.baseline_lambda_o() - bl["lambda_o"]) <= TOL * max(1, bl["lambda_o"])
    assert val.baseline_critical_count() == bl["critical"]
    assert np.array_equal(val.ctx.case_converged, bl["case_converged"])
    assert _rel(val.ctx.case_energy, bl["case_energy"]) <= TOL
    genomes = np.concatenate([np.full((1, 5), -1, np.int32), orc.random_genomes(200, 3, 2, seed=11)])
    _compare_cases(val, oac, genomes)


@pytest.mark.parametrize("seed,n_nodes,extra", [(3, 24, 12), (5, 40, 20), (8, 61, 30), (13, 110, 60)])
def test_random_grids_cases_vs_oracle(seed, n_nodes, extra):
    """shared-memory (64 / 256-thread) and HBM-scratch (512-thread, > 200 KB) workspaces"""
    text = _ac_json(random_grid_json(seed, n_nodes=n_nodes, extra_edges=extra, n_outages=8, n_stations=4,
                                     multi=True, injection=True))
    val, dc, orc, oac = _pair(text)
    genomes = np.concatenate([np.full((1, 5), -1, np.int32), orc.random_genomes(24, 3, 2, seed=seed)])
    got, ref = _compare_cases(val, oac, genomes)
    assert ref["converged"].mean() > 0.5  # the family is solvable, not a vacuous comparison


def test_stages_vs_oracle(data_dir):
    """worst_k_check and full_validation verdicts (ac_validator.cpp:399-473) for DC-scored genomes"""
    import paper_2605_10128_b200 as P
    from paper_2605_10128_b200.ac import Candidate, RejectionReason

    for text in [open(os.path.join(data_dir, "grid14_congested.json")).read(), mini_congestion_json()]:
        val, dc, orc, oac = _pair(text)
        genomes = np.concatenate([np.full((1, 5), -1, np.int32), orc.random_genomes(120, 3, 2, seed=21)])
        sc = dc.evaluate_arrays(genomes, 3, 2)
        reason = val.ctx.worst_k_check_arrays(genomes, sc.worst_idx, sc.worst_n, 3, 2)
        ref = oac.worst_k_check(genomes, 3, 2, sc.worst_idx, sc.worst_n)
        assert np.array_equal(reason, ref)
        r2, acc, lo = val.ctx.full_validation_arrays(genomes, 3, 2)
        q2, qacc, qlo = oac.full_validation(genomes, 3, 2)
        assert np.array_equal(r2, q2) and np.array_equal(acc, qacc)
        assert _rel(lo, qlo) <= TOL
        # validate_queue == validate() in sequence
        cands = [Candidate(P.Genome(g[:3].tolist(), g[3:].tolist()), sc.score(i)) for i, g in enumerate(genomes[:40])]
        recs = val.validate_queue(cands)
        for i, rec in enumerate(recs):
            if reason[i] != RejectionReason.None_:
                assert rec.stage == 1 and rec.reason == reason[i]
            else:
                assert rec.stage == 2 and rec.reason == r2[i] and rec.accepted == acc[i]
        assert len(val.records()) == 40
        assert val.ctx.kernel_launches() > 0


def test_pipeline_snapshot_to_ac_hand_off(data_dir):
    """The consumer side of the hot path (pipeline.cpp:380-425): the DC loop's
    snapshots feed the AC validator — candidates deduplicated by canonical key,
    eliminate(), the queue validated (two device batches), pruned ones
    recorded — and every verdict equals the oracle's worst_k_check /
    full_validation of the same genome."""
    import paper_2605_10128_b200 as P
    from paper_2605_10128_b200.ac import Candidate, RejectionReason, ValidationStage, record_to_json

    text = open(os.path.join(data_dir, "grid14_congested.json")).read()
    val, dc, orc, oac = _pair(text)
    snaps = []
    P.run_optimizer(dc, P.QdConfig(seed=3, batch_size=64, iters_per_epoch=5, max_evaluations=641),
                    sink=lambda s: snaps.append(s))
    assert snaps and snaps[-1].final
    resolved = set()
    n_val = 0
    for snap in snaps:
        cands, seen = [], set()
        for e in snap.entries:
            if e.genome.is_empty():
                continue
            key = e.genome.canonical_key()
            if key in resolved or key in seen:
                continue
            seen.add(key)
            cands.append(Candidate(e.genome, e.score))
        if not cands:
            continue
        out = val.eliminate(cands)
        queue = [cands[i] for i in out.queue]
        recs = val.validate_queue(queue)
        for c, rec in zip(queue, recs):
            g = np.array([c.genome.action_slots + c.genome.disconnection_slots], np.int32)
            wi = np.array([[k for k, _ in c.dc_score.worst_contingencies] or [-1]], np.int32)
            wn = np.array([len(c.dc_score.worst_contingencies)], np.int32)
            early = int(oac.worst_k_check(g, 3, 2, wi, wn)[0])
            if early != RejectionReason.None_:
                assert rec.stage == ValidationStage.WorstK and int(rec.reason) == early
            else:
                reason, acc, lo = oac.full_validation(g, 3, 2)
                assert rec.stage == ValidationStage.FullN1 and int(rec.reason) == int(reason[0])
                assert rec.accepted == bool(acc[0])
                assert abs(rec.ac_lambda_o - lo[0]) <= TOL * max(1.0, abs(lo[0]))
            json.loads(record_to_json(rec, val.grid, val.actions))
            resolved.add(c.genome.canonical_key())
            n_val += 1
        for i, why in out.pruned:
            val.record_elimination(cands[i], why)
            resolved.add(cands[i].genome.canonical_key())
    assert n_val > 0 and len(val.records()) == len(resolved)
