"""GPU parity of the MapElites loop: device mutation / crossover replay the
reference's RNG stream bit for bit (qd_optimizer.cpp:202-277), the device
archive equals a sequential Repertoire::insert replay (qd_optimizer.cpp:281-303,
replay oracle of test_qd_optimizer.cpp:234-288), and whole run_optimizer runs
match the oracle (qd_optimizer.cpp:344-417)."""
import json
import math
import os

import numpy as np
import pytest

import paper_2605_10128_b200 as P
from oracle.oracle import OracleContext, qd_config, random_grid_json

pytestmark = pytest.mark.gpu

MINI = {"nodes": [{"id": "a"}, {"id": "m"}, {"id": "f"}],
        "branches": [{"id": "af", "from": "a", "to": "f", "x_pu": 0.3, "limit_mw": 200.0},
                     {"id": "am", "from": "a", "to": "m", "x_pu": 0.05, "limit_mw": 130.0},
                     {"id": "mf", "from": "m", "to": "f", "x_pu": 0.05, "limit_mw": 45.0},
                     {"id": "mf2", "from": "m", "to": "f", "x_pu": 0.2, "limit_mw": 130.0}],
        "injections": [{"id": "g", "node": "a", "p_mw": 100.0, "kind": "generator", "v_setpoint_pu": 1.02},
                       {"id": "load", "node": "f", "p_mw": 100.0, "q_mvar": 20.0, "kind": "load"}],
        "contingencies": [{"id": "o-af", "branches": ["af"]}, {"id": "o-am", "branches": ["am"]}],
        "substations": [{"node": n, "busbars": ["B1", "B2"], "couplers": [["B1", "B2"]],
                         "terminals": [{"element": e, "reachable": ["B1", "B2"], "default": "B1"} for e in el]}
                        for n, el in [("a", ["af", "am", "g"]), ("m", ["am", "mf", "mf2"]),
                                      ("f", ["af", "mf", "mf2", "load"])]],
        "slack": "a"}


def _grids(data_dir):
    yield json.dumps(MINI)
    yield open(os.path.join(data_dir, "grid14_congested.json")).read()
    yield random_grid_json(99, n_nodes=25, extra_edges=20, n_outages=4, n_stations=3)


def _ctx(text):
    g = P.grid_from_json_text(text)
    return P.DcContext(g, P.build_action_set(g)), OracleContext(text)


def _parents(orc, n, seed):
    g = orc.random_genomes(n, 3, 2, seed=seed)
    g[:7] = -1  # empty parents exercise the forced add (qd_optimizer.cpp:170-172)
    return g


def test_mutation_replays_reference_stream(data_dir):
    for text in _grids(data_dir):
        ctx, orc = _ctx(text)
        for kw in ({}, {"mutation_mean": 5.5}, {"p_action": (0.0, 0.5, 0.5, 0.0)}):
            cfg = P.QdConfig(**kw)
            ocfg = qd_config(**kw)
            par = _parents(orc, 300, 3)
            seeds = np.arange(300, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15) + np.uint64(17)
            got = P.mutate_lanes(ctx, cfg, par, seeds)
            for i in range(len(par)):
                want, _ = orc.mutate(ocfg, par[i], int(seeds[i]))
                assert got[i].tolist() == want.tolist(), (i, par[i], got[i], want)


def test_crossover_replays_reference_stream(data_dir):
    for text in _grids(data_dir):
        ctx, orc = _ctx(text)
        for pc1 in (0.75, 1.0, 0.3):
            cfg = P.QdConfig(p_crossover_parent1=pc1)
            ocfg = qd_config(p_crossover_parent1=pc1)
            p1 = _parents(orc, 200, 5)
            p2 = _parents(orc, 200, 6)[::-1].copy()
            seeds = np.arange(200, dtype=np.uint64) * np.uint64(7919) + np.uint64(3)
            got = P.crossover_lanes(ctx, cfg, p1, p2, seeds)
            for i in range(len(p1)):
                want = orc.crossover(ocfg, p1[i], p2[i], int(seeds[i]))
                assert got[i].tolist() == want.tolist(), (i, p1[i], p2[i], got[i], want)


def _replay_oracle(stream, cfg):
    """Naive list replay of Repertoire::insert (test_qd_optimizer.cpp:262-277)."""
    cells = {}
    results = []
    for genome, sc in stream:
        if not math.isfinite(sc["fitness"]):
            results.append(False)
            continue
        cell = P.descriptor_to_cell(sc["lambda_d"], sc["lambda_s"], sc["lambda_r"], cfg)
        lst = cells.setdefault(cell, [])
        key = P.Genome(list(genome[:cfg.n_a]), list(genome[cfg.n_a:])).canonical_key()
        if any(k == key for k, _, _ in lst):
            results.append(False)
            continue
        if len(lst) >= cfg.cell_capacity and sc["fitness"] <= lst[-1][1]:
            results.append(False)
            continue
        pos = 0
        while pos < len(lst) and not (sc["fitness"] > lst[pos][1]):
            pos += 1
        lst.insert(pos, (key, sc["fitness"], list(genome)))
        if len(lst) > cfg.cell_capacity:
            lst.pop()
        results.append(True)
    return results, cells


def test_archive_replay_matches_sequential_insert(data_dir):
    ctx, orc = _ctx(open(os.path.join(data_dir, "grid14_congested.json")).read())
    rng = np.random.default_rng(99)
    for cap in (3, 4, 1):
        cfg = P.QdConfig(cell_capacity=cap)
        n = 2000
        g = np.full((n, 5), -1, np.int32)
        g[:, 3] = rng.integers(-1, 5, n)
        g[:, 4] = rng.integers(-1, 5, n)
        g[g[:, 3] == g[:, 4], 4] = -1
        g[:, 0] = rng.integers(-1, 6, n)
        sc = P.ScoreArrays(n, 20)
        sc.lambda_d[:] = (g[:, 3:] >= 0).sum(1)
        sc.lambda_s[:] = (g[:, :3] >= 0).sum(1)
        sc.lambda_r[:] = rng.integers(0, 4, n)
        # coarse fitness values force exact ties (arrival order decides)
        sc.fitness[:] = np.round(rng.uniform(-100, 0, n), 0)
        sc.fitness[rng.random(n) < 0.05] = -np.inf
        ins, snap = P.archive_replay(ctx, cfg, g, sc)
        stream = [(g[i].tolist(), dict(fitness=sc.fitness[i], lambda_d=int(sc.lambda_d[i]),
                                        lambda_s=int(sc.lambda_s[i]), lambda_r=int(sc.lambda_r[i])))
                  for i in range(n)]
        want_ins, cells = _replay_oracle(stream, cfg)
        assert ins.tolist() == want_ins
        got = {}
        for e in snap.entries:
            got.setdefault(e.cell, []).append((e.genome.canonical_key(), e.score.fitness,
                                               e.genome.action_slots + e.genome.disconnection_slots))
        assert got == {c: v for c, v in cells.items() if v}


def _compare_runs(res, ref, cfg):
    assert res.stats.evaluations == ref["stats"]["evaluations"]
    assert res.stats.epochs == ref["stats"]["epochs"]
    rt = ref["stats"]["fitness_trace"]
    assert len(res.stats.fitness_trace) == len(rt)
    for (ev, b), (rev, rb) in zip(res.stats.fitness_trace, rt):
        assert ev == rev and abs(b - rb) <= 1e-9 * max(1.0, abs(rb))
    last = ref["snapshots"][-1]
    want = [(e[0], e[1], e[2]) for e in last["entries"]]
    got = [(e.cell, e.genome.action_slots + e.genome.disconnection_slots, e.score.fitness)
           for e in res.repertoire.entries]
    assert len(got) == len(want)
    for (c, g, f), (rc, rg, rf) in zip(got, want):
        assert c == rc and g == rg and abs(f - rf) <= 1e-9 * max(1.0, abs(rf))


def test_optimizer_matches_reference_grid14_congested(data_dir):
    # BASELINE config 1: grid14_congested, batch 64, 50 generations (max_evaluations 3201)
    text = open(os.path.join(data_dir, "grid14_congested.json")).read()
    ctx, orc = _ctx(text)
    for seed, ipe in ((1, 500), (777, 7)):
        kw = dict(seed=seed, batch_size=64, iters_per_epoch=ipe, max_evaluations=3201)
        snaps = []
        res = P.run_optimizer(ctx, P.QdConfig(**kw), sink=snaps.append)
        ref = orc.run_optimizer(qd_config(**kw), all_snapshots=True)
        _compare_runs(res, ref, P.QdConfig(**kw))
        assert len(snaps) == len(ref["snapshots"]) and snaps[-1].final
        for s, rs in zip(snaps, ref["snapshots"]):
            assert s.epoch == rs["epoch"] and s.evaluations == rs["evaluations"]


def test_optimizer_mini_grid_semantics():
    # test_qd_optimizer.cpp:291-369
    ctx, orc = _ctx(json.dumps(MINI))
    kw = dict(seed=11, batch_size=16, iters_per_epoch=10)
    res = P.run_optimizer(ctx, P.QdConfig(max_evaluations=1, **kw))
    assert res.stats.evaluations == 1 and len(res.repertoire.entries) == 1
    assert res.repertoire.entries[0].genome.is_empty()
    res = P.run_optimizer(ctx, P.QdConfig(max_evaluations=4000, **kw))
    assert abs(res.repertoire.best_fitness) < 1e-9  # the clearing disconnection is found
    ref = orc.run_optimizer(qd_config(max_evaluations=4000, **kw))
    _compare_runs(res, ref, P.QdConfig(max_evaluations=4000, **kw))
    with pytest.raises(P.ConfigError):
        P.run_optimizer(ctx, P.QdConfig(batch_size=0))
