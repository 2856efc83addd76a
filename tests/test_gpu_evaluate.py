"""GPU parity of DcContext::evaluate_batch through the C ABI against the CPU
oracle (reference restatement). Cases follow the reference's own tests:
test_dc_engine.cpp:26-526 and acceptance.cpp:51-108."""
import json
import os

import numpy as np
import pytest

from oracle.oracle import random_grid_json
from tests.parity import compare_flows, compare_scores, grid_with_stations, make_pair

pytestmark = pytest.mark.gpu


def _all_singles(ctx, n_a=3, n_d=2):
    rows = [[-1] * (n_a + n_d)]
    for a in range(ctx.actions.n_actions):
        rows.append([a] + [-1] * (n_a + n_d - 1))
    for d in range(len(ctx.actions.disconnectables)):
        r = [-1] * (n_a + n_d)
        r[n_a] = d
        rows.append(r)
    return np.array(rows, np.int32)


def _check(ctx, orc, genomes, n_a=3, n_d=2, flows=True):
    sc, fr = ctx.evaluate_arrays(genomes, n_a, n_d, flows=True)
    ref = orc.evaluate(genomes, n_a, n_d, flows=True)
    lim = ctx.grid.branch_limit
    errs = compare_scores(sc, ref, ctx.config.worst_k, lim)
    if flows:
        errs.update(compare_flows(fr, ref))
    # the fast (scores-only) sweep must agree with the full-flows sweep
    fast = ctx.evaluate_arrays(genomes, n_a, n_d)
    compare_scores(fast, ref, ctx.config.worst_k, lim)
    return errs


def test_grid14_congested_singles_and_random(data_dir):
    text = open(os.path.join(data_dir, "grid14_congested.json")).read()
    ctx, orc = make_pair(text)
    pre = ctx.pre_optimization_score()
    assert abs(pre.fitness - orc.info["pre_score"]["fitness"]) <= 1e-9 * max(1, abs(pre.fitness))
    assert abs(ctx.lambda_b_pre() - orc.info["lambda_b_pre"]) <= 1e-9 * max(1, ctx.lambda_b_pre())
    _check(ctx, orc, _all_singles(ctx))
    _check(ctx, orc, orc.random_genomes(400, seed=5))


def test_grid14_split_station_vs_rebuild(data_dir):
    # test_dc_engine.cpp:50-81: station grafted on bus 4 of the 14-bus grid
    text = grid_with_stations(open(os.path.join(data_dir, "grid14.json")).read(), ["4"])
    ctx, orc = make_pair(text)
    _check(ctx, orc, orc.random_genomes(200, seed=7))


def test_acceptance1_random_grids():
    # acceptance.cpp:51-88 grid family (criterion 1), 20 genomes each
    for trial in range(0, 50, 3):
        text = random_grid_json(1000 + trial, n_nodes=10 + (trial * 7) % 51, extra_edges=6 + trial % 13,
                                n_outages=3 + trial % 5, n_stations=2 + trial % 2)
        ctx, orc = make_pair(text)
        _check(ctx, orc, orc.random_genomes(40, seed=4242 + trial))


def test_scratch_case_grids_multi_injection_busbar():
    # test_dc_engine.cpp:366-431: multi-branch, injection and busbar outages with islanding
    seen_isl = 0
    for seed in range(600, 612):
        text = random_grid_json(seed, n_nodes=14 + seed % 20, extra_edges=10 + seed % 7, n_outages=6, n_stations=2,
                                multi=True, injection=True, busbar=True)
        ctx, orc = make_pair(text, islanding_penalty_mw=7777.0)
        g = orc.random_genomes(60, seed=808 + seed)
        _check(ctx, orc, g)
        seen_isl += int(orc.evaluate(g, 3, 2)["islanded_outages"].sum())
    assert seen_isl > 0


def test_reference_kat_scenarios():
    tri = {"nodes": [{"id": "a"}, {"id": "b"}, {"id": "c"}],
           "branches": [{"id": "ab", "from": "a", "to": "b", "x_pu": 0.2, "limit_mw": 100.0},
                        {"id": "ac", "from": "a", "to": "c", "x_pu": 0.2, "limit_mw": 100.0},
                        {"id": "bc", "from": "b", "to": "c", "x_pu": 0.2, "limit_mw": 100.0}],
           "injections": [{"id": "g", "node": "a", "p_mw": 90.0, "kind": "generator"},
                          {"id": "l", "node": "c", "p_mw": 90.0, "kind": "load"}],
           "contingencies": [{"id": "o-ab", "branches": ["ab"]}], "slack": "c"}
    ctx, orc = make_pair(json.dumps(tri))
    import paper_2605_10128_b200 as P
    fr = ctx.screen(P.Genome.empty(3, 2))
    assert abs(fr.max_contingency[0, 1] - 90.0) < 1e-9 and abs(fr.max_contingency[0, 0]) < 1e-9
    # islanding contingency penalty (test_dc_engine.cpp:197-235)
    j = {"nodes": [{"id": x} for x in "abcd"],
         "branches": [{"id": i, "from": i[0], "to": i[1], "x_pu": 0.1, "limit_mw": 100.0}
                      for i in ["ab", "bc", "bd", "cd", "da", "ac"]],
         "injections": [{"id": "g", "node": "b", "p_mw": 50.0, "kind": "generator"},
                        {"id": "l", "node": "d", "p_mw": 50.0, "kind": "load"}],
         "contingencies": [{"id": "ab-out", "branches": ["ab"]}], "slack": "a"}
    ctx, orc = make_pair(json.dumps(j), islanding_penalty_mw=2500.0)
    names = [ctx.grid.n_branches]
    disc = ctx.actions.disconnectables.tolist()
    order = ["ab", "bc", "bd", "cd", "da", "ac"]
    g = P.Genome([-1, -1, -1], [disc.index(order.index("bc")), disc.index(order.index("bd"))])
    s = ctx.evaluate(g)
    assert not s.islanded and abs(s.lambda_o - 2500.0) < 1e-9
    assert len(s.worst_contingencies) == 1 and abs(s.worst_contingencies[0][1] - 2500.0) < 1e-9
    del names
    # genome islanding sentinel (test_dc_engine.cpp:497-526)
    j2 = {"nodes": [{"id": x} for x in "abcd"],
          "branches": [{"id": i, "from": i[0], "to": i[1], "x_pu": 0.1, "limit_mw": 100.0}
                       for i in ["ab", "bc", "ca", "bd", "cd"]],
          "injections": [{"id": "g", "node": "a", "p_mw": 40.0, "kind": "generator"},
                         {"id": "l", "node": "d", "p_mw": 40.0, "kind": "load"}], "slack": "a"}
    ctx, orc = make_pair(json.dumps(j2))
    s = ctx.evaluate(P.Genome([-1, -1, -1], [3, 4]))
    assert s.islanded and s.fitness == -np.inf
    # busbar outage + variant 2 (test_dc_engine.cpp:297-335)
    j3 = {"nodes": [{"id": x} for x in "abcd"],
          "branches": [{"id": i, "from": i[0], "to": i[1], "x_pu": 0.1, "limit_mw": 100.0}
                       for i in ["ab", "ac", "ad", "bc", "cd"]],
          "injections": [{"id": "g", "node": "a", "p_mw": 60.0, "kind": "generator"},
                         {"id": "l", "node": "c", "p_mw": 60.0, "kind": "load"}],
          "substations": [{"node": "a", "busbars": ["B1", "B2"], "couplers": [["B1", "B2"]],
                           "terminals": [{"element": e, "reachable": ["B1", "B2"], "default": "B1"}
                                         for e in ["ab", "ac", "ad", "g"]]}],
          "busbar_outages": [{"id": "bo", "substation": "a", "busbar": "B1"}], "slack": "c"}
    ctx, orc = make_pair(json.dumps(j3), fitness_variant=2, islanding_penalty_mw=5000.0)
    assert abs(ctx.lambda_b_pre() - 5000.0) < 1e-9 and abs(ctx.pre_optimization_score().fitness) < 1e-9
    _check(ctx, orc, _all_singles(ctx))


def test_slack_station_split():
    # test_dc_engine.cpp:433-471
    j = {"nodes": [{"id": x} for x in "sbcde"],
         "branches": [{"id": i, "from": i[0], "to": i[1], "x_pu": x, "limit_mw": 100.0}
                      for i, x in [("sb", .1), ("sc", .1), ("sd", .1), ("se", .1), ("bc", .2), ("cd", .2),
                                   ("de", .2), ("eb", .2)]],
         "injections": [{"id": "g", "node": "s", "p_mw": 80.0, "kind": "generator"},
                        {"id": "l", "node": "d", "p_mw": 80.0, "kind": "load"}],
         "substations": [{"node": "s", "busbars": ["B1", "B2"], "couplers": [["B1", "B2"]],
                          "terminals": [{"element": e, "reachable": ["B1", "B2"], "default": "B1"}
                                        for e in ["sb", "sc", "sd", "se", "g"]]}],
         "slack": "s"}
    ctx, orc = make_pair(json.dumps(j))
    _check(ctx, orc, _all_singles(ctx))


def test_batch_purity_and_padding(data_dir):
    # test_dc_engine.cpp:337-364: batch == single, order independence
    text = random_grid_json(400, n_nodes=20, extra_edges=12, n_outages=5, n_stations=2)
    ctx, orc = make_pair(text)
    g = orc.random_genomes(17, seed=9)
    a = ctx.evaluate_arrays(g, 3, 2)
    b = ctx.evaluate_arrays(g[::-1].copy(), 3, 2)
    assert np.array_equal(a.fitness, b.fitness[::-1])
    for i in range(len(g)):
        one = ctx.evaluate_arrays(g[i:i + 1], 3, 2)
        assert one.fitness[0] == a.fitness[i] and one.lambda_o[0] == a.lambda_o[i]


def test_high_rank_genomes_four_splits_four_disconnections():
    """n_a = n_d = 4 genomes reach update ranks 8..11 (k_sweep_hi); parity with
    the oracle and no capacity error."""
    import paper_2605_10128_b200 as P
    from tools.synth_grid import synth_grid

    text = json.dumps(synth_grid(300, n_stations=24, seed=31))
    ctx, orc = make_pair(text)
    g = orc.random_genomes(600, 4, 4, seed=77)
    sc = ctx.evaluate_arrays(g, 4, 4)
    ranks = P.batch_ranks(ctx, len(g))
    assert (ranks >= 8).sum() > 10, np.bincount(ranks[ranks >= 0])
    compare_scores(sc, orc.evaluate(g, 4, 4, flows=True), ctx.config.worst_k, ctx.grid.branch_limit)
    fast = ctx.evaluate_arrays(g, 4, 4)
    dense, _ = ctx.evaluate_arrays(g, 4, 4, flows=True)
    assert np.array_equal(fast.fitness, dense.fitness) and np.array_equal(fast.worst_idx, dense.worst_idx)


def test_worst_list_with_many_overloaded_contingencies():
    """Every contingency overloads something (limits x 0.3): more positive
    outage energies than k_finish's shared list holds, so the worst-k
    selection takes its histogram path (dc_engine.cpp:400-420 order: energy
    desc, index asc)."""
    from tools.synth_grid import synth_grid

    doc = synth_grid(400, n_stations=10, seed=41)
    for br in doc["branches"]:
        br["limit_mw"] *= 0.3
    for wk in (20, 3):
        ctx, orc = make_pair(json.dumps(doc), worst_k=wk)
        g = orc.random_genomes(120, seed=6)
        ref = orc.evaluate(g, 3, 2, flows=True)
        assert ((ref["energy"] > 0).sum(1) > 256).sum() > 50
        compare_scores(ctx.evaluate_arrays(g, 3, 2), ref, wk, ctx.grid.branch_limit)
