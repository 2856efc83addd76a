"""Timestep extension (BASELINE.json configs[2]: 24 timesteps). The reference
evaluates one injection vector (grid_model.hpp:36-46); with a 'timesteps' key
the engine evaluates every profile and aggregates (model.hpp, engine.cu
k_accum_t / k_finish_agg). Pinned against the oracle run once per timestep on
the single-profile grids, aggregated by tests/parity.py:oracle_timesteps."""
import json

import numpy as np
import pytest

import paper_2605_10128_b200 as P
from oracle.oracle import OracleContext
from tests.parity import compare_scores, oracle_timesteps, timestep_grids
from tools.synth_grid import synth_grid

pytestmark = pytest.mark.gpu


def _ctx(text):
    g = P.grid_from_json_text(text)
    return P.DcContext(g, P.build_action_set(g))


def test_timesteps_match_oracle_per_timestep_sum():
    for seed, n, T in ((11, 60, 4), (12, 120, 6)):
        text = json.dumps(synth_grid(n, n_stations=6, seed=seed, n_timesteps=T))
        ctx = _ctx(text)
        orcs = [OracleContext(t) for t in timestep_grids(text)]
        assert len(orcs) == T
        genomes = orcs[0].random_genomes(200, 3, 2, seed=seed)
        sc = ctx.evaluate_arrays(genomes, 3, 2)
        ref = oracle_timesteps(orcs, genomes, 3, 2)
        compare_scores(sc, ref, 20)
        # the pre-optimization score is the aggregated empty genome
        pre = oracle_timesteps(orcs, np.full((1, 5), -1, np.int32), 3, 2)
        assert abs(ctx.pre_optimization_score().fitness - pre["fitness"][0]) <= 1e-9 * max(1.0, abs(pre["fitness"][0]))


def test_single_timestep_profile_is_the_reference():
    base = synth_grid(80, n_stations=5, seed=21)
    one = dict(base)
    one["timesteps"] = {"count": 1, "injections": {i["id"]: [i["p_mw"]] for i in base["injections"]}}
    a, b = _ctx(json.dumps(base)), _ctx(json.dumps(one))
    genomes = OracleContext(json.dumps(base)).random_genomes(100, 3, 2, seed=3)
    sa, sb = a.evaluate_arrays(genomes, 3, 2), b.evaluate_arrays(genomes, 3, 2)
    for f in ("fitness", "lambda_o", "lambda_c", "lambda_c0", "worst_n", "worst_idx", "worst_energy"):
        assert np.array_equal(getattr(sa, f), getattr(sb, f)), f


def test_timestep_scale_equals_sum_of_single_profile_contexts():
    """2k-bus grid (configs[2] size), 3 profiles: the aggregated device
    evaluation of 1024 loop candidates equals the per-profile device
    evaluations summed (each of those is reference semantics)."""
    text = json.dumps(synth_grid(2000, n_stations=100, seed=3, n_timesteps=3))
    ctx = _ctx(text)
    sess = P.QdSession(ctx, P.QdConfig(batch_size=1024, seed=5, iters_per_epoch=1 << 30))
    sess.step(3)
    genomes = sess.offspring()
    agg = ctx.evaluate_arrays(genomes, 3, 2)
    parts = [_ctx(t).evaluate_arrays(genomes, 3, 2) for t in timestep_grids(text)]
    isl = np.zeros(len(genomes), bool)
    for p in parts:
        isl |= p.islanded.astype(bool)
    assert np.array_equal(agg.islanded.astype(bool), isl)
    live = ~isl
    for f in ("lambda_c", "lambda_c0", "islanded_outages"):
        assert np.array_equal(getattr(agg, f)[live], sum(getattr(p, f) for p in parts)[live]), f
    for f in ("lambda_o", "lambda_b"):
        want = sum(getattr(p, f) for p in parts)[live]
        got = getattr(agg, f)[live]
        assert np.max(np.abs(got - want) / np.maximum(1.0, np.abs(want))) <= 1e-12, f


def test_more_profiles_than_one_masked_launch():
    """10 profiles: the masked sweep runs kMaskProfiles (8) profiles per launch,
    so this covers a full launch plus a partial one; against the oracle run per
    timestep and summed."""
    text = json.dumps(synth_grid(150, n_stations=8, seed=31, n_timesteps=10))
    ctx = _ctx(text)
    orcs = [OracleContext(t) for t in timestep_grids(text)]
    assert len(orcs) == 10
    genomes = orcs[0].random_genomes(300, 3, 2, seed=7)
    sc = ctx.evaluate_arrays(genomes, 3, 2)
    ref = oracle_timesteps(orcs, genomes, 3, 2)
    compare_scores(sc, ref, 20)


def test_cfg3_against_the_oracle_per_profile():
    """The bench's configs[2] grid itself (2k buses, 100 split stations, 24
    timesteps: mask pass + three masked launches of 8 profiles) on 64 MapElites
    loop candidates, against the oracle run on each of the 24 single-profile
    grids and aggregated (not only against the engine's own per-profile path)."""
    from tools.synth_grid import config_json

    text = config_json("cfg3")
    ctx = _ctx(text)
    sess = P.QdSession(ctx, P.QdConfig(batch_size=512, seed=9, iters_per_epoch=1 << 30))
    sess.step(3)
    genomes = sess.offspring()[:64]
    sc = ctx.evaluate_arrays(genomes, 3, 2)
    orcs = [OracleContext(t) for t in timestep_grids(text)]
    assert len(orcs) == 24
    ref = oracle_timesteps(orcs, genomes, 3, 2)
    compare_scores(sc, ref, 20)
