"""Parity at the headline configuration (BASELINE.json configs[3]: the
TSO-scale 7k-bus / 10.5k-branch grid with 500 splittable stations) and on the
cfg2 grid's action table, against the CPU oracle (the reference restatement).

* loop candidates: a full 16384-lane MapElites generation on the device
  (the bench's genome distribution); the scores the skipping sweep gives for
  the whole batch agree with the oracle on a 96-lane sample (1e-9, counts
  exact off the knife edge), and the FlowResult path (base flows, N-1 maxima,
  outage energies) agrees on the same sample (dc_engine.cpp:285-422);
* the archive the loop built: every entry's recorded score equals the
  oracle's evaluation of its genome (the scores the loop inserted);
* mutation / crossover replay the reference's mt19937_64 stream bit for bit
  on the 7292-action cfg4 table and the 870-action cfg2 table, with archive
  parents (qd_optimizer.cpp:21-277): the add-pool / change-pool ranks there
  span thousands of ids.
"""
import numpy as np
import pytest

import paper_2605_10128_b200 as P
from oracle.oracle import OracleContext, qd_config
from tests.parity import compare_flows, compare_scores
from tools.synth_grid import config_json

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tso():
    text = config_json("cfg4")
    g = P.grid_from_json_text(text)
    a = P.build_action_set(g)
    ctx = P.DcContext(g, a)
    orc = OracleContext(text)
    assert a.n_actions == orc.info["n_actions"]
    assert a.disconnectables.tolist() == orc.info["disconnectables"]
    return ctx, orc


@pytest.fixture(scope="module")
def tso_loop(tso):
    ctx, _ = tso
    cfg = P.QdConfig(batch_size=16384, seed=5, iters_per_epoch=1 << 30)
    sess = P.QdSession(ctx, cfg)
    sess.step(3)
    return sess, cfg


def test_tso_loop_candidates_match_oracle(tso, tso_loop):
    ctx, orc = tso
    sess, _ = tso_loop
    genomes = sess.offspring()
    full = ctx.evaluate_arrays(genomes, 3, 2)  # the whole 16384-lane batch, scores-only skipping sweep
    assert np.isfinite(full.fitness).mean() > 0.9
    pick = np.random.default_rng(41).choice(len(genomes), 96, replace=False)
    sub = genomes[pick]
    ref = orc.evaluate(sub, 3, 2, flows=True)
    sc, fr = ctx.evaluate_arrays(sub, 3, 2, flows=True)
    compare_scores(sc, ref, ctx.config.worst_k, ctx.grid.branch_limit)
    compare_flows(fr, ref)
    for f in ("fitness", "lambda_o", "lambda_c", "lambda_c0", "lambda_b", "islanded", "worst_n", "worst_idx",
              "worst_energy"):
        assert np.array_equal(getattr(full, f)[pick], getattr(sc, f)), f"{f}: full batch vs sample batch"


def test_tso_archive_scores_match_oracle(tso, tso_loop):
    ctx, orc = tso
    sess, cfg = tso_loop
    snap = sess.fetch()
    assert len(snap.entries) > 50
    rng = np.random.default_rng(3)
    pick = rng.choice(len(snap.entries), min(48, len(snap.entries)), replace=False)
    ents = [snap.entries[i] for i in pick]
    g = np.array([e.genome.action_slots + e.genome.disconnection_slots for e in ents], np.int32)
    ref = orc.evaluate(g, 3, 2)
    tol = lambda a, b: abs(a - b) <= 1e-9 * max(1.0, abs(b))  # noqa: E731
    for i, e in enumerate(ents):
        s = e.score
        assert (s.lambda_d, s.lambda_s, s.lambda_r) == (ref["lambda_d"][i], ref["lambda_s"][i], ref["lambda_r"][i])
        assert e.cell == P.descriptor_to_cell(s.lambda_d, s.lambda_s, s.lambda_r, cfg)
        assert tol(s.lambda_o, ref["lambda_o"][i]) and tol(s.lambda_b, ref["lambda_b"][i])
        # counts decide on |f| > limit; the synthetic limits keep flows off the knife edge
        assert (s.lambda_c, s.lambda_c0) == (ref["lambda_c"][i], ref["lambda_c0"][i])
        assert tol(s.fitness, ref["fitness"][i])
        assert [k for k, _ in s.worst_contingencies] == ref["worst_idx"][i, :ref["worst_n"][i]].tolist()


def _replay_table(ctx, orc, parents, n):
    for kw in ({}, {"mutation_mean": 4.0}):
        cfg, ocfg = P.QdConfig(**kw), qd_config(**kw)
        seeds = np.arange(n, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15) + np.uint64(101)
        par = parents[np.arange(n) % len(parents)]
        got = P.mutate_lanes(ctx, cfg, par, seeds)
        for i in range(n):
            want, _ = orc.mutate(ocfg, par[i], int(seeds[i]))
            assert got[i].tolist() == want.tolist(), (i, par[i], got[i], want)
    for pc1 in (0.75, 0.3):
        cfg, ocfg = P.QdConfig(p_crossover_parent1=pc1), qd_config(p_crossover_parent1=pc1)
        seeds = np.arange(n, dtype=np.uint64) * np.uint64(7919) + np.uint64(5)
        p1 = parents[np.arange(n) % len(parents)]
        p2 = parents[(np.arange(n) * 7 + 3) % len(parents)]
        got = P.crossover_lanes(ctx, cfg, p1, p2, seeds)
        for i in range(n):
            want = orc.crossover(ocfg, p1[i], p2[i], int(seeds[i]))
            assert got[i].tolist() == want.tolist(), (i, p1[i], p2[i], got[i], want)


def _parents(snap, orc, seed):
    arch = np.array([e.genome.action_slots + e.genome.disconnection_slots for e in snap.entries], np.int32)
    rnd = orc.random_genomes(200, 3, 2, seed=seed)
    rnd[:5] = -1  # empty parents: the forced add (qd_optimizer.cpp:170-172)
    return np.concatenate([arch, rnd])


def test_tso_rng_replay_on_action_table(tso, tso_loop):
    ctx, orc = tso
    sess, _ = tso_loop
    assert orc.info["n_actions"] > 5000
    _replay_table(ctx, orc, _parents(sess.fetch(), orc, 13), 400)


def test_cfg2_rng_replay_on_action_table():
    text = config_json("cfg2")
    g = P.grid_from_json_text(text)
    ctx = P.DcContext(g, P.build_action_set(g))
    orc = OracleContext(text)
    assert orc.info["n_actions"] > 500
    sess = P.QdSession(ctx, P.QdConfig(batch_size=4096, seed=9, iters_per_epoch=1 << 30))
    sess.step(4)
    _replay_table(ctx, orc, _parents(sess.fetch(), orc, 17), 600)
