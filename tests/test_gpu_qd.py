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
from tests.parity import compare_scores, replay_inserts

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


_replay_oracle = replay_inserts


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


def _scores_from_trace(entries, worst_k=20):
    n = len(entries)
    sc = P.ScoreArrays(n, worst_k)
    for i, e in enumerate(entries):
        fit, ld, ls, lr, lo, lc, lc0, lb, wn, wi, wv = e
        sc.fitness[i] = -np.inf if fit <= -1e299 else fit
        sc.lambda_d[i], sc.lambda_s[i], sc.lambda_r[i] = ld, ls, lr
        sc.lambda_o[i], sc.lambda_c[i], sc.lambda_c0[i], sc.lambda_b[i] = lo, lc, lc0, lb
        sc.worst_n[i] = wn
        sc.worst_idx[i, :wn] = wi
        sc.worst_energy[i, :wn] = wv
    return sc


def test_lockstep_loop_matches_reference(data_dir):
    """BASELINE config 1 (grid14_congested, batch 64, 50 generations): per
    generation the device offspring equal the reference's bit for bit, the
    device scores match within 1e-9, and with the reference's scores inserted
    the device archive equals the reference archive exactly (given equal
    fitness, the archive contents are bit-identical)."""
    text = open(os.path.join(data_dir, "grid14_congested.json")).read()
    ctx, orc = _ctx(text)
    for seed in (1, 777):
        kw = dict(seed=seed, batch_size=64, iters_per_epoch=500, max_evaluations=3201)
        trace = orc.run_optimizer_trace(qd_config(**kw))
        assert len(trace["iters"]) == 50
        sess = P.QdSession(ctx, P.QdConfig(**kw))
        for it in trace["iters"]:
            ref_g = np.array(it["genomes"], np.int32)
            got_g = sess.offspring()
            assert np.array_equal(got_g, ref_g), f"offspring differ at iteration {it['it']}"
            ref_sc = _scores_from_trace(it["scores"])
            # device scores of the same lanes: 1e-9, counts exact off the knife edge
            mine = ctx.evaluate_arrays(got_g, 3, 2)
            compare_scores(mine, orc.evaluate(got_g, 3, 2, flows=True), 20, ctx.grid.branch_limit)
            sess.insert(got_g, ref_sc)
        snap = sess.fetch(final=True)
        got = [[e.cell, e.genome.action_slots + e.genome.disconnection_slots, e.score.fitness] for e in snap.entries]
        want = [[c, g, f] for c, g, f in trace["final"]]
        # the seed entry (cell 0) carries the device's own score of the empty genome
        assert got[0][:2] == want[0][:2] and abs(got[0][2] - want[0][2]) <= 1e-9 * abs(want[0][2])
        assert got[1:] == want[1:]


def test_optimizer_run_grid14_congested(data_dir):
    """Free-running device loop on config 1: same evaluation count, epochs and
    best fitness as the reference; elitism per cell across snapshots."""
    text = open(os.path.join(data_dir, "grid14_congested.json")).read()
    ctx, orc = _ctx(text)
    kw = dict(seed=1, batch_size=64, iters_per_epoch=7, max_evaluations=3201)
    snaps = []
    res = P.run_optimizer(ctx, P.QdConfig(**kw), sink=snaps.append)
    ref = orc.run_optimizer(qd_config(**kw), all_snapshots=True)
    assert res.stats.evaluations == ref["stats"]["evaluations"] == 3201
    assert res.stats.epochs == ref["stats"]["epochs"]
    assert abs(res.repertoire.best_fitness - ref["snapshots"][-1]["best_fitness"]) <= 1e-6
    assert len(snaps) == len(ref["snapshots"]) and snaps[-1].final
    best = {}
    for s in snaps:
        now = {}
        for e in s.entries:
            assert e.cell == P.descriptor_to_cell(e.score.lambda_d, e.score.lambda_s, e.score.lambda_r, P.QdConfig())
            now[e.cell] = max(now.get(e.cell, -np.inf), e.score.fitness)
        for c, f in best.items():
            assert now[c] >= f - 1e-12
        best = now


def test_optimizer_mini_grid_semantics():
    # test_qd_optimizer.cpp:291-369
    ctx, orc = _ctx(json.dumps(MINI))
    kw = dict(seed=11, batch_size=16, iters_per_epoch=10)
    res = P.run_optimizer(ctx, P.QdConfig(max_evaluations=1, **kw))
    assert res.stats.evaluations == 1 and len(res.repertoire.entries) == 1
    assert res.repertoire.entries[0].genome.is_empty()
    res = P.run_optimizer(ctx, P.QdConfig(max_evaluations=4000, **kw))
    assert abs(res.repertoire.best_fitness) < 1e-9  # the clearing disconnection is found
    res = P.run_optimizer(ctx, P.QdConfig(max_evaluations=10000, **kw))
    assert any(e.score.lambda_s >= 1 for e in res.repertoire.entries)
    assert any(e.score.lambda_d >= 1 for e in res.repertoire.entries)
    with pytest.raises(P.ConfigError):
        P.run_optimizer(ctx, P.QdConfig(batch_size=0))


def test_island_merge_matches_sequential_insert(data_dir):
    """Island exchange: two islands (own contexts, own seeds)
    pack their archives on the device, the blobs are concatenated as an
    allgather would, and the device merge equals a sequential
    Repertoire::insert replay of island 0's entries then island 1's (cell
    order, position order). Both islands end with the same archive; the
    host mirror of the blob layout decodes the device blob; the loop keeps
    running after a merge."""
    import torch

    from paper_2605_10128_b200.islands import BlobLayout, IslandExchange, pack_entries, unpack_blob

    text = open(os.path.join(data_dir, "grid14_congested.json")).read()
    sess, snaps = [], []
    for seed in (3, 4):
        ctx, _ = _ctx(text)
        s = P.QdSession(ctx, P.QdConfig(seed=seed, batch_size=64, cell_capacity=3))
        s.step(6)
        sess.append(s)
        snaps.append(s.fetch())
    cfg = sess[0].cfg
    lay = BlobLayout(P.cell_count(cfg), cfg.cell_capacity, cfg.n_a + cfg.n_d, 20)
    assert sess[0].blob_bytes() == lay.nbytes
    blobs = torch.empty(2 * lay.nbytes, dtype=torch.uint8, device="cuda")
    for i, s in enumerate(sess):
        s.pack(blobs[i * lay.nbytes:].data_ptr())
    torch.cuda.synchronize()
    host = blobs.cpu().numpy()
    # the host mirror decodes the device blob into the fetched snapshot
    for i, snap in enumerate(snaps):
        dec = unpack_blob(lay, host[i * lay.nbytes:(i + 1) * lay.nbytes])
        assert [(d["cell"], d["genome"], d["fitness"]) for d in dec] == [
            (e.cell, e.genome.action_slots + e.genome.disconnection_slots, e.score.fitness) for e in snap.entries]
        assert [d["worst"] for d in dec] == [[(k, v) for k, v in e.score.worst_contingencies] for e in snap.entries]
        # ... and the host encoder reproduces the device blob byte for byte
        assert np.array_equal(pack_entries(lay, snap.entries), host[i * lay.nbytes:(i + 1) * lay.nbytes])
    stream = [(e.genome.action_slots + e.genome.disconnection_slots,
               dict(fitness=e.score.fitness, lambda_d=e.score.lambda_d, lambda_s=e.score.lambda_s,
                    lambda_r=e.score.lambda_r)) for snap in snaps for e in snap.entries]
    _, cells = replay_inserts(stream, cfg)
    want = {c: v for c, v in cells.items() if v}
    merged = []
    for s in sess:
        s.merge(blobs.data_ptr(), 2)
        m = s.fetch()
        got = {}
        for e in m.entries:
            got.setdefault(e.cell, []).append((e.genome.canonical_key(), e.score.fitness,
                                               e.genome.action_slots + e.genome.disconnection_slots))
        assert got == want
        merged.append([(e.cell, e.genome.action_slots + e.genome.disconnection_slots, e.score.fitness,
                        e.score.lambda_o, e.score.worst_contingencies) for e in m.entries])
    assert merged[0] == merged[1]
    assert max(snaps[0].best_fitness, snaps[1].best_fitness) == sess[0].fetch().best_fitness
    # a single island merging its own blob is unchanged; the loop continues after merges
    ex = IslandExchange(sess[0])
    before = sess[0].fetch().entries
    ex.exchange()
    after = sess[0].fetch().entries
    assert [(e.cell, e.score.fitness) for e in before] == [(e.cell, e.score.fitness) for e in after]
    sess[0].step(3)
    assert sess[0].fetch().best_fitness >= snaps[0].best_fitness


def _valid(ctx, g, n_a=3):
    # genome_valid, genome.cpp:49-63
    acts = [a for a in g[:n_a] if a >= 0]
    disc = [d for d in g[n_a:] if d >= 0]
    st = [ctx.actions.substation_of(a) for a in acts]
    return (len(set(st)) == len(st) and len(set(disc)) == len(disc) and all(a < ctx.actions.n_actions for a in acts)
            and all(d < len(ctx.actions.disconnectables) for d in disc))


def test_philox_mode_valid_and_distributed_like_replay(data_dir):
    """Counter-based lane RNG (north_star item 1; extension): valid offspring,
    the same operator statistics as the reference stream (two-sample
    chi-square on the changed-slot counts), a working optimizer."""
    text = open(os.path.join(data_dir, "grid14_congested.json")).read()
    ctx, orc = _ctx(text)
    par = _parents(orc, 20000, 8)
    seeds = np.arange(len(par), dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15) + np.uint64(99)
    hist = {}
    for rng in ("replay", "philox"):
        kids = P.mutate_lanes(ctx, P.QdConfig(rng=rng), par, seeds)
        assert all(_valid(ctx, k) for k in kids)
        changed = (kids != par).sum(1)
        hist[rng] = np.bincount(changed, minlength=6)[:6].astype(float)
        x = P.crossover_lanes(ctx, P.QdConfig(rng=rng), par, par[::-1].copy(), seeds)
        assert all(_valid(ctx, k) for k in x)
    a, b = hist["replay"], hist["philox"]
    keep = (a + b) > 20
    chi2 = float((((a - b) ** 2)[keep] / (a + b)[keep]).sum())
    assert chi2 < 25.0, (a, b)   # 5 dof, p ~ 1e-4
    assert not np.array_equal(P.mutate_lanes(ctx, P.QdConfig(rng="philox"), par[:64], seeds[:64]),
                              P.mutate_lanes(ctx, P.QdConfig(rng="replay"), par[:64], seeds[:64]))
    kw = dict(seed=3, batch_size=64, iters_per_epoch=50, max_evaluations=1 + 64 * 150)
    rep = P.run_optimizer(ctx, P.QdConfig(**kw))
    phi = P.run_optimizer(ctx, P.QdConfig(rng="philox", **kw))
    assert phi.stats.evaluations == rep.stats.evaluations
    assert phi.repertoire.best_fitness >= rep.repertoire.best_fitness - 0.05 * abs(rep.repertoire.best_fitness)
    with pytest.raises(P.ConfigError):
        P.QdConfig(rng="xorshift").to_c()


def test_optimizer_feeds_native_channel_asynchronously(data_dir):
    """Snapshot -> AC hand-off: epoch snapshots are
    packed on the device and copied asynchronously; fed into a native
    SnapshotChannel while a consumer thread pops them, they equal the
    synchronous sink's snapshots (make_snapshot order, last one final)."""
    import threading

    text = open(os.path.join(data_dir, "grid14_congested.json")).read()
    ctx, _ = _ctx(text)
    kw = dict(seed=9, batch_size=64, iters_per_epoch=5, max_evaluations=1 + 64 * 42)
    via_sink = []
    P.run_optimizer(ctx, P.QdConfig(**kw), sink=via_sink.append)
    ch = P.SnapshotChannel(0)
    got = []

    def consumer():
        while (s := ch.pop()) is not None:
            got.append(s)

    t = threading.Thread(target=consumer)
    t.start()
    res = P.run_optimizer(ctx, P.QdConfig(**kw), channel=ch)
    ch.close()
    t.join(timeout=60)
    assert len(got) == len(via_sink) == res.stats.epochs and got[-1].final
    for a, b in zip(got, via_sink):
        assert (a.epoch, a.evaluations, a.best_fitness, a.final) == (b.epoch, b.evaluations, b.best_fitness, b.final)
        assert [(e.cell, e.genome.action_slots + e.genome.disconnection_slots, e.score.fitness,
                 e.score.worst_contingencies) for e in a.entries] == \
            [(e.cell, e.genome.action_slots + e.genome.disconnection_slots, e.score.fitness,
              e.score.worst_contingencies) for e in b.entries]
    # bounded channel: the producer never blocks, the final snapshot survives
    ch2 = P.SnapshotChannel(1)
    P.run_optimizer(ctx, P.QdConfig(**kw), channel=ch2)
    last = ch2.try_pop()
    assert last is not None and last.final and ch2.dropped() == res.stats.epochs - 1


def test_batch_sharded_generations_equal_one_gpu(data_dir):
    """SURVEY.md 8(e) parity mode: two 'ranks' (own contexts, same seed) draw
    the same offspring, each evaluates half of the lanes, the score slices are
    exchanged as device blobs and both insert all lanes: after 6 generations
    both archives equal the unsharded run's bit for bit."""
    import torch

    text = open(os.path.join(data_dir, "grid14_congested.json")).read()
    kw = dict(seed=12, batch_size=64, iters_per_epoch=1 << 30)
    ref_ctx, _ = _ctx(text)
    ref = P.QdSession(ref_ctx, P.QdConfig(**kw))
    ref.step(6)
    want = [(e.cell, e.genome.action_slots + e.genome.disconnection_slots, e.score.fitness, e.score.lambda_o,
             e.score.worst_contingencies) for e in ref.fetch().entries]
    ranks = []
    for _ in range(2):
        ctx, _ = _ctx(text)
        ranks.append(P.QdSession(ctx, P.QdConfig(**kw)))
    half = 32
    nb = ranks[0].scores_blob_bytes(half)
    blobs = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(2)]
    for _ in range(6):
        for r, s in enumerate(ranks):
            s.generation_begin()
            s.evaluate_lanes(r * half, (r + 1) * half)
            s.scores_pack(r * half, (r + 1) * half, blobs[r].data_ptr())
        torch.cuda.synchronize()
        for r, s in enumerate(ranks):
            o = 1 - r
            s.scores_unpack(o * half, (o + 1) * half, blobs[o].data_ptr())
            s.generation_end()
    for s in ranks:
        got = [(e.cell, e.genome.action_slots + e.genome.disconnection_slots, e.score.fitness, e.score.lambda_o,
                e.score.worst_contingencies) for e in s.fetch().entries]
        assert got == want
