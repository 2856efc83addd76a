"""The engine's own NCCL exchange (tg_islands_*, host/islands.cpp) on one GPU:
a one-rank communicator runs the real ncclCommInitRank / ncclAllGather path
on the context stream. (Two NCCL ranks cannot share one device; the N>1 host
logic is covered by tests/test_islands_gloo.py and the driver's multi-GPU run.)

* island mode: pack -> ncclAllGather -> merge after every generation gives the
  archive of the torch-side IslandExchange on an identically seeded session;
* shard mode: batch-sharded generations through the native path equal plain
  generations (one population, lane-order insert).
"""
import os

import pytest

import paper_2605_10128_b200 as P
from paper_2605_10128_b200.islands import IslandExchange, NativeIslands

pytestmark = pytest.mark.gpu


def _sessions(data_dir, **kw):
    text = open(os.path.join(data_dir, "grid14_congested.json")).read()
    out = []
    for _ in range(2):
        g = P.grid_from_json_text(text)
        ctx = P.DcContext(g, P.build_action_set(g))
        out.append(P.QdSession(ctx, P.QdConfig(**kw)))
    return out


def _archive(sess):
    return [(e.cell, e.genome.action_slots + e.genome.disconnection_slots, e.score.fitness,
             e.score.worst_contingencies) for e in sess.fetch().entries]


def test_native_island_exchange_matches_torch_exchange(data_dir):
    a, b = _sessions(data_dir, seed=7, batch_size=64, cell_capacity=3)
    nat = NativeIslands(a)
    ref = IslandExchange(b)
    nat.step(5, merge_every=1)
    for _ in range(5):
        b.step(1)
        ref.exchange()
    assert nat.exchanges == 5
    assert _archive(a) == _archive(b)
    nat.exchange()
    a.step(2)
    b.step(2)
    assert _archive(a) == _archive(b)


def test_native_shard_step_equals_plain_generations(data_dir):
    a, b = _sessions(data_dir, seed=9, batch_size=64)
    nat = NativeIslands(a)
    nat.shard_step(4)
    b.step(4)
    assert _archive(a) == _archive(b)
