"""SnapshotChannel (native, channel.hpp:15-79): the reference's channel
semantics tests (test_pipeline.cpp:44-79) on the C-ABI channel; host-only, no GPU."""
import threading

import paper_2605_10128_b200 as P


def tagged(epoch, final=False, n_entries=1):
    entries = [P.SnapshotEntry(3 + i, P.Genome([i, -1, -1], [-1, -1]),
                               P.ScoreVector(1.5 * i, i, 0, 0.0, 0, 1, 2, -10.0 * (i + 1), False, [(4, 2.5)]))
               for i in range(n_entries)]
    return P.RepertoireSnapshot(epoch, 64 * epoch, -10.0, final, entries)


def test_bounded_channel_drops_oldest_non_final():
    ch = P.SnapshotChannel(2)
    for e in (1, 2, 3):
        ch.push(tagged(e))
    assert ch.dropped() == 1
    a, b = ch.try_pop(), ch.try_pop()
    assert (a.epoch, b.epoch) == (2, 3)
    assert ch.try_pop() is None


def test_final_snapshot_survives_overflow():
    ch = P.SnapshotChannel(2)
    ch.push(tagged(1))
    ch.push(tagged(2, True))
    ch.push(tagged(3))
    epochs = []
    while (s := ch.try_pop()) is not None:
        epochs.append(s.epoch)
    assert 2 in epochs


def test_pop_blocks_until_close():
    ch = P.SnapshotChannel(0)
    seen = []

    def consumer():
        while (s := ch.pop()) is not None:
            seen.append(s.epoch)

    t = threading.Thread(target=consumer)
    t.start()
    for i in range(1, 6):
        ch.push(tagged(i, i == 5))
    ch.close()
    t.join(timeout=30)
    assert seen == [1, 2, 3, 4, 5]


def test_snapshot_round_trip():
    ch = P.SnapshotChannel(0)
    s = tagged(7, True, n_entries=3)
    ch.push(s)
    got = ch.pop()
    assert got.epoch == 7 and got.final and got.evaluations == 448
    assert [(e.cell, e.genome.action_slots, e.score.fitness, e.score.worst_contingencies) for e in got.entries] == \
        [(e.cell, e.genome.action_slots, e.score.fitness, e.score.worst_contingencies) for e in s.entries]
