"""Action cache interoperability with the reference (CPU).

grid_content_hash (grid_model.cpp:494-503) is FNV-1a over the canonical dump
grid_to_json_text (grid_model.cpp:423-485); the action cache of
save_action_set / load_action_set (importer.cpp:407-479) is keyed by it. The
engine's host model restates both, so a cache written by `topopt import` loads
in the engine and the reverse. Checked against the oracle (the reference
restatement, same nlohmann/json library) on the bundled grids, random grids
with busbar outages / injections / multi-branch contingencies, and the cfg2
synthetic grid.
"""
import os

import pytest

import paper_2605_10128_b200 as P
from oracle.oracle import OracleContext, random_grid_json
from tools.synth_grid import config_json

DATA = os.path.join(os.path.dirname(__file__), "golden", "data")


def _grids():
    for name in ("grid14.json", "grid14_congested.json"):
        yield name, open(os.path.join(DATA, name)).read()
    for s in range(4):
        yield f"random{s}", random_grid_json(100 + s, 30, 15, 6, 3, multi=True, injection=True, busbar=True)
    yield "cfg2", config_json("cfg2")


@pytest.mark.parametrize("name,text", list(_grids()), ids=lambda x: x if isinstance(x, str) and len(x) < 40 else "")
def test_canonical_dump_and_hash_match_reference(name, text):
    orc = OracleContext(text)
    g = P.grid_from_json_text(text)
    assert g.to_json_text() == orc.grid_json()
    assert g.content_hash() == orc.grid_hash()


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_action_cache_round_trips_between_engine_and_reference(tmp_path, seed):
    text = random_grid_json(200 + seed, 30, 15, 6, 3, multi=True, injection=True, busbar=True)
    orc = OracleContext(text)
    g = P.grid_from_json_text(text)
    a = P.build_action_set(g)
    # engine -> reference: the reference's load_action_set accepts the engine's cache
    assert orc.load_action_cache(a.to_json_text()) == a.n_actions == orc.info["n_actions"]
    # reference -> engine: the engine loads the reference's cache with the same ids
    path = tmp_path / "actions.json"
    path.write_text(orc.action_cache() + "\n")
    b = P.load_action_set(g, str(path))
    assert b is not None and b.n_actions == a.n_actions
    assert b.substation.tolist() == a.substation.tolist() and b.groups == a.groups
    assert b.disconnectables.tolist() == a.disconnectables.tolist()
    # a cache of another grid is rejected (hash mismatch)
    other = P.grid_from_json_text(random_grid_json(999, 30, 15, 6, 3, busbar=True))
    assert P.load_action_set(other, str(path)) is None
