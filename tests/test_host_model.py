"""CPU tests of the engine's host side (no GPU): grid loading and validation,
import step (action ids must equal the reference's), C-ABI exports."""
import ctypes
import json
import os
import re

import numpy as np
import pytest

import paper_2605_10128_b200 as P
from oracle.oracle import OracleContext, random_grid_json

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_every_declared_symbol_is_exported():
    header = open(os.path.join(ROOT, "include", "topopt_b200.h")).read()
    names = set(re.findall(r"\b(tg_[a-z0-9_]+)\s*\(", header))
    assert len(names) >= 24
    lib = ctypes.CDLL(P.api.L.LIB_PATH)
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing


def _action_parity(text, seed=0, cap=1 << 23):
    g = P.grid_from_json_text(text)
    a = P.build_action_set(g, seed=seed, cap=cap)
    orc = OracleContext(text, enum_seed=seed, enum_cap=cap)
    assert a.n_actions == orc.info["n_actions"]
    assert a.disconnectables.tolist() == orc.info["disconnectables"]
    for i, act in enumerate(orc.info["actions"]):
        assert int(a.substation[i]) == act["substation"]
        assert a.groups[i] == act["group"]
        assert int(a.lambda_r[i]) == act["lambda_r"]
    return a


def test_action_ids_match_reference_on_fixtures(data_dir):
    for name in ("grid14.json", "grid14_congested.json"):
        _action_parity(open(os.path.join(data_dir, name)).read())


@pytest.mark.parametrize("seed", list(range(50, 59)) + list(range(600, 606)) + [70, 99, 300, 400, 500])
def test_action_ids_match_reference_on_random_grids(seed):
    text = random_grid_json(seed, n_nodes=16 + seed % 17, extra_edges=10 + seed % 9, n_outages=4, n_stations=3,
                            multi=seed % 2 == 0, injection=seed % 3 == 0, busbar=True)
    _action_parity(text)


def test_downsampled_enumeration_matches_reference():
    # importer.cpp:256-274: std::sample with derive_seed(seed, 0x5741, station)
    text = random_grid_json(99, n_nodes=25, extra_edges=20, n_stations=3)
    _action_parity(text, seed=42, cap=4)


def test_grid14_congested_import(data_dir):
    g = P.load_grid(os.path.join(data_dir, "grid14_congested.json"))
    a = P.build_action_set(g)
    assert (g.n_nodes, g.n_branches, g.n_contingencies, g.n_busbar_outages) == (14, 20, 10, 1)
    assert a.n_actions == 38 and a.disconnectables.tolist() == [3, 6, 8, 11, 18]
    assert a.station_ranges == {0: (0, 24), 1: (24, 32), 2: (32, 38)}


def test_grid_errors_follow_reference_kinds():
    with pytest.raises(P.ParseError):
        P.grid_from_json_text("{not json")
    with pytest.raises(P.ParseError):
        P.grid_from_json_text('{"nodes": []}')
    zero = {"nodes": [{"id": "a"}, {"id": "b"}],
            "branches": [{"id": "ab", "from": "a", "to": "b", "x_pu": 0.0, "limit_mw": 100.0}], "slack": "a"}
    with pytest.raises(P.ValidationError):
        P.grid_from_json_text(json.dumps(zero))
    isl = {"nodes": [{"id": "a"}, {"id": "b"}, {"id": "c"}],
           "branches": [{"id": "ab", "from": "a", "to": "b", "x_pu": 0.1, "limit_mw": 100.0},
                        {"id": "bc", "from": "b", "to": "c", "x_pu": 0.1, "limit_mw": 100.0}],
           "contingencies": [{"id": "o1", "branches": ["ab"]}], "slack": "a"}
    with pytest.raises(P.IslandedContingency):
        P.grid_from_json_text(json.dumps(isl))
    with pytest.raises(P.IoError):
        P.load_grid("/nonexistent/grid.json")


def test_action_cache_round_trip(tmp_path):
    text = random_grid_json(70, n_nodes=20, extra_edges=14, n_outages=3, n_stations=2)
    g = P.grid_from_json_text(text)
    a = P.build_action_set(g)
    path = str(tmp_path / "cache.json")
    P.save_action_set(a, g, path)
    b = P.load_action_set(g, path)
    assert b is not None and b.n_actions == a.n_actions and b.groups == a.groups
    assert b.disconnectables.tolist() == a.disconnectables.tolist()
    other = P.grid_from_json_text(random_grid_json(71, n_nodes=20, extra_edges=14))
    assert P.load_action_set(other, path) is None


def test_descriptor_kats():
    cfg = P.QdConfig()
    assert P.descriptor_to_cell(0, 0, 0, cfg) == 0
    assert P.descriptor_to_cell(1, 2, 0, cfg) == 7
    assert P.descriptor_to_cell(2, 3, 45, cfg) == 551
    assert P.cell_count(cfg) == 552
    assert P.descriptor_to_cell(0, 0, 99, cfg) == P.descriptor_to_cell(0, 0, 45, cfg)
    hits = np.zeros(P.cell_count(cfg), int)
    for d in range(cfg.d_max + 1):
        for s in range(cfg.s_max + 1):
            for r in range(cfg.r_max + 1):
                hits[P.descriptor_to_cell(d, s, r, cfg)] += 1
    assert (hits == 1).all()
