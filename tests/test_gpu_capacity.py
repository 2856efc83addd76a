"""Compile-time capacities never truncate (dc_engine.cpp:319-356, 373-386
handle any outage size): an outage larger than the engine's capacity is a
CapacityError, an outage inside it matches the oracle. Capacity errors that
happen inside the device loop are sticky and surface on the next host call."""
import json

import numpy as np
import pytest

import paper_2605_10128_b200 as P
from tests.parity import compare_flows, compare_scores, make_pair
from tools.synth_grid import synth_grid

pytestmark = pytest.mark.gpu


def _wheel(n_spokes: int) -> dict:
    """A hub with n_spokes branches to a ring of rim nodes (no bridges), the
    hub a 2-busbar substation whose busbar B1 carries every spoke."""
    nodes = [{"id": "hub"}] + [{"id": f"r{i}"} for i in range(n_spokes)]
    br = [{"id": f"s{i}", "from": "hub", "to": f"r{i}", "x_pu": 0.1 + 0.01 * i, "limit_mw": 60.0}
          for i in range(n_spokes)]
    br += [{"id": f"c{i}", "from": f"r{i}", "to": f"r{(i + 1) % n_spokes}", "x_pu": 0.2, "limit_mw": 80.0}
           for i in range(n_spokes)]
    inj = [{"id": "g", "node": "r0", "p_mw": 300.0, "kind": "generator"}]
    inj += [{"id": f"l{i}", "node": f"r{i}", "p_mw": 10.0, "kind": "load"} for i in range(1, n_spokes)]
    return {"nodes": nodes, "branches": br, "injections": inj,
            "contingencies": [{"id": f"o{i}", "branches": [f"c{i}"]} for i in range(0, n_spokes, 3)],
            "busbar_outages": [{"id": "bo-hub-B1", "substation": "hub", "busbar": "B1"}],
            "substations": [{"node": "hub", "busbars": ["B1", "B2"], "couplers": [["B1", "B2"]],
                             "terminals": [{"element": f"s{i}", "reachable": ["B1", "B2"], "default": "B1"}
                                           for i in range(n_spokes)]}],
            "slack": "r0"}


def test_busbar_implied_set_over_capacity_is_an_error():
    g = P.grid_from_json_text(json.dumps(_wheel(30)))
    with pytest.raises(P.CapacityError):
        P.DcContext(g, P.build_action_set(g))


def test_busbar_implied_set_inside_capacity_matches_oracle():
    text = json.dumps(_wheel(12))
    ctx, orc = make_pair(text)
    genomes = orc.random_genomes(64, 3, 2, seed=3)
    sc, fr = ctx.evaluate_arrays(genomes, 3, 2, flows=True)
    ref = orc.evaluate(genomes, 3, 2, flows=True)
    compare_scores(sc, ref, ctx.config.worst_k, ctx.grid.branch_limit)
    compare_flows(fr, ref)


def _many_injection_outage(n_inj: int) -> str:
    doc = synth_grid(60, seed=11, n_stations=6)
    loads = [i["id"] for i in doc["injections"] if i["kind"] == "load"][:n_inj]
    assert len(loads) == n_inj
    doc["contingencies"].append({"id": "o-many-loads", "branches": [], "injections": loads})
    doc["contingencies"].append({"id": "o-branch-and-loads", "branches": [doc["contingencies"][0]["branches"][0]],
                                 "injections": loads[: n_inj // 2]})
    return json.dumps(doc)


def test_twenty_injection_contingency_matches_oracle():
    text = _many_injection_outage(20)
    ctx, orc = make_pair(text)
    genomes = orc.random_genomes(128, 3, 2, seed=4)
    sc, fr = ctx.evaluate_arrays(genomes, 3, 2, flows=True)
    ref = orc.evaluate(genomes, 3, 2, flows=True)
    compare_scores(sc, ref, ctx.config.worst_k, ctx.grid.branch_limit)
    compare_flows(fr, ref)
    # the injection outages carry energy: they are evaluated, not dropped
    k = orc.info["n_contingencies"] - 2
    assert np.array_equal(fr.outage_energy[:, k] > 0, ref["energy"][:, k] > 0)


def test_injection_outage_over_capacity_is_an_error():
    g = P.grid_from_json_text(_many_injection_outage(40))
    with pytest.raises(P.CapacityError):
        P.DcContext(g, P.build_action_set(g))
