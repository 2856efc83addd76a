"""build_ptdf (importer.cpp:358-401) on the device, against the oracle's
restatement and the reference's own PTDF tests (test_importer.cpp:269-320):
single-branch and triangle known answers, the angle formulation on the
14-bus fixture, nodal balance on random grids, and the full matrix at cfg2
scale (1k nodes / 1.5k branches)."""
import json
import os

import numpy as np
import pytest

import paper_2605_10128_b200 as P
from oracle.oracle import OracleContext, random_grid_json
from tools.synth_grid import config_json

pytestmark = pytest.mark.gpu

TWO_NODE = {"nodes": [{"id": "a"}, {"id": "b"}],
            "branches": [{"id": "ab", "from": "a", "to": "b", "x_pu": 0.1, "limit_mw": 150.0}],
            "injections": [{"id": "g", "node": "a", "p_mw": 100.0, "kind": "generator"},
                           {"id": "l", "node": "b", "p_mw": 100.0, "kind": "load"}], "slack": "b"}
TRIANGLE = {"nodes": [{"id": "a"}, {"id": "b"}, {"id": "c"}],
            "branches": [{"id": "ab", "from": "a", "to": "b", "x_pu": 0.2, "limit_mw": 100.0},
                         {"id": "ac", "from": "a", "to": "c", "x_pu": 0.2, "limit_mw": 100.0},
                         {"id": "bc", "from": "b", "to": "c", "x_pu": 0.2, "limit_mw": 100.0}],
            "injections": [{"id": "g", "node": "a", "p_mw": 90.0, "kind": "generator"},
                           {"id": "l", "node": "c", "p_mw": 90.0, "kind": "load"}], "slack": "c"}


def _p(text):
    d = json.loads(text)
    ids = [n["id"] for n in d["nodes"]]
    p = np.zeros(len(ids))
    for i in d.get("injections", []):
        p[ids.index(i["node"])] += i["p_mw"] if i["kind"] == "generator" else -i["p_mw"]
    p[ids.index(d["slack"])] -= p.sum()  # base_power_vector, grid_model.cpp:505-510
    return p


def test_ptdf_known_answers():
    g = P.grid_from_json_text(json.dumps(TWO_NODE))
    m = P.build_ptdf(g)
    assert m[0, 0] == pytest.approx(1.0) and m[0, 1] == pytest.approx(0.0)
    assert (m @ _p(json.dumps(TWO_NODE)))[0] == pytest.approx(100.0)
    t = P.grid_from_json_text(json.dumps(TRIANGLE))
    f = P.build_ptdf(t) @ _p(json.dumps(TRIANGLE))
    assert f == pytest.approx([30.0, 60.0, 30.0])


def test_ptdf_matches_oracle_and_balances(data_dir):
    texts = [open(os.path.join(data_dir, n)).read() for n in ("grid14.json", "grid14_congested.json")]
    texts += [random_grid_json(seed, 30, 15, 6, 3) for seed in range(60, 67)]
    texts.append(config_json("cfg2"))
    for text in texts:
        g = P.grid_from_json_text(text)
        got = P.build_ptdf(g)
        want = OracleContext(text).build_ptdf()
        assert got.shape == want.shape
        assert np.max(np.abs(got - want)) <= 1e-9 * max(1.0, np.max(np.abs(want)))
        # nodal balance (test_importer.cpp:295-311): flows reproduce the injections
        d = json.loads(text)
        ids = {n["id"]: i for i, n in enumerate(d["nodes"])}
        p = _p(text)
        f = got @ p
        res = np.zeros(len(ids))
        for e, br in enumerate(d["branches"]):
            res[ids[br["from"]]] += f[e]
            res[ids[br["to"]]] -= f[e]
        keep = np.arange(len(ids)) != ids[d["slack"]]
        assert np.max(np.abs(res[keep] - p[keep])) < 1e-9 * max(1.0, np.max(np.abs(p)))
        assert np.all(got[:, ids[d["slack"]]] == 0.0)
