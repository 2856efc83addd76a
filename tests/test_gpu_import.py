"""Device islanding validation of candidate splits (tg_actionset_build_device,
SURVEY §8(f) row 3) against the host path and the oracle restatement of
importer.cpp:239-356: the action ids, groups and realizations must be equal
(exact: the validation is a graph property)."""
import time

import pytest

from oracle.oracle import OracleContext, random_grid_json

pytestmark = pytest.mark.gpu


def _same(a, b):
    assert a.n_actions == b.n_actions
    assert a.substation.tolist() == b.substation.tolist()
    assert a.groups == b.groups
    assert a.lambda_r.tolist() == b.lambda_r.tolist()
    assert a.disconnectables.tolist() == b.disconnectables.tolist()


@pytest.mark.parametrize("seed", [1, 2, 3, 5, 8, 13, 21, 34])
def test_random_grids_device_equals_host_and_oracle(seed):
    import paper_2605_10128_b200 as P

    text = random_grid_json(seed, n_nodes=12 + 5 * seed % 40, extra_edges=4 + seed % 9, n_outages=6,
                            n_stations=4, multi=seed % 2 == 0, injection=seed % 3 == 0)
    g = P.grid_from_json_text(text)
    dev = P.build_action_set(g, device=0)
    host = P.build_action_set(g)
    _same(dev, host)
    orc = OracleContext(text)
    assert dev.n_actions == orc.info["n_actions"]
    for i, act in enumerate(orc.info["actions"]):
        assert dev.substation[i] == act["substation"] and dev.groups[i] == act["group"]


@pytest.mark.parametrize("cfg", ["cfg2", "cfg4"])
def test_synthetic_configs_device_equals_host(cfg):
    import paper_2605_10128_b200 as P
    from tools.synth_grid import config_json

    g = P.grid_from_json_text(config_json(cfg))
    t0 = time.perf_counter()
    dev = P.build_action_set(g, device=0)
    t1 = time.perf_counter()
    host = P.build_action_set(g)
    t2 = time.perf_counter()
    _same(dev, host)
    print(f"{cfg}: {dev.n_actions} actions, device build {t1 - t0:.2f} s, host build {t2 - t1:.2f} s")
