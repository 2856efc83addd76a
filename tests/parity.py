"""Shared parity helpers: run the same genomes through the B200 engine (C ABI)
and the CPU oracle, and compare with the tolerances stated in BASELINE.md §3
(FP64: 1e-9 relative with scale max(1, |x|); counts and encodings exact)."""
from __future__ import annotations

import json

import numpy as np

from oracle.oracle import OracleContext

TOL = 1e-9


def rel_err(got, want) -> float:
    got = np.asarray(got, float)
    want = np.asarray(want, float)
    if got.size == 0:
        return 0.0
    fin = np.isfinite(want)
    assert np.array_equal(np.isfinite(got), fin)
    if not fin.any():
        return 0.0
    return float(np.max(np.abs(got[fin] - want[fin]) / np.maximum(1.0, np.abs(want[fin]))))


def make_pair(grid_json: str, **dc):
    """(product DcContext, oracle context) for one grid; asserts equal action ids."""
    import paper_2605_10128_b200 as P

    g = P.grid_from_json_text(grid_json)
    a = P.build_action_set(g)
    cfg = P.DcConfig(**{k: v for k, v in dc.items() if k in P.DcConfig.__dataclass_fields__})
    ctx = P.DcContext(g, a, cfg)
    orc = OracleContext(grid_json, penalty=cfg.islanding_penalty_mw, worst_k=cfg.worst_k, weight_c0=cfg.weight_c0,
                        weight_c=cfg.weight_c, variant=cfg.fitness_variant)
    assert a.n_actions == orc.info["n_actions"]
    assert a.disconnectables.tolist() == orc.info["disconnectables"]
    for i, act in enumerate(orc.info["actions"]):
        assert a.substation[i] == act["substation"] and a.groups[i] == act["group"]
        assert a.lambda_r[i] == act["lambda_r"]
    return ctx, orc


def knife_edges(values, limits, tol=TOL):
    """Branches whose value sits on its limit within tolerance: the reference's
    strict '>' comparisons (dc_engine.cpp:396-397) are decided there by
    rounding, so counts may legitimately differ by these."""
    v = np.asarray(values, float)
    lim = np.asarray(limits, float)
    return np.abs(v - lim) <= tol * np.maximum(1.0, lim)


def compare_scores(sc, ref: dict, worst_k: int, limits=None, weights=(200.0, 50.0)) -> dict:
    """Asserts parity of a ScoreArrays batch against oracle output; returns error stats.

    Counts must be exact except on knife edges; when `limits` is given and the
    oracle output carries flows ('fmax', 'base'), a lambda_c / lambda_c0
    difference is accepted if it is covered by branches on their limit and
    the fitness differs by exactly the corresponding weights."""
    n = len(sc.fitness)
    assert np.array_equal(sc.islanded, ref["islanded"]), "islanded flags differ"
    for k in ("lambda_d", "lambda_s", "lambda_r"):
        assert np.array_equal(getattr(sc, k), ref[k]), k
    live = ref["islanded"] == 0
    assert np.array_equal(sc.islanded_outages[live], ref["islanded_outages"][live]), "islanded outages"
    assert np.array_equal(sc.islanded_busbar_outages[live], ref["islanded_busbar"][live]), "islanded busbar"
    fit_adj = np.array(ref["fitness"], float).copy()
    ties = 0
    for i in np.nonzero(live)[0]:
        dc = int(sc.lambda_c[i]) - int(ref["lambda_c"][i])
        dc0 = int(sc.lambda_c0[i]) - int(ref["lambda_c0"][i])
        if dc == 0 and dc0 == 0:
            continue
        assert limits is not None and "fmax" in ref, f"lane {i}: lambda_c {dc:+d} lambda_c0 {dc0:+d} without flows"
        edge_c = int(knife_edges(ref["fmax"][i], limits).sum())
        edge_c0 = int(knife_edges(np.abs(ref["base"][i]), limits).sum())
        assert abs(dc) <= edge_c and abs(dc0) <= edge_c0, f"lane {i}: count difference off the knife edge"
        fit_adj[i] -= weights[0] * dc0 + weights[1] * dc
        ties += 1
    errs = {k: rel_err(getattr(sc, k), ref[k]) for k in ("lambda_o", "lambda_b")}
    errs["fitness"] = rel_err(sc.fitness, fit_adj)
    errs["knife_edge_lanes"] = ties
    for k in ("lambda_o", "lambda_b", "fitness"):
        assert errs[k] <= TOL, f"{k} rel err {errs[k]:.3e}"
    werr = 0.0
    for i in range(n):
        if not live[i]:
            continue
        # an outage energy that is exactly 0 in exact arithmetic (|f| == limit)
        # enters the list (energy > 0, dc_engine.cpp:414) on rounding alone:
        # compare the entries above the knife edge
        gw, rw = int(sc.worst_n[i]), int(ref["worst_n"][i])
        gmask = sc.worst_energy[i, :gw] > 1e-7
        rmask = ref["worst_val"][i, :rw] > 1e-7
        gi, ri = sc.worst_idx[i, :gw][gmask], ref["worst_idx"][i, :rw][rmask]
        gv, rv = sc.worst_energy[i, :gw][gmask], ref["worst_val"][i, :rw][rmask]
        if gw == worst_k or rw == worst_k:  # truncated lists: compare the common prefix
            m = min(len(gi), len(ri))
            gi, ri, gv, rv = gi[:m], ri[:m], gv[:m], rv[:m]
        assert len(gi) == len(ri), f"worst list length lane {i}: {gw} vs {rw}"
        # each contingency id carries its own energy: an id in both lists has
        # the same energy; an id in one list only must be a tie swap (an entry
        # of the other list with an equal energy that is itself missing here,
        # e.g. equal energies cut by the worst_k truncation)
        rmap = dict(zip(ri.tolist(), rv.tolist()))
        gmap = dict(zip(gi.tolist(), gv.tolist()))
        r_only = [rmap[k] for k in rmap if k not in gmap]
        for k, e in gmap.items():
            if k in rmap:
                assert abs(e - rmap[k]) <= TOL * max(1.0, abs(rmap[k])), f"worst lane {i} id {k}: {e} vs {rmap[k]}"
            else:
                assert any(abs(e - x) <= TOL * max(1.0, abs(x)) for x in r_only), \
                    f"worst list lane {i}: id {k} ({e}) not in the reference list and not a tie: {gi} vs {ri}"
        # both lists are ranked (energy desc, id asc), dc_engine.cpp:412-420
        assert all(gv[j] >= gv[j + 1] for j in range(len(gv) - 1)), f"worst list lane {i} not ranked"
        werr = max(werr, rel_err(gv, rv))
    assert werr <= TOL, f"worst energies rel err {werr:.3e}"
    errs["worst"] = werr
    return errs


def compare_flows(fr, ref: dict) -> dict:
    live = ref["islanded"] == 0
    out = {}
    for mine, theirs in (("base", "base"), ("max_contingency", "fmax"), ("max_busbar", "fbus"),
                         ("outage_energy", "energy")):
        e = rel_err(getattr(fr, mine)[live], ref[theirs][live])
        assert e <= TOL, f"{mine} rel err {e:.3e}"
        out[mine] = e
    return out


def grid_with_stations(base_json: str, buses) -> str:
    """Graft 2-busbar stations (helpers.hpp:65-78 station_json) onto buses."""
    doc = json.loads(base_json)
    ids = {b["id"]: b for b in doc["branches"]}
    doc.setdefault("substations", [])
    for bus in buses:
        el = [b["id"] for b in doc["branches"] if b["from"] == bus or b["to"] == bus]
        el += [i["id"] for i in doc.get("injections", []) if i["node"] == bus]
        doc["substations"].append({"node": bus, "busbars": ["B1", "B2"], "couplers": [["B1", "B2"]],
                                   "terminals": [{"element": e, "reachable": ["B1", "B2"], "default": "B1"}
                                                 for e in el]})
    del ids
    return json.dumps(doc)


def replay_inserts(stream, cfg):
    """Naive list replay of Repertoire::insert (test_qd_optimizer.cpp:262-277):
    stream of (genome, {fitness, lambda_d, lambda_s, lambda_r}) -> (inserted
    flags, {cell: [(key, fitness, genome)]})."""
    import math

    from paper_2605_10128_b200 import Genome, descriptor_to_cell

    cells = {}
    results = []
    for genome, sc in stream:
        if not math.isfinite(sc["fitness"]):
            results.append(False)
            continue
        cell = descriptor_to_cell(sc["lambda_d"], sc["lambda_s"], sc["lambda_r"], cfg)
        lst = cells.setdefault(cell, [])
        key = Genome(list(genome[:cfg.n_a]), list(genome[cfg.n_a:])).canonical_key()
        if any(k == key for k, _, _ in lst):
            results.append(False)
            continue
        if len(lst) >= cfg.cell_capacity and sc["fitness"] <= lst[-1][1]:
            results.append(False)
            continue
        pos = 0
        while pos < len(lst) and not (sc["fitness"] > lst[pos][1]):
            pos += 1
        lst.insert(pos, (key, sc["fitness"], list(genome)))
        if len(lst) > cfg.cell_capacity:
            lst.pop()
        results.append(True)
    return results, cells


def timestep_grids(grid_json: str):
    """The single-profile grids of a grid with a 'timesteps' key (model.hpp):
    grid t = the grid with every profiled injection's p_mw replaced by its t-th
    value (what the reference evaluates for that timestep)."""
    doc = json.loads(grid_json)
    ts = doc.pop("timesteps", None)
    if not ts:
        return [json.dumps(doc)]
    out = []
    for t in range(int(ts["count"])):
        d = json.loads(json.dumps(doc))
        for inj in d.get("injections", []):
            prof = ts.get("injections", {}).get(inj["id"])
            if prof is not None:
                inj["p_mw"] = prof[t]
        out.append(json.dumps(d))
    return out


def oracle_timesteps(orcs, genomes, n_a, n_d, worst_k=20, weights=(200.0, 50.0)):
    """Aggregated evaluation over timesteps (the extension's definition, on top
    of the reference's per-timestep evaluate): lambda_o/c/c0/b and islanded
    counts summed, energies summed per contingency and ranked (energy desc,
    index asc, first worst_k), islanded at any timestep = islanded (fitness
    -inf). Variant 1 fitness."""
    per = [o.evaluate(genomes, n_a, n_d, flows=True) for o in orcs]
    n = len(genomes)
    out = {k: sum(p[k] for p in per) for k in ("lambda_o", "lambda_c", "lambda_c0", "lambda_b",
                                               "islanded_outages", "islanded_busbar")}
    for k in ("lambda_d", "lambda_s", "lambda_r"):
        out[k] = per[0][k]
    isl = np.zeros(n, bool)
    for p in per:
        isl |= p["islanded"].astype(bool)
    out["islanded"] = isl.astype(np.uint8)
    energy = sum(p["energy"] for p in per)
    out["fitness"] = -(out["lambda_o"] + weights[0] * out["lambda_c0"] + weights[1] * out["lambda_c"])
    out["fitness"][isl] = -np.inf
    wi = np.zeros((n, max(worst_k, 1)), np.int32)
    wv = np.zeros((n, max(worst_k, 1)))
    wn = np.zeros(n, np.int32)
    for i in range(n):
        if isl[i]:
            for k in ("lambda_o", "lambda_b"):
                out[k][i] = 0.0
            for k in ("lambda_c", "lambda_c0", "islanded_outages", "islanded_busbar"):
                out[k][i] = 0
            continue
        pos = [(-energy[i, k], k) for k in range(energy.shape[1]) if energy[i, k] > 0]
        pos.sort()
        for j, (v, k) in enumerate(pos[:worst_k]):
            wi[i, j], wv[i, j] = k, -v
        wn[i] = min(len(pos), worst_k)
    out.update(worst_idx=wi, worst_val=wv, worst_n=wn)
    return out
