"""Seeded synthetic transmission grids in the reference's JSON format.

Recipe of SURVEY.md §8(d): a connected, meshed, planar-like graph (nearest-
neighbour spanning tree plus short chords, mean degree ~3), reactances
U(0.05, 0.5) p.u. (helpers.hpp:469), generators on ~20% of the nodes
U(50, 250) MW and loads U(10, 90) MW scaled to balance (the slack takes the
residual, grid_model.cpp:508), limits from the base-case DC flows
|f0|*U(1.15, 1.6) + margin with a few percent tightened so N-1 overloads exist,
single-branch contingencies on every non-bridge branch outside a reserved
disconnectable pool (importer.cpp:53-56 excludes contingency branches from
disconnection), and 2-busbar substations on nodes with 3..10 terminals.
The output loads unchanged in the reference, the oracle and the engine.
"""
from __future__ import annotations

import json
import sys

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


def _bridges(n: int, edges: np.ndarray) -> set:
    adj = [[] for _ in range(n)]
    for e, (a, b) in enumerate(edges):
        adj[a].append((b, e))
        adj[b].append((a, e))
    tin = [-1] * n
    low = [0] * n
    out = set()
    t = 0
    for r in range(n):
        if tin[r] >= 0:
            continue
        tin[r] = low[r] = t
        t += 1
        stack = [(r, -1, 0)]
        while stack:
            v, via, i = stack[-1]
            if i < len(adj[v]):
                stack[-1] = (v, via, i + 1)
                w, e = adj[v][i]
                if e == via:
                    continue
                if tin[w] < 0:
                    tin[w] = low[w] = t
                    t += 1
                    stack.append((w, e, 0))
                else:
                    low[v] = min(low[v], tin[w])
            else:
                stack.pop()
                if stack:
                    p = stack[-1][0]
                    low[p] = min(low[p], low[v])
                    if low[v] > tin[p]:
                        out.add(via)
    return out


def synth_grid(n_nodes: int, seed: int = 0, branch_ratio: float = 1.5, n_stations: int = 50,
               disc_fraction: float = 0.1, tight_fraction: float = 0.03, max_terminals: int = 10,
               n_timesteps: int = 1) -> dict:
    rng = np.random.default_rng(seed)
    n = n_nodes
    pos = rng.random((n, 2))
    order = rng.permutation(n)
    edges = []
    have = set()
    # nearest-neighbour tree over a random insertion order
    placed = [order[0]]
    placed_pos = pos[[order[0]]]
    for k in range(1, n):
        v = order[k]
        d = np.sum((placed_pos - pos[v]) ** 2, axis=1)
        u = placed[int(np.argmin(d))]
        edges.append((u, v))
        have.add((min(u, v), max(u, v)))
        placed.append(v)
        placed_pos = np.vstack([placed_pos, pos[v]]) if k < 2000 else placed_pos
        if k >= 2000:
            # large grids: rebuild the candidate array in blocks to stay O(n^2 / block)
            placed_pos = pos[placed]
    # chords between near neighbours
    target = int(round(branch_ratio * n))
    knn = 6
    cand = []
    block = 1024
    for s in range(0, n, block):
        d = np.sum((pos[s:s + block, None, :] - pos[None, :, :]) ** 2, axis=2)
        nb = np.argsort(d, axis=1)[:, 1:knn + 1]
        for i in range(nb.shape[0]):
            for j in nb[i]:
                a, b = s + i, int(j)
                cand.append((min(a, b), max(a, b)))
    cand = sorted(set(cand) - have)
    rng.shuffle(cand)
    for a, b in cand:
        if len(edges) >= target:
            break
        edges.append((a, b))
        have.add((a, b))
    edges = np.array(edges, dtype=np.int64)
    E = len(edges)
    x = rng.uniform(0.05, 0.5, E)

    # injections
    n_gen = max(1, n // 5)
    gen_nodes = np.sort(rng.choice(n, n_gen, replace=False))
    is_gen = np.zeros(n, bool)
    is_gen[gen_nodes] = True
    gen_p = rng.uniform(50.0, 250.0, n_gen)
    load_nodes = np.nonzero(~is_gen)[0]
    load_p = rng.uniform(10.0, 90.0, len(load_nodes))
    load_p *= 0.97 * gen_p.sum() / load_p.sum()
    slack = int(gen_nodes[0])

    # base-case DC flows for the limits
    p = np.zeros(n)
    p[gen_nodes] += gen_p
    p[load_nodes] -= load_p
    p[slack] -= p.sum()
    keep = np.ones(n, bool)
    keep[slack] = False
    red = -np.ones(n, np.int64)
    red[keep] = np.arange(n - 1)
    b = 1.0 / x
    rows, cols, vals = [], [], []
    for e, (i, j) in enumerate(edges):
        ri, rj = red[i], red[j]
        if ri >= 0:
            rows.append(ri), cols.append(ri), vals.append(b[e])
        if rj >= 0:
            rows.append(rj), cols.append(rj), vals.append(b[e])
        if ri >= 0 and rj >= 0:
            rows += [ri, rj]
            cols += [rj, ri]
            vals += [-b[e], -b[e]]
    B = sp.csc_matrix((vals, (rows, cols)), shape=(n - 1, n - 1))
    th = np.zeros(n)
    th[keep] = spla.spsolve(B, p[keep])
    f0 = b * (th[edges[:, 0]] - th[edges[:, 1]])

    # contingencies: all non-bridges outside the reserved disconnectable pool
    br = _bridges(n, edges)
    nonbridge = np.array([e for e in range(E) if e not in br])
    reserve = set(rng.choice(nonbridge, int(disc_fraction * E), replace=False).tolist()) if len(nonbridge) else set()
    conts = [int(e) for e in nonbridge if int(e) not in reserve]

    # limits: the base case is N-1 secure with margin U(1.02, 1.35) except a
    # tight_fraction of branches set below their N-1 peak (congestion to fix)
    X = np.linalg.inv(B.toarray())
    Xf = np.zeros((n, n - 1))
    Xf[keep] = X
    ptdf = b[:, None] * (Xf[edges[:, 0]] - Xf[edges[:, 1]])       # E x (n-1)
    kc = np.array(conts, dtype=np.int64)
    fmax = np.abs(f0).copy()
    for s in range(0, len(kc), 512):
        ks = kc[s:s + 512]
        T = ptdf[:, red[edges[ks, 0]].clip(0)] * (red[edges[ks, 0]] >= 0) - \
            ptdf[:, red[edges[ks, 1]].clip(0)] * (red[edges[ks, 1]] >= 0)  # E x k LODF numerators
        den = 1.0 - T[ks, np.arange(len(ks))]
        f1 = f0[:, None] + T * (f0[ks] / den)[None, :]
        f1[ks, np.arange(len(ks))] = 0.0
        fmax = np.maximum(fmax, np.abs(f1).max(axis=1))
    del X, Xf, ptdf
    lim = fmax * rng.uniform(1.02, 1.35, E) + 5.0
    tight = rng.random(E) < tight_fraction
    lim[tight] = np.maximum(np.abs(f0[tight]) * 1.1 + 2.0, fmax[tight] * rng.uniform(0.8, 0.98, tight.sum()))

    # stations
    deg = np.zeros(n, np.int64)
    np.add.at(deg, edges[:, 0], 1)
    np.add.at(deg, edges[:, 1], 1)
    n_inj = np.ones(n, np.int64)  # every node carries one injection
    terms = deg + n_inj
    eligible = np.nonzero((deg >= 3) & (terms <= max_terminals))[0]
    stations = np.sort(rng.choice(eligible, min(n_stations, len(eligible)), replace=False))

    inj_id = {}
    injections = []
    for k, v in enumerate(gen_nodes):
        inj_id[int(v)] = f"g{v}"
        injections.append({"id": f"g{v}", "node": f"n{v}", "p_mw": float(gen_p[k]), "kind": "generator"})
    for k, v in enumerate(load_nodes):
        inj_id[int(v)] = f"l{v}"
        injections.append({"id": f"l{v}", "node": f"n{v}", "p_mw": float(load_p[k]), "kind": "load"})
    incident = [[] for _ in range(n)]
    for e, (i, j) in enumerate(edges):
        incident[i].append(e)
        incident[j].append(e)
    subs = []
    for v in stations:
        el = [f"e{e}" for e in incident[v]] + [inj_id[int(v)]]
        subs.append({"node": f"n{v}", "busbars": ["B1", "B2"], "couplers": [["B1", "B2"]],
                     "terminals": [{"element": t, "reachable": ["B1", "B2"],
                                    "default": "B2" if rng.random() < 0.5 else "B1"} for t in el]})
    doc = {
        "nodes": [{"id": f"n{v}"} for v in range(n)],
        "branches": [{"id": f"e{e}", "from": f"n{i}", "to": f"n{j}", "x_pu": float(x[e]),
                      "limit_mw": float(lim[e])} for e, (i, j) in enumerate(edges)],
        "injections": injections,
        "contingencies": [{"id": f"o{e}", "branches": [f"e{e}"]} for e in conts],
        "substations": subs,
        "busbar_outages": [],
        "slack": f"n{slack}",
    }
    if n_timesteps > 1:
        # daily profile (extension key, ignored by the reference loader): loads
        # follow 0.8 + 0.25 sin(pi (t - 6) / 12) with 3 % noise, generators the
        # same curve with 5 % noise; the slack absorbs the residual
        t = np.arange(n_timesteps)
        curve = 0.8 + 0.25 * np.sin(np.pi * (t - 6) / 12.0)
        prof = {}
        for k, v in enumerate(gen_nodes):
            prof[f"g{v}"] = [float(x) for x in gen_p[k] * curve * rng.uniform(0.95, 1.05, n_timesteps)]
        for k, v in enumerate(load_nodes):
            prof[f"l{v}"] = [float(x) for x in load_p[k] * curve * rng.uniform(0.97, 1.03, n_timesteps)]
        doc["timesteps"] = {"count": int(n_timesteps), "injections": prof}
    return doc


# BASELINE.json configs
CONFIGS = {
    "cfg2": dict(n_nodes=1000, n_stations=50, seed=2),      # 1k-bus / 1.5k-branch, B=4096
    "cfg3": dict(n_nodes=2000, n_stations=100, seed=3, n_timesteps=24),  # 2k-bus, 100 split stations, 24 steps
    "cfg4": dict(n_nodes=7000, n_stations=500, seed=4),     # TSO scale ~7k / 10k / 500 stations
}


def config_json(name: str) -> str:
    return json.dumps(synth_grid(**CONFIGS[name]))


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    print(config_json(name))


def with_ac_data(grid: dict, r_ratio: float = 0.1, charging: float = 0.02, q_ratio: float = 0.25,
                 v_set: float = 1.02, p_scale: float = 0.5) -> dict:
    """AC fields for a synthetic grid (the configs above are DC-only): r = r_ratio x,
    line charging, load q = q_ratio p, generators regulate to v_set (PV buses), every
    injection scaled by p_scale (the DC configs load their branches near the limits;
    at full load most of them have no AC solution)."""
    g = json.loads(json.dumps(grid))
    for inj in g["injections"]:
        inj["p_mw"] *= p_scale
    for b in g["branches"]:
        b["r_pu"] = r_ratio * b["x_pu"]
        b["b_pu"] = charging
    for inj in g["injections"]:
        if inj["kind"] == "load":
            inj["q_mvar"] = q_ratio * inj["p_mw"]
        else:
            inj["v_setpoint_pu"] = v_set
    return g
