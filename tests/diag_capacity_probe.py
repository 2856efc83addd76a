"""Diagnostic (not collected by pytest): capacity errors of random genomes at n_a/n_d = 3/2 and 4/4 on cfg2, the failing ones checked against the oracle. Run on a GPU: python tests/diag_capacity_probe.py"""
import sys, json, numpy as np
sys.path.insert(0, '.')
import paper_2605_10128_b200 as P
from tools.synth_grid import config_json
from oracle.oracle import OracleContext
for cfg in ("cfg2",):
    text = config_json(cfg)
    g = P.grid_from_json_text(text); ctx = P.DcContext(g, P.build_action_set(g))
    orc = OracleContext(text)
    for na, nd in ((3, 2), (4, 4)):
        G = orc.random_genomes(65536, na, nd, seed=5)
        bad = 0; badg = []
        for i in range(0, len(G), 256):
            try:
                ctx.evaluate_arrays(G[i:i+256], na, nd)
            except P.CapacityError:
                for j in range(i, i + 256):
                    try:
                        ctx.evaluate_arrays(G[j:j+1], na, nd)
                    except P.CapacityError:
                        bad += 1; badg.append(G[j].tolist())
        print(cfg, na, nd, "capacity errors", bad, "of", len(G), badg[:3], flush=True)
    # loop genomes
    sess = P.QdSession(ctx, P.QdConfig(batch_size=4096, seed=3, iters_per_epoch=1<<30))
    sess.step(200)
    print("200 loop generations ok")
