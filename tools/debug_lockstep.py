import os, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_10128_b200 as P
from oracle.oracle import OracleContext, qd_config
text = open("tests/golden/data/grid14_congested.json").read()
g = P.grid_from_json_text(text); ctx = P.DcContext(g, P.build_action_set(g)); orc = OracleContext(text)
kw = dict(seed=1, batch_size=64, iters_per_epoch=500, max_evaluations=3201)
trace = orc.run_optimizer_trace(qd_config(**kw))
bad = []
for it in trace["iters"]:
    gg = np.array(it["genomes"], np.int32)
    mine = ctx.evaluate_arrays(gg, 3, 2)
    ref = orc.evaluate(gg, 3, 2)
    for i in range(len(gg)):
        a, b = mine.fitness[i], ref["fitness"][i]
        if np.isfinite(b) and abs(a - b) > 1e-9 * max(1, abs(b)):
            bad.append(gg[i].tolist())
uniq = sorted(set(map(tuple, bad)))
print("mismatching genomes:", len(uniq), uniq[:20])
for gen in uniq[:5]:
    arr = np.array([gen], np.int32)
    sc, fr = ctx.evaluate_arrays(arr, 3, 2, flows=True)
    ref = orc.evaluate(arr, 3, 2, flows=True)
    print("genome", gen, "gpu fit", sc.fitness[0], "ref", ref["fitness"][0])
    for k in ("lambda_o", "lambda_c", "lambda_c0", "lambda_b", "islanded_outages"):
        print("  ", k, getattr(sc, k)[0], ref[k if k != "islanded_outages" else "islanded_outages"][0])
    print("   base err", np.max(np.abs(fr.base[0] - ref["base"][0])), "fmax err", np.max(np.abs(fr.max_contingency[0] - ref["fmax"][0])),
          "fbus err", np.max(np.abs(fr.max_busbar[0] - ref["fbus"][0])), "energy err", np.max(np.abs(fr.outage_energy[0] - ref["energy"][0])))
    print("   fbus gpu", np.round(fr.max_busbar[0], 3).tolist())
    print("   fbus ref", np.round(ref["fbus"][0], 3).tolist())
    print("   isl bus", sc.islanded_busbar_outages[0], ref["islanded_busbar"][0])
    print("   energy gpu", np.round(fr.outage_energy[0],3).tolist(), "\n   energy ref", np.round(ref["energy"][0],3).tolist())
