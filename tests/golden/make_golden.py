"""Regenerates tests/golden/grid14_congested_golden.json: fixed genomes on the
bundled grid14_congested.json and their scores from the CPU oracle (the
restatement of the reference's DcContext::evaluate, pinned by the reference's
own known-answer tests in oracle/kats). The GPU engine and the oracle are both
checked against this file, so a change in either shows up as a diff.

usage: python tests/golden/make_golden.py
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import OracleContext  # noqa: E402


def main():
    text = open(os.path.join(HERE, "data", "grid14_congested.json")).read()
    orc = OracleContext(text)
    genomes = orc.random_genomes(48, 3, 2, seed=20261017)
    # plus every single action and every single disconnection
    rows = [[-1] * 5]
    rows += [[a, -1, -1, -1, -1] for a in range(orc.info["n_actions"])]
    rows += [[-1, -1, -1, d, -1] for d in range(len(orc.info["disconnectables"]))]
    rows += genomes.tolist()
    import numpy as np
    g = np.array(rows, np.int32)
    ref = orc.evaluate(g, 3, 2, flows=True)
    out = {"grid": "data/grid14_congested.json", "n_a": 3, "n_d": 2, "genomes": g.tolist(), "scores": []}
    for i in range(len(g)):
        wn = int(ref["worst_n"][i])
        out["scores"].append({
            "fitness": float(ref["fitness"][i]), "lambda_o": float(ref["lambda_o"][i]),
            "lambda_c": int(ref["lambda_c"][i]), "lambda_c0": int(ref["lambda_c0"][i]),
            "lambda_b": float(ref["lambda_b"][i]), "lambda_d": int(ref["lambda_d"][i]),
            "lambda_s": int(ref["lambda_s"][i]), "lambda_r": int(ref["lambda_r"][i]),
            "islanded": int(ref["islanded"][i]),
            "worst": [[int(ref["worst_idx"][i][j]), float(ref["worst_val"][i][j])] for j in range(wn)],
            "base": [float(x) for x in ref["base"][i]], "fmax": [float(x) for x in ref["fmax"][i]]})
    json.dump(out, open(os.path.join(HERE, "grid14_congested_golden.json"), "w"), indent=0)
    print(f"{len(g)} genomes written")


if __name__ == "__main__":
    main()
