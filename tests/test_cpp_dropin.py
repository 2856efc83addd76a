"""The C++ drop-in (include/topopt_b200.hpp, the reference's C++ surface over
the C ABI) driven from a compiled C++ test binary (tests/cpp/dropin_test.cpp):

* host mode (CPU): grid load / canonical hash / action cache round trip,
  genome helpers, descriptor_to_cell KATs and the mapping of every error kind
  to its exception type (errors.hpp:9-34);
* gpu mode: DcContext::evaluate_batch / evaluate / evaluate_flows against the
  golden vectors (1e-9), mixed slot counts in one batch, pre-optimization
  score, run_optimizer with a sink, the std::atomic<bool> stop flag,
  ConfigError and sink exceptions; the optimizer run is compared here with the
  oracle's run_optimizer (qd_optimizer.cpp:344-417); AcValidator (baseline,
  worst-k and full N-1 verdicts of the golden genomes, validate_queue) against the
  oracle's ac_validator.cpp restatement.
"""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "dropin_test")
GOLDEN = os.path.join(ROOT, "tests", "golden", "grid14_congested_golden.json")


def _binary():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    return BIN


def test_cpp_dropin_host():
    r = subprocess.run([_binary(), "host", GOLDEN], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


@pytest.mark.gpu
def test_cpp_dropin_gpu(tmp_path):
    from oracle.oracle import OracleContext, qd_config

    out = tmp_path / "dropin.json"
    r = subprocess.run([_binary(), "gpu", GOLDEN, str(out)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
    got = json.loads(out.read_text())
    text = open(os.path.join(ROOT, "tests", "golden", "data", "grid14_congested.json")).read()
    ref = OracleContext(text).run_optimizer(qd_config(seed=1, batch_size=64, iters_per_epoch=7,
                                                      max_evaluations=3201), all_snapshots=False)
    assert got["evaluations"] == ref["stats"]["evaluations"] == 3201
    assert got["epochs"] == ref["stats"]["epochs"] == got["n_snapshots"]
    assert abs(got["best_fitness"] - ref["snapshots"][-1]["best_fitness"]) <= 1e-6
    # AcValidator through the C++ API vs the oracle's restatement of ac_validator.cpp
    import numpy as np
    from oracle.oracle import OracleAc
    gold = json.loads(open(GOLDEN).read())
    orc = OracleContext(text)
    oac = OracleAc(orc)
    ac = got["ac"]
    assert abs(ac["baseline_lambda_o"] - oac.baseline["lambda_o"]) <= 1e-8 * max(1.0, oac.baseline["lambda_o"])
    assert ac["baseline_critical"] == oac.baseline["critical"]
    gen = np.array(gold["genomes"], np.int32)
    n_a = gold["n_a"]
    n_d = gen.shape[1] - n_a
    sc = orc.evaluate(gen, n_a, n_d)
    assert ac["worst_k"] == oac.worst_k_check(gen, n_a, n_d, sc["worst_idx"], sc["worst_n"]).tolist()
    reason, acc, lo = oac.full_validation(gen, n_a, n_d)
    assert ac["full_reason"] == reason.tolist()
    assert np.allclose(ac["full_lambda_o"], lo, rtol=1e-8, atol=1e-8)
