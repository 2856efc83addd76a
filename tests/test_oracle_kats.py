"""Pins the CPU oracle to the reference's own known-answer tests (ported in
oracle/kats/kats.cpp from proj/tests/*.cpp and acceptance criteria 1-7)."""
import os
import subprocess

from oracle.oracle import KATS_PATH, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_oracle_known_answer_tests():
    if not os.path.exists(KATS_PATH):
        build()
    data = os.path.join(ROOT, "tests", "golden", "data")
    out = subprocess.run([KATS_PATH, data], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-2000:]
    assert "0 failed" in out.stdout
