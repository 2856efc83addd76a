"""The reference-side shim (integration/dc_engine_b200.hpp)
compiles against the reference's own headers (CPU, this container only: the
reference tree is not shipped to the GPU box). The headers name Eigen types;
integration/eigen_stub declares them (Eigen is absent here)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not present")
def test_shim_compiles_against_reference_headers():
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Wextra", "-Werror",
                        "-I", os.path.join(ROOT, "include"), "-I", os.path.join(ROOT, "integration", "eigen_stub"),
                        "-I", REF_INC, os.path.join(ROOT, "integration", "check_shim.cpp")],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr


def test_cpp_api_header_compiles_standalone():
    """include/topopt_b200.hpp needs nothing but the C header and the standard library."""
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Wextra", "-Werror", "-x", "c++",
                        "-I", os.path.join(ROOT, "include"), "-"], input='#include "topopt_b200.hpp"\n',
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
