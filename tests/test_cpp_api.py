"""The C++ mirror of the reference API (include/dg2d_b200/dg2d.hpp): it compiles on its own
(CPU), and the C++ parity harness tests/cpp/parity.cpp — reference solver and B200 path side by
side in one binary, built by `make -C oracle cpptest` — passes on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "parity_cpp")


def test_cpp_header_compiles_standalone(tmp_path):
    src = tmp_path / "use.cpp"
    src.write_text('#include "dg2d_b200/dg2d.hpp"\n'
                   "int main() { dg2d_b200::SolverOptions o; o.rk_order = 2;\n"
                   "  dg2d_b200::CoefficientArray c(4, 3, 10); c.at(1, 2, 3) = 1.0;\n"
                   "  return o.scheme_id() == 2 && c.data[(1 * 3 + 2) * 10 + 3] == 1.0 ? 0 : 1; }\n")
    for std in ("c++17", "gnu++20"):
        r = subprocess.run(["g++", f"-std={std}", "-fsyntax-only", "-Wall", "-Wextra",
                            "-I", os.path.join(ROOT, "include"), str(src)], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr


@pytest.mark.gpu
def test_cpp_parity_harness_against_reference():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/parity_cpp not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0 and "ALL PASSED" in r.stdout, r.stdout + r.stderr
