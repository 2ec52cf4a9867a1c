"""The C++ facade's verify_equivalence / compare_gradients / backward_full /
run_plan (include/chunkflow_b200.hpp) on the GPU, compiled as a reference-
style C++ caller (tests/cpp/verify_facade_test.cpp)."""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_facade_verify_equivalence(tmp_path):
    lib = os.path.join(ROOT, "paper_2503_02356_b200")
    exe = tmp_path / "verify_facade_test"
    subprocess.run(["g++", "-std=c++17", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "verify_facade_test.cpp"), f"-L{lib}", "-lchunkflow_b200",
                    f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    lines = out.splitlines()
    # VerifyReport::to_text layout (plan_runner.hpp:352-365)
    assert lines[0].startswith("chunks: ") and lines[1].startswith("events: ")
    assert re.match(r"embedding max_abs_diff=\d\.\d{6}e[+-]\d+ rel_err=\d\.\d{6}e[+-]\d+$", lines[2])
    assert "result: PASS" in lines
    assert "k1_vs_k3 max_rel_err=0 loss_rel_err=0" in out, out
    assert "ValidationError: execution plan is invalid: chunk" in out and "never backwarded" in out, out
    assert "backward_full tensors=21" in out, out
