"""The C++ facade (include/chunkflow_b200.hpp) compiles against the C-ABI
library and reproduces the reference's worked-batch plan (a C++ caller of the
reference swaps the include and link line, nothing else)."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_facade_builds_and_plans(tmp_path):
    exe = tmp_path / "facade_test"
    lib = os.path.join(ROOT, "paper_2503_02356_b200")
    subprocess.run(["g++", "-std=c++17", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "facade_test.cpp"), f"-L{lib}", "-lchunkflow_b200",
                    f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    assert "chunks=4 events=9 peak=2 recompute=2 groups=1" in out
    assert "edited_violations=" in out and "without a live retain-forward" in out
    assert "hand=backward of chunk 0 without a live retain-forward" in out
    assert "ValidationError: chunk_size must be at least 1" in out
    assert "makespans=56,54,46 bubble=55.56 stage0_ops=9" in out
    assert "base=34.8714 resid=0.59524" in out  # test_memory_model.cpp: 34.8717 +- 1e-3
    assert "tuner best=2,2 evals=4" in out
    assert "json=1 set=2,7,3" in out
