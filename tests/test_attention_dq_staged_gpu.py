"""The register-staged persistent dQ kernel (dq_persist_kernel, which fuses
D = rowsum(dO * O) into its Q / dO staging; attention_tc_bwd.cu) on every
attention case.  The default is the TMA-fed dq_persist_tma_kernel with D from
dsum_rows_kernel; CF_DQ_PERSIST=1 selects this one in a child process (the
switch is read once per process): fp32-reference numerics
(test_attention_gpu.py), the bitwise synchronisation stress
(test_attention_stress_gpu.py) and the GPU-vs-oracle gradient parity of
run_plan (test_parity_gpu.py)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def test_staged_dq_kernel_passes_the_attention_and_parity_suites():
    env = dict(os.environ, CF_DQ_PERSIST="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(HERE, "test_attention_gpu.py"), os.path.join(HERE, "test_attention_stress_gpu.py"),
                        os.path.join(HERE, "test_parity_gpu.py")],
                       cwd=os.path.dirname(HERE), env=env, capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
