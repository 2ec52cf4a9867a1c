"""The 128-key-tile dQ kernel (dq_wide_kernel, attention_tc_bwd.cu) on every
attention case: the launch choice is made per call from the launch's keys per
query (long-context chunks take it), so the operator-level tests run it by
forcing CF_DQ_WIDE=1 in a child process (the switch is read once per
process): fp32-reference numerics (test_attention_gpu.py) and the bitwise
synchronisation stress (test_attention_stress_gpu.py)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def test_wide_dq_kernel_passes_the_attention_suites():
    env = dict(os.environ, CF_DQ_WIDE="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(HERE, "test_attention_gpu.py"), os.path.join(HERE, "test_attention_stress_gpu.py"),
                        "-k", "backward or stress"],
                       cwd=os.path.dirname(HERE), env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
