"""bench.py --gpus N without torchrun env re-launches itself as N ranks
(VERDICT r1 next #2).  On CPU the --dry-run mode runs the same rank wiring
over gloo: WORLD_SIZE must equal --gpus, every rank builds the global plan
and takes its DP partition, and rank 0 checks that the ranks' chunks
partition the global plan with whole dependent groups on one rank."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(out):
    rows = [json.loads(l) for l in out.splitlines() if l.startswith("{")]
    assert len(rows) == 1, out
    return rows[0]


def test_bench_self_spawns_two_gloo_ranks():
    p = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--dry-run"], cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    line = _line(p.stdout)
    assert line["n_gpus"] == 2 and line["backend"] == "gloo"
    assert line["partition_ok"] is True
    assert sum(line["tokens_per_rank"]) == line["global_tokens"] > 2 * 250000
    assert line["config"]["parallelism"] == "dp2"


def test_bench_rejects_world_size_mismatch():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1", MASTER_PORT="29533")
    p = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--dry-run"], cwd=ROOT, capture_output=True,
                       text=True, timeout=300, env=env)
    assert p.returncode != 0
    assert "WORLD_SIZE=1" in (p.stderr + p.stdout)
