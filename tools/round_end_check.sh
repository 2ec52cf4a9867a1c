#!/bin/bash
# Full-state GPU evidence: A/B bench of two library builds (alternating, same
# box), the full GPU suite, smoke(), and the default bench line.
# Usage: tools/round_end_check.sh old.so new.so
mkdir -p gpurun_out
bash tools/ab_bench.sh $1 $2 2 2>&1 | tee gpurun_out/ab_bench.txt
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; tail -3 gpurun_out/gputests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 600 gpurun_out/bench.json
