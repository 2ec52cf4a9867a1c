#!/bin/bash
# Final-state check after the default kernel changes: GPU suite, smoke,
# compute-sanitizer on the smoke step and the attention suite, bench line.
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gputests_final.log 2>&1; tail -2 gpurun_out/gputests_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
for tool in memcheck synccheck; do
  timeout 900 $S --tool $tool --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize_${tool}_smoke_s4.log 2>&1
  echo "$tool smoke rc=$?"; tail -2 gpurun_out/sanitize_${tool}_smoke_s4.log
done
timeout 1200 $S --tool memcheck --error-exitcode 9 python -m pytest -x -q -m gpu tests/test_attention_gpu.py tests/test_attention_stress_gpu.py \
  > gpurun_out/sanitize_memcheck_attention_s4.log 2>&1
echo "memcheck attention rc=$?"; tail -2 gpurun_out/sanitize_memcheck_attention_s4.log
timeout 1200 python bench.py > gpurun_out/bench_final_s4.json 2> gpurun_out/bench_final_s4.err; tail -c 200 gpurun_out/bench_final_s4.json
