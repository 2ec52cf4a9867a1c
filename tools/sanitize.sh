#!/bin/bash
# compute-sanitizer passes over the smoke step and the small
# parity / PP / kernel tests; summaries to gpurun_out/sanitize_*.log.
set -u
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck initcheck; do
  timeout 900 $S --tool $tool --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" \
    > gpurun_out/sanitize_${tool}_smoke.log 2>&1
  echo "$tool smoke rc=$?"
done
timeout 1200 $S --tool memcheck --error-exitcode 9 python -m pytest -x -q -m gpu \
  tests/test_parity_gpu.py tests/test_pp_gpu.py tests/test_attention_gpu.py -k "toy or llama-small or p2 or forward or backward" \
  > gpurun_out/sanitize_memcheck_tests.log 2>&1
echo "memcheck tests rc=$?"
# the fused epilogues (SwiGLU / RoPE + KV copy), cross-entropy row kernel,
# attention backward readouts and the segment operators
timeout 1500 $S --tool memcheck --error-exitcode 9 python -m pytest -x -q -m gpu \
  tests/test_gemm_gpu.py tests/test_parity_gpu.py tests/test_segment_gpu.py tests/test_attention_stress_gpu.py \
  -k "forced or v32000 or v97 or dh128 or segment or compose or single_chunk or stress" \
  > gpurun_out/sanitize_memcheck_fused.log 2>&1
echo "memcheck fused rc=$?"
timeout 900 $S --tool racecheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" \
  > gpurun_out/sanitize_racecheck_smoke.log 2>&1
echo "racecheck smoke rc=$?"
