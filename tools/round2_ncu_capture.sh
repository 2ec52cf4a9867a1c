#!/bin/bash
# Round-2 ncu evidence on one B200: --set full captures of the attention
# kernels at chunk 2 of the C2 long group (bench.py --workload long) and of
# two CTA-pair GEMM launches of a short-workload step (the gate|up forward
# and a grouped weight-gradient launch), summarised with tools/ncu_summary.py;
# plus the GEMM DRAM-traffic capture (tools/gemm_traffic_quick.py).
set -x
mkdir -p gpurun_out
for k in attn_fwd_pp_kernel dq_wide_kernel dkv_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 70 --launch-count 1 \
    -o /tmp/r2_$k python bench.py --workload long --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
done
# gate|up forward of layer 1 (launch 6 of the step) and the grouped o + q|k|v weight gradient of layer 31
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_pair --launch-skip 6 --launch-count 1 \
  -o /tmp/r2_gemm_gateup_fwd python bench.py --workload short --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_pair --launch-skip 136 --launch-count 1 \
  -o /tmp/r2_gemm_oqkv_wgrad python bench.py --workload short --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
(cd /tmp && python $GRAFT_REPO_ROOT/tools/ncu_summary.py $GRAFT_REPO_ROOT/gpurun_out/r2_ncu_summary.json \
  r2_attn_fwd_pp_kernel.ncu-rep r2_dq_wide_kernel.ncu-rep r2_dkv_kernel.ncu-rep r2_gemm_gateup_fwd.ncu-rep \
  r2_gemm_oqkv_wgrad.ncu-rep)
cp /tmp/r2_dq_wide_kernel.ncu-rep gpurun_out/
python tools/gemm_traffic_quick.py gpurun_out/r2_gemm_traffic.json CF_GEMM_SERP=1 > gpurun_out/r2_gemm_traffic.log 2>&1
tail -20 gpurun_out/r2_gemm_traffic.log
cat gpurun_out/r2_ncu_summary.json | head -80
