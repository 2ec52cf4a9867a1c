#!/bin/bash
# Short-chunk attention evidence: timings of the three tcgen05 attention
# kernels on packed C2 short chunks, then ncu --set full of one launch each
# (reports kept under gpurun_out/ for ncu -i here).
mkdir -p gpurun_out
for c in 0 14 27; do timeout 300 python tools/attn_short_bench.py $c 2>&1 | grep -E "T=|tcgen05"; done
for k in attn_fwd_pp_kernel dq_persist_kernel dkv_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 3 --launch-count 1 \
    -o gpurun_out/ncu_short_$k python tools/attn_short_bench.py 14 > gpurun_out/ncu_short_$k.log 2>&1
  tail -2 gpurun_out/ncu_short_$k.log
done
