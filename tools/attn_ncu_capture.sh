#!/bin/bash
# ncu --set full of one launch each of the attention kernels at chunk 2 of the
# C2 long group (T = 8192 queries, KV prefix 16,384), plus the long-workload
# launch list; summaries land in gpurun_out/ (the .ncu-rep files stay in /tmp).
set -x
mkdir -p gpurun_out
for k in attn_fwd_pp_kernel dq_kernel dkv_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 70 --launch-count 1 \
    -o /tmp/ncu_$k python bench.py --workload long --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
done
(cd /tmp && python $GRAFT_REPO_ROOT/tools/ncu_summary.py $GRAFT_REPO_ROOT/gpurun_out/attn_ncu.json \
  ncu_attn_fwd_pp_kernel.ncu-rep ncu_dq_kernel.ncu-rep ncu_dkv_kernel.ncu-rep)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_long.csv \
  python bench.py --workload long --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python profiles/summarize_launches.py gpurun_out/launches_long.csv > gpurun_out/launches_long.txt
gzip -f gpurun_out/launches_long.csv
