#!/bin/bash
# Session-4 evidence on one B200: GPU suite, smoke, the bench line, the C2
# launch list (ncu gpu__time_duration, later part of a step), and ncu --set
# full of one launch each of the persistent attention kernels in the step.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputests_s4.log 2>&1; tail -2 gpurun_out/gputests_s4.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_s4.log 2>&1; tail -1 gpurun_out/smoke_s4.log
timeout 1200 python bench.py > gpurun_out/bench_s4.json 2> gpurun_out/bench_s4.err; tail -c 300 gpurun_out/bench_s4.json
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 60000 -c 24000 --csv \
  --log-file gpurun_out/launches_s4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python profiles/summarize_launches.py gpurun_out/launches_s4.csv > gpurun_out/launches_s4.txt; head -20 gpurun_out/launches_s4.txt
gzip -f gpurun_out/launches_s4.csv
for k in attn_fwd_pp_persist_kernel dkv_persist_kernel dq_persist_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 40 --launch-count 1 \
    -o gpurun_out/ncu_s4_$k python bench.py --workload short --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
done
ls -la gpurun_out/*.ncu-rep
