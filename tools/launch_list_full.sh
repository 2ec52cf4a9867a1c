#!/bin/bash
# Whole-step C2 launch list (ncu gpu__time_duration.sum, --clock-control none):
# the first step of bench.py with no warm-up, ~23.7K launches.
mkdir -p gpurun_out
timeout 3300 ncu --metrics gpu__time_duration.sum --clock-control none -c 25000 --csv \
  --log-file gpurun_out/launches_full.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
python profiles/summarize_launches.py gpurun_out/launches_full.csv > gpurun_out/launches_full.txt; head -24 gpurun_out/launches_full.txt
gzip -f gpurun_out/launches_full.csv
