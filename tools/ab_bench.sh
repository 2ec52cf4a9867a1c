#!/bin/bash
# A/B of two library builds on the same box, alternating: tools/ab_bench.sh a.so b.so [rounds]
A=$1; B=$2; R=${3:-2}
for i in $(seq 1 $R); do
  for L in $A $B; do
    CF_LIB=$L python bench.py --no-cpu-baseline --steps 3 --warmup 2 2>/dev/null > gpurun_out/ab.json
    python - "$L" <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab.json"))
print(sys.argv[1].split("/")[-1], round(d["ms_per_step"], 1), "ms", d["clocks"]["sm_mhz"], "MHz", round(d["value"]))
PY
  done
done
