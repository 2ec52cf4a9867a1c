#!/bin/bash
# GEMM raster-group sweep on the C2 bench (CF_GEMM_GROUP overrides the M-blocks per group).
for g in "$@"; do
  CF_GEMM_GROUP=$g python bench.py --no-cpu-baseline --steps 3 --warmup 2 2>/dev/null > gpurun_out/group_$g.json
  python - "$g" <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/group_{sys.argv[1]}.json"))
print("group", sys.argv[1], round(d["ms_per_step"], 1), d["clocks"]["sm_mhz"], round(d["roofline"]["achieved"], 1))
PY
done
