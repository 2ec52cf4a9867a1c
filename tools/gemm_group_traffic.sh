#!/bin/bash
# DRAM bytes and time per GEMM shape vs the raster group size (CF_GEMM_GROUP).
# Usage: bash tools/gemm_group_traffic.sh 8 16 32 ...
mkdir -p gpurun_out
for g in "$@"; do
  CF_GEMM_GROUP=$g GEMM_BENCH_ONCE=1 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:gemm --csv python tools/gemm_bench.py > gpurun_out/gt_$g.csv 2>/dev/null
  CF_GEMM_GROUP=$g python tools/gemm_bench.py > gpurun_out/gb_$g.txt 2>&1
  python - "$g" <<'PY'
import csv, io, sys, json
g = sys.argv[1]
txt = open(f"gpurun_out/gt_{g}.csv").read()
shapes = [json.loads(l) for l in txt.splitlines() if l.startswith("{")]
rows = [l for l in txt.splitlines() if l.startswith('"')]
rd = list(csv.DictReader(io.StringIO("\n".join(rows))))
per = {}
for r in rd:
    per.setdefault(r["ID"], {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
times = {l.split()[0] + " " + l.split()[1]: l for l in open(f"gpurun_out/gb_{g}.txt") if "TFLOP" in l}
for s, (k, m) in zip(shapes, sorted(per.items(), key=lambda x: int(x[0]))):
    dram = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
    tf = [l for l in open(f"gpurun_out/gb_{g}.txt") if l.startswith(s["shape"])]
    print(f"g={g:3s} {s['shape']:15s} dram/alg {dram / s['algorithmic_bytes']:5.2f}  |  {tf[0].split('K=')[1].strip() if tf else ''}")
PY
done
