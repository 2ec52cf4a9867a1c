#!/bin/bash
# Round-end evidence on one B200: GPU tests, smoke, the bench line, the C2
# launch list and ncu --set full captures of the forward / backward GEMMs of
# one chunk (summarised on the box; the .ncu-rep files stay under 64 MiB).
set -x
mkdir -p gpurun_out
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputests_final.log 2>&1; tail -2 gpurun_out/gputests_final.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
fi
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -c 300 gpurun_out/bench_final.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_c2.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python profiles/summarize_launches.py gpurun_out/launches_c2.csv > gpurun_out/launches_c2.txt
gzip -f gpurun_out/launches_c2.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_pair --launch-count 8 -o /tmp/gemm_fwd \
  python bench.py --workload short --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_pair --launch-skip 129 --launch-count 8 \
  -o /tmp/gemm_bwd python bench.py --workload short --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
(cd /tmp && python $GRAFT_REPO_ROOT/tools/ncu_summary.py $GRAFT_REPO_ROOT/gpurun_out/ncu_gemm_summary.json gemm_fwd.ncu-rep gemm_bwd.ncu-rep)
cp /tmp/gemm_fwd.ncu-rep gpurun_out/
ls -la gpurun_out/
