#!/bin/bash
# Per-kernel device time, tensor-pipe activity and SM clock of the attention
# kernels at the calibration shape (tools/attn_calib.py T) for the default
# library and the CF_BWD_DIAG builds given as arguments (build_ab/lib_diag<v>.so).
T=${T:-16384}
run() {
  ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:"dq_kernel|dkv_kernel" -s 2 -c 2 --csv python tools/attn_calib.py $T 2>/dev/null |
    python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>14 and r[0]!='ID']
for r in rows: print('  %-12s %-70s %14s %s'%(r[4].split('(')[0].split('::')[-1], r[12], r[14], r[13]))"
}
echo "== base"; NO_SDPA=1 run
for v in "$@"; do echo "== diag$v"; CF_LIB=$PWD/build_ab/lib_diag$v.so NO_SDPA=1 run; done
