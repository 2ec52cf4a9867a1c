#!/bin/bash
# Ring-depth sweep of the attention backward (CF_DQ_KS / CF_DQ_VS / CF_DKV_QS
# builds in build_ab/lib_bwd_<KS><VS><QS>.so): long-chunk and short-chunk times.
for v in "$@"; do
  L=$PWD/build_ab/lib_bwd_$v.so
  a=$(CF_LIB=$L python tools/attn_bench.py 2>&1 | grep "bwd tcgen05 pipelined" | awk '{print $4}')
  b=$(CF_LIB=$L python tools/attn_short_bench.py 2>&1 | grep "bwd tcgen05" | head -1 | awk '{print $3}')
  echo "$v long_ms=$a short_us=$b"
done
