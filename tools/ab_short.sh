#!/bin/bash
# A/B of two library builds on the packed short-chunk attention shapes and the
# attention-backward GPU parity tests: tools/ab_short.sh old.so new.so
A=$1; B=$2
for c in 0 14 22 26 27; do
  for L in $A $B; do
    echo "== $(basename $L) chunk $c"
    CF_LIB=$L timeout 300 python tools/attn_short_bench.py $c 2>&1 | grep -E "ping-pong|bwd tcgen05"
  done
done
