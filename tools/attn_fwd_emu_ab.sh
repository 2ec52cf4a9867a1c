#!/bin/bash
# Forward-attention exp2 offload A/B (CF_FWD_EMU builds in build_ab/lib_emu<v>.so):
# calibration shape (T = 16384 and 2048) for each variant.
for T in 16384 2048; do
  for v in "$@"; do
    echo "== emu$v T=$T"; CF_LIB=$PWD/build_ab/lib_emu$v.so NO_SDPA=1 python tools/attn_calib.py $T
  done
done
