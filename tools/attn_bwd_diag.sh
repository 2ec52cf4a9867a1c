# Attention-backward bottleneck diagnostics (builds in build_ab/lib_diag<v>.so,
# CF_BWD_DIAG=v): 1 softmax math skipped, 2 softmax side skipped, 3 = 2 + only
# the TS (A-in-TMEM) MMAs, 4 = 3 without operand loads, 5 = 3 with half the loads
for T in 16384 2048; do
echo "== T=$T base"; NO_SDPA=1 python tools/attn_calib.py $T
for v in "$@"; do echo "== diag$v"; CF_LIB=$PWD/build_ab/lib_diag$v.so NO_SDPA=1 python tools/attn_calib.py $T; done
done
