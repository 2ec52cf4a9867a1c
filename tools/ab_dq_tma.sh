#!/bin/bash
# A/B of the TMA-fed persistent dQ kernel (CF_DQ_PERSIST=2) against the
# register-staged one (=1): tests, operator-level packed chunks, the engine's
# short workload.
timeout 1500 python -m pytest tests/test_attention_dq_tma_gpu.py -x -q 2>&1 | tail -2
for c in 0 14 22 27; do for v in 1 2; do echo "== chunk $c CF_DQ_PERSIST=$v"; CF_DQ_PERSIST=$v timeout 300 python tools/attn_short_bench.py $c 2>&1 | grep -E "bwd tcgen05"; done; done
for v in 1 2 1 2; do echo "== short CF_DQ_PERSIST=$v"; CF_DQ_PERSIST=$v timeout 600 python bench.py --workload short --steps 2 --warmup 1 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; b=r['attention_bwd']; print(round(d['ms_per_step'],1), d['clocks']['sm_mhz'], 'bwd', round(b['achieved'],1), round(b['share_of_step'],4))"; done
