"""DRAM bytes per GEMM launch vs algorithmic bytes for the 16 GEMM shapes of
tools/gemm_traffic.py (one chunk's layers 0-1 forward, head + layer 31
backward), from a light ncu pass (dram bytes + duration only), for the
environment variants given: e.g. CF_GEMM_SERP=0 CF_GEMM_SERP=1.
Usage: python tools/gemm_traffic_quick.py out.json VAR=VAL [VAR=VAL ...]"""
import csv
import io
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gemm_traffic import BWD, FWD, algorithmic  # noqa: E402

METRICS = "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"


def capture(env, skip):
    cmd = ["ncu", "--metrics", METRICS, "--clock-control", "none", "-k", "regex:gemm_pair", "--launch-skip",
           str(skip), "--launch-count", "8", "--csv", "python", "bench.py", "--workload", "short", "--steps", "1",
           "--warmup", "1", "--no-cpu-baseline"]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900).stdout
    rows = [r for r in csv.reader(io.StringIO(out)) if len(r) > 14 and r[0].isdigit()]
    per = {}
    for r in rows:
        per.setdefault(r[0], {})[r[12]] = float(r[14]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
                                                           "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
                                                           "nsecond": 1e-9, "msecond": 1e-3}.get(r[13], 1.0)
    return [per[k] for k in sorted(per, key=int)]


def main():
    res = {}
    for var in sys.argv[2:]:
        k, v = var.split("=")
        env = dict(os.environ, **{k: v})
        launches = capture(env, 0) + capture(env, 129)
        rows = []
        for (name, M, N, K, epi), l in zip(FWD + BWD, launches):
            dram = l["dram__bytes_read.sum"] + l["dram__bytes_write.sum"]
            a = algorithmic(M, N, K, epi)
            rows.append({"shape": name, "M": M, "N": N, "K": K if K is not None else M[0][2], "dram_bytes": dram,
                         "algorithmic_bytes": a,
                         "ratio": dram / a, "duration_us": l["gpu__time_duration.sum"] * 1e6})
        tot_d = sum(r["dram_bytes"] for r in rows)
        tot_a = sum(r["algorithmic_bytes"] for r in rows)
        res[var] = {"mean_ratio": tot_d / tot_a, "mean_dram_bytes_per_launch": tot_d / len(rows),
                    "mean_algorithmic_bytes_per_launch": tot_a / len(rows),
                    "sum_duration_us": sum(r["duration_us"] for r in rows), "launches": rows}
        print(f"== {var}: dram/alg {tot_d / tot_a:.3f}, sum of durations {res[var]['sum_duration_us']:.0f} us")
        for r in rows:
            print(f"  {r['shape']:15s} {r['duration_us']:8.1f} us  dram {r['dram_bytes'] / 1e6:8.1f} MB  "
                  f"alg {r['algorithmic_bytes'] / 1e6:8.1f} MB  x{r['ratio']:.2f}")
    json.dump(res, open(sys.argv[1], "w"), indent=1)


if __name__ == "__main__":
    main()
