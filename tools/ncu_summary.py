"""Summarises ncu --set full captures (.ncu-rep) into JSON: per launch the
kernel, duration, DRAM bytes read/written, tensor-pipe activity and SM clock.
Usage: python tools/ncu_summary.py out.json a.ncu-rep [b.ncu-rep ...]"""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_active_pct",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "launch__grid_size": "grid",
    "launch__registers_per_thread": "regs",
}
# reported when the capture has them (--set full does)
OPTIONAL = {
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pct",
    "sm__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.per_cycle_active": "warps_active",
}
SCALE = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "nsecond": 1e-9,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "hz": 1.0, "Khz": 1e3, "Mhz": 1e6,
         "Ghz": 1e9, "%": 1.0, "": 1.0, "register/thread": 1.0}


def read(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join({**METRICS, **OPTIONAL})],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    idx = {k: i for i, k in enumerate(head)}
    launches = []
    for r in rows[2:]:
        rec = {"kernel": r[idx["Kernel Name"]].split("(")[0].replace("(anonymous namespace)::", "")}
        for m, key in METRICS.items():
            rec[key] = float(r[idx[m]].replace(",", "")) * SCALE.get(units[idx[m]], 1.0)
        for m, key in OPTIONAL.items():
            if m in idx and r[idx[m]] not in ("", "n/a"):
                rec[key] = float(r[idx[m]].replace(",", "")) * SCALE.get(units[idx[m]], 1.0)
        rec["dram_bytes"] = rec["dram_read"] + rec["dram_write"]
        launches.append(rec)
    return launches


def main():
    res = {}
    for rep in sys.argv[2:]:
        res[rep.split("/")[-1]] = read(rep)
    json.dump(res, open(sys.argv[1], "w"), indent=1)
    for k, ls in res.items():
        print(k)
        for r in ls:
            print(f"  {r['kernel'][:48]:48s} {r['duration']*1e6:9.1f} us  dram {r['dram_bytes']/1e6:9.1f} MB  "
                  f"tensor {r['tensor_active_pct']:5.1f}%  {r['sm_clock']/1e9:.2f} GHz")


if __name__ == "__main__":
    main()
