"""Headline metrics of committed ncu --set full captures -> profiles/<round>/ncu_summary.json
(read by bench.py for the roofline `traffic` field).
Usage: ncu_json.py OUT.json NAME=REP|CMD|WORKLOAD ..."""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "gpu_time_ms": ("gpu__time_duration.sum", 1.0),
    "dram_bytes_read": ("dram__bytes_read.sum", None),
    "dram_bytes_write": ("dram__bytes_write.sum", None),
    "fp64_pipe_active_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed", 1.0),
    "issue_active_pct": ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", 1.0),
    "warps_active_per_sm": ("sm__warps_active.avg.per_cycle_active", 1.0),
    "registers_per_thread": ("launch__registers_per_thread", 1.0),
    "smem_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1.0),
    "sm_clock_ghz": ("sm__cycles_elapsed.avg.per_second", 1.0),
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def read(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    kern = vals[hdr.index("Kernel Name")]
    out = {}
    for key, (metric, _) in METRICS.items():
        i = hdr.index(metric)
        v = float(vals[i].replace(",", ""))
        if key.startswith("dram_bytes"):
            v = int(round(v * SCALE.get(units[i], 1)))
        out[key] = round(v, 3) if isinstance(v, float) else v
    return kern, out


def main():
    dst, specs = sys.argv[1], sys.argv[2:]
    res = {}
    for spec in specs:
        name, rest = spec.split("=", 1)
        rep, cmd, workload = rest.split("|")
        kern, m = read(rep)
        res[name] = {"capture": rep, "kernel": kern.split("(")[0], "command": cmd,
                     "workload": workload, **m}
    with open(dst, "w") as fh:
        json.dump(res, fh, indent=1)
        fh.write("\n")
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
