#!/usr/bin/env python3
"""Summarise ncu reports for profiles/: for every <name>.ncu-rep given,
write <outdir>/<name>_exec_kernel_details.csv (the details page) and
<outdir>/<name>_raw_key.json (the key raw metrics), and print one line.

usage: python tools/ncu_summary.py OUTDIR report.ncu-rep [...]
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
        "launch__occupancy_limit_registers", "sm__cycles_active.avg", "gpc__cycles_elapsed.max",
        "lts__t_sector_hit_rate.pct"]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout


def main():
    out = sys.argv[1]
    os.makedirs(out, exist_ok=True)
    for rep in sys.argv[2:]:
        name = os.path.basename(rep)[:-len(".ncu-rep")]
        with open(os.path.join(out, f"{name}_exec_kernel_details.csv"), "w") as f:
            f.write(ncu("-i", rep, "--page", "details", "--csv"))
        rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(KEYS)))))
        hdr, units, vals = rows[0], rows[1], rows[2]
        key = {h: [v, u] for h, u, v in zip(hdr, units, vals) if h in KEYS}
        json.dump(key, open(os.path.join(out, f"{name}_raw_key.json"), "w"), indent=1)

        def num(k, scale):
            v, u = key[k]
            v = float(v.replace(",", ""))
            return v * scale.get(u, 1.0)
        g = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
        t = num("gpu__time_duration.sum", {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "msecond": 1e-3, "usecond": 1e-6})
        rd, wr = num("dram__bytes_read.sum", g), num("dram__bytes_write.sum", g)
        print(json.dumps({"report": name, "us": round(t * 1e6, 1), "dram_read_GB": round(rd / 1e9, 4),
                          "dram_write_GB": round(wr / 1e9, 4), "dram_bytes": int(rd + wr),
                          "dram_TBps": round((rd + wr) / t / 1e12, 3),
                          "dram_pct_peak": key.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", ["?"])[0],
                          "grid": key["launch__grid_size"][0], "regs": key["launch__registers_per_thread"][0]}))


if __name__ == "__main__":
    main()
