"""Key per-kernel metrics of an ncu --set full report as JSON (for
profiles/kernel_metrics.json, read by bench.py's compute rooflines):
issue activity, SIMD efficiency, L2 / L1 hit rates, occupancy, DRAM bytes."""
import csv
import json
import subprocess
import sys

WANT = {
    "duration_ns": "gpu__time_duration.sum",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "thread_inst_per_warp_inst": "smsp__thread_inst_executed_per_inst_executed.ratio",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "l1_hit_pct": "l1tex__t_sector_hit_rate.pct",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "registers": "launch__registers_per_thread",
}


def metrics(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, units = r[0], r[1]
    out = []
    for row in r[2:]:
        d = dict(zip(h, row))
        m = {"kernel": d.get("Kernel Name", "")}
        for k, name in WANT.items():
            if name in d and d[name] not in ("", "n/a"):
                v = float(d[name].replace(",", ""))
                u = units[h.index(name)]
                if u == "Kbyte":
                    v *= 1e3
                elif u == "Mbyte":
                    v *= 1e6
                elif u == "Gbyte":
                    v *= 1e9
                elif u == "usecond":
                    v *= 1e3
                elif u == "msecond":
                    v *= 1e6
                m[k] = v
        if "thread_inst_per_warp_inst" in m:
            m["simd_efficiency"] = m["thread_inst_per_warp_inst"] / 32.0
        out.append(m)
    return out


if __name__ == "__main__":
    # ncu_metrics.py <report> <key>                    first kernel of the report
    # ncu_metrics.py <report> <key> <kernel-substring>  first kernel whose name contains the substring
    ms = metrics(sys.argv[1])
    if len(sys.argv) > 3:
        ms = [m for m in ms if sys.argv[3] in m["kernel"]]
    print(json.dumps({sys.argv[2]: ms[0]}))
