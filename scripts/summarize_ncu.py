"""Summarise ncu --set full captures into profiles/r01_<name>_ncu_summary.txt."""
import csv
import subprocess
import sys

KEYS = ['Kernel Name', 'launch__grid_size', 'launch__block_size', 'launch__registers_per_thread',
        'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_sector_hit_rate.pct',
        'l1tex__t_sector_hit_rate.pct', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__thread_inst_executed_per_inst_executed.ratio', 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum']


def summarize(rep, out, header):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, units = r[0], r[1]
    lines = ["# " + l for l in header.splitlines()]
    for row in r[2:]:
        d = dict(zip(h, row))
        lines.append("# --- launch")
        for k in KEYS:
            if k in d:
                lines.append("%s\t%s\t%s" % (k, d[k], units[h.index(k)]))
        st = [(int(float(d[k])), k) for k in h if k.startswith('smsp__pcsamp_warps_issue_stalled')
              and not k.endswith('not_issued') and d[k] not in ('', 'n/a')]
        lines.append("# top stall reasons (pc samples)")
        for c, k in sorted(st, reverse=True)[:6]:
            lines.append("%s\t%d" % (k, c))
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    summarize(sys.argv[1], sys.argv[2], sys.argv[3])
