"""Summarise .ncu-rep captures into a markdown table (run here, no GPU needed).
usage: python tools/ncu_summary.py OUT.md REP [REP ...]"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__cycles_active.avg", "SMSP active cycles"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem"),
]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    return hdr, units, r[2:]


def main():
    dst, reps = sys.argv[1], sys.argv[2:]
    lines = []
    for rep in reps:
        hdr, units, data = rows(rep)
        for d in data:
            name = d[hdr.index("Kernel Name")][:90]
            lines.append(f"### {name}  ({rep.split('/')[-1]})\n")
            lines.append("| metric | value | unit |\n|---|---|---|")
            for key, label in METRICS:
                if key in hdr:
                    i = hdr.index(key)
                    lines.append(f"| {label} (`{key}`) | {d[i]} | {units[i]} |")
            stalls = [(h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), d[i])
                      for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_")]
            def f(x):
                try:
                    return float(x)
                except ValueError:
                    return 0.0
            stalls.sort(key=lambda x: -f(x[1]))
            lines.append("\nTop stall reasons (warps per issue): " +
                         ", ".join(f"{k} {float(v):.2f}" for k, v in stalls[:6]) + "\n")
    open(dst, "w").write("\n".join(lines) + "\n")
    print(dst)


if __name__ == "__main__":
    main()
