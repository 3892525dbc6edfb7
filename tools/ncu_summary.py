"""Summarise ncu reports (run here, no GPU): key metrics + top stalled SASS lines.

usage: python tools/ncu_summary.py report1.ncu-rep [...]   > profiles/<name>.md
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("launch__occupancy_limit_registers", "occ. limit regs"),
    ("launch__occupancy_limit_shared_mem", "occ. limit smem"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
]


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def summarize(rep):
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")][:90]
        out.append(f"### {name}\n")
        out.append("| metric | value |\n|---|---|")
        for key, label in METRICS:
            if key in hdr:
                i = hdr.index(key)
                out.append(f"| {label} (`{key}`) | {r[i]} {units[i]} |")
        st = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")]
        tot = float(r[hdr.index("smsp__pcsamp_sample_count")] or 1)
        top = sorted(((float(r[hdr.index(h)] or 0), h) for h in st), reverse=True)[:6]
        out.append("| top stall reasons (pc sampling) | " + ", ".join(
            f"{h.replace('smsp__pcsamp_warps_issue_stalled_', '')} {v / tot:.0%}" for v, h in top) + " |")
        out.append("")
    src = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    if len(src) > 2:
        h = src[1]
        try:
            i_s, i_src = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
            data = []
            for r in src[2:]:
                try:
                    data.append((float(r[i_s] or 0), r[i_src]))
                except (ValueError, IndexError):
                    pass
            tot = sum(d[0] for d in data) or 1
            out.append("Top stalled SASS instructions (share of samples):\n")
            for v, s in sorted(data, reverse=True)[:8]:
                out.append(f"    {v / tot:6.1%}  {s.strip()[:100]}")
            out.append("")
        except ValueError:
            pass
    return "\n".join(out)


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        print(f"## {rep.split('/')[-1]}\n")
        print(summarize(rep))
