"""Per-source-line instruction counts and stall samples from an ncu report.

usage: python tools/ncu_lines.py report.ncu-rep [file-substring] [top]
"""
import csv
import io
import subprocess
import os
import sys


def main():
    rep = sys.argv[1]
    want = sys.argv[2] if len(sys.argv) > 2 else ""
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    path = None
    rows = []
    hdr = None
    for rec in csv.reader(io.StringIO(out)):
        if not rec:
            continue
        if rec[0] == "File Path":
            path = rec[1]
            continue
        if rec[0] == "Line No":
            hdr = rec
            continue
        if hdr is None or rec[0] in ("Function Name",) or not rec[0].isdigit():
            continue
        d = dict(zip(["line", "src"] + hdr[2:], rec))
        if want and want not in (path or ""):
            continue
        try:
            inst = int(d.get("Instructions Executed", "0") or 0)
            samp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            continue
        rows.append((path.rsplit("/", 1)[-1], int(rec[0]), inst, samp, rec[1].strip()[:90]))
    ti = sum(r[2] for r in rows) or 1
    ts = sum(r[3] for r in rows) or 1
    print(f"total warp-inst {ti:,}  samples {ts:,}")
    key = 3 if os.environ.get("BY_STALL") else 2
    for r in sorted(rows, key=lambda r: -r[key])[:top]:
        print(f"{r[0]}:{r[1]:<5} inst {100 * r[2] / ti:5.1f}%  stall {100 * r[3] / ts:5.1f}%  {r[4]}")


if __name__ == "__main__":
    main()
