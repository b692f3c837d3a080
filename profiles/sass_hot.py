"""Hottest SASS instructions of one kernel in an ncu report (source page).

    python profiles/sass_hot.py <file.ncu-rep> <kernel regex> [top]
"""
import csv
import io
import subprocess
import sys


def main(path, regex, top=30):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--kernel-name", f"regex:{regex}",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hdr]
    si, ni, ei = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    body = [r for r in rows[hdr + 1:] if len(r) > ei and r[0] and r[0] != "Address"]
    tot_s = sum(float(r[ni] or 0) for r in body) or 1.0
    tot_i = sum(float(r[ei] or 0) for r in body) or 1.0
    print(f"samples {tot_s:.0f}, warp instructions {tot_i:.3g}")
    for r in sorted(body, key=lambda r: -float(r[ni] or 0))[:top]:
        print(f"{r[0]:>6} {float(r[ni] or 0) / tot_s:6.3f} {float(r[ei] or 0) / tot_i:6.3f}  {r[si]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
