"""Top CUDA source lines by warp-stall samples / executed instructions from an .ncu-rep.

    python tools/ncu_lines.py report.ncu-rep [N] [function-substring]
"""
import csv
import subprocess
import sys


def main(path, n=25, func=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    allrows = []
    fname, fn = "", ""
    i = 0
    while i < len(rows):
        r = rows[i]
        if r and r[0] in ("File Name", "File Path"):
            fname = r[1].split("/")[-1]
        if r and r[0] in ("Function Name", "Kernel Name"):
            fn = r[1]
        if r and r[0] == "Line No" and "Warp Stall Sampling (All Samples)" in r:
            h = r
            si = h.index("Warp Stall Sampling (All Samples)")
            ii = h.index("Instructions Executed")
            i += 1
            while i < len(rows) and rows[i] and rows[i][0] not in ("Line No", "File Name", "File Path", "Address",
                                                                  "Function Name", "Kernel Name"):
                x = rows[i]
                if func is None or func in fn:
                    try:
                        allrows.append((int(x[si] or 0), int(x[ii] or 0), fname, x[0], x[1].strip()[:95]))
                    except (ValueError, IndexError):
                        pass
                i += 1
            continue
        i += 1
    ts = sum(a[0] for a in allrows) or 1
    ti = sum(a[1] for a in allrows) or 1
    print(f"{'stall%':>7} {'inst%':>6}  file:line  source")
    for s, ins, f, ln, src in sorted(allrows, key=lambda t: -(t[0] / ts + t[1] / ti))[:n]:
        print(f"{100*s/ts:6.1f}% {100*ins/ti:5.1f}%  {f}:{ln}  {src}")
    print(f"total warp-instructions {ti}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25, sys.argv[3] if len(sys.argv) > 3 else None)
