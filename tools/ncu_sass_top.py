"""Top SASS instructions of one kernel by warp-stall samples (ncu source page).

    python tools/ncu_sass_top.py report.ncu-rep kernel-regex [N]
"""
import csv
import subprocess
import sys


def main(path, kregex, n=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass",
                          "--kernel-name", "regex:" + kregex], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = next(r for r in rows if r and r[0] == "Address")
    si = h.index("Warp Stall Sampling (All Samples)")
    ii = h.index("Instructions Executed")
    data = []
    for r in rows:
        if len(r) == len(h) and r[0] != "Address":
            try:
                data.append((int(r[si] or 0), int(r[ii] or 0), r[0], r[1]))
            except ValueError:
                pass
    tot = sum(d[0] for d in data) or 1
    for s, ins, addr, src in sorted(data, key=lambda d: -d[0])[:n]:
        print(f"{100 * s / tot:5.1f}% {ins:>10d}  {addr}  {src[:100]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
