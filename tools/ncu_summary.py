"""Summarise an .ncu-rep (details page) into the handful of numbers we track."""
import csv, subprocess, sys
KEEP = ("Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Compute (SM) Throughput",
        "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread", "Executed Ipc Active",
        "Issue Slots Busy", "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler",
        "Dynamic Shared Memory Per Block", "Grid Size", "Block Size", "Avg. Active Threads Per Warp",
        "Block Limit Shared Mem", "Block Limit Registers", "SM Frequency", "L2 Cache Throughput")
def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = csv.reader(out.splitlines()); h = next(r)
    cur = None
    for row in r:
        d = dict(zip(h, row))
        k = d.get("Kernel Name", "")[:80]
        if k != cur:
            print("==", k); cur = k
        if d.get("Metric Name") in KEEP:
            print(f"   {d['Metric Name']:40s} {d['Metric Value']} {d.get('Metric Unit','')}")
if __name__ == "__main__":
    main(sys.argv[1])
