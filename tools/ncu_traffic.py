"""Scan-stage DRAM traffic per search from an ncu capture of one search step.

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
        --log-file gpurun_out/traffic_c3.csv python tools/prof_search.py --config c3 --nprobe 8 --reps 1
    python tools/ncu_traffic.py gpurun_out/traffic_c3.csv c3 8 > profiles/round1/traffic_c3.json

Sums the kernels of the last search (scan-stage kernels: everything launched by
ivrq_search_scan); the per-kernel split is kept for DESIGN.md.
"""
import csv
import json
import sys

SCAN = ("scan_", "first_", "ip_", "tc_", "pair_", "qhat", "cs_", "group_prefix", "rda_", "lf_max", "rd_radius")


def main(path, cfg, nprobe):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    idi = h.index("ID")
    per = {}
    for r in rows[1:]:
        k = r[ki]
        per.setdefault(int(r[idi]), {"name": k})[r[mi]] = (float(r[vi].replace(",", "")), r[ui])
    ids = sorted(per)
    # the last search: from the last rotate GEMM (StoreF64 epilogue) on
    last = max(i for i in ids if "StoreF64" in per[i]["name"] or "RowMajor<float>, gemm::RowMajor<float>" in per[i]["name"])
    tot, kern = 0.0, {}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for i in ids:
        if i <= last:
            continue
        name = per[i]["name"].split("(")[0].replace("void ", "")
        if not any(t in name for t in SCAN):
            continue
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            v, u = per[i].get(m, (0.0, "byte"))
            b += v * scale.get(u, 1)
        tot += b
        kern[name] = kern.get(name, 0.0) + b
    print(json.dumps({"config": cfg, "n_probe": int(nprobe), "dram_bytes": int(tot),
                      "kernels": {k: int(v) for k, v in sorted(kern.items(), key=lambda kv: -kv[1])}}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3])
