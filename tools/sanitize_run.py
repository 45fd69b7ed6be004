"""Small searches that exercise the tcgen05 / TMA / mbarrier kernels, for compute-sanitizer."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2602_23999_b200 as iv  # noqa: E402


def run(n, d, nlist, bits, nprobe, k, mode="bitwise"):
    rng = np.random.default_rng(d)
    x = rng.standard_normal((n, d)).astype(np.float32)
    q = rng.standard_normal((64, d)).astype(np.float32)
    ix = iv.build_index(x, iv.BuildParams(n_clusters=nlist, quant=iv.QuantizationParams(bits=bits), kmeans_iters=2))
    res = iv.search_batch(q, ix, iv.SearchParams(k=k, n_probe=nprobe, ip_mode=mode))
    print(f"n={n} d={d} bits={bits}: {sum(r[0].size for r in res)} results")


if __name__ == "__main__":
    import os

    os.environ.setdefault("IVRQ_TC_IP", "1")
    os.environ.setdefault("IVRQ_TC_REFINE", "1")
    run(4000, 768, 16, 8, 4, 10)   # tc_refine (fused stage 1), scan_rda, rda_final, tc_probe
    run(4000, 512, 16, 4, 4, 10)   # tc_refine nibble producers, tc_ip
    run(3000, 96, 12, 3, 3, 7)     # ip_list / warp path
