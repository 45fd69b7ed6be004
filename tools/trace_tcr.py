"""Summarise a tc_refine CTA-0 timeline (dev builds with -DIVRQ_TCR_TRACE): per tag a 4096-slot
array of clock64 stamps indexed by the event's counter (0 = not recorded)."""
import sys

import numpy as np

NAMES = {1: "P", 2: "M", 3: "A", 4: "B", 5: "E0", 6: "E1", 7: "L", 8: "Mi"}


def main(path):
    a = np.fromfile(path, dtype=np.uint64).reshape(16, 4096).astype(np.int64)
    t0 = a[a > 0].min()
    ev = {t: {i: int(a[t, i] - t0) for i in np.flatnonzero(a[t])} for t in NAMES}
    span = max(max(v.values()) for v in ev.values() if v)
    print(f"{path}: span {span} clk; stages {len(ev[2])} tiles {len(ev[3])} groups {len(ev[4])}")

    def pairs(t1, t2):
        return [ev[t2][i] - ev[t1][i] for i in ev[t1] if i in ev[t2]]

    def show(label, xs):
        if xs:
            print(f"  {label:38s} median {np.median(xs):8.0f} mean {np.mean(xs):8.0f}")

    show("MMA issue of one stage (M->Mi)", pairs(2, 8))
    show("MMA stage-to-stage", list(np.diff(sorted(ev[2].values()))))
    show("producer issue -> MMA start (P->M)", pairs(1, 2))
    show("producer stage-to-stage", list(np.diff(sorted(ev[1].values()))))
    show("epilogue per tile (E0->E1)", pairs(5, 6))
    show("MMA tile start gap (A)", list(np.diff(sorted(ev[3].values()))))
    show("B issue -> bfull (L->B)", pairs(7, 4))
    # empty round trip: MMA issue done for stage i -> producer issue of stage i + NST
    for nst in (3, 4, 5, 6):
        x = [ev[1][i + nst] - ev[8][i] for i in ev[8] if i + nst in ev[1]]
        if x and np.median(x) > 0:
            show(f"commit(empty) -> producer (NST={nst})", x)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
