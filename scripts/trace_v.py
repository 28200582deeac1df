"""Analyse a DFX_VTRACE dump of the G-stationary V kernel (experiment builds, -DDFX_TRACE).
  python scripts/trace_v.py gpurun_out/vtrace.bin
Per-CTA %globaltimer stamps (ns): 0 entry, 1 after the cluster sync, 2 G slice issued, 3 MMA saw
the G slice, 4 MMA saw the first B stage, 5 MMA issued the last commit, 6 epilogue had its B
slice, 7 epilogue saw the accumulator, 8 ba_sq stored, 9 epilogue done (finisher included)."""
import sys

import numpy as np

CTA, EV = 148, 10
NAMES = ["entry", "synced", "G issued", "G landed", "B0 landed", "last commit", "B regs",
         "acc ready", "stored", "done"]


def main(path):
    raw = open(path, "rb").read()
    rec = 32 + CTA * EV * 8
    for k in range(len(raw) // rec):
        hdr = np.frombuffer(raw[k * rec:k * rec + 32], dtype=np.int32)
        ctas = int(hdr[0])
        t = np.frombuffer(raw[k * rec + 32:(k + 1) * rec], dtype=np.uint64).reshape(CTA, EV)
        t = t[:min(ctas, CTA)].astype(np.float64)
        t0 = t[:, 0][t[:, 0] > 0].min()
        print(f"launch {k}: ctas {ctas} stages {hdr[1]} kx {hdr[2]} bn {hdr[3]} nsl {hdr[4]} tiles {hdr[5]}")
        for e in range(EV):
            v = t[:, e]
            v = v[v > 0] - t0
            if len(v):
                p = np.percentile(v, [0, 50, 100]) / 1e3
                print(f"  {e} {NAMES[e]:12s} min/med/max us after first entry: {p[0]:7.2f} {p[1]:7.2f} {p[2]:7.2f}")


if __name__ == "__main__":
    main(sys.argv[1])
