"""Analyse a DFX_TRACE dump of the pair W.A^T kernel (experiment builds, -DDFX_TRACE).
  python scripts/trace_u.py gpurun_out/trace.bin
Events per CTA and ring stage (ns, %globaltimer): 0 producer issued stage j, 1 MMA saw stage i
full (leader), 2 MMA released stage i (leader), 3 producer saw stage j's slot empty."""
import sys

import numpy as np

N, EV, CTA = 128, 4, 148


def main(path):
    raw = open(path, "rb").read()
    rec = 32 + CTA * EV * N * 8
    for k in range(len(raw) // rec):
        hdr = np.frombuffer(raw[k * rec:k * rec + 32], dtype=np.int32)
        ctas, stages, kbps, nh, bn, ka, tiles, ks = hdr
        t = np.frombuffer(raw[k * rec + 32:(k + 1) * rec], dtype=np.uint64).reshape(CTA, EV, N).astype(np.float64)
        n = min(N, kbps // max(ka, 1))
        print(f"launch {k}: ctas {ctas} stages {stages} kb/split {kbps} nh {nh} bn {bn} ka {ka} tiles {tiles}")
        lat, period, relwait, emptylat, full_gap = [], [], [], [], []
        for c in range(0, ctas, 2):
            iss = np.maximum(t[c, 0, :n], t[c + 1, 0, :n])
            full, rel, emp = t[c, 1, :n], t[c, 2, :n], t[c, 3, :n]
            if full[0] == 0:
                continue
            lat.append(full - iss)                         # issue (later CTA) -> MMA sees full
            period.append(np.diff(full))                    # consumption period
            emptylat.append(emp[stages:] - rel[:n - stages])  # release -> producer sees the slot
            full_gap.append(full[1:] - rel[:-1])            # MMA waits for the next stage
        q = lambda a: np.percentile(np.concatenate(a), [10, 50, 90]).round(0)
        print("  TMA latency (issue -> full seen) p10/50/90 ns:", q(lat))
        print("  stage period (full_i -> full_i+1):", q(period))
        print("  release -> producer sees empty:", q(emptylat))
        print("  MMA idle (release_i -> full_i+1):", q(full_gap))
        print("  tile time (first issue -> last release) median us:",
              round(float(np.median([t[c, 2, n - 1] - t[c, 0, 0] for c in range(0, ctas, 2) if t[c, 1, 0] > 0])) / 1e3, 2))


if __name__ == "__main__":
    main(sys.argv[1])
