"""Analyse a DFX_TRACE dump of the pair W.A^T kernel (experiment builds, -DDFX_TRACE).
  python scripts/trace_u.py gpurun_out/trace.bin
Per CTA: ev0 = producer issues fill j, ev1 = MMA sees stage i full (leader), ev2 = MMA
issued + committed stage i (leader), ev3 = chain finished stage i.  Times in ns."""
import sys

import numpy as np

N, EV, CTA = 256, 4, 148


def main(path):
    raw = open(path, "rb").read()
    rec = 32 + CTA * EV * N * 8
    for k in range(len(raw) // rec):
        hdr = np.frombuffer(raw[k * rec:k * rec + 32], dtype=np.int32)
        ctas, stages, kbps, nh, bn, cg, tiles, ks = hdr
        t = np.frombuffer(raw[k * rec + 32:(k + 1) * rec], dtype=np.uint64).reshape(CTA, EV, N).astype(np.float64)
        n = min(N, kbps)
        t0 = t[:ctas, 0, 0][t[:ctas, 0, 0] > 0].min()
        print(f"launch {k}: ctas {ctas} stages {stages} kb/split {kbps} nh {nh} bn {bn} commit_every {cg} tiles {tiles} ks {ks}")
        lat, mma_gap, issue_lag, chain_lag, starts, ends = [], [], [], [], [], []
        for c in range(0, ctas, 2):           # leaders
            iss = t[c, 0, :n] - t0
            iss_p = t[c + 1, 0, :n] - t0
            full = t[c, 1, :n] - t0
            mma = t[c, 2, :n] - t0
            ch = t[c, 3, :n] - t0
            if full[0] <= -t0 + 1:
                continue
            starts.append(iss[0]); ends.append(mma[n - 1])
            lat.append(full - np.maximum(iss, iss_p))            # issue -> MMA sees full
            mma_gap.append(np.diff(mma))                           # MMA stage-to-stage period
            issue_lag.append(iss[stages:] - mma[:n - stages])      # producer reissue vs consumption
            if ch.max() > 0:
                chain_lag.append(ch - mma)
        q = lambda a: np.percentile(np.concatenate(a), [10, 50, 90]).round(0) if a else None
        print("  first issue (ns, rel. to earliest CTA):", np.percentile(starts, [0, 50, 100]).round(0))
        print("  last MMA stage done:", np.percentile(ends, [0, 50, 100]).round(0))
        print("  issue->full latency p10/50/90:", q(lat))
        print("  MMA stage period p10/50/90:", q(mma_gap))
        print("  refill(j) - mma(j-S) p10/50/90:", q(issue_lag))
        print("  chain done - mma issued p10/50/90:", q(chain_lag))
        # where does the MMA wait: time from previous mma issue to this full arrival
        waits = [np.maximum(0, (t[c, 1, 1:n] - t[c, 2, :n - 1])) for c in range(0, ctas, 2) if t[c, 1, 0] > 0]
        print("  MMA idle per stage (full - prev issue) p10/50/90:", q(waits), " total per CTA (us) median:",
              round(float(np.median([w.sum() for w in waits])) / 1e3, 2))


if __name__ == "__main__":
    main(sys.argv[1])
