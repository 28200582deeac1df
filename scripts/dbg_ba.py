"""Debug helper: per-tile error of the norm terms vs the oracle, and run-to-run determinism."""
import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle'); sys.path.insert(0, 'tests')
import pyoracle, paper_2603_22276_b200 as P
from conftest import to_dev
o = pyoracle.Oracle(); dfx = P.Dfx(0)
shapes = [tuple(map(int, a.split(','))) for a in sys.argv[1:]] or [(128, 4096, 512), (1024, 1024, 384)]
for (d_out, d_in, r) in shapes:
    W = o.seeded_gaussian(d_out, d_in, 1, 1); A = o.seeded_gaussian(r, d_in, 2, 1); B = o.seeded_gaussian(d_out, r, 3, 1)
    s = 2 / np.sqrt(r); cs, _ = o.plan_chunks(d_out, d_in)
    want = o.norm_terms(W, A, B, s, cs)
    w, a, b = to_dev(W, 1), to_dev(A, 1), to_dev(B, 1)
    prev = None
    for rep in range(3):
        out = torch.empty(3, d_out, device='cuda')
        dfx.norm_terms(w, a, b, s, cs, out[0], out[1], out[2]); torch.cuda.synchronize()
        t = out.cpu().numpy()
        sc = np.sqrt(want[0] * want[2])
        e = [np.abs(t[0] - want[0]).max(), (np.abs(t[1] - want[1]) / sc).max(), (np.abs(t[2] - want[2]) / want[2]).max()]
        det = None if prev is None else [bool(np.array_equal(prev[i], t[i])) for i in range(3)]
        print(d_out, d_in, r, 'rep', rep, 'err base/cross/ba', ['%.2e' % x for x in e], 'same-as-prev', det,
              'worst ba tile', int(np.argmax(np.abs(t[2] - want[2]) / want[2]) // 128))
        prev = t
