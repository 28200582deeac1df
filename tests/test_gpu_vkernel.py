"""Both V = B [G_hi | G_lo] kernels of the bf16 / fp16 tensor-core norm against the oracle.

The planner picks the V kernel per shape and SM budget (generic tc_rowdot that re-streams its
G slice per tile, or the G-stationary pair kernel tc_pair_gstat); DFX_V_GSTAT pins the choice
for the process, so each mode runs in a child process here.  ba_sq follows the reference's
rowsum((B G) (.) B) (factored_norm.cpp:104-117) to fp32 accumulation order; base_sq is
bitwise the reference's serial chain in both runs; the finished norms agree within the
bf16 / fp16 bar."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (d_out, d_in, r, dtype code): ragged rows, r not a multiple of 64, several N slices
# (pyoracle codes: 1 = bf16, 2 = fp16)
SHAPES = [(300, 512, 64, 1), (1000, 1024, 96, 1), (777, 640, 384, 1), (2048, 1024, 512, 1),
          (513, 512, 1024, 1), (1000, 1024, 384, 2), (256, 4096, 200, 1)]

CHILD = r"""
import json, sys, numpy as np, torch
sys.path[:0] = [sys.argv[1], sys.argv[1] + "/oracle"]
import paper_2603_22276_b200 as P, pyoracle
o = pyoracle.Oracle(); dfx = P.Dfx(0)
out = {}
for (d_out, d_in, r, dt) in json.loads(sys.argv[2]):
    tdt = {1: torch.bfloat16, 2: torch.float16}[dt]
    W = o.seeded_gaussian(d_out, d_in, 11, dt); A = o.seeded_gaussian(r, d_in, 12, dt)
    B = o.seeded_gaussian(d_out, r, 13, dt)
    cs, _ = o.plan_chunks(d_out, d_in)
    dev = lambda x: torch.from_numpy(x).cuda().to(tdt)
    t = torch.empty(3, d_out, device="cuda")
    wn = torch.empty(d_out, device="cuda")
    s = 2.0 / np.sqrt(r)
    dfx.row_norm(dev(W), dev(A), dev(B), s, cs, wn, terms=t)
    torch.cuda.synchronize()
    out[f"{d_out}x{d_in}x{r}x{dt}"] = {"terms": t.cpu().numpy().tolist(), "wn": wn.cpu().numpy().tolist()}
print(json.dumps(out))
"""


def _run(mode):
    env = dict(os.environ, DFX_V_GSTAT=str(mode))
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT, json.dumps(SHAPES)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_v_kernels_match_oracle(dfx, oracle):
    o = oracle
    runs = {m: _run(m) for m in (0, 1)}
    for (d_out, d_in, r, dt) in SHAPES:
        key = f"{d_out}x{d_in}x{r}x{dt}"
        W = o.seeded_gaussian(d_out, d_in, 11, dt)
        A = o.seeded_gaussian(r, d_in, 12, dt)
        B = o.seeded_gaussian(d_out, r, 13, dt)
        cs, _ = o.plan_chunks(d_out, d_in)
        s = 2.0 / np.sqrt(r)
        ref_base, ref_cross, ref_ba = o.norm_terms(W, A, B, s, cs)
        ref_wn = o.row_norm(dt, W, A, B, s, cs)
        t0 = np.asarray(runs[0][key]["terms"], np.float32)
        t1 = np.asarray(runs[1][key]["terms"], np.float32)
        for t in (t0, t1):
            assert np.array_equal(t[0].view(np.uint32), np.asarray(ref_base, np.float32).view(np.uint32)), key
            assert np.all(np.abs(t[2] - ref_ba) <= 1e-4 * np.abs(ref_ba) + 1e-6 * ref_ba.max()), key
        # the two V kernels: the same ba_sq up to fp32 accumulation order
        assert np.all(np.abs(t0[2] - t1[2]) <= 1e-4 * np.abs(t0[2]) + 1e-6 * t0[2].max()), key
        ulp = np.spacing(ref_wn.astype(np.float32)) * (2 ** 16 if dt == 1 else 2 ** 13)
        for m in (0, 1):
            wn = np.asarray(runs[m][key]["wn"], np.float32)
            assert np.all(np.abs(wn - ref_wn) <= ulp), (key, m)
