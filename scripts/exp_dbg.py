import ctypes as C, math, os, sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2603_22276_b200 as P
dfx = P.Dfx(0)
d_out = d_in = 8192; r = 384; s = 2 / math.sqrt(r)
W = torch.randn(d_out, d_in, device='cuda').bfloat16(); A = torch.randn(r, d_in, device='cuda').bfloat16()
B = torch.randn(d_out, r, device='cuda').bfloat16(); wn = torch.empty(d_out, device='cuda')
for _ in range(3): dfx.row_norm(W, A, B, s, 8192, wn)
torch.cuda.synchronize()
buf = (C.c_longlong * 4096)()
dfx.lib.dfx_exp_dbg.argtypes = [C.c_void_p, C.c_int]
dfx.lib.dfx_exp_dbg(buf, 256)
t = np.array(buf[:256], dtype=np.int64)
before, after = t[0::2], t[1::2]
print("total cycles (first wait -> last wait)", after[-1] - before[0])
print("wait cycles per k-block (first 20):", (after - before)[:20].tolist())
print("issue->next cycles per k-block (first 20):", (before[1:] - after[:-1])[:20].tolist())
print("median block period", np.median(np.diff(before)), "median wait", np.median(after - before))
