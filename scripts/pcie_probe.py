import torch, time
n_up, n_dn = 348160000, 201392128
hu = torch.empty(n_up, dtype=torch.uint8).pin_memory(); du = torch.empty(n_up, dtype=torch.uint8, device="cuda")
hd = torch.empty(n_dn, dtype=torch.uint8).pin_memory(); dd = torch.empty(n_dn, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
up = lambda: du.copy_(hu, non_blocking=True)
dn = lambda: hd.copy_(dd, non_blocking=True)
def both():
    with torch.cuda.stream(s1): du.copy_(hu, non_blocking=True)
    with torch.cuda.stream(s2): hd.copy_(dd, non_blocking=True)
tu, td, tb = t(up), t(dn), t(both)
print(f"H2D {n_up/tu/1e9:.1f} GB/s ({tu*1e3:.2f} ms), D2H {n_dn/td/1e9:.1f} GB/s ({td*1e3:.2f} ms), both {tb*1e3:.2f} ms -> floor {1/tb:.1f} steps/s")
