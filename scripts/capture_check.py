import torch, paper_2603_22276_b200 as P
dfx = P.Dfx(0)
st = torch.cuda.Stream()
b = torch.randn(256, 1024, device="cuda").bfloat16(); l = torch.randn_like(b); g = torch.ones(1024, device="cuda"); d = torch.empty_like(b)
with torch.cuda.stream(st):
    dfx.compose_fwd(b, l, g, 0.5, d)
torch.cuda.synchronize()
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr, stream=st):
    dfx.compose_fwd(b, l, g, 0.5, d)
gr.replay(); torch.cuda.synchronize(); print("capture ok")
