import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_15524_b200 import hs
nh, d, ctx, B = 32, 128, 576, 1
nblk = B * ((ctx + 15) // 16) + 4
pool = torch.randn(nblk, 2, nh, 16, d, device="cuda").to(torch.bfloat16)
maxb = (ctx + 15) // 16 + 1
tables = torch.arange(B * maxb, device="cuda", dtype=torch.int32).reshape(B, maxb) % nblk
seqs = torch.tensor([[i, 1, ctx - 1, i] for i in range(B)], dtype=torch.int32, device="cuda")
q = torch.randn(B, nh * d, device="cuda").to(torch.bfloat16)
o = torch.empty_like(q)
ws = torch.empty(B * nh * 64 * (d + 2), dtype=torch.float32, device="cuda")
for _ in range(5):
    hs.k_attention(q, pool, seqs, 1, ctx, tables, o, nh, d, True, ws)
torch.cuda.synchronize()
