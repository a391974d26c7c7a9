"""Determinism check of the prefill attention kernel (HS_ATTN_TC selects the kernel): the same
paged-attention call repeated 20 times must give identical bytes."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_15524_b200 import hs  # noqa: E402

torch.manual_seed(0)
for (nh, d, lens) in ((4, 64, (32, 17, 100)), (8, 128, (300, 129, 64)), (32, 128, (512,))):
    n = len(lens)
    T = sum(lens)
    nb = sum((l + 15) // 16 for l in lens) + 4
    q = (torch.randn(T, nh * d, device="cuda") * 0.5).to(torch.bfloat16)
    pool = (torch.randn(nb, 2, nh, 16, d, device="cuda") * 0.5).to(torch.bfloat16)
    max_blocks = max((l + 15) // 16 for l in lens)
    tables = torch.zeros(n, max_blocks, dtype=torch.int32, device="cuda")
    seqs = torch.zeros(n, 4, dtype=torch.int32, device="cuda")
    b, qs = 0, 0
    for i, l in enumerate(lens):
        k = (l + 15) // 16
        tables[i, :k] = torch.arange(b, b + k, dtype=torch.int32)
        seqs[i] = torch.tensor([qs, l, 0, i], dtype=torch.int32)
        b += k
        qs += l
    outs = []
    for it in range(20):
        o = torch.zeros(T, nh * d, dtype=torch.bfloat16, device="cuda")
        hs.k_attention(q, pool, seqs, max(lens), max(lens), tables, o, nh, d, False)
        torch.cuda.synchronize()
        outs.append(o.view(torch.int16).cpu().numpy())
    same = all(np.array_equal(outs[0], x) for x in outs[1:])
    ndiff = max(int((outs[0] != x).sum()) for x in outs[1:])
    print(f"nh={nh} d={d} lens={lens}: deterministic={same} max differing elements={ndiff}")
