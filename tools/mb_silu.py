import sys, os, json, torch
sys.path.insert(0, "/root/repo")
from paper_2502_15524_b200 import hs
ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
M, K, N = 22016, 4096, 512
Ws = [torch.randn(M, K, device="cuda").to(torch.bfloat16) * K ** -0.5 for _ in range(3)]
X = torch.randn(N, K, device="cuda").to(torch.bfloat16)
for epi, ocols in ((0, M), (2, M // 2)):
    out = torch.empty(N, ocols, device="cuda", dtype=torch.bfloat16)
    for i in range(3): hs.k_gemm(Ws[i % 3], X, N, epi, out, ws=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(20): hs.k_gemm(Ws[i % 3], X, N, epi, out, ws=ws)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    print(json.dumps({"epi": epi, "us": round(us, 1), "tflops": round(2 * M * N * K / us / 1e6, 1)}))
