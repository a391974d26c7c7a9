import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2502_15524_b200 import hs
sys.path.insert(0, "tests"); from test_kernels_gpu import attention_ref, rand_bf16, dev_bf16, host_bits
from oracle.numerics import bf16_value, bf16_bits
rng = np.random.default_rng(0)
for nh, d, ctx in [(1, 128, 37), (1, 128, 130), (2, 64, 100)]:
    nblk = 16
    pool = np.zeros((nblk, 2, nh, 16, d), dtype=np.uint16)
    K, V = rand_bf16(rng, (ctx, nh, d)), rand_bf16(rng, (ctx, nh, d))
    tab = list(range(nblk))[::-1]
    for p in range(ctx):
        pool[tab[p // 16], 0, :, p % 16] = K[p]; pool[tab[p // 16], 1, :, p % 16] = V[p]
    q = rand_bf16(rng, (ctx, nh, d))
    ref = attention_ref(bf16_value(q), bf16_value(K), bf16_value(V), np.arange(ctx))
    o = torch.empty((ctx, nh * d), dtype=torch.bfloat16, device="cuda")
    tables = torch.tensor([tab + [0] * 8], dtype=torch.int32, device="cuda")
    seqs = torch.tensor([[0, ctx, 0, 0]], dtype=torch.int32, device="cuda")
    hs.k_attention(dev_bf16(q.reshape(ctx, nh * d)), dev_bf16(pool), seqs, ctx, ctx, tables, o, nh, d, False, None)
    torch.cuda.synchronize()
    g = bf16_value(host_bits(o)).reshape(ctx, nh, d)
    err = np.abs(g - ref).max(axis=(1, 2))
    print(nh, d, ctx, "bad rows:", [(i, round(float(e), 3)) for i, e in enumerate(err) if e > 0.05][:20])
    bad = np.abs(g - ref) > 0.05
    if bad.any():
        r = np.where(bad.any(axis=(1, 2)))[0][0]
        print(" row", r, "bad dims", np.where(bad[r].any(axis=0))[0][:40])
# multi-sequence packed case (as tests/test_kernels_gpu.py::test_attention_paged)
for nh, d in [(4, 64), (8, 128)]:
    rng = np.random.default_rng(nh + d)
    lens = [37, 1, 130, 16]
    nblk, maxb = 64, 48
    free = list(rng.permutation(nblk))
    pool = np.zeros((nblk, 2, nh, 16, d), dtype=np.uint16)
    seqs, tables, qs, outs_ref, t0 = [], np.zeros((len(lens), maxb), np.int32), [], [], 0
    for i, n in enumerate(lens):
        ctx = n
        nb = (ctx + 15) // 16
        tab = [free.pop() for _ in range(nb)]
        tables[i, :nb] = tab
        K, V = rand_bf16(rng, (ctx, nh, d)), rand_bf16(rng, (ctx, nh, d))
        for p in range(ctx):
            pool[tab[p // 16], 0, :, p % 16] = K[p]
            pool[tab[p // 16], 1, :, p % 16] = V[p]
        q = rand_bf16(rng, (n, nh, d))
        outs_ref.append(attention_ref(bf16_value(q), bf16_value(K), bf16_value(V), np.arange(ctx - n, ctx)))
        qs.append(q)
        seqs.append([t0, n, ctx - n, i])
        t0 += n
    q = np.concatenate(qs).reshape(t0, nh * d)
    o = torch.zeros((t0, nh * d), dtype=torch.bfloat16, device="cuda")
    hs.k_attention(dev_bf16(q), dev_bf16(pool), torch.tensor(seqs, dtype=torch.int32, device="cuda"),
                   max(lens), max(lens), torch.from_numpy(tables).cuda(), o, nh, d, False, None)
    torch.cuda.synchronize()
    g = bf16_value(host_bits(o)).reshape(t0, nh, d)
    ref = np.concatenate(outs_ref)
    err = np.abs(g - ref).max(axis=2)
    rows = np.where(err.max(axis=1) > 0.05)[0]
    print("packed", nh, d, "bad rows", rows[:40], "heads", np.where(err.max(axis=0) > 0.05)[0])
