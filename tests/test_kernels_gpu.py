"""Op-level parity of every sm_100a kernel (through the C ABI, include/hs_kernels.h) against
the CPU oracle's definition of the op, on seeded inputs spanning several tiles and ragged
tails.  Tolerances: bf16 outputs may differ from the fp64
oracle by at most 1 bf16 ulp (the GPU accumulates in fp32) on a small fraction of elements;
byte copies must be bit-exact; argmax must be exact (same fp32 inputs on both sides)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.numerics import bf16, bf16_bits, bf16_value, rmsnorm, rope, rope_cos_sin, silu  # noqa: E402

if torch.cuda.is_available():
    from paper_2502_15524_b200 import hs  # noqa: E402


def dev_bf16(bits: np.ndarray):
    return torch.from_numpy(bits.view(np.int16)).cuda().view(torch.bfloat16)


def host_bits(t) -> np.ndarray:
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def rand_bf16(rng, shape, scale=1.0):
    return bf16_bits(rng.standard_normal(shape) * scale)


def ulp_diff(a_bits, b_bits):
    """Distance in bf16 ulps between two bf16 bit arrays (monotone integer mapping)."""
    def key(b):
        b = b.astype(np.int32)
        return np.where(b & 0x8000, 0x8000 - (b & 0x7FFF), 0x8000 + b)
    return np.abs(key(a_bits) - key(b_bits))


def check_bf16(gpu_bits, ref_vals, max_frac=0.02, scale=None, rel=2.0 ** -20):
    """<= 1 bf16 ulp from the exactly rounded fp64 value, except where cancellation makes the
    result tiny: there |gpu - ref| <= rel * scale (accumulation error of the terms; 2^-20 for
    an fp32 sum, 2^-16 for tensor-core attention with P split into two bf16 halves)."""
    d = ulp_diff(gpu_bits, bf16_bits(ref_vals))
    if scale is not None:
        close = np.abs(bf16_value(gpu_bits) - ref_vals) <= rel * scale
        d = np.where(close, np.minimum(d, 1), d)
    assert d.max() <= 1, f"max ulp diff {d.max()}"
    assert (d > 0).mean() <= max_frac, f"{(d > 0).mean():.4f} of elements differ by 1 ulp"


def tiled(W):
    """A [M, K] weight as the library stores it (include/hs.h): 128 x 64 blocks, each contiguous,
    block (i, j) at i * K/64 + j (same shape, permuted memory)."""
    M, K = W.shape
    return W.view(M // 128, 128, K // 64, 64).permute(0, 2, 1, 3).contiguous().view(M, K)


GEMM_CASES = [  # (M, K, N)
    (256, 256, 1), (256, 256, 16), (384, 256, 37), (256, 512, 64), (512, 256, 130),
    (768, 256, 300), (256, 768, 1100), (128, 64, 5),
    (2048, 4096, 7), (1536, 2048, 64), (4096, 11008, 3),  # stream-K (decode) path when ws is given
    (4096, 4096, 128), (2048, 1024, 200),                 # prefill chunks: tiled split-K / persistent
    (12288, 1024, 512), (22016, 1024, 300),               # CTA-pair kernel (256 x 256 tiles, ragged N)
    (4096, 8192, 512),                                    # CTA pairs with split-K + reduction (ws given)
]


@pytest.mark.parametrize("M,K,N", GEMM_CASES)
@pytest.mark.parametrize("split", [False, True])
def test_gemm_epilogues(M, K, N, split):
    rng = np.random.default_rng(M * 7 + K + N)
    Wb, Xb = rand_bf16(rng, (M, K), K ** -0.5), rand_bf16(rng, (N + 3, K))
    Rb = rand_bf16(rng, (N, M))
    W, X, R = tiled(dev_bf16(Wb)), dev_bf16(Xb), dev_bf16(Rb)
    ws = torch.empty(16 << 20, dtype=torch.uint8, device="cuda") if split else None
    acc = bf16_value(Xb[:N]) @ bf16_value(Wb).T  # [N, M] float64
    out = torch.empty((N, M), dtype=torch.bfloat16, device="cuda")
    hs.k_gemm(W, X, N, 0, out, ws=ws)
    torch.cuda.synchronize()
    check_bf16(host_bits(out), acc, scale=np.abs(bf16_value(Xb[:N])) @ np.abs(bf16_value(Wb)).T)
    hs.k_gemm(W, X, N, 1, out, resid=R, ws=ws)
    torch.cuda.synchronize()
    absacc = np.abs(bf16_value(Xb[:N])) @ np.abs(bf16_value(Wb)).T
    check_bf16(host_bits(out), bf16_value(Rb) + acc, scale=absacc + np.abs(bf16_value(Rb)))
    outf = torch.empty((N, M), dtype=torch.float32, device="cuda")
    hs.k_gemm(W, X, N, 3, outf, ws=ws)
    torch.cuda.synchronize()
    assert np.abs(outf.cpu().numpy() - acc).max() <= 1e-4 * max(1.0, np.abs(acc).max())
    # gate/up interleaved by 16 rows -> silu(g) * u  [N, M/2]
    outh = torch.empty((N, M // 2), dtype=torch.bfloat16, device="cuda")
    hs.k_gemm(W, X, N, 2, outh, ws=ws)
    torch.cuda.synchronize()
    rows = np.arange(M).reshape(-1, 32)
    gi, ui = rows[:, :16].ravel(), rows[:, 16:].ravel()
    g, u = acc[:, gi], acc[:, ui]
    # propagate the fp32 accumulation error of g and u through silu(g) * u (|silu'| <= 1.1)
    check_bf16(host_bits(outh), silu(g) * u, scale=1.1 * np.abs(u) * absacc[:, gi] + np.abs(silu(g)) * absacc[:, ui])


def test_gemm_llama_shapes_decode_and_prefill():
    """7B shapes: gate_up (M=22016, K=4096) at decode N=1 (split-K) and O-proj at N=512."""
    rng = np.random.default_rng(5)
    for (M, K, N) in ((22016, 4096, 1), (4096, 4096, 512), (4096, 11008, 16)):
        Wb, Xb = rand_bf16(rng, (M, K), K ** -0.5), rand_bf16(rng, (N, K))
        out = torch.empty((N, M), dtype=torch.float32, device="cuda")
        ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
        hs.k_gemm(tiled(dev_bf16(Wb)), dev_bf16(Xb), N, 3, out, ws=ws)
        torch.cuda.synchronize()
        sel = rng.choice(M, 64, replace=False)
        ref = bf16_value(Xb) @ bf16_value(Wb[sel]).T
        assert np.abs(out.cpu().numpy()[:, sel] - ref).max() <= 2e-3 * max(1.0, np.abs(ref).max())


@pytest.mark.parametrize("T,H", [(1, 256), (7, 4096), (33, 5120), (5, 256)])
def test_rmsnorm(T, H):
    rng = np.random.default_rng(T + H)
    xb, wb = rand_bf16(rng, (T, H), 3.0), bf16_bits(1 + 0.1 * rng.standard_normal(H))
    y = torch.empty((T, H), dtype=torch.bfloat16, device="cuda")
    hs.k_rmsnorm(dev_bf16(xb), dev_bf16(wb), y, 1e-5)
    torch.cuda.synchronize()
    check_bf16(host_bits(y), rmsnorm(bf16_value(xb), bf16_value(wb), 1e-5, rnd=lambda v: v), max_frac=0.01)
    rows = torch.tensor([T - 1, 0], dtype=torch.int32, device="cuda")
    y2 = torch.empty((2, H), dtype=torch.bfloat16, device="cuda")
    hs.k_rmsnorm(dev_bf16(xb), dev_bf16(wb), y2, 1e-5, rows=rows)
    torch.cuda.synchronize()
    assert np.array_equal(host_bits(y2), host_bits(y)[[T - 1, 0]])


def rope_table(max_pos, d, theta=1e4):
    c, s = rope_cos_sin(np.arange(max_pos), d, theta)
    return torch.from_numpy(np.stack([c, s], -1).astype(np.float32)).cuda()


@pytest.mark.parametrize("nh,d", [(4, 64), (32, 128)])
def test_rope_kv_write(nh, d):
    rng = np.random.default_rng(nh)
    T, H, nblk = 21, nh * d, 8
    qkv = rand_bf16(rng, (T, 3 * H))
    pos = np.arange(T, dtype=np.int32) + 5
    blocks = np.array([6, 1, 3], dtype=np.int32)
    slot = np.array([blocks[p // 16] * 16 + p % 16 for p in pos], dtype=np.int32)
    pool = torch.zeros((nblk, 2, nh, 16, d), dtype=torch.bfloat16, device="cuda")
    q = torch.empty((T, H), dtype=torch.bfloat16, device="cuda")
    hs.k_rope_kv(dev_bf16(qkv), torch.from_numpy(pos).cuda(), torch.from_numpy(slot).cuda(), rope_table(64, d),
                 q, pool, nh, d)
    torch.cuda.synchronize()
    c, s = rope_cos_sin(pos, d, 1e4)
    v = bf16_value(qkv).reshape(T, 3, nh, d)
    ref_q = rope(v[:, 0], c, s, rnd=lambda a: a)
    ref_k = rope(v[:, 1], c, s, rnd=lambda a: a)
    check_bf16(host_bits(q).reshape(T, nh, d), ref_q, max_frac=0.01)
    P = host_bits(pool)
    for t in range(T):
        blk, off = slot[t] // 16, slot[t] % 16
        check_bf16(P[blk, 0, :, off, :], ref_k[t], max_frac=0.05)
        assert np.array_equal(P[blk, 1, :, off, :], qkv.reshape(T, 3, nh, d)[t, 2])


def attention_ref(q, K, V, pos, want_scale=False):
    """Causal softmax attention (float64): q [n, nh, d] at positions pos over K, V [ctx, nh, d].
    With want_scale also returns sum_j p_j |v_j| (the magnitude of the terms)."""
    d = q.shape[-1]
    out = np.empty_like(q)
    scale = np.empty_like(q)
    for i, p in enumerate(pos):
        sc = np.einsum("hd,khd->hk", q[i], K[: p + 1]) / np.sqrt(d)
        e = np.exp(sc - sc.max(-1, keepdims=True))
        out[i] = np.einsum("hk,khd->hd", e, V[: p + 1]) / e.sum(-1)[:, None]
        scale[i] = np.einsum("hk,khd->hd", e, np.abs(V[: p + 1])) / e.sum(-1)[:, None]
    return (out, scale) if want_scale else out


@pytest.mark.parametrize("nh,d", [(4, 64), (8, 128)])
@pytest.mark.parametrize("decode", [False, True])
def test_attention_paged(nh, d, decode):
    rng = np.random.default_rng(nh + d + decode)
    lens = [37, 1, 130, 16] if not decode else [1, 1, 1, 1]
    ctxs = [37, 1, 130, 16] if not decode else [37, 1, 1100, 16]  # 1100: two 1024-token splits
    nblk, maxb = 128, 80
    free = list(rng.permutation(nblk))
    pool = np.zeros((nblk, 2, nh, 16, d), dtype=np.uint16)
    seqs, tables, qs, outs_ref, t0 = [], np.zeros((len(lens), maxb), np.int32), [], [], 0
    for i, (n, ctx) in enumerate(zip(lens, ctxs)):
        nb = (ctx + 15) // 16
        tab = [free.pop() for _ in range(nb)]
        tables[i, :nb] = tab
        K, V = rand_bf16(rng, (ctx, nh, d)), rand_bf16(rng, (ctx, nh, d))
        for p in range(ctx):
            pool[tab[p // 16], 0, :, p % 16] = K[p]
            pool[tab[p // 16], 1, :, p % 16] = V[p]
        q = rand_bf16(rng, (n, nh, d))
        pos = np.arange(ctx - n, ctx)
        outs_ref.append(attention_ref(bf16_value(q), bf16_value(K), bf16_value(V), pos, want_scale=True))
        qs.append(q)
        seqs.append([t0, n, ctx - n, i])
        t0 += n
    q = np.concatenate(qs).reshape(t0, nh * d)
    o = torch.empty((t0, nh * d), dtype=torch.bfloat16, device="cuda")
    ws = torch.empty(len(lens) * nh * 64 * (d + 2), dtype=torch.float32, device="cuda")
    hs.k_attention(dev_bf16(q), dev_bf16(pool), torch.tensor(seqs, dtype=torch.int32, device="cuda"),
                   max(lens), max(ctxs), torch.from_numpy(tables).cuda(), o, nh, d, decode, ws)
    torch.cuda.synchronize()
    ref = np.concatenate([r[0] for r in outs_ref]).reshape(t0, nh * d)
    sc = np.concatenate([r[1] for r in outs_ref]).reshape(t0, nh * d)
    check_bf16(host_bits(o), ref, max_frac=0.05, scale=sc, rel=2.0 ** -16)


def test_argmax_ties_lowest_id():
    rng = np.random.default_rng(9)
    L = rng.standard_normal((5, 32000)).astype(np.float32)
    L[1, 7] = L[1, 31999] = L[1].max() + 1  # tie: lowest id wins
    L[2, :] = 0.5                            # all equal -> 0
    L[3, 1023] = 1e30
    t = torch.empty(5, dtype=torch.int32, device="cuda")
    hs.k_argmax(torch.from_numpy(L).cuda(), t)
    torch.cuda.synchronize()
    assert t.cpu().tolist() == [int(np.argmax(r)) for r in L]
    assert t.cpu().tolist()[1:4] == [7, 0, 1023]


def test_embed_and_span_copy_bit_exact():
    rng = np.random.default_rng(11)
    E = rand_bf16(rng, (1000, 256))
    tok = rng.integers(0, 1000, 77).astype(np.int32)
    x = torch.empty((77, 256), dtype=torch.bfloat16, device="cuda")
    hs.k_embed(torch.from_numpy(tok).cuda(), dev_bf16(E), x)
    torch.cuda.synchronize()
    assert np.array_equal(host_bits(x), E[tok])
    span = 256 * 1024
    a = torch.randint(0, 255, (40 * span,), dtype=torch.uint8, device="cuda")
    b = torch.zeros_like(a)
    perm = rng.permutation(40)[:25]
    src = torch.tensor([a.data_ptr() + int(i) * span for i in perm], dtype=torch.int64, device="cuda")
    dst = torch.tensor([b.data_ptr() + int(i) * span for i in range(25)], dtype=torch.int64, device="cuda")
    hs.k_span_copy(src, dst, span)
    torch.cuda.synchronize()
    A, B = a.cpu().numpy().reshape(40, span), b.cpu().numpy().reshape(40, span)
    assert np.array_equal(B[:25], A[perm]) and not B[25:].any()


def test_tmem_a_operand_probe():
    """tcgen05.cp (smem -> TMEM) + tcgen05.mma with A from TMEM equals the shared-memory A path
    bit for bit, and both equal the fp32 reference (the A-in-TMEM staging of the decode stack's
    deep weight ring)."""
    torch.manual_seed(0)
    K = 256
    A = (torch.randn(128, K, device="cuda") * 0.1).to(torch.bfloat16)
    B = torch.randn(16, K, device="cuda").to(torch.bfloat16)
    ss, ts = hs.tmem_a_gemm(A, B)
    ref = (B.float() @ A.float().t())
    assert torch.allclose(ss, ref, rtol=1e-4, atol=1e-4), (ss - ref).abs().max()
    assert torch.equal(ss, ts), (ss - ts).abs().max()
