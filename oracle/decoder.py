"""Oracle decoder: paged-KV Llama-2 forward, pipeline-parallel partition, consolidation.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain and slow on purpose: every step
follows SURVEY §8(c)'s algorithm in the paper's order; numpy matmuls are the only library
primitive used for arithmetic.

Paper passages followed:
  * KV cache: "the key and value vectors of previous tokens remain unchanged during
    iterations ... cache these vectors"; prefill stores the prompt's KV,
    decoding "reuses the key-value cache and generates one token at a time".
  * Pipeline parallelism: "distributes a model's layers across multiple workers, with
    intermediate results transmitted sequentially between workers"; the
    hand-off is one hidden vector per token ("8 KB of inter-layer results per token",
    PAPER.md:355 -> 4096 * 2 bytes).
  * Consolidation / KV migration: "stop scheduling ... wait for all on-the-fly batches ...
    query the cache block manager to obtain the blocks that are used by existing requests,
    and then collect these blocks from all workers with a gather operation.  Blocks are
    gathered to the worker with whole model and placed at different layers, according to
    which worker it comes from."; the worker "continues to generate
    tokens with whole model while other workers are terminated".
"""
from __future__ import annotations

import heapq

import numpy as np

import hsgen

from .numerics import (argmax_lowest, bf16, bf16_bits, bf16_value, linear, rmsnorm, rmsnorm_split, rope,
                       rope_cos_sin, silu)

BLOCK = 16  # tokens per KV block (reading R6)


# ---------------------------------------------------------------- weights ------------------
class Weights:
    """Logical weights drawn by the shared generator (float64 values of bf16 draws).
    Layers are produced lazily; ``cache`` keeps them (tiny models)."""

    def __init__(self, cfg: dict, seed: int = hsgen.WEIGHT_SEED, cache: bool = True, nthreads: int = 0):
        self.cfg, self.seed, self.cache, self.nthreads = cfg, seed, cache, nthreads
        self._layers: dict[int, dict] = {}
        self._misc: dict[str, np.ndarray] = {}

    def _t(self, tid):
        return bf16_value(hsgen.tensor_bf16(self.cfg, self.seed, tid, self.nthreads))

    def layer(self, l: int) -> dict:
        if l in self._layers:
            return self._layers[l]
        T = lambda k: self._t(hsgen.layer_tensor(l, k))  # noqa: E731
        w = dict(attn_norm=T(hsgen.ATTN_NORM)[0], wq=T(hsgen.WQ), wk=T(hsgen.WK), wv=T(hsgen.WV),
                 wo=T(hsgen.WO), ffn_norm=T(hsgen.FFN_NORM)[0], wg=T(hsgen.WG), wu=T(hsgen.WU),
                 wd=T(hsgen.WD))
        if self.cache:
            self._layers[l] = w
        return w

    def _get(self, name, tid):
        if name not in self._misc:
            self._misc[name] = self._t(tid)
        return self._misc[name]

    def embed_rows(self, tokens) -> np.ndarray:
        """x[t] = E[tok_t] (the model takes a sequence of tokens)."""
        H = self.cfg["hidden"]
        if self.cfg["vocab"] * H <= (1 << 24):
            return self._get("embed", hsgen.EMBED)[np.asarray(tokens)]
        out = np.empty((len(tokens), H), dtype=np.uint16)
        L = hsgen.lib()
        c = hsgen.cfg_struct(self.cfg)
        import ctypes as C
        for i, t in enumerate(tokens):
            L.hsgen_tensor_bf16(C.byref(c), self.seed, hsgen.EMBED, int(t) * H, H,
                                out[i].ctypes.data, 1)
        return bf16_value(out)

    def final_norm(self):
        return self._get("final_norm", hsgen.FINAL_NORM)[0]

    def lm_head(self):
        return self._get("lm_head", hsgen.LM_HEAD)


def layer_param_bytes(cfg) -> int:
    H, F = cfg["hidden"], cfg["ffn"]
    return 2 * (2 * H + 4 * H * H + 3 * F * H)


def embed_param_bytes(cfg) -> int:
    return 2 * cfg["vocab"] * cfg["hidden"]


def final_param_bytes(cfg) -> int:
    return 2 * (cfg["hidden"] + cfg["vocab"] * cfg["hidden"])


def kv_block_bytes(cfg) -> int:
    """One 16-token block of one layer: K and V, all heads: 16 * 2 * H * 2 bytes."""
    return BLOCK * 2 * cfg["n_heads"] * cfg["head_dim"] * 2


# ---------------------------------------------------------------- block manager ------------
class BlockManager:
    """Centralised cache block manager ("query the cache block manager").
    Blocks of 16 tokens, lowest free id first; the same ids serve every stage's layers."""

    def __init__(self, num_blocks: int):
        self.free = list(range(num_blocks))
        heapq.heapify(self.free)
        self.tables: dict[int, list[int]] = {}
        self.ctx: dict[int, int] = {}

    def append(self, seq: int, n_new: int) -> list[tuple[int, int]]:
        """Reserve slots for n_new tokens of seq; returns (block, offset) per new token."""
        tab = self.tables.setdefault(seq, [])
        c0 = self.ctx.get(seq, 0)
        out = []
        for p in range(c0, c0 + n_new):
            if p // BLOCK >= len(tab):
                if not self.free:
                    raise MemoryError("KV blocks exhausted")
                tab.append(heapq.heappop(self.free))
            out.append((tab[p // BLOCK], p % BLOCK))
        self.ctx[seq] = c0 + n_new
        return out

    def release(self, seq: int):
        for b in self.tables.pop(seq, []):
            heapq.heappush(self.free, b)
        self.ctx.pop(seq, None)

    def slot(self, seq: int, pos: int) -> tuple[int, int]:
        return self.tables[seq][pos // BLOCK], pos % BLOCK


# ---------------------------------------------------------------- worker -------------------
class Worker:
    """One pipeline stage: owns layers [b, e) and their KV pools
    (pool[l] : [num_blocks, 2 (K|V), n_heads, 16, head_dim] bf16 bits)."""

    def __init__(self, cfg, weights: Weights, b: int, e: int, num_blocks: int, rnd=bf16, acc=np.float64):
        self.cfg, self.w, self.rnd = cfg, weights, rnd
        self.lin = (lambda x, W: linear(x, W, acc))
        self.layers = list(range(b, e))
        self.num_blocks = num_blocks
        nh, d = cfg["n_heads"], cfg["head_dim"]
        self.kv = {l: np.zeros((num_blocks, 2, nh, BLOCK, d), dtype=np.uint16) for l in self.layers}
        self.is_first = b == 0
        self.is_last = e == cfg["n_layers"]

    def add_layers(self, layers):
        nh, d = self.cfg["n_heads"], self.cfg["head_dim"]
        for l in layers:
            if l not in self.kv:
                self.kv[l] = np.zeros((self.num_blocks, 2, nh, BLOCK, d), dtype=np.uint16)
        self.layers = sorted(set(self.layers) | set(layers))
        self.is_first = 0 in self.layers
        self.is_last = self.cfg["n_layers"] - 1 in self.layers

    def layer_forward(self, l: int, x: np.ndarray, batch, trace: dict | None = None) -> np.ndarray:
        """One decoder layer over the packed tokens of ``batch`` (list of (seq, positions,
        slots, table) per sequence, in packing order).  x: float64 bf16 values [T, H].
        ``trace`` (optional dict) receives the layer's materialised intermediates (n, q', k', v,
        o, h, n2, a) for the layer-level parity tests' error bounds; it changes nothing."""
        h = self.attention_half(l, x, batch, trace)                                # steps 4.1-4.6
        return self.mlp_half(l, h, trace)                                            # steps 4.7-4.9

    def attention_half(self, l: int, x: np.ndarray, batch, trace: dict | None = None) -> np.ndarray:
        """Steps 4.1-4.6 of layer l: h = x + Attention(RMSNorm(x)) W_o^T (writes the batch's
        K/V into the layer's pool)."""
        cfg, rnd, W = self.cfg, self.rnd, self.w.layer(l)
        nh, d, eps = cfg["n_heads"], cfg["head_dim"], cfg["rms_eps"]
        T = x.shape[0]
        n, r = rmsnorm_split(x, W["attn_norm"], eps, rnd)                          # step 4.1 (R10b)
        q = rnd(r * self.lin(n, W["wq"])).reshape(T, nh, d)                           # step 4.2
        k = rnd(r * self.lin(n, W["wk"])).reshape(T, nh, d)
        v = rnd(r * self.lin(n, W["wv"])).reshape(T, nh, d)
        pos = np.concatenate([np.asarray(p) for (_, p, _, _) in batch])
        c, s = rope_cos_sin(pos, d, cfg["rope_theta"], table_f32=rnd is bf16)      # step 4.3
        q, k = rope(q, c, s, rnd), rope(k, c, s, rnd)
        pool = self.kv[l]
        t0 = 0
        o = np.empty((T, nh, d))
        for (seq, p, slots, table) in batch:                                        # step 4.4
            m = len(p)
            for i, (blk, off) in enumerate(slots):
                pool[blk, 0, :, off, :] = bf16_bits(k[t0 + i]) if rnd is bf16 else 0
                pool[blk, 1, :, off, :] = bf16_bits(v[t0 + i]) if rnd is bf16 else 0
            # visible keys: positions 0 .. max(p) of this sequence, read through the table
            n_keys = int(p[-1]) + 1
            if rnd is bf16:
                Kc = np.empty((n_keys, nh, d))
                Vc = np.empty((n_keys, nh, d))
                for j in range(n_keys):
                    blk, off = table[j // BLOCK], j % BLOCK
                    Kc[j] = bf16_value(pool[blk, 0, :, off, :])
                    Vc[j] = bf16_value(pool[blk, 1, :, off, :])
            else:  # exact mode keeps an unrounded dense cache per sequence
                cache = self._exact_cache.setdefault((l, seq), {})
                for i in range(m):
                    cache[int(p[i])] = (k[t0 + i], v[t0 + i])
                Kc = np.stack([cache[j][0] for j in range(n_keys)])
                Vc = np.stack([cache[j][1] for j in range(n_keys)])
            # step 4.5: causal softmax attention, query at position p sees keys 0..p
            sc = np.einsum("thd,khd->htk", q[t0:t0 + m], Kc) / np.sqrt(d)
            mask = np.arange(n_keys)[None, :] > np.asarray(p)[:, None]
            sc = np.where(mask[None], -np.inf, sc)
            mx = sc.max(axis=-1, keepdims=True)
            e = np.exp(sc - mx)
            o[t0:t0 + m] = rnd(np.einsum("htk,khd->thd", e, Vc) / e.sum(axis=-1).T[:, :, None])
            t0 += m
        h = rnd(x + self.lin(o.reshape(T, nh * d), W["wo"]))                          # step 4.6
        if trace is not None:
            trace.update(n=n, q=q, k=k, v=v, o=o, h=h)
        return h

    def mlp_half(self, l: int, h: np.ndarray, trace: dict | None = None) -> np.ndarray:
        """Steps 4.7-4.9 of layer l: x' = h + (silu(n2 W_g^T) * (n2 W_u^T)) W_d^T, n2 = RMSNorm(h)
        (as r2 (h * w) W^T: reading R10b)."""
        rnd, W = self.rnd, self.w.layer(l)
        n2, r2 = rmsnorm_split(h, W["ffn_norm"], self.cfg["rms_eps"], rnd)         # step 4.7
        a = rnd(silu(r2 * self.lin(n2, W["wg"])) * (r2 * self.lin(n2, W["wu"])))      # step 4.8
        out = rnd(h + self.lin(a, W["wd"]))                                           # step 4.9
        if trace is not None:
            trace.update(n2=n2, a=a, out=out)
        return out

    _exact_cache: dict = {}

    def forward(self, x, batch):
        for l in self.layers:
            x = self.layer_forward(l, x, batch)
        return x

    def head(self, x_last: np.ndarray) -> np.ndarray:
        """Final RMSNorm + lm_head -> float64 logits (unrounded)."""
        nf = rmsnorm(x_last, self.w.final_norm(), self.cfg["rms_eps"], self.rnd)
        return self.lin(nf, self.w.lm_head())


# ---------------------------------------------------------------- group --------------------
def split_layers(n_layers: int, pp: int) -> list[tuple[int, int]]:
    """Contiguous ranges, floor(L/pp) layers each, remainder to the earliest stages
    (reading R2; "partitions LLM layers across servers")."""
    base, rem = divmod(n_layers, pp)
    out, b = [], 0
    for k in range(pp):
        e = b + base + (1 if k < rem else 0)
        out.append((b, e))
        b = e
    return out


class Group:
    """A pipeline-parallel worker group over stage ranges; stage k runs after stage k-1 and
    receives a byte copy of its hidden states."""

    def __init__(self, cfg: dict, weights: Weights | None = None, pp: int = 1,
                 ranges=None, num_blocks: int = 256, rnd=bf16, acc=np.float64):
        self.cfg = cfg
        self.w = weights or Weights(cfg)
        self.ranges = ranges or split_layers(cfg["n_layers"], pp)
        self.workers = [Worker(cfg, self.w, b, e, num_blocks, rnd, acc) for (b, e) in self.ranges]
        self.bm = BlockManager(num_blocks)
        self.rnd = rnd
        self.handoff_bytes = 0
        Worker._exact_cache = {}

    def _run(self, seq_ids, toks_per_seq):
        batch, tokens = [], []
        for sid, toks in zip(seq_ids, toks_per_seq):
            c0 = self.bm.ctx.get(sid, 0)
            slots = self.bm.append(sid, len(toks))
            batch.append((sid, np.arange(c0, c0 + len(toks)), slots, self.bm.tables[sid]))
            tokens.extend(int(t) for t in toks)
        x = self.w.embed_rows(tokens)                                   # stage 0 (a5)
        for k, wk in enumerate(self.workers):
            if k > 0:  # hand-off: one bf16 hidden vector per token, a byte copy
                bits = bf16_bits(x) if self.rnd is bf16 else None
                self.handoff_bytes += x.shape[0] * x.shape[1] * 2
                x = bf16_value(bits.copy()) if bits is not None else x.copy()
            x = wk.forward(x, batch)
        last = np.cumsum([len(t) for t in toks_per_seq]) - 1
        logits = self.workers[-1].head(x[last])                          # last stage (a14)
        return [argmax_lowest(r) for r in logits], logits               # (a15)

    def prefill(self, seq_ids, prompts):
        for s in seq_ids:
            if s in self.bm.tables:
                raise ValueError("sequence already live")
        return self._run(seq_ids, prompts)

    def decode(self, seq_ids, in_tokens):
        return self._run(seq_ids, [[t] for t in in_tokens])

    def release(self, seq_id):
        self.bm.release(seq_id)

    def owner(self, layer: int) -> Worker:
        for wk in self.workers:
            if layer in wk.layers:
                return wk
        raise KeyError(layer)

    def read_kv(self, seq: int, layer: int, pos0: int, n: int) -> np.ndarray:
        """[n, 2, n_heads, head_dim] bf16 bits of positions pos0.. of seq at layer."""
        pool = self.owner(layer).kv[layer]
        out = []
        for p in range(pos0, pos0 + n):
            blk, off = self.bm.slot(seq, p)
            out.append(pool[blk, :, :, off, :])
        return np.stack(out)

    def consolidate(self, target: int):
        """Scale down to ``target``: gather every other stage's layers (weights + the used KV
        blocks of live sequences, same block ids) into it; returns (weight_bytes, kv_bytes)."""
        cfg = self.cfg
        tgt = self.workers[target]
        moved = [l for l in range(cfg["n_layers"]) if l not in tgt.layers]
        wbytes = len(moved) * layer_param_bytes(cfg)
        if not tgt.is_first:
            wbytes += embed_param_bytes(cfg)
        if not tgt.is_last:
            wbytes += final_param_bytes(cfg)
        kvb = 0
        srcs = {l: self.owner(l) for l in moved}
        tgt.add_layers(moved)
        for l in moved:
            for seq, table in self.bm.tables.items():
                for blk in table:                      # pool_tau[l][b] <- pool_owner(l)[l][b]
                    tgt.kv[l][blk] = srcs[l].kv[l][blk]
                    kvb += kv_block_bytes(cfg)
        self.workers = [tgt]
        self.ranges = [(0, cfg["n_layers"])]
        return wbytes, kvb

    def scale_up(self, owner: dict):
        """Scale up ("converting all cold-start workers into individual serving
        endpoints"): every worker becomes a standalone endpoint holding the whole model; live
        sequence s continues on endpoint owner[s], and its KV blocks of the layers that endpoint
        did not hold are gathered from their owners at the same block ids.
        Returns (endpoints, weight_bytes, kv_bytes): endpoint k is a one-worker Group whose block
        manager holds only its sequences (the other blocks are free).  Consumes this group."""
        cfg = self.cfg
        L = cfg["n_layers"]
        srcs = {l: self.owner(l) for l in range(L)}
        live = sorted(self.bm.tables)
        eps, wbytes, kvb = [], 0, 0
        for k, wk in enumerate(self.workers):
            have = set(wk.layers)
            moved = [l for l in range(L) if l not in have]
            wbytes += len(moved) * layer_param_bytes(cfg)
            if not wk.is_first:
                wbytes += embed_param_bytes(cfg)
            if not wk.is_last:
                wbytes += final_param_bytes(cfg)
            mine = [sq for sq in live if owner[sq] == k]
            e = Group.__new__(Group)
            e.cfg, e.w, e.rnd, e.handoff_bytes = cfg, self.w, self.rnd, 0
            e.ranges = [(0, L)]
            ew = Worker(cfg, self.w, 0, L, wk.num_blocks, self.rnd)
            ew.lin = wk.lin
            for l in range(L):
                if l in have:                          # its own layers: the pools as they are
                    ew.kv[l] = wk.kv[l].copy()
                else:                                  # pool_k[l][b] <- pool_owner(l)[l][b]
                    for sq in mine:
                        for blk in self.bm.tables[sq]:
                            ew.kv[l][blk] = srcs[l].kv[l][blk]
                            kvb += kv_block_bytes(cfg)
            e.workers = [ew]
            bm = BlockManager(wk.num_blocks)
            used = set()
            for sq in mine:
                bm.tables[sq] = list(self.bm.tables[sq])
                bm.ctx[sq] = self.bm.ctx[sq]
                used |= set(bm.tables[sq])
            bm.free = [b for b in range(wk.num_blocks) if b not in used]
            heapq.heapify(bm.free)
            e.bm = bm
            eps.append(e)
        self.workers = []
        return eps, wbytes, kvb
