"""CPU oracle for the HydraServe cold-start data path (arXiv 2502.15524).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product path
(``paper_2502_15524_b200``) never imports it and shares no code with it; the only common
dependency is the seeded input generator ``hsgen`` (random draws + image byte layout, no
arithmetic of the method).

What it computes (the plain definition — the method "reaches exactly the unpartitioned
model's result"):
  * ``numerics``  — bf16 rounding, RMSNorm, Linear, RoPE, causal softmax attention, SiLU
                    (Llama-2 decoder; PAPER.md:817 names the Llama2 series), evaluated in
                    float64 with bf16 rounding at the points DESIGN.md "Numerics contract"
                    fixes.
  * ``decoder``   — a decoder forward over a paged KV cache ("the key and value vectors of
                    previous tokens remain unchanged ... cache these vectors", PAPER.md:127-
                    130), a pipeline-parallel wrapper whose stages own contiguous layer
                    ranges and hand over one hidden vector per token ("distributes a model's
                    layers across multiple workers, with intermediate results transmitted
                    sequentially"; "8 KB of inter-layer results per token",
                    PAPER.md:355), and scale-down consolidation ("migrate all existing
                    requests to that worker along with their key-value cache", PAPER.md:
                    602-606; "Blocks are gathered to the worker with whole model and placed
                    at different layers, according to which worker it comes from",
                    PAPER.md:633-634) and scale-up (every worker becomes an endpoint,
                    PAPER.md:608-612).  ``Worker.attention_half`` / ``mlp_half`` are the two
                    halves of ``layer_forward`` (the layer-level parity harness feeds each the
                    GPU's own input).
  * ``plan``      — stage planning: contiguous layer split, stage byte counts, the paper's
                    predictors Eq. 1, Eq. 2, Eq. 5
                    (PAPER.md:579-584), server selection, Algorithm 1
                    (PAPER.md:424-452), the Eq. 3 / Eq. 4 contention registry (PAPER.md:
                    469-502) and the contention-aware placement of a cold start (R20).

Pins (tests/test_oracle_*.py, test_placement.py, test_layerwise_harness.py): HF transformers'
Llama in float64 (architecture), torch fp64 library routines, closed forms, brute-force dense
recompute, PP-split == unsplit, consolidation and scale-up == the single worker, the paper's
printed sizes (12.5 GB / 24.2 GB, 8 KB/token), SPEC.md's worked predictor and Eq. 3/4 values,
an exhaustive Alg. 1.  ``place_cold_start`` is our reading R20 written out step by step: pinned
through its parts (Alg. 1's selection and Eq. 3/4, both pinned) and hand-checkable cases (a
burst on equal links), not by a value the paper prints.
"""
