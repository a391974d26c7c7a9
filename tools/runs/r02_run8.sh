#!/bin/bash
# round-2 GPU run 8: decode-stack changes (per-slot activation producer, K/V L2 prefetch): parity
# of the decode paths, traces A/B, bench N=1
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke8.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke8.log
timeout 1500 python -m pytest tests/test_group_gpu.py tests/test_fullsize_gpu.py -q -rA --timeout 1200 -k "decode_stack or tiny_layerwise or 7b_layerwise or pp_invariance or decode_steps" > gpurun_out/gputest8.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest8.log
for V in "" "HS_DSTACK_KVPF=0"; do
  echo "== $V" >> gpurun_out/exp8.txt
  env $V timeout 300 python tools/trace_dstack.py > gpurun_out/t8.txt 2>&1
  head -2 gpurun_out/t8.txt >> gpurun_out/exp8.txt
  grep -E '"(B0 qkv act|qkv published|attn flags ok|attn kv done|E attn done|B1 o act|E o done|o grid-last|B2 gu act|E gu done|B3 down act|B3 down act end|E down done|d grid-last)"' gpurun_out/t8.txt >> gpurun_out/exp8.txt
  env $V timeout 300 python tools/trace_dstack.py llama2-13b --batch 16 > gpurun_out/t8b.txt 2>&1
  head -2 gpurun_out/t8b.txt >> gpurun_out/exp8.txt
done
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench8.json 2> gpurun_out/bench8.err; echo "bench rc=$?" >> gpurun_out/bench8.err
