#!/bin/bash
# round-2 GPU run 4: decode_steps fix check, decode-stack A/B experiments
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_group_gpu.py -q -rA --timeout 300 -k "decode_steps or prefetch" > gpurun_out/gputest4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest4.log
for V in "" "HS_DSTACK_NOMMA=1" "HS_DSTACK_L2AHEAD=8" "HS_DSTACK_L2AHEAD=24" "HS_DSTACK_BACKOFF=64" "HS_DSTACK_BACKOFF=1024"; do
  echo "== $V" >> gpurun_out/exp4.txt
  env $V timeout 300 python tools/trace_dstack.py > gpurun_out/t4.txt 2>&1
  head -2 gpurun_out/t4.txt >> gpurun_out/exp4.txt
  grep -E '"(B0 qkv act|qkv published|attn flags ok|E attn done|B1 o act|E o done|o grid-last|B2 gu act|E gu done|B3 down act|B3 down act end|E down done|d grid-last)"' gpurun_out/t4.txt >> gpurun_out/exp4.txt
done
