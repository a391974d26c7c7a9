#!/bin/bash
# round-2 GPU run 13: single-pass tcgen05 prefill attention (HS_ATTN_TC=1): parity + timing A/B
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build13.log 2>&1
HS_ATTN_TC=1 timeout 1200 python -m pytest tests/test_kernels_gpu.py tests/test_group_gpu.py -q -rA --timeout 600 -x -k "attention or varlen or chunked or tiny_layerwise or readiness or pp_split" > gpurun_out/gputest13.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest13.log
for V in "HS_ATTN_TC=1" "HS_ATTN_TC=0"; do
  echo "== prefill $V" >> gpurun_out/exp13.txt
  env $V timeout 300 python tools/prefill_prof.py 512 >> gpurun_out/exp13.txt 2>&1
  env $V timeout 300 python tools/prefill_prof.py 2048 >> gpurun_out/exp13.txt 2>&1
done
true
