#!/bin/bash
# round-2 GPU run 11: tcgen05 prefill attention: op-level + layer-level parity, timing A/B
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke11.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke11.log
timeout 1200 python -m pytest tests/test_kernels_gpu.py tests/test_group_gpu.py -q -rA --timeout 600 -x -k "attention or varlen or chunked or tiny_layerwise or readiness or pp_split" > gpurun_out/gputest11.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest11.log
for V in "" "HS_ATTN_TC=0"; do
  echo "== prefill $V" >> gpurun_out/exp11.txt
  env $V timeout 300 python tools/prefill_prof.py 512 >> gpurun_out/exp11.txt 2>&1
  env $V timeout 300 python tools/prefill_prof.py 2048 >> gpurun_out/exp11.txt 2>&1
done
timeout 1200 python -m pytest tests/test_fullsize_gpu.py -q -rA --timeout 1000 -k "7b_layerwise and 1" > gpurun_out/gputest11b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest11b.log
