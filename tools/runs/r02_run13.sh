#!/bin/bash
# round-2 GPU run 13: single-pass tcgen05 prefill attention (HS_ATTN_TC=1): parity + timing A/B
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build13.log 2>&1
HS_ATTN_TC=1 python tools/attn_det.py > gpurun_out/attn_det.txt 2>&1
for i in 1 2 3; do HS_ATTN_TC=1 timeout 600 python -m pytest tests/test_group_gpu.py -q --timeout 300 -k "pp_split" >> gpurun_out/gputest13.log 2>&1; done
for V in "HS_ATTN_TC=1"; do
  echo "== prefill $V" >> gpurun_out/exp13.txt
  env $V timeout 300 python tools/prefill_prof.py 512 >> gpurun_out/exp13.txt 2>&1
  env $V timeout 300 python tools/prefill_prof.py 2048 >> gpurun_out/exp13.txt 2>&1
done
true
