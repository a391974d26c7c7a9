#!/bin/bash
# round-2 GPU run 47: tcgen05 prefill attention with Q read through L2 (__ldcg) instead of the
# non-coherent path — the PP-split / background-load tests in 30 processes with HS_ATTN_TC=1
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build47.log 2>&1
for r in $(seq 1 30); do
  HS_ATTN_TC=1 timeout 300 python -m pytest tests/test_group_gpu.py -q --timeout 200 -k "background_host_load or pp_split" >> gpurun_out/bg47_tc.log 2>&1; echo "tc rc=$?" >> gpurun_out/bg47_summary.txt
done
