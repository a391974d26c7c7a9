#!/bin/bash
# round-2 GPU run 48: attn_tc nondeterminism — the same tests with programmatic dependent launch off
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build48.log 2>&1
for r in $(seq 1 20); do
  HS_ATTN_TC=1 HS_PDL=0 timeout 300 python -m pytest tests/test_group_gpu.py -q --timeout 200 -k "background_host_load or pp_split" >> gpurun_out/bg48_tc_nopdl.log 2>&1; echo "tc_nopdl rc=$?" >> gpurun_out/bg48_summary.txt
done
