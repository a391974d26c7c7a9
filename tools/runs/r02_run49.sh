#!/bin/bash
# round-2 GPU run 49: attn_tc with griddepcontrol.wait before the metadata reads — the PP-split /
# background-load tests in 30 processes with HS_ATTN_TC=1, then the full GPU suite with it
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build49.log 2>&1
for r in $(seq 1 30); do
  HS_ATTN_TC=1 timeout 300 python -m pytest tests/test_group_gpu.py -q --timeout 200 -k "background_host_load or pp_split" >> gpurun_out/bg49_tc.log 2>&1; echo "tc rc=$?" >> gpurun_out/bg49_summary.txt
done
HS_ATTN_TC=1 timeout 2400 python -m pytest tests -m gpu -q -rA --timeout 1200 > gpurun_out/gputest49_tc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest49_tc.log
HS_ATTN_TC=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench49_tc.json 2> gpurun_out/bench49_tc.err
