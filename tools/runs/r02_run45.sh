#!/bin/bash
# round-2 GPU run 45: is the run-43 background-load mismatch the tcgen05 prefill attention?
# the test 12x with each attention kernel, then the full GPU suite twice more (final code)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build45.log 2>&1
for r in $(seq 1 12); do
  HS_ATTN_TC=1 timeout 300 python -m pytest tests/test_group_gpu.py -q --timeout 200 -k "background_host_load or pp_split" >> gpurun_out/bg45_tc.log 2>&1; echo "tc rc=$?" >> gpurun_out/bg45_summary.txt
  timeout 300 python -m pytest tests/test_group_gpu.py -q --timeout 200 -k "background_host_load or pp_split" >> gpurun_out/bg45_mma.log 2>&1; echo "mma rc=$?" >> gpurun_out/bg45_summary.txt
done
for r in 1 2; do
  timeout 2400 python -m pytest tests -m gpu -q -rA --timeout 1200 > gpurun_out/gputest45_$r.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest45_$r.log
done
