#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the tiny config-1 smoke (prefill
# kernels, the decode stack, hand-off, consolidation copy list) and the chunked-prefill +
# pipelined-decode tests; logs under gpurun_out/sanitizer_*.log
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for T in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $T --error-exitcode 9 --print-limit 50 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_${T}_smoke.log 2>&1
  echo "exit=$?" >> gpurun_out/sanitizer_${T}_smoke.log
done
timeout 1500 $CS --tool memcheck --error-exitcode 9 --print-limit 50 python -m pytest tests/test_group_gpu.py -q -x -k "decode_steps_micro_batched_equals_stepwise and 2-8-2 or chunked_prefill_layerwise and True or consolidation_bit_exact and 2-0" > gpurun_out/sanitizer_memcheck_tests.log 2>&1
echo "exit=$?" >> gpurun_out/sanitizer_memcheck_tests.log
