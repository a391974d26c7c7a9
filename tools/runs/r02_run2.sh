#!/bin/bash
# round-2 GPU run 2: full-size parity, bench, decode-stack trace with L2 prefetch distances
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build2.log 2>&1
timeout 1500 python -m pytest tests/test_fullsize_gpu.py -q -rA --timeout 1400 > gpurun_out/fullsize2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/fullsize2.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "bench rc=$?" >> gpurun_out/bench2.err
for A in 0 8 16 32 64; do
  HS_DSTACK_L2AHEAD=$A timeout 300 python tools/trace_dstack.py > gpurun_out/trace7b_ahead$A.txt 2>&1
done
for A in 0 16 32; do
  HS_DSTACK_L2AHEAD=$A timeout 300 python tools/trace_dstack.py llama2-13b --batch 16 > gpurun_out/trace13b_b16_ahead$A.txt 2>&1
done
