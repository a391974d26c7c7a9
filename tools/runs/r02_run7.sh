#!/bin/bash
# round-2 GPU run 7 (tiled weight layout): full GPU suite, bench N=1, decode-stack trace
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke7.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke7.log
timeout 2400 python -m pytest tests -m gpu -q -rA --timeout 1500 > gpurun_out/gputest7.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest7.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench7.json 2> gpurun_out/bench7.err; echo "bench rc=$?" >> gpurun_out/bench7.err
timeout 300 python tools/trace_dstack.py > gpurun_out/trace7b_tiled.txt 2>&1
timeout 300 python tools/trace_dstack.py llama2-13b --batch 16 > gpurun_out/trace13b_b16_tiled.txt 2>&1
