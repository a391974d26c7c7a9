#!/bin/bash
# round-2 GPU run 16: full regression (smoke, every GPU test, bench N=1)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke16.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke16.log
timeout 2700 python -m pytest tests -m gpu -q -rA --timeout 1500 > gpurun_out/gputest16.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest16.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench16.json 2> gpurun_out/bench16.err; echo "bench rc=$?" >> gpurun_out/bench16.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench16_ref.json 2> gpurun_out/bench16_ref.err; echo "ref rc=$?" >> gpurun_out/bench16_ref.err
