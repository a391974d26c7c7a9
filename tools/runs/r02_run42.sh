#!/bin/bash
# round-2 GPU run 42: spin timeouts on SM cycles (clock64) instead of %globaltimer — full GPU
# suite twice, smoke twice, bench N=1, two-groups stress
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build42.log 2>&1
nvidia-smi -q -d CLOCK > gpurun_out/clocks42.txt 2>&1
for r in 1 2; do
  timeout 2400 python -m pytest tests -m gpu -q -rA --timeout 1200 > gpurun_out/gputest42_$r.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest42_$r.log
  timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke42_$r.log 2>&1
done
timeout 900 python bench.py > gpurun_out/bench42.json 2> gpurun_out/bench42.err
for r in 1 2; do timeout 300 python tools/stress_dstack.py --steps 600 --both > gpurun_out/st42_both$r.json 2> gpurun_out/st42_both$r.err; echo "both$r rc=$?" >> gpurun_out/st42_summary.txt; done
