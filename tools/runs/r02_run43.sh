#!/bin/bash
# round-2 GPU run 43: tcgen05 prefill attention as the default — full GPU suite twice, smoke,
# bench N=1, two-groups decode stress
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build43.log 2>&1
for r in 1 2; do
  timeout 2400 python -m pytest tests -m gpu -q -rA --timeout 1200 > gpurun_out/gputest43_$r.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest43_$r.log
done
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke43.log 2>&1
timeout 900 python bench.py > gpurun_out/bench43.json 2> gpurun_out/bench43.err
timeout 300 python tools/stress_dstack.py --steps 600 --both > gpurun_out/st43_both.json 2> gpurun_out/st43_both.err; echo "both rc=$?" >> gpurun_out/st43_summary.txt
