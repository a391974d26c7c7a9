#!/bin/bash
# round-2 GPU run 40: robustness of the final code — the full GPU suite twice more, smoke twice
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build40.log 2>&1
for r in 1 2; do
  timeout 2400 python -m pytest tests -m gpu -q -rA --timeout 1200 > gpurun_out/gputest40_$r.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest40_$r.log
  timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke40_$r.log 2>&1
done
