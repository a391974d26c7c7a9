#!/bin/bash
# round-2 GPU run 50: final code as shipped (tcgen05 prefill attention default) — full GPU suite + smoke
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build50.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rA --timeout 900 > gpurun_out/gputest50.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest50.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke50.log 2>&1
