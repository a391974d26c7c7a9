#!/bin/bash
# Final check of HEAD: full GPU suite, smoke, default bench.
mkdir -p gpurun_out/rs6
timeout 900 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/rs6/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/rs6/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/rs6/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/rs6/bench_b1.json 2> gpurun_out/rs6/bench_b1.err; echo "bench n1 rc=$?"
echo done
