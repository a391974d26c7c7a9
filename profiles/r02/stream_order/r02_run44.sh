#!/bin/bash
# round-2 GPU run 44: the stream-order regression test against the fixed library and against
# the build before the fix (libhs_prefix.so = 23ce69d; expected to fail there)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build44.log 2>&1
for r in 1 2; do
  timeout 900 python -m pytest tests/test_group_gpu.py -q -rA --timeout 600 -k "stream_order" > gpurun_out/gputest44_fixed_$r.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest44_fixed_$r.log
  HS_LIB_VARIANT=libhs_prefix.so timeout 900 python -m pytest tests/test_group_gpu.py -q -rA --timeout 600 -k "stream_order" > gpurun_out/gputest44_prefix_$r.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest44_prefix_$r.log
done
timeout 2400 python -m pytest tests -m gpu -q -rA --timeout 1200 > gpurun_out/gputest44_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest44_full.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke44.log 2>&1
