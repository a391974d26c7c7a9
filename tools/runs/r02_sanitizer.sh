#!/bin/bash
# compute-sanitizer, ONE tool per gpurun call (B200_PROFILING.md): bash tools/r02_sanitizer.sh memcheck|racecheck|synccheck
# over the tiny config-1 smoke: prefill kernels, the decode stack (cooperative, flag-polling),
# stage hand-off, consolidation copy list.  Log: gpurun_out/sanitizer_<tool>_smoke.log
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=$1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_plain.log 2>&1 &&
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $T --error-exitcode 9 --print-limit 50 \
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_${T}_smoke.log 2>&1
echo "exit=$?" >> gpurun_out/sanitizer_${T}_smoke.log
