#!/bin/bash
# round-2 GPU run 41: intermittent decode-stack trap (run 40) — failure records + env A/B stress
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build41.log 2>&1
timeout 900 python -m pytest tests/test_fullsize_gpu.py -q -rA --timeout 600 -k "7b and not pp8" > gpurun_out/gputest41.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest41.log
run() { tag=$1; shift; env "$@" timeout 300 python tools/stress_dstack.py --steps 400 > gpurun_out/st41_$tag.json 2> gpurun_out/st41_$tag.err; echo "$tag rc=$?" >> gpurun_out/st41_summary.txt; }
for r in 1 2 3; do run def$r HS_X=0; done
for r in 1 2; do run nopdl$r HS_PDL=0; done
for r in 1 2; do run noearly$r HS_DSTACK_EARLYPARTS=0; done
for r in 1 2; do run flag1_$r HS_DSTACK_FLAGPAD=1; done
