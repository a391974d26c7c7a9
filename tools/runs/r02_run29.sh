#!/bin/bash
# round-2 GPU run 29: flag-poll back-off A/B of the decode stack (B=1 and 13B B=16)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build29.log 2>&1
for r in 1 2; do
  for B in 64 128 256 512; do
    HS_DSTACK_BACKOFF=$B timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b29_bo${B}_$r.json 2> gpurun_out/b29_bo${B}_$r.err
  done
done
for B in 64 256; do
  HS_DSTACK_BACKOFF=$B timeout 900 python bench.py --config 4 --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b29_c4_bo$B.json 2> gpurun_out/b29_c4_bo$B.err
done
