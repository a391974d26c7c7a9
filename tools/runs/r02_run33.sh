#!/bin/bash
# round-2 GPU run 33 (script r02_run32.sh re-run): same-box A/B of two builds: libhs_base.so (HEAD 1ad56cc) vs libhs.so (half-CTA
# attention units for batches, compile-time barrier ids)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for r in 1 2 3; do
  HS_LIB_VARIANT=libhs_base.so timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b33_base_$r.json 2> gpurun_out/b33_base_$r.err
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b33_new_$r.json 2> gpurun_out/b33_new_$r.err
done
HS_LIB_VARIANT=libhs_base.so timeout 900 python bench.py --config 4 --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b33_c4_base.json 2> gpurun_out/b33_c4_base.err
timeout 900 python bench.py --config 4 --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b33_c4_new.json 2> gpurun_out/b33_c4_new.err
