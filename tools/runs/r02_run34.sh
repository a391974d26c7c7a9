#!/bin/bash
# round-2 GPU run 34: same-box A/B of two builds: libhs_base.so (HEAD 1ad56cc) vs libhs.so (half-CTA
# attention units for batches, compile-time barrier ids, compiled into the batched kernels only)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for r in 1 2 3; do
  HS_LIB_VARIANT=libhs_base.so timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b34_base_$r.json 2> gpurun_out/b34_base_$r.err
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b34_new_$r.json 2> gpurun_out/b34_new_$r.err
done
HS_LIB_VARIANT=libhs_base.so timeout 900 python bench.py --config 4 --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b34_c4_base.json 2> gpurun_out/b34_c4_base.err
timeout 900 python bench.py --config 4 --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b34_c4_new.json 2> gpurun_out/b34_c4_new.err
