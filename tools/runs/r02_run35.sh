#!/bin/bash
# round-2 GPU run 35: same-box A/B: libhs_base.so (HEAD 1ad56cc) vs libhs.so (half-CTA units for batches;
# workspace sized as before for max_seqs = 1) with flags packed / one 128-byte line each (HS_DSTACK_FLAGPAD)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build35.log 2>&1
for r in 1 2; do
  HS_LIB_VARIANT=libhs_base.so timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b35_base_$r.json 2> gpurun_out/b35_base_$r.err
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b35_new_$r.json 2> gpurun_out/b35_new_$r.err
  HS_DSTACK_FLAGPAD=32 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b35_pad_$r.json 2> gpurun_out/b35_pad_$r.err
done
timeout 900 python bench.py --config 4 --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b35_c4_new.json 2> gpurun_out/b35_c4_new.err
HS_DSTACK_FLAGPAD=32 timeout 900 python bench.py --config 4 --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b35_c4_pad.json 2> gpurun_out/b35_c4_pad.err
