#!/bin/bash
# After the collective-destroy fix: SPMD GPU tests, PP2/PP4 repeat loop with the consolidation breakdown.
mkdir -p gpurun_out/rs3
timeout 900 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/rs3/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/rs3/tests.log
for r in 1 2 3 4 5; do
  for n in 2 4; do
    HS_DEBUG_CONS=1 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29700 + 10 * r + n)) bench.py --gpus $n --steps 3 --warmup 2 --decode-steps 16 --no-cpu-baseline \
      > gpurun_out/rs3/r${r}_$n.json 2> gpurun_out/rs3/r${r}_$n.err
    echo "run $r pp $n rc=$? $(grep -o 'HsError.*' gpurun_out/rs3/r${r}_$n.err | head -1)"
  done
done
echo done
