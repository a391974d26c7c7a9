#!/bin/bash
# Released-stage teardown deferred to the release point: SPMD/group GPU tests, PP4/PP2 pause breakdown x2.
mkdir -p gpurun_out/rs5
timeout 600 python -m pytest tests/test_spmd_gpu.py tests/test_group_gpu.py -q -m gpu --timeout 500 > gpurun_out/rs5/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/rs5/tests.log
for r in 1 2; do
  for n in 4 2; do
    HS_DEBUG_CONS=1 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29900 + 10 * r + n)) bench.py --gpus $n --steps 3 --warmup 3 --no-cpu-baseline \
      > gpurun_out/rs5/r${r}_$n.json 2> gpurun_out/rs5/r${r}_$n.err
    echo "run $r pp $n rc=$? $(grep -o 'HsError.*' gpurun_out/rs5/r${r}_$n.err | head -1)"
  done
done
echo done
