#!/bin/bash
# Config 4 with the consolidation pause split into list / copy / barrier.
mkdir -p gpurun_out/rs8
HS_DEBUG_CONS=1 timeout 700 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29539 \
  bench.py --gpus 4 --config 4 --steps 3 --warmup 3 > gpurun_out/rs8/c4.json 2> gpurun_out/rs8/c4.err; echo "c4 rc=$?"
echo done
