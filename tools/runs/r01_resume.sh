#!/bin/bash
# Resume-session check on one 4-GPU box: GPU tests, bench N=1/2/4, config 4, consolidation repro loop.
mkdir -p gpurun_out/rs
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/rs/smi.txt
timeout 900 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/rs/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/rs/tests.log
timeout 600 python bench.py > gpurun_out/rs/b1.json 2> gpurun_out/rs/b1.err; echo "b1 rc=$?"
for n in 2 4; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$n bench.py --gpus $n --steps 3 --warmup 2 > gpurun_out/rs/pp$n.json 2> gpurun_out/rs/pp$n.err; echo "pp$n rc=$?"; done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29539 bench.py --gpus 4 --config 4 --steps 2 --warmup 1 > gpurun_out/rs/c4.json 2> gpurun_out/rs/c4.err; echo "c4 rc=$?"
bash tools/cons_race4.sh
echo done
