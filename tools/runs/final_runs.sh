set -x
timeout 900 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/final_tests.log 2>&1; tail -2 gpurun_out/final_tests.log
timeout 600 python bench.py > gpurun_out/final_b1.json 2> gpurun_out/final_b1.err
for n in 2 4; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$n bench.py --gpus $n --steps 3 --warmup 2 > gpurun_out/final_pp$n.json 2> gpurun_out/final_pp$n.err; done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29529 bench.py --gpus 4 --config 4 --steps 2 --warmup 1 > gpurun_out/final_c4.json 2> gpurun_out/final_c4.err
timeout 900 python bench.py --config 5 > gpurun_out/final_c5.json 2> gpurun_out/final_c5.err
echo done
