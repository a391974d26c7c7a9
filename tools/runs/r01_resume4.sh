#!/bin/bash
# Re-entry check of HEAD (peer-memory release after consolidation): full GPU suite, smoke, default bench, PP2/PP4 x2.
mkdir -p gpurun_out/rs4
timeout 900 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/rs4/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/rs4/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/rs4/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/rs4/bench_b1.json 2> gpurun_out/rs4/bench_b1.err; echo "bench n1 rc=$?"
for r in 1 2; do
  for n in 2 4; do
    HS_DEBUG_CONS=1 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29800 + 10 * r + n)) bench.py --gpus $n --steps 3 --warmup 3 --no-cpu-baseline \
      > gpurun_out/rs4/r${r}_$n.json 2> gpurun_out/rs4/r${r}_$n.err
    echo "run $r pp $n rc=$? $(grep -o 'HsError.*' gpurun_out/rs4/r${r}_$n.err | head -1)"
  done
done
echo done
