#!/bin/bash
# round-2 GPU run 25: early reads of the held tile's parts/residual + cached K/V read before the q/k/v flags
# (tagged o / a words removed) — full GPU suite, A/B, trace
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build25.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x -rA --timeout 1200 > gpurun_out/gputest25.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest25.log
for r in 1 2; do
  for V in 0 1; do
    HS_DSTACK_KVEARLY=$V timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/b25_kve${V}_$r.json 2> gpurun_out/b25_kve${V}_$r.err
  done
done
timeout 900 python bench.py --config 4 --gpus 1 --steps 3 --warmup 3 > gpurun_out/b25_c4.json 2> gpurun_out/b25_c4.err
HS_DSTACK_TRACE_K=0 TRACE_NPZ=gpurun_out/trace25_7b_k0.npz timeout 600 python tools/trace_dstack.py > gpurun_out/trace25_7b_k0.txt 2>&1
