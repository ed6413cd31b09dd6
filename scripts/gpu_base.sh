#!/bin/bash
# quick state check: smoke, gpu tests, C2..C5 bench lines
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/nvsmi.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
for cfg in ${CFGS:-C2}; do
  timeout 600 python bench.py --config $cfg --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_$cfg.json 2>> gpurun_out/bench.err; echo "bench $cfg rc=$?"
  cat gpurun_out/bench_$cfg.json | cut -c1-600
done
