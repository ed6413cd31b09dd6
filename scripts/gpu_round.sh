#!/bin/bash
# One GPU session: parity tests, bench, ncu launch list + full capture of the dominant kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/nvsmi.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json
for cfg in ${EXTRA_CFGS}; do
  timeout 600 python bench.py --config $cfg --no-cpu-baseline > gpurun_out/bench_$cfg.json 2>> gpurun_out/bench.err; echo "bench $cfg rc=$?"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>> gpurun_out/ncu.err; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_assemble|k_merge_rows|k_xh1_fill" -s 3 -c 2 -f -o gpurun_out/prof_c2 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>> gpurun_out/ncu.err; echo "ncu full rc=$?"
