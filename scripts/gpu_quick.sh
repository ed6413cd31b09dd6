#!/bin/bash
# quick iteration: parity sweep, C2 bench, ncu full capture of k_assemble
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python scripts/debug_2d.py > gpurun_out/debug2d.log 2>&1; timeout 900 python scripts/gpu_check.py ${CHECK_ARGS} > gpurun_out/check.log 2>&1; echo "check rc=$?"; grep -c PASS gpurun_out/check.log; grep -A3 FAIL gpurun_out/check.log | head -30
timeout 600 python bench.py --steps 20 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
if [ -z "${NO_NCU}" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_assemble -s 5 -c 1 -f -o gpurun_out/prof_C2 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > /dev/null 2> gpurun_out/ncu.err; echo "ncu rc=$?"
fi
