#!/bin/bash
# iteration loop: parity sweep, phase timing, C2 bench, ncu capture of k_assemble
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python scripts/gpu_check.py ${CHECK_ARGS} > gpurun_out/check.log 2>&1; echo "check rc=$?"; grep -c PASS gpurun_out/check.log; grep -A3 FAIL gpurun_out/check.log | head -30
LOR_PHASE_TIMING=1 timeout 300 python scripts/phase_timing.py 32 4 h1 2>&1 | tail -9
timeout 600 python bench.py --steps 20 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('value', d['value'], 'k_assemble ms', d['roofline']['avg_launch_ms'], 'frac', d['roofline']['frac'], 'phases', d['phases_ms'], 'e2e', d['e2e']['value'])"
tail -3 gpurun_out/bench.err
if [ -z "${NO_NCU}" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_assemble -s 5 -c 1 -f -o gpurun_out/prof_C2 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > /dev/null 2> gpurun_out/ncu.err; echo "ncu rc=$?"
fi
