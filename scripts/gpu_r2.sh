#!/bin/bash
# round-2 iteration: selected GPU tests, C2/C3 bench lines, optional ncu of the fill
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest ${TESTS:-tests/test_gpu_xframe.py tests/test_gpu_boundary.py} -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_r2.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_r2.log | grep -E "passed|failed|Error|assert" | head -20
for cfg in ${CFGS:-C2 C3}; do
  timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 30 ${BENCH_ARGS} > gpurun_out/bench_$cfg.json 2>> gpurun_out/bench.err; echo "bench $cfg rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/bench_$cfg.json')); print('$cfg', 'value %.1f'%d['value'], 'ms %.4f'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'], 'phases', {k: round(v,4) for k,v in d['phases_ms'].items()})" 2>&1 | tail -2
done
tail -3 gpurun_out/bench.err
if [ -n "${NCU}" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_xh1_fill}" -s ${SKIP:-4} -c 1 -f -o gpurun_out/prof_${NCU} \
    python bench.py --config ${NCU} --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2> gpurun_out/ncu.err; echo "ncu rc=$?"
fi
