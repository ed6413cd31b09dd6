#!/bin/bash
# End-of-round GPU session: smoke, parity tests, bench lines (C2 default + C3/C4/C5), reference arm,
# ncu launch list of the default bench, ncu --set full captures of the timed-step kernels.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/nvsmi.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json
for cfg in ${EXTRA_CFGS}; do
  timeout 600 python bench.py --config $cfg --no-cpu-baseline > gpurun_out/bench_$cfg.json 2>> gpurun_out/bench.err; echo "bench $cfg rc=$?"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>> gpurun_out/ncu.err; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_xh1_fill -s 2 -c 1 -f -o gpurun_out/prof_C2 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>> gpurun_out/ncu.err; echo "ncu C2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_xh1_fill -s 2 -c 1 -f -o gpurun_out/prof_C3 \
  python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>> gpurun_out/ncu.err; echo "ncu C3 rc=$?"
for sp in 1 2; do
  cfg=$([ $sp = 1 ] && echo C4 || echo C5)
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"_ZN4lorb10k_assembleILi3ELi${sp}E|k_merge_rows" -s 3 -c 2 -f -o gpurun_out/prof_$cfg \
    python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>> gpurun_out/ncu.err; echo "ncu $cfg rc=$?"
done
