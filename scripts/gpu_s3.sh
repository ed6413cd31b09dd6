#!/bin/bash
# round-2 session-3 baseline: smoke, GPU tests, C4 bench on both ND paths, ncu of the ND xv fill
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
if [ -z "${NO_TESTS}" ]; then
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
fi
for v in 0 1; do
LOR_XV_ND=$v timeout 600 python bench.py --config C4 --steps 10 --no-cpu-baseline --no-e2e --no-reassembly > gpurun_out/c4_$v.json 2>gpurun_out/c4_$v.err; echo "c4 xv=$v rc=$?"
python -c "import json; d=json.load(open('gpurun_out/c4_$v.json')); print('xv=$v', d['ms_per_step'], d['phases_ms'], d['roofline']['frac'])"
done
LOR_XV_ND=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_xv_fill" -s 1 -c 1 -f -o gpurun_out/prof_nd \
  python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-reassembly > /dev/null 2> gpurun_out/ncu.err; echo "ncu rc=$?"
