#!/bin/bash
# xframe tuning round trip: parity (xframe tests), phase clocks, C2/C3 bench lines, one ncu capture
TAG=${1:-x}
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 400 python -m pytest tests/test_gpu_xframe.py -x -q > gpurun_out/t_$TAG.log 2>&1; tail -3 gpurun_out/t_$TAG.log
timeout 200 python scripts/phase_timing_x.py 32 4 2>&1 | tail -6
for c in C2 C3; do
  timeout 200 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b${TAG}_$c.json 2> gpurun_out/b${TAG}_$c.err
  python -c "import json;d=json.loads(open('gpurun_out/b${TAG}_$c.json').read().strip().splitlines()[-1]);print('$c',d['phases_ms'],d['roofline']['frac'])"
done
[ -z "$NO_NCU" ] && ncu --set full --import-source on --clock-control none -k regex:k_xh1_fill -c 1 -o gpurun_out/ncu_$TAG python bench.py --config C2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$TAG.log 2>&1; tail -1 gpurun_out/ncu_$TAG.log
