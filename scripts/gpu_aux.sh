#!/bin/bash
# post-assembly steps (NEXT-1 A3 layout + A4, NEXT-2 coordinate vectors): bench lines + DRAM bytes
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r02_v3}
for cfg in ${CFGS:-C2-A4 C4-A4 C5-A4 C2-X}; do
  timeout 600 python bench.py --config $cfg > gpurun_out/bench_${TAG}_$cfg.json 2>> gpurun_out/bench_aux.err; echo "bench $cfg rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_$cfg.json')); print('$cfg', round(d['value'],1), d['unit'], 'ms', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3), 'launches', d['gpu_launches'])"
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active \
    --clock-control none --csv --log-file gpurun_out/dram_${TAG}_$cfg.csv -k regex:"k_pc|k_bc|k_coords" \
    python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>> gpurun_out/ncu_aux.err; echo "ncu $cfg rc=$?"
done
