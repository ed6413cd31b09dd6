#!/bin/bash
# bench lines for every config (C2 with cpu_baseline), reference arm, launch list of the default run
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/nvsmi.txt
timeout 900 python bench.py > gpurun_out/bench_C2.json 2> gpurun_out/bench.err; echo "bench C2 rc=$?"
for cfg in ${CFGS:-C3 C4 C5 C4-G C5-C}; do
  timeout 600 python bench.py --config $cfg ${EXTRA} > gpurun_out/bench_$cfg.json 2>> gpurun_out/bench.err; echo "bench $cfg rc=$?"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err; echo "ref rc=$?"
for f in gpurun_out/bench_*.json; do python -c "
import json,sys; d=json.load(open('$f'))
r=d.get('roofline') or {}; re=d.get('reassembly') or {}; c=d.get('cpu_baseline') or {}; e=d.get('e2e') or {}
print('$f'.split('/')[-1], 'value %.1f'%d['value'], 'ms %.4f'%d['ms_per_step'], 'frac %.3f'%r.get('frac',0), 'fill_ms %.4f'%r.get('avg_launch_ms',0), 'reasm %.1f'%(re.get('value') or 0), 'setup_ms %.0f'%(d.get('setup_ms') or 0), 'cpu %s'%c.get('value'), 'e2e %.1f'%(e.get('value') or 0), d.get('phases_ms'))
" 2>&1 | tail -1; done
tail -3 gpurun_out/bench.err
if [ -z "${NO_LAUNCHES}" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-reassembly > /dev/null 2>> gpurun_out/ncu.err; echo "ncu list rc=$?"
fi
