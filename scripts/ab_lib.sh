#!/bin/bash
# A/B timing of alternative builds of the library: for each alt/lib_*.so, copy it in place and run the
# C2 / C3 bench lines (kernel experiments; alt/ is scratch, git-ignored)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for lib in alt/lib_*.so; do
  cp $lib paper_2210_12253_b200/liblor_b200.so
  for cfg in ${CFGS:-C2}; do
    timeout 300 python bench.py --config $cfg --steps 30 --no-cpu-baseline --no-e2e --no-reassembly > /tmp/b.json 2>/dev/null
    python -c "import json; d=json.load(open('/tmp/b.json')); print('$lib $cfg', 'ms %.4f'%d['ms_per_step'], 'fill %.4f'%d['roofline']['avg_launch_ms'])"
  done
done
