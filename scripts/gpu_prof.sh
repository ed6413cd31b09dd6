#!/bin/bash
# ncu full capture of the dominant kernel (and k_count) for one config
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CFG=${CFG:-C2}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_assemble -s 5 -c 1 -f -o gpurun_out/prof_${CFG} \
  python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2> gpurun_out/ncu_${CFG}.err; echo "ncu full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_count -s 3 -c 1 -f -o gpurun_out/prof_count_${CFG} \
  python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>> gpurun_out/ncu_${CFG}.err; echo "ncu count rc=$?"
ls -la gpurun_out/
