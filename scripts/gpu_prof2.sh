#!/bin/bash
# targeted ncu captures: the timed-step kernels of C2 / C3 (k_xh1_fill) and C4 (k_assemble, k_merge_rows)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for cfg in ${CFGS:-C2}; do
  timeout 900 ncu --set full --clock-control none --import-source on ${NCU_ARGS} -k regex:"${KREGEX:-k_xh1_fill|k_assemble|k_merge_rows|k_scan}" -s ${SKIP:-6} -c ${CNT:-3} -f -o gpurun_out/prof_$cfg \
    python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2> gpurun_out/ncu_$cfg.err; echo "ncu $cfg rc=$?"
done
