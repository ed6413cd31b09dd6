#!/bin/bash
# Round-2 v4: re-measure the configs the vector-space prefetch changed, DRAM bytes of their fills
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=r02_v3
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_r02_v6.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_r02_v6.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02_v6.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_r02_v6.log
for cfg in C4 C5 C4-J C5-J C5-V; do
  timeout 900 python bench.py --config $cfg > gpurun_out/bench_${TAG}_$cfg.json 2>> gpurun_out/bench.err; echo "bench $cfg rc=$?"
done
for cfg in C4 C5; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active \
    --clock-control none --csv --log-file gpurun_out/dram_${TAG}_$cfg.csv -k regex:"k_xh1|k_xv|k_assemble|k_merge|k_scan|k_count|k_discrete|k_rowptr" \
    python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-reassembly > /dev/null 2>> gpurun_out/ncu.err; echo "ncu dram $cfg rc=$?"
done
for c in C4 C5; do timeout 900 python scripts/emulated_scaling.py $c 1 2 4 8 > gpurun_out/emulated_scaling_r02_$c.jsonl 2>> gpurun_out/emu.err; echo "emu $c rc=$?"; done
