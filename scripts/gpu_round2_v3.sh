#!/bin/bash
# Round-2 v3 measurement session: smoke, GPU tests, every bench line (cpu_baseline included),
# reference arm, ncu launch list + DRAM bytes + one full capture, size and p sweeps.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r02_v3}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/nvsmi.txt
if [ -z "${NO_TESTS}" ]; then
  timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_${TAG}.log
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest rc=$?"
  tail -2 gpurun_out/pytest_gpu_${TAG}.log
fi
for cfg in ${CFGS:-C2 C3 C4 C5 C4-G C5-C C2-J C4-J C5-J C2-V C4-V C2-L C2-A4 C4-A4 C5-A4 C2-X}; do
  timeout 900 python bench.py --config $cfg > gpurun_out/bench_${TAG}_$cfg.json 2>> gpurun_out/bench.err; echo "bench $cfg rc=$?"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_${TAG}_ref.json 2>> gpurun_out/bench.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_C2.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-reassembly > /dev/null 2>> gpurun_out/ncu.err; echo "ncu list rc=$?"
for cfg in C2 C3 C4 C5 C4-G C5-C; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active \
    --clock-control none --csv --log-file gpurun_out/dram_${TAG}_$cfg.csv -k regex:"k_xh1|k_xv|k_assemble|k_merge|k_scan|k_count|k_discrete|k_rowptr" \
    python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-reassembly > /dev/null 2>> gpurun_out/ncu.err; echo "ncu dram $cfg rc=$?"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_xh1_fill" -s 2 -c 1 -f -o gpurun_out/prof_${TAG}_C2 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-reassembly > /dev/null 2>> gpurun_out/ncu.err; echo "ncu full C2 rc=$?"
timeout 900 python scripts/size_sweep.py > gpurun_out/size_sweep_${TAG}.jsonl 2>> gpurun_out/sweep.err; echo "size sweep rc=$?"
timeout 900 python scripts/legacy_sweep.py 96 > gpurun_out/legacy_sweep_${TAG}.jsonl 2>> gpurun_out/sweep.err; echo "legacy sweep rc=$?"
ls gpurun_out
