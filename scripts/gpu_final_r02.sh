#!/bin/bash
# final state of round 2: GPU tests, smoke, the default bench line and the reference arm
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02_v10.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_r02_v10.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_r02_v10.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_r02_v10.log
timeout 900 python bench.py > gpurun_out/bench_r02_v10_C2.json 2> gpurun_out/bench_v5.err; echo "bench rc=$?"; cut -c1-400 gpurun_out/bench_r02_v10_C2.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_r02_v10_ref.json 2>> gpurun_out/bench_v5.err; echo "ref rc=$?"
