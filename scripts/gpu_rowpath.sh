# p = 1 per-row path + vector routing: build, GPU tests of the touched paths, smoke, sweeps
mkdir -p gpurun_out
python -c "from paper_2210_12253_b200 import build; build.build()" > gpurun_out/b.log 2>&1 || exit 9
timeout 1200 python -m pytest tests/test_gpu_rowpath.py tests/test_gpu_xframe.py tests/test_gpu_legacy.py tests/test_gpu_boundary.py tests/test_gpu_xv.py -x -q -m gpu > gpurun_out/pt_rowpath.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_rowpath.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_rowpath.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_rowpath.log
timeout 900 python scripts/legacy_sweep.py 96 > gpurun_out/legacy_sweep_r02_v4.jsonl 2> gpurun_out/sweep.err; echo "legacy sweep rc=$?"
env -u LOR_XV timeout 900 python scripts/vector_sweep.py 96 h1 1,2,3,4,5,6,7,8 > gpurun_out/vector_sweep_r02_v4_h1.jsonl 2>> gpurun_out/sweep.err; echo "h1 sweep rc=$?"
python - <<'P'
import json
for f in ("legacy_sweep_r02_v4.jsonl", "vector_sweep_r02_v4_h1.jsonl"):
    for l in open("gpurun_out/" + f):
        d = json.loads(l); print(f[:6], {k: (round(v, 3) if isinstance(v, float) else v) for k, v in d.items() if not isinstance(v, (list, dict))})
P
