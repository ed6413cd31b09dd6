# p = 1 per-row path of ND / RT: build, tests, p = 1 sweeps (default vs LOR_ROWPATH=0)
mkdir -p gpurun_out
python -c "from paper_2210_12253_b200 import build; build.build()" > gpurun_out/b.log 2>&1 || exit 9
timeout 1200 python -m pytest tests/test_gpu_rowpath.py tests/test_gpu_xv.py tests/test_gpu_coef.py tests/test_gpu_xframe.py -x -q -m gpu > gpurun_out/pt_rowpath2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_rowpath2.log
env -u LOR_XV timeout 600 python scripts/vector_sweep.py 96 nd,rt 1,2 > gpurun_out/vector_sweep_r02_v5_p1.jsonl 2> gpurun_out/vs5.err; echo "sweep rc=$?"
LOR_ROWPATH=0 timeout 600 python scripts/vector_sweep.py 96 nd,rt 1 > gpurun_out/vector_sweep_r02_v5_p1_off.jsonl 2>> gpurun_out/vs5.err; echo "sweep off rc=$?"
tail -3 gpurun_out/vs5.err
python - <<'P'
import json
for f in ("vector_sweep_r02_v5_p1.jsonl", "vector_sweep_r02_v5_p1_off.jsonl"):
    for l in open("gpurun_out/" + f):
        d = json.loads(l); print(f[-12:], d["space"], d["p"], round(d["call_ms"], 3), round(d["mdofs"]), d["fill_path"], [round(x, 3) for x in d["phases_ms"]])
P
