python -c "from paper_2210_12253_b200 import build; build.build()" > gpurun_out/b.log 2>&1 || exit 9
timeout 900 python -m pytest tests/test_gpu_xv.py tests/test_gpu_parity.py tests/test_gpu_coef.py -x -q -m gpu > gpurun_out/pt_route.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_route.log
VS_TAG=vector_sweep_r02_v4 VS_N=96 VS_SP=nd,rt VS_P=1,2,3,4,5,6,7,8 bash scripts/vs_ab.sh
