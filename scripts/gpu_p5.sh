bash scripts/gpu_final_r02.sh
# H1 p = 4 / 5 fill kernels side by side (launch time, occupancy, stall reasons)
cat > /tmp/p5.py <<'P'
import sys, torch
sys.path.insert(0, ".")
from paper_2210_12253_b200 import meshgen as mg
from paper_2210_12253_b200.lor import LOR
p = int(sys.argv[1]); n = 96 // p
m = mg.box_mesh(3, (n, n, n), p)
ctx = LOR(m, spaces=("h1",))
out = ctx.assemble("h1", 1.0, 1.0, "vertex")
for _ in range(3):
    ctx.reassemble("h1", 1.0, 1.0, "vertex", out=out)
torch.cuda.synchronize()
P
for p in 4 5 6; do
timeout 600 ncu --set full --clock-control none -k regex:"k_xh1_fill" -s 2 -c 1 --csv --page raw python /tmp/p5.py $p > gpurun_out/ncu_h1_p$p.csv 2>gpurun_out/ncu_h1_p$p.err; echo "ncu p$p rc=$?"
done
