cd $GRAFT_REPO_ROOT
cat > /tmp/gat2.py <<'PY'
import sys, os, torch
sys.path.insert(0, os.getcwd())
from paper_2308_12093_b200 import device as d
n = 169343
src, dst = d.synthetic_graph(n, 1166243 / n, 1)
P = d.Pattern.gat_pattern(n, src, dst)
X = d.random_uniform(n, 128, 12)
m = d.Model("gat2", 128, 32, 40, heads=8, gat_level="full", seed=14)
t = d.random_uniform(n, 320, 13)
for _ in range(3): m.train_step(P, X, t)
torch.cuda.synchronize()
PY
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread --clock-control none --csv -k regex:"k_|gemm|split" python /tmp/gat2.py > gpurun_out/gat2_launch.csv 2>/dev/null
