cd $GRAFT_REPO_ROOT
cat > /tmp/tf.py <<'PY'
import sys, os, torch
sys.path.insert(0, os.getcwd())
from paper_2308_12093_b200 import device as d
n = 169343
src, dst = d.synthetic_graph(n, 1166243 / n, 1)
A = d.Adjacency.gcn_operator(n, src, dst, torch.float32, "csc")
X = d.random_uniform(n, 128, 12)
th, b = d.gcn_params(128, 1024, 14)
G = d.random_uniform(n, 1024, 13)
sch = d.resolve_scheme("transform-first", 128, 1024, True, False)
for _ in range(2):
    out, c = d.gcn_forward(A, X, th, b, sch); d.gcn_backward(A, G, th, c, True)
torch.cuda.synchronize()
PY
ncu --metrics gpu__time_duration.sum,launch__registers_per_thread,launch__grid_size --clock-control none --csv -k regex:"k_|gemm|split" python /tmp/tf.py > gpurun_out/tf_launch.csv 2>/dev/null
