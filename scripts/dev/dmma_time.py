import os, sys, time, torch
sys.path.insert(0, os.getcwd())
from paper_2308_12093_b200 import device as d
for (n, m, k, ta) in [(169343, 128, 256, False), (128, 169343, 256, True), (20000, 500, 512, False)]:
    A = torch.randn((m, n) if ta else (n, m), dtype=torch.float64, device="cuda")
    B = torch.randn(m, k, dtype=torch.float64, device="cuda")
    for _ in range(3): d.gemm(A, B, ta, False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [d.gemm(A, B, ta, False) for _ in range(10)]; e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    ref = (A.t() if ta else A) @ B
    err = ((d.gemm(A, B, ta, False) - ref).abs().max() / ref.abs().max()).item()
    print(f"{'simt' if os.environ.get('SGNN_DMMA_OFF') else 'dmma'} n={n} m={m} k={k} ta={ta}: {ms:.3f} ms  {2*n*m*k/ms/1e9:.1f} TFLOP/s  err {err:.1e}")
