import torch, statistics
n = 169343
A = torch.randn(n, 128, device="cuda"); B = torch.randn(128, 256, device="cuda")
G = torch.randn(n, 256, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def t(fn, it=20):
    for _ in range(3): fn()
    ms = []
    for _ in range(it):
        flush.fill_(1); flush.view(torch.int64).sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
    return statistics.median(ms) * 1e3
for tf in (False, True):
    torch.backends.cuda.matmul.allow_tf32 = tf
    print("tf32" if tf else "fp32", "nn", round(t(lambda: A @ B), 1), "nt", round(t(lambda: G @ B.t()), 1), "tn", round(t(lambda: A.t() @ G), 1))
Ab, Bb, Gb = A.bfloat16(), B.bfloat16(), G.bfloat16()
print("bf16 nn", round(t(lambda: Ab @ Bb), 1), "nt", round(t(lambda: Gb @ Bb.t()), 1), "tn", round(t(lambda: Ab.t() @ Gb), 1))
print("copy 173MB", round(t(lambda: G.clone()), 1))
