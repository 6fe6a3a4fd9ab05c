"""Measure cuBLAS TF32 / bf16 dense GEMM throughput on this B200 (roofline
denominator for the 3xTF32 sparse DeltaConv: TF32 peak / 3)."""
import json, sys, torch
torch.backends.cuda.matmul.allow_tf32 = True
res = {}
for name, dt in (("tf32", torch.float32), ("bf16", torch.bfloat16)):
    n = 8192
    a = torch.randn(n, n, device="cuda", dtype=dt); b = torch.randn(n, n, device="cuda", dtype=dt)
    for _ in range(5): a @ b
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    it = 30
    s.record()
    for _ in range(it): a @ b
    e.record(); torch.cuda.synchronize()
    res[name + "_tflops"] = 2 * n ** 3 * it / (s.elapsed_time(e) / 1e3) / 1e12
res["note"] = "cuBLAS 8192^3 GEMM burst (30 iters), torch.matmul, allow_tf32=True; measured by tools/tf32_peak.py"
print(json.dumps(res))
if len(sys.argv) > 1: json.dump(res, open(sys.argv[1], "w"), indent=1)
