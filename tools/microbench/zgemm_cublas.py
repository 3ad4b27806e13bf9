"""cuBLAS ZGEMM / DGEMM yardsticks (non-hot-path) for the FP64 roofline."""
import json, torch
def bench(dtype, n, reps=10):
    a = torch.randn(n, n, dtype=dtype, device="cuda"); b = torch.randn(n, n, dtype=dtype, device="cuda")
    for _ in range(3): c = a @ b
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    mult = 8 if dtype.is_complex else 2
    return {"gemm": str(dtype), "n": n, "ms": best, "tflops": mult * n**3 / best / 1e9}
for dt, n in [(torch.float64, 8192), (torch.complex128, 4096), (torch.complex128, 8192)]:
    print(json.dumps(bench(dt, n)))
# batched zgemm shaped like the c1 middle-mode transform: 256 x (256x256) . (256x256)
x = torch.randn(256, 256, 256, dtype=torch.complex128, device="cuda"); m = torch.randn(256, 256, dtype=torch.complex128, device="cuda")
for _ in range(3): y = torch.matmul(m, x)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); 
for _ in range(10): y = torch.matmul(m, x)
e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1) / 10
print(json.dumps({"gemm": "batched c1 mode2", "ms": ms, "tflops": 8 * 256**4 / ms / 1e9}))
