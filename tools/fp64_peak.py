"""FP64 reference throughputs on this B200 (library numbers, for the roofline denominators):
cuBLAS DGEMM 8192^3 and ZGEMM at the config-5 shapes (4096 x 4096 x 64 / 128), via torch."""
import json
import torch

def bench(fn, flops, it=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(it):
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return flops / (best / 1e3) / 1e12, best

out = {}
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
out["dgemm_8192_tflops"], _ = bench(lambda: a @ b, 2 * 8192 ** 3)
A = torch.randn(4096, 4096, dtype=torch.complex128, device="cuda")
for c in (64, 128):
    X = torch.randn(4096, c, dtype=torch.complex128, device="cuda")
    out[f"zgemm_4096x4096x{c}_tflops"], out[f"zgemm_4096x4096x{c}_ms"] = bench(lambda: A @ X, 8 * 4096 * 4096 * c)
print(json.dumps(out))
