"""cuBLAS DGEMM yardstick (torch.matmul fp64) -- measurement tool only.

Measures native FP64 GEMM throughput on the box;
never on the product path.
"""
import json, sys, torch

def main():
    dev = torch.device("cuda:0")
    for n in (4096, 8192):
        a = torch.randn(n, n, dtype=torch.float64, device=dev)
        b = torch.randn(n, n, dtype=torch.float64, device=dev)
        for _ in range(3):
            torch.matmul(a, b)
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(5):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); torch.matmul(a, b); e1.record(); e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(json.dumps({"kind": "cublas_dgemm", "n": n, "ms": best, "tflops": 2 * n**3 / (best * 1e-3) / 1e12}))
    sys.stdout.flush()

if __name__ == "__main__":
    main()
