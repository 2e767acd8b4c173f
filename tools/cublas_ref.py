"""Dense fp16 cuBLAS (torch.matmul) on the 34B prefill shapes: the practical tensor
ceiling on this box for the same GEMM sizes (development reference, not the product)."""
import json
import torch

SHAPES = {"qkv": (8192, 10240), "o": (8192, 8192), "gate": (8192, 22016), "gate_up": (8192, 44032),
          "down": (22016, 8192)}
M = 2048
for name, (K, N) in SHAPES.items():
    a = torch.randn(M, K, device="cuda", dtype=torch.half)
    b = torch.randn(N, K, device="cuda", dtype=torch.half)
    for _ in range(3):
        c = a @ b.t()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        c = a @ b.t()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) * 1e-3 / reps
    print(json.dumps({"shape": name, "M": M, "us": t * 1e6, "TFLOPs": 2 * M * N * K / t / 1e12}), flush=True)
