"""Per-launch decode GEMM time inside a CUDA graph (no host overhead), rotating
weights > 4x L2 (development tool)."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_03788_b200 import sq  # noqa: E402

SHAPES = {"qkv": (8192, 10240), "o": (8192, 8192), "gate": (8192, 22016), "gate_up": (8192, 44032),
          "down": (22016, 8192), "7b-o": (4096, 4096), "7b-gu": (4096, 11008), "7b-down": (11008, 4096)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="o,gate,gate_up,down")
    ap.add_argument("--m", default="1,16")
    ap.add_argument("--launches", type=int, default=64)
    ap.add_argument("--tail", default="0")
    a = ap.parse_args()
    dev = "cuda"
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    peak = 6532.2
    for name in a.shapes.split(","):
        K, N = SHAPES[name]
        wb = K * N // 2 + 4 * N * K // 128
        copies = max(2, (4 * l2) // wb + 1)
        W = (torch.randn(N, K, device=dev) * 0.02).half()
        q0 = sq.quantize_pack_groupwise(W)
        del W
        qs = [q0] + [sq.QuantizedLinear(q0.Wq.clone(), q0.scales.clone(), q0.zeros.clone(), N, K)
                     for _ in range(copies - 1)]
        import ctypes
        L = sq.lib()
        L.sq_debug_set_decode_tail.argtypes = [ctypes.c_float]
        sq.set_option(sq.SQ_OPT_WEIGHTS_STATIC, 1)
        for M, tail in [(int(m), float(tf)) for m in a.m.split(",") for tf in a.tail.split(",")]:
            L.sq_debug_set_decode_tail(tail)
            x = torch.randn(M, K, device=dev).half()
            y = torch.empty(M, N, device=dev, dtype=torch.half)
            ws = sq.default_workspace(dev, sq.w4a16_gemm_workspace_bytes(M, N, K))
            for q in qs:
                sq.w4a16_gemm(x, q, out=y, workspace=ws, path=sq.SQ_PATH_DECODE)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for i in range(a.launches):
                    sq.w4a16_gemm(x, qs[i % len(qs)], out=y, workspace=ws, path=sq.SQ_PATH_DECODE)
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) * 1e-3 / (5 * a.launches)
            B = wb + 2 * M * K + 2 * M * N
            print(json.dumps({"shape": name, "M": M, "tail": tail, "us": t * 1e6, "GBs": B / t / 1e9,
                              "frac": B / t / 1e9 / peak}), flush=True)
        del qs, q0
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
