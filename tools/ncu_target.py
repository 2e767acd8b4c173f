"""Small ncu target: a few launches of one hot-path kernel on a 34B shape.

python tools/ncu_target.py decode|prefill|quant [--M 16] [--K 8192] [--N 22016]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_03788_b200 import sq  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("kind", choices=["decode", "prefill", "quant", "smooth"])
    ap.add_argument("--M", type=int, default=None)
    ap.add_argument("--K", type=int, default=8192)
    ap.add_argument("--N", type=int, default=22016)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--path", type=int, default=None, help="explicit SQ_PATH_*")
    ap.add_argument("--zeros-u4", action="store_true", help="packed u4 zero points (SQ_ZEROS_U4)")
    a = ap.parse_args()
    dev = "cuda"
    W = (torch.randn(a.N, a.K, device=dev) * 0.02).half()
    s = torch.rand(a.K, device=dev) + 0.5
    if a.kind == "quant":
        for _ in range(a.reps):
            sq.quantize_pack_groupwise(W, s, zeros_u4=a.zeros_u4)
    elif a.kind == "smooth":
        for _ in range(a.reps):
            sq.smooth_scales(W, s, 0.5)
    else:
        q = sq.quantize_pack_groupwise(W, s, zeros_u4=a.zeros_u4)
        M = a.M or (16 if a.kind == "decode" else 2048)
        x = torch.randn(M, a.K, device=dev).half()
        y = torch.empty(M, a.N, device=dev, dtype=torch.half)
        path = sq.SQ_PATH_DECODE if a.kind == "decode" else sq.SQ_PATH_PREFILL
        if a.path is not None:
            path = a.path
        nb = sq.w4a16_gemm_workspace_bytes(M, a.N, a.K)
        ws = torch.zeros(max(nb, 16), dtype=torch.uint8, device=dev)
        for _ in range(a.reps):
            sq.w4a16_gemm(x, q, out=y, path=path, workspace=ws)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
