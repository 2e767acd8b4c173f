"""Quick per-kernel timing sweep (development tool; bench.py is the contract).

python tools/quick_bench.py [--decode] [--prefill] [--quant] [--iters 50]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_03788_b200 import sq  # noqa: E402

PEAKS = {"hbm_gbs": 6532.2, "bf16_tflops": 1657.7}
try:
    PEAKS.update(json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json"))))
except Exception:
    pass

SHAPES_34B = [(8192, 10240, "qkv"), (8192, 8192, "o"), (8192, 22016, "gate/up"), (22016, 8192, "down")]
SHAPES_7B = [(4096, 4096, "7b-qkvo"), (4096, 11008, "7b-gate/up"), (11008, 4096, "7b-down")]


def make_weights(K, N, copies, dev):
    W = (torch.randn(N, K, device=dev) * 0.02).half()
    q = sq.quantize_pack_groupwise(W)
    del W
    out = [q]
    for _ in range(copies - 1):
        out.append(sq.QuantizedLinear(q.Wq.clone(), q.scales.clone(), q.zeros.clone(), q.N, q.K, static=True))
    return out


def time_calls(fn_list, iters):
    for f in fn_list[:3]:
        f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(iters):
        fn_list[i % len(fn_list)]()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e-3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--decode", action="store_true")
    ap.add_argument("--prefill", action="store_true")
    ap.add_argument("--quant", action="store_true")
    ap.add_argument("--iters", type=int, default=60)
    ap.add_argument("--m", type=str, default="1,4,16")
    ap.add_argument("--pm", type=str, default="2048")
    a = ap.parse_args()
    if not (a.decode or a.prefill or a.quant):
        a.decode = a.prefill = a.quant = True
    dev = torch.device("cuda")
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    res = []
    if a.decode:
        for K, N, name in SHAPES_34B + SHAPES_7B:
            wbytes = K * N // 2 + 4 * N * K // 128
            copies = max(2, (4 * l2) // wbytes + 1)
            ws = make_weights(K, N, copies, dev)
            for M in [int(x) for x in a.m.split(",")]:
                x = torch.randn(M, K, device=dev).half()
                y = torch.empty(M, N, device=dev, dtype=torch.half)
                fns = [lambda q=q: sq.w4a16_gemm(x, q, out=y, path=sq.SQ_PATH_DECODE) for q in ws]
                t = time_calls(fns, a.iters)
                B = wbytes + 2 * M * K + 2 * M * N
                r = dict(kind="decode", shape=name, M=M, K=K, N=N, us=t * 1e6, GBs=B / t / 1e9,
                         frac=B / t / 1e9 / PEAKS["hbm_gbs"])
                print(json.dumps(r), flush=True)
                res.append(r)
            del ws
            torch.cuda.empty_cache()
    if a.prefill:
        for K, N, name in SHAPES_34B:
            ws = make_weights(K, N, 2, dev)
            for M in [int(x) for x in a.pm.split(",")]:
                x = torch.randn(M, K, device=dev).half()
                y = torch.empty(M, N, device=dev, dtype=torch.half)
                fns = [lambda q=q: sq.w4a16_gemm(x, q, out=y, path=sq.SQ_PATH_PREFILL) for q in ws]
                t = time_calls(fns, max(10, a.iters // 4))
                F = 2 * M * N * K
                r = dict(kind="prefill", shape=name, M=M, K=K, N=N, us=t * 1e6, TFLOPs=F / t / 1e12,
                         frac=F / t / 1e12 / PEAKS["bf16_tflops"])
                print(json.dumps(r), flush=True)
                res.append(r)
            del ws
            torch.cuda.empty_cache()
    if a.quant:
        for K, N, name in SHAPES_34B:
            W = (torch.randn(N, K, device=dev) * 0.02).half()
            s = torch.rand(K, device=dev) + 0.5
            fns = [lambda: sq.quantize_pack_groupwise(W, s)]
            t = time_calls(fns, 10)
            B = 2 * N * K + N * K // 2 + 4 * N * K // 128 + 4 * K
            r = dict(kind="quant", shape=name, K=K, N=N, us=t * 1e6, GBs=B / t / 1e9)
            print(json.dumps(r), flush=True)
            fns = [lambda: sq.smooth_scales(W, s, 0.5)]
            t = time_calls(fns, 10)
            B = 2 * N * K
            print(json.dumps(dict(kind="smooth", shape=name, K=K, N=N, us=t * 1e6, GBs=B / t / 1e9)), flush=True)
            del W
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
