"""A/B timing of the quantize kernel (sq_quantize_pack_groupwise, fold + Eq. 1 + pack) from
several libsq builds in one process: python tools/ab_quant.py lib1.so lib2.so ...
AB_WHAT=absmax times the column abs-max instead (sq_act_absmax over W[N][K], 2NK bytes);
AB_DTYPE=bf16 quantizes bf16 weights."""
import ctypes
import json
import os
import sys

import torch


def main():
    libs = []
    for p in sys.argv[1:]:
        L = ctypes.CDLL(p)
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.sq_quantize_pack_groupwise.argtypes = [vp, i32, vp, i64, i64, i32, vp, vp, vp, vp, vp]
        L.sq_act_absmax.argtypes = [vp, i32, i64, i64, vp, i32, vp]
        libs.append((os.path.basename(p), L))
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"]
    dev = "cuda"
    if os.environ.get("AB_WHAT") == "absmax":
        return absmax(libs, peak, dev)
    for N, K in ((22016, 8192), (8192, 22016), (10240, 8192)):
        bf16 = os.environ.get("AB_DTYPE") == "bf16"
        W = (torch.randn(N, K, device=dev) * 0.02).to(torch.bfloat16 if bf16 else torch.float16)
        s = (torch.rand(K, device=dev) + 0.5).float()
        Wq = torch.empty(N, K // 2, dtype=torch.uint8, device=dev)
        sc = torch.empty(K // 128, N, dtype=torch.int16, device=dev)
        z = torch.empty(K // 128, N, dtype=torch.int16, device=dev)
        st = torch.cuda.current_stream().cuda_stream
        byts = N * K * 2 + N * K // 2 + 4 * N * (K // 128) + 4 * K
        for smooth in (True, False):
            row = {"N": N, "K": K, "smooth": smooth}
            times = {n: [] for n, _ in libs}
            for rnd in range(7):
                for n, L in libs:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(10):
                        assert L.sq_quantize_pack_groupwise(W.data_ptr(), 1 if bf16 else 0, s.data_ptr() if smooth else None, N, K,
                                                            128, Wq.data_ptr(), sc.data_ptr(), z.data_ptr(), None,
                                                            st) == 0
                    e1.record()
                    torch.cuda.synchronize()
                    times[n].append(e0.elapsed_time(e1) * 100.0)
            for n, ts in times.items():
                us = sorted(ts)[len(ts) // 2]
                row[n] = round(us, 1)
                row[n + "_frac"] = round(byts / (us * 1e-6) / 1e9 / peak, 3)
            print(json.dumps(row), flush=True)


def absmax(libs, peak, dev):
    for N, K in ((22016, 8192), (8192, 22016), (10240, 8192), (44032, 8192), (2048, 8192)):
        W = (torch.randn(N, K, device=dev) * 0.02).half()
        out = torch.empty(K, device=dev)
        st = torch.cuda.current_stream().cuda_stream
        row = {"N": N, "K": K}
        times = {n: [] for n, _ in libs}
        for rnd in range(7):
            for n, L in libs:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(10):
                    assert L.sq_act_absmax(W.data_ptr(), 0, N, K, out.data_ptr(), 0, st) == 0
                e1.record()
                torch.cuda.synchronize()
                times[n].append(e0.elapsed_time(e1) * 100.0)
        for n, ts in times.items():
            us = sorted(ts)[len(ts) // 2]
            row[n] = round(us, 1)
            row[n + "_frac"] = round(2 * N * K / (us * 1e-6) / 1e9 / peak, 3)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
