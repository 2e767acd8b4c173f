"""Sustained prefill A/B with SM clock and board power sampled (NVML) while each
library's CUDA graph replays back to back for ~1.5 s.
python tools/ab_clock.py lib1.so lib2.so ...  (shape: gate_up, M = 2048)"""
import os
import sys
import threading
import time

import pynvml
import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ab_decode import bind  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_03788_b200 import sq  # noqa: E402


def main():
    libs = [(os.path.basename(p), None if p == "cublas" else bind(p)) for p in sys.argv[1:]]
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    K, N, M = 8192, 44032, 2048
    q = sq.quantize_pack_groupwise((torch.randn(N, K, device="cuda") * 0.02).half())
    x = torch.randn(M, K, device="cuda").half()
    y = torch.empty(M, N, device="cuda", dtype=torch.half)
    ws = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
    w16 = (torch.randn(N, K, device="cuda") * 0.02).half() if any(L is None for _, L in libs) else None
    for rnd in range(2):
        for name, L in libs:
            def call(L=L):
                if L is None:
                    torch.matmul(x, w16.t(), out=y)
                    return
                st = L.sq_w4a16_gemm_path(x.data_ptr(), 0, q.Wq.data_ptr(), q.scales.data_ptr(), q.zeros.data_ptr(),
                                          y.data_ptr(), M, N, K, 128, ws.data_ptr(), ws.numel(), 2,
                                          torch.cuda.current_stream().cuda_stream)
                assert st == 0
            call()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(10):
                    call()
            samples, stop = [], [False]

            def sampler():
                while not stop[0]:
                    samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                    pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
                    time.sleep(0.02)
            g.replay()
            torch.cuda.synchronize()
            th = threading.Thread(target=sampler)
            th.start()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            n = 0
            t_end = time.time() + 1.5
            while time.time() < t_end:
                g.replay()
                n += 10
                if n % 50 == 0:
                    torch.cuda.synchronize()
            e1.record()
            torch.cuda.synchronize()
            stop[0] = True
            th.join()
            us = e0.elapsed_time(e1) * 1e3 / n
            s = sorted(samples[len(samples) // 4:])
            clk = sorted(c for c, _ in s)[len(s) // 2]
            pw = sorted(p for _, p in s)[len(s) // 2]
            tf = 2 * M * N * K / (us * 1e-6) / 1e12
            print(f"round {rnd} {name:24s} {us:8.1f} us  {tf:6.0f} TF/s  sm_clock {clk} MHz  power {pw:.0f} W  "
                  f"TF/s per GHz {tf / clk * 1e3:.0f}", flush=True)
            del g


if __name__ == "__main__":
    main()
