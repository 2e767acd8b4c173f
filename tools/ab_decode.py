"""A/B timing of decode GEMM kernels from several libsq builds in one process
(same box, interleaved rounds).  python tools/ab_decode.py lib1.so lib2.so ..."""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_03788_b200 import sq  # noqa: E402

def _peaks():
    try:
        d = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
        return d["hbm_gbs"], d["bf16_tflops"]
    except Exception:
        return 6433.0, 1618.0


PEAK_HBM, PEAK_TC = _peaks()
SHAPES = {"o": (8192, 8192), "gate": (8192, 22016), "gate_up": (8192, 44032), "down": (22016, 8192)}


def bind(path):
    """path[:opt=val,...] -- a library copy with its own process-wide options."""
    path, _, opts = path.partition(":")
    L = ctypes.CDLL(path)
    vp, i64, i32, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t
    L.sq_w4a16_gemm_path.argtypes = [vp, i32, vp, vp, vp, vp, i64, i64, i64, i32, vp, sz, i32, vp]
    if hasattr(L, "sq_w4a16_gemm_ex"):
        L.sq_w4a16_gemm_ex.argtypes = [vp, i32, vp, vp, vp, vp, i64, i64, i64, i32, vp, sz, i32, ctypes.c_uint, vp]
    L.sq_w4a16_gemm_workspace_bytes.argtypes = [i64, i64, i64, i32]
    L.sq_w4a16_gemm_workspace_bytes.restype = sz
    L.sq_set_option.argtypes = [i32, i32]
    if not hasattr(L, "sq_w4a16_gemm_ex"):
        L.sq_set_option(2, 1)  # version-1 libraries: process-wide "weights static"
    for kv in filter(None, opts.split(",")):
        k, v = kv.split("=")
        assert L.sq_set_option(int(k), int(v)) == 0
    return L


def main():
    args = sys.argv[1:]
    path, ms = 1, (1, 16)
    if args and args[0] == "--prefill":
        path, ms, args = 2, (2048,), args[1:]
    if args and args[0].startswith("--path="):  # SQ_PATH_*: 1 decode (mma.sync), 2 prefill (tcgen05)
        path, args = int(args[0][7:]), args[1:]
    if args and args[0].startswith("--ms="):
        ms, args = tuple(int(v) for v in args[0][5:].split(",")), args[1:]
    shapes = SHAPES
    if args and args[0].startswith("--shapes="):  # K:N,K:N,...
        shapes = {s: tuple(int(v) for v in s.split(":")) for s in args[0][9:].split(",")}
        args = args[1:]
    libs = [(os.path.basename(p), bind(p)) for p in args]  # name keeps any :opts suffix
    dev = "cuda"
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    cold = path == 1 or min(ms) < 512  # rotate weight copies (> 4 x L2) when HBM-bound
    if os.environ.get("AB_WARM_L2"):  # consumer-bound probe: one weight copy, L2-resident
        cold = False
    launches = 48 if cold or os.environ.get("AB_WARM_L2") else 8
    res = {}
    for name, (K, N) in shapes.items():
        wb = K * N // 2 + 4 * N * K // 128
        copies = max(2, (4 * l2) // wb + 1) if cold else (1 if os.environ.get("AB_WARM_L2") else 2)
        if os.environ.get("AB_COPIES"):  # working-set probe: this many distinct weight copies
            copies = int(os.environ["AB_COPIES"])
        W = (torch.randn(N, K, device=dev) * 0.02).half()
        q0 = sq.quantize_pack_groupwise(W)
        del W
        qs = [q0] + [sq.QuantizedLinear(q0.Wq.clone(), q0.scales.clone(), q0.zeros.clone(), N, K)
                     for _ in range(copies - 1)]
        for M in ms:
            x = torch.randn(M, K, device=dev).half()
            y = torch.empty(M, N, device=dev, dtype=torch.half)
            graphs = []
            for lname, L in libs:
                nb = L.sq_w4a16_gemm_workspace_bytes(M, N, K, 128)
                ws = torch.zeros(nb + 256, dtype=torch.uint8, device=dev)

                def call(q, L=L, ws=ws, nb=nb):
                    args = (x.data_ptr(), 0, q.Wq.data_ptr(), q.scales.data_ptr(), q.zeros.data_ptr(), y.data_ptr(),
                            M, N, K, 128, ws.data_ptr(), nb + 256, path)
                    if hasattr(L, "sq_w4a16_gemm_ex"):  # weights resident and final: SQ_GEMM_WEIGHTS_STATIC
                        st = L.sq_w4a16_gemm_ex(*args, 1, torch.cuda.current_stream().cuda_stream)
                    else:
                        st = L.sq_w4a16_gemm_path(*args, torch.cuda.current_stream().cuda_stream)
                    assert st == 0, st
                for q in qs:
                    call(q)
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    for i in range(launches):
                        call(qs[i % len(qs)])
                g.replay()
                torch.cuda.synchronize()
                graphs.append((lname, g, ws))
            times = {ln: [] for ln, _, _ in graphs}
            for rnd in range(6):
                for lname, g, _ in graphs:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    g.replay()
                    e1.record()
                    torch.cuda.synchronize()
                    times[lname].append(e0.elapsed_time(e1) * 1e3 / launches)
            # roofline time = max(bytes / HBM, flops / tensor peak), reported as HBM-equivalent bytes
            B = max(wb + 2 * M * K + 2 * M * N, 2 * M * N * K * PEAK_HBM / (PEAK_TC * 1e3))
            row = {"shape": name, "M": M}
            for ln, ts in times.items():
                ts = sorted(ts)[1:-1]
                us = sum(ts) / len(ts)
                row[ln] = round(us, 2)
                row[ln + "_frac"] = round(B / (us * 1e-6) / 1e9 / PEAK_HBM, 3)
            print(json.dumps(row), flush=True)
            del graphs
        del qs, q0
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
