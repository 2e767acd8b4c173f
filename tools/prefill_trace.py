"""Where does the prefill kernel's MMA issuer wait?  Needs a libsq built with
SQ_PRE_TRACE=1 (python -m paper_2312_03788_b200.build --name ptrace --define SQ_PRE_TRACE=1).
Prints, per shape, the mean over CTAs of the cycles spent in each barrier wait as a
fraction of the CTA's total cycles.   python tools/prefill_trace.py <lib.so> [M]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_03788_b200 import sq  # noqa: E402

SHAPES = {"o": (8192, 8192), "qkv": (8192, 10240), "gate_up": (8192, 44032), "down": (22016, 8192)}
NAMES = ["mma:d_empty", "mma:a_full", "mma:x_full", "mma:total", "dq:c_full", "dq:a_empty", "dq:d_full",
         "dq:epilogue"]


def main():
    L = ctypes.CDLL(sys.argv[1])
    M = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
    vp, i64, i32, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t
    L.sq_w4a16_gemm_path.argtypes = [vp, i32, vp, vp, vp, vp, i64, i64, i64, i32, vp, sz, i32, vp]
    L.sq_debug_prefill_trace.argtypes = [vp, i32]
    for name, (K, N) in SHAPES.items():
        q = sq.quantize_pack_groupwise((torch.randn(N, K, device="cuda") * 0.02).half())
        x = torch.randn(M, K, device="cuda").half()
        y = torch.empty(M, N, device="cuda", dtype=torch.half)
        ws = torch.zeros(max(1 << 20, sq.w4a16_gemm_workspace_bytes(M, N, K)), dtype=torch.uint8, device="cuda")
        for _ in range(3):
            st = L.sq_w4a16_gemm_path(x.data_ptr(), 0, q.Wq.data_ptr(), q.scales.data_ptr(), q.zeros.data_ptr(),
                                      y.data_ptr(), M, N, K, 128, ws.data_ptr(), ws.numel(), 2,
                                      torch.cuda.current_stream().cuda_stream)
            assert st == 0
        torch.cuda.synchronize()
        buf = np.zeros(1024 * 8, dtype=np.uint64)
        L.sq_debug_prefill_trace(buf.ctypes.data, buf.size)
        t = buf.reshape(1024, 8)[:148].astype(np.float64)
        lead = t[:, 3] > 0  # 2-CTA builds: only the cluster leader issues MMAs
        tot = t[np.arange(148) & ~(0 if lead.all() else 1), 3][:, None]
        frac = t / tot
        frac[~lead, :4] = np.nan
        tot = tot[lead]
        out = {n: round(float(np.nanmean(frac[:, i])), 4) for i, n in enumerate(NAMES)}
        out["total_cycles_mean"] = float(tot.mean())
        out["total_cycles_min_max"] = [float(tot.min()), float(tot.max())]
        print(name, out, flush=True)


if __name__ == "__main__":
    main()
