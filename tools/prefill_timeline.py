"""Per-stage timeline of CTA 0 of one prefill launch (SQ_PRE_TRACE=1 build).
python tools/prefill_timeline.py <lib.so> [K N M]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_03788_b200 import sq  # noqa: E402


def main():
    L = ctypes.CDLL(sys.argv[1])
    K, N, M = (int(v) for v in sys.argv[2:5]) if len(sys.argv) > 4 else (8192, 8192, 2048)
    vp, i64, i32, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t
    L.sq_w4a16_gemm_path.argtypes = [vp, i32, vp, vp, vp, vp, i64, i64, i64, i32, vp, sz, i32, vp]
    L.sq_debug_prefill_timeline.argtypes = [vp]
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
    t = np.zeros(16 * 1024, dtype=np.int64)
    L.sq_debug_prefill_timeline(t.ctypes.data)
    t = t.reshape(16, 1024)
    nkb = K // 64
    n = min(1024, 2 * nkb)
    t0 = t[0, 0]
    r = t[:, :n] - t0
    a_ok, x_ok, c_ok, ae_ok, c_iss, x_iss = r[0], r[1], r[2], r[3], r[4], r[5]
    ndq = int((t[6:14, 0] != 0).sum())
    arr = r[6:6 + ndq]
    iv = np.diff(x_ok)
    print("stage interval (MMA issue to issue) cycles: median %d  p10 %d  p90 %d  mean %.0f" %
          (np.median(iv), np.percentile(iv, 10), np.percentile(iv, 90), iv.mean()))
    late_a = np.maximum(0, a_ok[1:] - x_ok[:-1])
    late_x = np.maximum(0, x_ok[1:] - a_ok[1:])
    print("MMA wait per stage: a_full mean %.0f, x_full mean %.0f" % (late_a.mean(), late_x.mean()))
    print("dq warp0: a_empty ok -> arrive (st+wait+fence) mean %.0f" % (arr[0] - ae_ok).mean())
    print("a_full ok - last arrive: mean %.0f" % (a_ok - arr.max(0)).mean())
    rel = arr - arr.min(0)
    print("per-warp arrive lag behind the first warp (mean over stages):", [int(v) for v in rel.mean(1)])
    print("which warp is last (histogram):", np.bincount(arr.argmax(0), minlength=ndq).tolist())
    print("X TMA issue -> MMA sees it: median %.0f" % np.median(x_ok - x_iss))
    print("kb, a_ok, x_ok, x_iss, arrivals...")
    for kb in list(range(0, 24)) + list(range(nkb - 3, nkb + 6)):
        if kb < n:
            print(kb, a_ok[kb], x_ok[kb], x_iss[kb], arr[:, kb].tolist())


if __name__ == "__main__":
    main()
