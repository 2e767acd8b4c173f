"""Per-CTA timeline of one decode GEMM launch (development tool)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_03788_b200 import sq  # noqa: E402


def run(K, N, M, prev=True):
    dev = "cuda"
    W = (torch.randn(N, K, device=dev) * 0.02).half()
    q = sq.quantize_pack_groupwise(W)
    q2 = sq.QuantizedLinear(q.Wq.clone(), q.scales.clone(), q.zeros.clone(), N, K)
    x = torch.randn(M, K, device=dev).half()
    y = torch.empty(M, N, device=dev, dtype=torch.half)
    tr = torch.zeros(2048 * 8, dtype=torch.int64, device=dev)
    L = sq.lib()
    L.sq_debug_set_decode_trace.argtypes = [ctypes.c_void_p]
    sq.set_option(sq.SQ_OPT_WEIGHTS_STATIC, 1)
    for _ in range(3):
        sq.w4a16_gemm(x, q2, out=y, path=sq.SQ_PATH_DECODE)
        sq.w4a16_gemm(x, q, out=y, path=sq.SQ_PATH_DECODE)
    torch.cuda.synchronize()
    L.sq_debug_set_decode_trace(ctypes.c_void_p(tr.data_ptr()))
    sq.w4a16_gemm(x, q2, out=y, path=sq.SQ_PATH_DECODE)   # previous kernel
    sq.w4a16_gemm(x, q, out=y, path=sq.SQ_PATH_DECODE)    # traced (overwrites)
    torch.cuda.synchronize()
    L.sq_debug_set_decode_trace(None)
    t = tr.view(-1, 8).cpu().numpy().astype(np.float64)
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    rel = (t - t0) / 1000.0
    rel[t == 0] = np.nan
    names = ["start", "pdl_wait_done", "first_data", "seg1_end", "last_seg_end"]
    print(f"K={K} N={N} M={M}: {len(t)} CTAs")
    for i, n in enumerate(names):
        col = rel[:, i]
        col = col[~np.isnan(col)]
        if len(col):
            print(f"  {n:14s} min {col.min():7.2f}  p50 {np.median(col):7.2f}  max {col.max():7.2f} us")
    end = np.nanmax(rel[:, 3:5], axis=1)
    print(f"  end            min {np.nanmin(end):7.2f}  p50 {np.nanmedian(end):7.2f}  max {np.nanmax(end):7.2f} us")
    smid = t[:, 5].astype(int)
    nun = t[:, 6].astype(int)
    dur = end - rel[:, 2]
    rate = nun / dur
    print("  units/us by SM parity of smid:", [round(float(np.nanmean(rate[smid % 2 == p])), 3) for p in (0, 1)])
    order = np.argsort(smid)
    print("  per-SM rate (units/us), first 40 SMs:", np.round(rate[order][:80:2], 2).tolist())
    # correlation of the two CTAs sharing an SM
    by = {}
    for sm, r in zip(smid, rate):
        by.setdefault(sm, []).append(r)
    pairs = [v for v in by.values() if len(v) == 2]
    if pairs:
        pr = np.array(pairs)
        print("  same-SM CTA rate corr:", round(float(np.corrcoef(pr[:, 0], pr[:, 1])[0, 1]), 3),
              " sm-mean rate min/max:", round(float(pr.mean(1).min()), 3), round(float(pr.mean(1).max()), 3))
    sm_rates = {sm: np.mean(v) for sm, v in by.items()}
    lo = sorted(sm_rates, key=sm_rates.get)[:10]
    print("  slowest SMs:", lo)


if __name__ == "__main__":
    for (K, N) in [(8192, 8192), (8192, 22016), (8192, 44032)]:
        for M in (1, 16):
            run(K, N, M)
