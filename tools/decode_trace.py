"""Per-CTA timeline of back-to-back decode GEMM launches (development tool).

Needs a library built with -DSQ_DEC_TRACE=1, e.g.
  python paper_2312_03788_b200/build.py --define SQ_DEC_TRACE=1 --name trace
  SQ_LIB=paper_2312_03788_b200/_lib/variants/libsq_trace.so python tools/decode_trace.py 8192:8192 1
Prints, per launch (times in us relative to the first launch's first CTA start):
CTA start min/max, first data (p50/max), consumers done (p50/max), CTA end (p50/max).
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_03788_b200 import sq  # noqa: E402


def run(K, N, M, launches=6, graph=True):
    dev = "cuda"
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    wb = K * N // 2 + 4 * N * K // 128
    copies = max(2, (4 * l2) // wb + 1)
    W = (torch.randn(N, K, device=dev) * 0.02).half()
    q0 = sq.quantize_pack_groupwise(W)
    del W
    qs = [q0] + [sq.QuantizedLinear(q0.Wq.clone(), q0.scales.clone(), q0.zeros.clone(), N, K)
                 for _ in range(copies - 1)]
    x = torch.randn(M, K, device=dev).half()
    y = torch.empty(M, N, device=dev, dtype=torch.half)
    L = sq.lib()
    L.sq_debug_decode_trace.argtypes = [ctypes.c_void_p]
    sq.set_option(sq.SQ_OPT_WEIGHTS_STATIC, 1)
    tr = torch.zeros(launches * 2048 * 8, dtype=torch.int64, device=dev)

    def seq():
        for i in range(launches):
            sq.w4a16_gemm(x, qs[i % len(qs)], out=y, path=sq.SQ_PATH_DECODE)

    seq()
    torch.cuda.synchronize()
    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            seq()
        g.replay()
        torch.cuda.synchronize()
    L.sq_debug_decode_trace(ctypes.c_void_p(tr.data_ptr()))
    if graph:
        g.replay()
    else:
        seq()
    torch.cuda.synchronize()
    L.sq_debug_decode_trace(None)
    t = tr.view(-1, 8).cpu().numpy().astype(np.float64)
    n = int((t[:, 0] > 0).sum())
    P = n // launches
    t = t[:n]
    t0 = t[:, 0].min()
    print(f"K={K} N={N} M={M}: {P} CTAs x {launches} launches ({'graph' if graph else 'eager'})")
    print("  launch  start[min,max]   pdl_wait[p50,max]  first[p50,max]   cons_done[p50,max]   end[p50,max]   (us)")
    prev_end = None
    for li in range(launches):
        r = t[li * P:(li + 1) * P]
        rel = (r[:, :4] - t0) / 1000.0
        st, fd, cd, en = rel[:, 0], rel[:, 1], rel[:, 2], rel[:, 3]
        pw = (r[:, 6] - t0) / 1000.0
        gap = "" if prev_end is None else f"  (start - prev end max: {st.min() - prev_end:+.2f})"
        print(f"  {li:5d}  [{st.min():7.2f},{st.max():7.2f}]  [{np.median(pw):7.2f},{pw.max():7.2f}]"
              f"  [{np.median(fd):7.2f},{fd.max():7.2f}]"
              f"  [{np.median(cd):7.2f},{cd.max():7.2f}]  [{np.median(en):7.2f},{en.max():7.2f}]{gap}")
        prev_end = en.max()
        if li == launches - 2:
            dur = cd - fd
            q = [0, 10, 50, 90, 100]
            print("    first-data pct", np.round(np.percentile(fd - fd.min(), q), 2).tolist(),
                  " busy(us) pct", np.round(np.percentile(dur, q), 2).tolist(),
                  " done pct", np.round(np.percentile(cd - cd.min(), q), 2).tolist(),
                  " end-done pct", np.round(np.percentile(en - cd, q), 2).tolist())
            sm = r[:, 4].astype(int)
            slow = np.argsort(-dur)[:8]
            print("    slowest CTAs (blk, smid, busy):", [(int(r[i, 5]), int(sm[i]), round(float(dur[i]), 2)) for i in slow])
            print("    corr(busy, first-data):", round(float(np.corrcoef(dur, fd)[0, 1]), 3),
                  " busy by smid parity:", [round(float(dur[sm % 2 == k].mean()), 2) for k in (0, 1)],
                  " busy by blk parity:", [round(float(dur[r[:, 5].astype(int) % 2 == k].mean()), 2) for k in (0, 1)])
    span = (t[:, 3].max() - t0) / 1000.0
    print(f"  total span {span:.2f} us, {span / launches:.2f} us/launch, "
          f"{wb * launches / (span * 1e-6) / 1e9:.0f} GB/s")


if __name__ == "__main__":
    shape = sys.argv[1] if len(sys.argv) > 1 else "8192:8192"
    K, N = (int(v) for v in shape.split(":"))
    M = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    run(K, N, M, graph=True)
