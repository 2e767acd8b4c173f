"""Why the bench's per-shape chains run slower than tools/ab_decode.py on the same shape:
time the 34B gate|up decode chain (48 launches, one CUDA graph) on (a) the bench stack's
smoothed weights, (b) the same stack built without smoothing, (c) 48 fresh unsmoothed copies
quantized from N(0, 0.02), at M = 1 and 16, with the X of the bench and a plain randn X."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_03788_b200 import sq, stack, tp  # noqa: E402


def chain_us(qs, x, y, reps=10):
    def run():
        for q in qs:
            sq.w4a16_gemm(x, q, out=y)
    run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run()
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (reps * len(qs))


def main():
    dev = "cuda"
    model = tp.CODELLAMA_34B
    out = {}
    for smooth in (True, False):
        st = stack.build_stack(model, 48, 0, 1, dev, smooth=smooth)
        si = [i for i, sh in enumerate(st.shards) if sh.name == "gate_up"][0]
        sh = st.shards[si]
        qs = [row[si].q for row in st.layers]
        for M in (1, 16):
            b = stack.make_buffers(st, M, dev)
            x = b.x[sh.name]
            y = b.y[sh.name]
            out[f"stack smooth={smooth} M={M} benchX"] = chain_us(qs, x, y)
            xr = torch.randn(M, sh.K, device=dev).half()
            out[f"stack smooth={smooth} M={M} randnX"] = chain_us(qs, xr, y)
        del st, qs
        torch.cuda.empty_cache()
    N, K = 44032, 8192
    W = (torch.randn(N, K, device=dev) * 0.02).half()
    q0 = sq.quantize_pack_groupwise(W)
    del W
    qs = [q0] + [sq.QuantizedLinear(q0.Wq.clone(), q0.scales.clone(), q0.zeros.clone(), N, K, static=True)
                 for _ in range(47)]
    q0.mark_static()
    for M in (1, 16):
        x = torch.randn(M, K, device=dev).half()
        y = torch.empty(M, N, device=dev, dtype=torch.half)
        out[f"48 copies of one randn layer M={M}"] = chain_us(qs, x, y)
    for k, v in out.items():
        print(json.dumps({"case": k, "us_per_launch": round(v, 2)}), flush=True)


if __name__ == "__main__":
    main()
