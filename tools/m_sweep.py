"""C5 of SURVEY.md §8(d) / BASELINE.json configs[4]: M sweep 1..4096 at K = 8192, N = 22016
through sq_w4a16_gemm, both paths where legal, against the roofline min(HBM x I, TC).

Each point: a CUDA graph of `launches` back-to-back calls over rotating weight copies
(> 4 x L2 when the point is HBM-bound, so every call streams cold weights), median of
rounds, CUDA events.  Prints one JSON line per (M, path) and a summary line with the
measured crossover; `--out` also writes them to a file (profiles/msweep_r01.jsonl).

    python tools/m_sweep.py [--out profiles/msweep_r01.jsonl]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_03788_b200 import sq  # noqa: E402

MS = [1, 2, 4, 8, 16, 24, 32, 48, 64, 96, 128, 192, 256, 512, 1024, 2048, 4096]


def peaks():
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "MEASURED_PEAKS.json"
    except Exception:
        return 7700.0, 2250.0, "B200_PROFILING.md fallback (7.7 TB/s, 2.25 PF/s)"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--K", type=int, default=8192)
    ap.add_argument("--N", type=int, default=22016)
    ap.add_argument("--ms", default=",".join(map(str, MS)))
    ap.add_argument("--rounds", type=int, default=7)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    K, N = a.K, a.N
    hbm, tc, src = peaks()
    dev = "cuda"
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    wb = K * N // 2 + 4 * N * K // 128
    copies = max(2, (4 * l2) // wb + 1)
    W = (torch.randn(N, K, device=dev) * 0.02).half()
    q0 = sq.quantize_pack_groupwise(W)
    del W
    qs = [q0] + [sq.QuantizedLinear(q0.Wq.clone(), q0.scales.clone(), q0.zeros.clone(), N, K, static=True)
                 for _ in range(copies - 1)]
    rows = []
    best = {}
    for M in (int(v) for v in a.ms.split(",")):
        x = torch.randn(M, K, device=dev).half()
        y = torch.empty(M, N, device=dev, dtype=torch.half)
        B = wb + 2 * M * K + 2 * M * N
        F = 2.0 * M * N * K
        t_roof = max(B / (hbm * 1e9), F / (tc * 1e12))
        bound = "hbm" if B / (hbm * 1e9) >= F / (tc * 1e12) else "tensor"
        paths = [sq.SQ_PATH_DECODE, sq.SQ_PATH_PREFILL] if M <= sq.decode_max_m() else [sq.SQ_PATH_PREFILL]
        for path in paths:
            ws = torch.zeros(sq.w4a16_gemm_workspace_bytes(M, N, K) + 256, dtype=torch.uint8, device=dev)
            launches = 32 if F < 2e11 else 8
            for q in qs:
                sq.w4a16_gemm(x, q, out=y, workspace=ws, path=path)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for i in range(launches):
                    sq.w4a16_gemm(x, qs[i % len(qs)], out=y, workspace=ws, path=path)
            g.replay()
            torch.cuda.synchronize()
            ts = []
            for _ in range(a.rounds):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3 / launches)
            us = sorted(ts)[len(ts) // 2]
            row = {"M": M, "K": K, "N": N, "path": "decode" if path == sq.SQ_PATH_DECODE else "prefill",
                   "us": round(us, 2), "GB/s": round(B / (us * 1e-6) / 1e9, 1),
                   "TFLOP/s": round(F / (us * 1e-6) / 1e12, 1), "bound": bound,
                   "roofline_us": round(t_roof * 1e6, 2), "frac_roofline": round(t_roof * 1e6 / us, 3)}
            rows.append(row)
            print(json.dumps(row), flush=True)
            if M not in best or us < best[M][0]:
                best[M] = (us, row["path"])
            del g, ws
    cross = [M for M in sorted(best) if best[M][1] == "prefill" and M <= sq.decode_max_m()]
    summary = {"summary": True, "peaks": {"hbm_gbs": hbm, "tensor_tflops": tc, "source": src},
               "ridge_M": round((tc * 1e12) / (hbm * 1e9) * 0.53125 / 2, 1),
               "decode_max_m": sq.decode_max_m(),
               "M_where_prefill_beats_decode": cross,
               "best_path": {str(M): best[M][1] for M in sorted(best)}}
    print(json.dumps(summary), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            for r in rows + [summary]:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
