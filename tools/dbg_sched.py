import sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_2312_03788_b200 import sq, synth
SH = [(8192, 8192), (8192, 22016), (10240, 8192), (4096, 8192)] if len(sys.argv) > 1 else [(8192, 4096), (1024, 1024), (8192, 8192), (4096, 4096)]
for N, K in SH:
    W = synth.weights(N, K, seed=77)
    ref = oracle.quantize_pack(W, None)
    q = sq.quantize_pack_groupwise(torch.from_numpy(W).cuda())
    for M in (1, 5, 16):
        X = synth.activations(M, K, seed=78).astype(np.float16)
        x = torch.from_numpy(X).cuda()
        y_ref = oracle.gemm(X, ref["Wq"], ref["scales"], ref["zeros"], 128, "f16")
        for sched in (1, 2):
            try:
                sq.set_option(sq.SQ_OPT_DECODE_SCHEDULE, sched)
            except Exception:
                if sched == 2:
                    continue
            ys = [sq.w4a16_gemm(x, q, path=sq.SQ_PATH_DECODE).float().cpu().numpy() for _ in range(3)]
            errs = [np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref) for y in ys]
            det = all(np.array_equal(ys[0], y) for y in ys[1:])
            bad = np.argwhere(np.abs(ys[0] - y_ref) > 1e-2 * np.abs(y_ref).max())
            print(N, K, M, "sched", sched, "errs", [f"{e:.2e}" for e in errs], "det", det,
                  "bad", len(bad), bad[:5].tolist() if len(bad) else "", flush=True)

