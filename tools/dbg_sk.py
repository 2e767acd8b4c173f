import sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_2312_03788_b200 import sq, synth
N, K, M = 8192, 8192, 1
W = synth.weights(N, K, seed=77)
ref = oracle.quantize_pack(W, None)
q = sq.quantize_pack_groupwise(torch.from_numpy(W).cuda())
X = synth.activations(M, K, seed=78).astype(np.float16)
x = torch.from_numpy(X).cuda()
# per-group reference partials: y_g[n][g]
Wd = oracle.dequant(ref["Wq"], ref["scales"], ref["zeros"], 128) if hasattr(oracle, "dequant") else None
y_ref = oracle.gemm(X, ref["Wq"], ref["scales"], ref["zeros"], 128, "f16")[0]
sq.set_option(sq.SQ_OPT_DECODE_SCHEDULE, 1)
for pdl in (1, 0):
    sq.set_option(sq.SQ_OPT_PDL, pdl)
    y = sq.w4a16_gemm(x, q, path=sq.SQ_PATH_DECODE).float().cpu().numpy()[0]
    rel = np.abs(y - y_ref).reshape(-1, 64).max(1) / np.abs(y_ref).max()
    badrb = np.nonzero(rel > 1e-2)[0]
    print("pdl", pdl, "bad row blocks", len(badrb), badrb[:10], badrb[-5:])
    # try to explain: per-unit (4-group) contributions
    xd = X.astype(np.float64)[0]
    Wdq = Wd if Wd is not None else None
    if Wdq is not None:
        G = K // 128
        contrib = (Wdq.reshape(N, G // 4, 512) * xd.reshape(G // 4, 512)).sum(2)  # N x upb
        for rb in badrb[:3]:
            rows = slice(rb * 64, rb * 64 + 64)
            d = (y[rows] - y_ref[rows])
            # least squares: d ~ sum_u a_u contrib[rows, u]
            A = contrib[rows]
            coef, *_ = np.linalg.lstsq(A, d, rcond=None)
            print("rb", rb, "diff as units:", np.round(coef, 2))
