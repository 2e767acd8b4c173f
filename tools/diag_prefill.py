"""Diagnose the prefill kernel's numerics pattern (development tool)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2312_03788_b200 import sq, synth  # noqa: E402


def main():
    dev = "cuda"
    for (N, K, M) in [(128, 128, 128), (256, 256, 128)]:
        W = synth.weights(N, K, seed=1)
        q = sq.quantize_pack_groupwise(torch.from_numpy(W).to(dev))
        ref = oracle.quantize_pack(W, None)
        What = oracle.dequant(ref["Wq"], ref["scales"], ref["zeros"])  # [N][K]
        X = np.zeros((M, K), np.float16)
        for m in range(M):
            X[m, m % K] = 1.0
        y = sq.w4a16_gemm(torch.from_numpy(X).to(dev), q, path=sq.SQ_PATH_PREFILL).float().cpu().numpy()
        exp = np.stack([What[:, m % K] for m in range(M)]).astype(np.float16).astype(np.float32)
        ok = (y == exp)
        print(f"N={N} K={K} M={M}: exact frac {ok.mean():.3f}, zero frac {(y == 0).mean():.3f}")
        row_ok = ok.mean(axis=0)
        print(" per n (first 128):", "".join("#" if v > 0.99 else ("." if v < 0.01 else "+") for v in row_ok[:128]))
        k_ok = ok.mean(axis=1)
        print(" per m (k idx)    :", "".join("#" if v > 0.99 else ("." if v < 0.01 else "+") for v in k_ok[:128]))
        # where wrong, is y equal to the expected value of some other k?
        bad = np.argwhere(~ok)[:8]
        for m, n in bad:
            cands = np.where(What[n].astype(np.float16).astype(np.float32) == y[m, n])[0]
            print(f"  m={m} n={n} got {y[m, n]:.6f} exp {exp[m, n]:.6f}; matches W[n][k] for k in {cands[:8]}")
    # random case error by k-quarter
    N, K, M = 128, 256, 64
    W = synth.weights(N, K, seed=2)
    q = sq.quantize_pack_groupwise(torch.from_numpy(W).to(dev))
    ref = oracle.quantize_pack(W, None)
    What = oracle.dequant(ref["Wq"], ref["scales"], ref["zeros"])
    X = synth.activations(M, K, seed=3).astype(np.float16)
    y = sq.w4a16_gemm(torch.from_numpy(X).to(dev), q, path=sq.SQ_PATH_PREFILL).double().cpu().numpy()
    yref = X.astype(np.float64) @ What.T
    print("rand rel err", np.linalg.norm(y - yref) / np.linalg.norm(yref))
    for lo, hi in ((0, 16), (16, 32), (32, 48), (48, 64), (0, 64), (64, 128), (128, 256)):
        part = X[:, lo:hi].astype(np.float64) @ What[:, lo:hi].T
        c = np.sum(part * y) / np.sum(part * part)
        print(f"  k[{lo},{hi}) regression coef of y on partial: {c:.3f}")
    for r0 in range(0, 128, 32):
        e = np.linalg.norm(y[:, r0:r0 + 32] - yref[:, r0:r0 + 32]) / np.linalg.norm(yref[:, r0:r0 + 32])
        print(f"  rows [{r0},{r0+32}) rel err {e:.3f}")


if __name__ == "__main__":
    main()
