"""P9 brute-force reference: a second, independent CPU
implementation of the Conv-LIF layer for tiny images, written directly from the
update lines -- Eq. (1), Algorithm 1 and
Algorithm 2 -- with explicit Python loops over time, output
channel, output pixel and kernel tap, vectorised only over the batch (numpy
fp64).  It shares no code with oracle/ (the C oracle) or with the CUDA path; the
exhaustive-batch tests compare all three on every binary input of a 2x2 image.

TEST INFRASTRUCTURE ONLY (imported by tests/).
"""
import numpy as np


def layer(S, W, bias, *, K, mode, beta, v_th, reset="subtract", v_reset=0.0, pad=1):
    """S u8 [T,B,1..C,H,W]; W [Co,Ci,3,3]; returns (out u8 [T_out,B,Co,Ho,Wo], V [B,Co,Ho,Wo])."""
    S = np.asarray(S, np.float64)
    T, B, Ci, H, Wd = S.shape
    Co, _, R, Sk = W.shape
    Ho, Wo = H + 2 * pad - R + 1, Wd + 2 * pad - Sk + 1
    if mode == "dense":
        K = 1
    G = T // K
    beta = float(np.float32(beta))
    v_th = float(np.float32(v_th))
    v_reset = float(np.float32(v_reset))
    W = np.asarray(W, np.float32).astype(np.float64)
    b = np.zeros(Co) if bias is None else np.asarray(bias, np.float32).astype(np.float64)
    T_out = G if mode == "tac" else T
    out = np.zeros((T_out, B, Co, Ho, Wo), np.uint8)
    V = np.zeros((B, Co, Ho, Wo))
    prev = np.zeros((B, Co, Ho, Wo), bool)
    for k in range(G):
        # aggregate of the group: sum_j beta^(K-1-j) S_(kK+j)
        A = np.zeros((B, Ci, H, Wd))
        for j in range(K):
            A = A + beta ** (K - 1 - j) * S[k * K + j]
        # one convolution of the aggregate (cross-correlation, zero padding)
        Y = np.zeros((B, Co, Ho, Wo))
        for co in range(Co):
            for y in range(Ho):
                for x in range(Wo):
                    acc = np.full(B, b[co])
                    for ci in range(Ci):
                        for r in range(R):
                            for s in range(Sk):
                                yi, xi = y + r - pad, x + s - pad
                                if 0 <= yi < H and 0 <= xi < Wd:
                                    acc = acc + W[co, ci, r, s] * A[:, ci, yi, xi]
                    Y[:, co, y, x] = acc
        steps = K if mode == "tactp" else 1
        decay = beta ** K if mode == "tac" else beta
        for j in range(steps):
            V = decay * V + Y
            if reset == "delayed":
                V = V - v_th * prev
            s = V >= v_th
            if reset == "subtract":
                V = np.where(s, V - v_th, V)
            elif reset == "hard":
                V = np.where(s, v_reset, V)
            prev = s
            out[k if mode == "tac" else k * K + j] = s
    return out, V
