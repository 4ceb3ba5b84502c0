"""Plaintext-slot shadow of Alg. enroller_bsgs + Alg. sender-bsgs (test helper).

Written independently of oracle/ in numpy: the same schedule on real slot
vectors with exact cyclic shifts (np.roll), used to pin the oracle's layout
and scan schedule.  Rot_r(x)[t] = x[t + r] (R7).
"""
import numpy as np


def rot(x, r):
    return np.roll(x, -r)


def shadow_enroll(U, N, ns, n1, a, k):
    M = ns // N
    K = U.shape[0]
    ks = k if k < N // 2 else k - N
    j = ks // n1                      # floor (R3)
    shift = (n1 * j) % N
    z = np.zeros(ns)
    for b in range(M // 2):
        g = a * (M // 2) + b
        diag = np.zeros(N)
        for t in range(N):
            v = g * N + t
            if v < K:
                diag[t] = U[v, (t + k) % N]
        z[b * 2 * N: b * 2 * N + N] = np.roll(diag, shift)   # right pre-shift within the block
    return z


def shadow_scan(U, u_query, N, ns, n1, a):
    zq = np.tile(u_query, ns // N)
    r = [rot(zq, i) for i in range(n1)]
    jmin, jmax = -(N // 2) // n1, (N // 2 - 1) // n1
    y = np.zeros(ns)
    for j in range(jmin, jmax + 1):
        lo, hi = max(0, -j * n1 - N // 2), min(n1 - 1, N // 2 - 1 - j * n1)
        if lo > hi:
            continue
        S = np.zeros(ns)
        for i in range(lo, hi + 1):
            S += r[i] * shadow_enroll(U, N, ns, n1, a, (j * n1 + i) % N)
        y += rot(S, (n1 * j) % N)
    return y + rot(y, ns - N)          # fold by Rot_{-N} (R2)


def scores_from_slots(z, N, ns, a, K):
    M = ns // N
    out = []
    for b in range(M // 2):
        for t in range(N):
            v = (a * (M // 2) + b) * N + t
            if v < K:
                out.append(z[b * 2 * N + t])
    return np.array(out)
