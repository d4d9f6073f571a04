"""Numpy model of the restructured basis conversion used by the GPU kernels (k_basis.cu).

The reference conversion (proj/src/basis_convert.cpp) is build_schedule's fold-pass sequence.  Its
recursion is conv(2^K) = C_rows(conv(t)) o C_cols(conv(D)) o L1(t, D): view the array as D rows of
t bits (t = digit_size), L1 is the radix-y Taylor expansion in y = x^t + x (the level passes),
C_cols converts the row index, C_rows each row.  L1 has the closed form (Lucas):
    G_k = sum_{d superset of k} x^(d-k) F_d           (subset-zeta over row bits, with shifts)
    g_k = (G_k mod x^t) + x (G_k div x^t) + (G_{k-1} div x^t)   (one carry level, needs D <= t)
and its inverse  F'_d = sum_{k superset of d} x^(k-d) g_k ;  F_d = (F'_d mod x^t) + (F'_{d-1} div x^t).
This model checks that restatement against the pass schedule bit for bit."""
import numpy as np


def digit_size(c):
    t = 2
    while t <= (c // 2) // t:
        t *= t
    return t


def build(out, c, u):
    if c <= 2:
        return
    t = digit_size(c)
    s = c
    while s >= 2 * t:
        out.append((s * u, (s // 2 - s // (2 * t)) * u))
        s //= 2
    build(out, c // t, u * t)
    build(out, t, u)


def passes_conv(bits, inverse=False):
    """Reference semantics: fold passes on a 0/1 numpy vector."""
    n = bits.size
    sched = []
    build(sched, n, 1)
    x = bits.copy()
    seq = sched[::-1] if inverse else sched
    for S, D in seq:
        src = x.copy()
        for base in range(0, n, S):
            q = np.arange(S // 2 - D, S - D)
            v = src[base + q + D].copy()
            if not inverse:
                m = q + 2 * D < S
                v[m] ^= src[base + q[m] + 2 * D]
            x[base + q] ^= v
    return x


def zeta_shift(rows, t, D):
    """G_k = sum_{d >= k (superset)} x^(d-k) F_d, rows widened to t + D bits."""
    W = t + D
    G = np.zeros((D, W), np.uint8)
    G[:, :t] = rows
    b = 1
    while b < D:
        for d in range(D):
            if not d & b:
                G[d, b:] ^= G[d | b, : W - b]   # x^b * G_{d|b}
        b <<= 1
    return G


def L1_fwd(F, t, D):
    G = zeta_shift(F.reshape(D, t), t, D)
    lo, hi = G[:, :t], G[:, t:]
    g = lo.copy()
    hw = hi.shape[1]
    g[:, 1:1 + hw] ^= hi[:, : t - 1] if hw > t - 1 else hi           # x * H_k
    g[1:, :hw] ^= hi[:-1, :]                                          # H_{k-1}
    assert not hi[:, t - 1:].any() if hw > t - 1 else True
    return g.reshape(-1)


def L1_inv(g, t, D):
    Fp = zeta_shift(g.reshape(D, t), t, D)
    F = Fp[:, :t].copy()
    hw = Fp.shape[1] - t
    F[1:, :hw] ^= Fp[:-1, t:]
    return F.reshape(-1)


def conv(bits, inverse=False):
    n = bits.size
    if n <= 2:
        return bits.copy()
    t = digit_size(n)
    D = n // t
    assert D <= t, (n, t, D)
    x = bits.copy()
    if not inverse:
        x = L1_fwd(x, t, D)
        M = x.reshape(D, t)
        M = np.stack([conv(M[:, j]) for j in range(t)], axis=1)   # C_cols: row index
        M = np.stack([conv(M[i]) for i in range(D)], axis=0)      # C_rows
        return M.reshape(-1)
    M = x.reshape(D, t)
    M = np.stack([conv(M[i], True) for i in range(D)], axis=0)
    M = np.stack([conv(M[:, j], True) for j in range(t)], axis=1)
    return L1_inv(M.reshape(-1), t, D)


if __name__ == "__main__":
    rng = np.random.default_rng(1)
    for K in range(1, 15):
        n = 1 << K
        for trial in range(3):
            f = rng.integers(0, 2, n).astype(np.uint8)
            ref = passes_conv(f)
            got = conv(f)
            assert np.array_equal(ref, got), ("fwd", K)
            assert np.array_equal(conv(got, True), f), ("inv", K)
            assert np.array_equal(passes_conv(ref, True), f)
        print("K", K, "ok", "t", digit_size(n), "D", n // digit_size(n))
