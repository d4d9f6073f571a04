"""Numpy model of the round-2 basis conversion (k_basis2.cu), checked bit for bit against the
reference's fold-pass schedule (bc_model.passes_conv = build_schedule, proj/src/basis_convert.cpp).

conv(2^K), LT < K <= 2 LT, t = 2^LT (16 on the GPU), D = 2^(K-LT) rows of t bits, row index
d = (A, B) with B the low LB = LT/2 bits:

  conv = [T_d (x) T_r] o L1,   L1 = Taylor expansion in y = x^t + x (one carry level, D <= t)
  L1   = L1_inner o L1_outer   (y^D digits = z^A y^B with z = y^(2^LB) = x^(t 2^LB) + x^(2^LB)):
     L1_outer: Taylor in z over chunks of t 2^LB bits: zeta over A with skews of 2^LB bits
     L1_inner: Taylor in y inside every chunk: zeta over B with skews of 1 bit
  T_r  = conv(t) of every row;  T_d = conv(D) over the row index (rows as units).

Generic step (any two-term z = x^T + x^s, R digits, s R <= T):
  forward  G_e = sum_{c superset e} x^(s(c-e)) f_c ;  F_e = (G_e mod x^T) + x^s (G_e div x^T) + (G_{e-1} div x^T)
  inverse  F'_c = sum_{e superset c} x^(s(e-c)) F_e ; f_c = (F'_c mod x^T) + (F'_{c-1} div x^T)
In the skewed absolute frame (row c shifted by s c) the subset sums are plain XOR butterflies; each
row's part beyond its own window [s e, s e + T) is the carry/overflow ("side") that lands in the
first s R bits of rows e (+ s) and e + 1 (forward) / row c + 1 (inverse)."""
import numpy as np

from bc_model import passes_conv


def two_term_step(rows, s, inverse):
    """rows: R x T 0/1 array (R a power of two); the generic step above, via the absolute frame."""
    R, T = rows.shape
    W = T + s * R
    Z = np.zeros((R, W), np.uint8)
    for c in range(R):
        Z[c, s * c:s * c + T] = rows[c]
    for b in range(R.bit_length() - 1):  # superset sums over the row index
        for c in range(R):
            if not c >> b & 1:
                Z[c] ^= Z[c | 1 << b]
    out = np.zeros_like(rows)
    side = np.zeros((R, s * R), np.uint8)  # beyond-window part of row e, offset o = q - (s e + T)
    for e in range(R):
        out[e] = Z[e, s * e:s * e + T]
        tail = Z[e, s * e + T:]
        side[e, :tail.size] = tail[: s * R]
    for e in range(R):  # fix-up of the first s R bits
        if not inverse:
            out[e, s:s * R] ^= side[e, : s * R - s]
            if e:
                out[e, : s * R] ^= side[e - 1]
        elif e:
            out[e, : s * R] ^= side[e - 1]
    return out


def conv_units(x2d, inverse):
    """conv over the row index of a (D, width) array: the same map on every bit column."""
    D = x2d.shape[0]
    if D <= 2:
        return x2d.copy()
    out = np.empty_like(x2d)
    for col in range(x2d.shape[1]):
        out[:, col] = passes_conv(x2d[:, col], inverse)
    return out


def conv_model(x, K, LT, inverse=False):
    t = 1 << LT
    LB = LT // 2
    D = 1 << (K - LT)
    M = x.reshape(D, t).copy()
    lgD = K - LT
    if not inverse:
        if lgD > LB:  # L1_outer over A: chunks of t 2^LB bits, skew 2^LB per digit
            DA = D >> LB
            M = two_term_step(M.reshape(DA, t << LB), 1 << LB, False).reshape(D, t)
        RB = min(D, 1 << LB)
        for ch in range(D // RB):  # L1_inner in every chunk
            M[ch * RB:(ch + 1) * RB] = two_term_step(M[ch * RB:(ch + 1) * RB], 1, False)
        M = np.stack([passes_conv(r, False) for r in M])          # T_r
        M = conv_d(M, LB, False)                                    # T_d
    else:
        M = conv_d(M, LB, True)
        M = np.stack([passes_conv(r, True) for r in M])
        RB = min(D, 1 << LB)
        for ch in range(D // RB):
            M[ch * RB:(ch + 1) * RB] = two_term_step(M[ch * RB:(ch + 1) * RB], 1, True)
        if lgD > LB:
            DA = D >> LB
            M = two_term_step(M.reshape(DA, t << LB), 1 << LB, True).reshape(D, t)
    return M.reshape(-1)


def conv_d(M, LB, inverse):
    """T_d = conv(D) over the row index, rows of t bits as units:  D <= 2^LB: conv over B;  else
    L1 (digits of 2^LB units: zeta over A, unit skew) then conv over A (x) conv over B."""
    D, t = M.shape
    if D <= 1 << LB:
        return conv_units(M, inverse)
    DA, RB = D >> LB, 1 << LB
    if not inverse:
        Y = two_term_step_units(M.reshape(DA, RB, t), False)
        Y = np.stack([conv_units(Y[:, b, :], False) for b in range(RB)], 1)   # over A
        Y = np.stack([conv_units(Y[a], False) for a in range(DA)])            # over B
    else:
        Y = np.stack([conv_units(M.reshape(DA, RB, t)[a], True) for a in range(DA)])
        Y = np.stack([conv_units(Y[:, b, :], True) for b in range(RB)], 1)
        Y = two_term_step_units(Y, True)
    return Y.reshape(D, t)


def two_term_step_units(Y, inverse):
    """The generic step with digits of RB units (s = 1 unit): every bit column independently."""
    DA, RB, t = Y.shape
    out = np.empty_like(Y)
    for col in range(t):
        out[:, :, col] = two_term_step(Y[:, :, col], 1, inverse)
    return out


def main():
    rng = np.random.default_rng(1)
    for LT in (4, 8):
        for K in range(LT + 1, 2 * LT + 1):
            if LT == 8 and K > 14:
                continue  # (slow in pure numpy; K <= 14 covers A of up to 2 bits)
            x = rng.integers(0, 2, 1 << K, dtype=np.uint8)
            want = passes_conv(x, False)
            got = conv_model(x, K, LT, False)
            assert np.array_equal(got, want), ("fwd", LT, K)
            back = conv_model(want, K, LT, True)
            assert np.array_equal(back, x), ("inv", LT, K)
            print("ok", LT, K, flush=True)


if __name__ == "__main__":
    main()
