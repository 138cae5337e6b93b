"""NumPy emulation of the p2 axis-0 chunk algebra (plane pass exports, local
forward elimination, carries, back substitution) against a plain Thomas
solve, on random load vectors.  Development aid for csrc/fused_p2.cu."""
import numpy as np


def thomas_aux(m):
    w = np.zeros(m)
    idv = np.zeros(m)
    dd = 2.0 / 3.0
    idv[0] = 1.0 / dd
    for i in range(1, m):
        wi = (1.0 / 3.0) / dd
        w[i] = wi
        dd = (2.0 / 3.0 if i + 1 == m else 4.0 / 3.0) - wi * (1.0 / 3.0)
        idv[i] = 1.0 / dd
    return w, idv


def thomas(f, w, idv):
    f = f.copy()
    m = len(f)
    for i in range(1, m):
        f[i] -= w[i] * f[i - 1]
    f[m - 1] *= idv[m - 1]
    for i in range(m - 2, -1, -1):
        f[i] = (f[i] - (1.0 / 3.0) * f[i + 1]) * idv[i]
    return f


def load0(P, m0):
    """axis-0 load stencil of fine planes P[p] (p < n0) -> coarse y[k]."""
    n0 = len(P)
    y = np.zeros(m0)
    for k in range(m0):
        acc = 0.0
        if k >= 1:
            acc += P[2 * k - 2] / 12 + 0.5 * P[2 * k - 1]
        acc += (5 / 12 if k in (0, m0 - 1) else 5 / 6) * P[2 * k]
        if 2 * k + 1 < n0:
            acc += 0.5 * P[2 * k + 1]
        if 2 * k + 2 < n0:
            acc += P[2 * k + 2] / 12
        y[k] = acc
    return y


def emulate(P, C):
    n0 = len(P)
    m0 = (n0 + 1) // 2
    w0, id0 = thomas_aux(m0)
    NC = max(1, (m0 - 1) // C)
    C = min(C, m0 - 1)
    NC = max(1, (m0 - 1) // C)
    G = np.zeros(m0)
    S = np.zeros(NC)
    EU = np.zeros(NC)
    ED = np.zeros(NC)
    A0 = np.zeros(m0)
    gam = np.zeros(m0)
    ch = np.zeros((NC, 5))
    for c in range(NC):
        a0 = c * C
        a1 = m0 if c == NC - 1 else a0 + C
        Ap = 1.0
        Gp = 1.0
        SG = 0.0
        for i in range(a0, a1):
            if i > a0:
                Ap *= -w0[i]
            A0[i] = Ap
            g_ = id0[i] * Gp
            gam[i] = g_
            SG += g_ * Ap
            Gp *= -(1.0 / 3.0) * id0[i]
        ch[c] = [A0[a1 - 1], SG, gam[a1 - 1], Gp, w0[a1] if c + 1 < NC else 0.0]
    # plane pass (state machine of k_p2_plane)
    for c in range(NC):
        a0 = c * C
        a1 = m0 if c == NC - 1 else a0 + C
        pend = n0 if c == NC - 1 else 2 * a1
        A = B = 0.0
        gprev = 0.0
        s = 0.0

        def reg(k, y):
            nonlocal gprev, s
            gl = y if k == a0 else y - w0[k] * gprev
            gprev = gl
            s = gam[k] * gl if k == a0 else s + gam[k] * gl
            G[k] = gl
            if k == a1 - 1:
                S[c] = s

        for p in range(2 * a0, pend):
            H = P[p]
            k = p >> 1
            if p % 2 == 0:
                wk = 5 / 12 if k in (0, m0 - 1) else 5 / 6
                ev = A + H / 12
                A = B + wk * H
                B = H / 12
                if k > a0:
                    reg(k - 1, ev)
                elif c > 0:
                    EU[c] = ev
                if p == n0 - 1:
                    reg(k, A)
            else:
                A += 0.5 * H
                B += 0.5 * H
                if c < NC - 1 and p == 2 * a1 - 1:
                    reg(k, A)
                    ED[c] = B
    # carries
    X = np.zeros(NC)
    XB = np.zeros(NC)
    Xc = 0.0
    for c in range(NC):
        X[c] = Xc
        if c + 1 < NC:
            a1 = (c + 1) * C
            gend = G[a1 - 1] + ch[c, 0] * Xc + EU[c + 1]
            Xc = ED[c] - ch[c, 4] * gend
    xn = 0.0
    for c in range(NC - 1, -1, -1):
        XB[c] = xn
        eu = EU[c + 1] if c + 1 < NC else 0.0
        xn = S[c] + ch[c, 1] * X[c] + ch[c, 2] * eu + ch[c, 3] * xn
    # column pass
    z = np.zeros(m0)
    for c in range(NC):
        a0 = c * C
        a1 = m0 if c == NC - 1 else a0 + C
        xn = XB[c]
        eu = EU[c + 1] if c + 1 < NC else 0.0
        for i in range(a1 - 1, a0 - 1, -1):
            gg = G[i] + A0[i] * X[c] + (eu if i == a1 - 1 else 0.0)
            zz = (gg - (1.0 / 3.0) * xn) * id0[i]
            xn = zz
            z[i] = zz
    return z


if __name__ == "__main__":
    rng = np.random.default_rng(0)
    worst = 0.0
    for n0 in (5, 9, 17, 33, 65, 129, 257, 41, 513):
        P = rng.standard_normal(n0)
        m0 = (n0 + 1) // 2
        w0, id0 = thomas_aux(m0)
        ref = thomas(load0(P, m0), w0, id0)
        for C in (1, 2, 3, 5, 8, 16):
            if C > m0 - 1:
                continue
            z = emulate(P, C)
            err = np.max(np.abs(z - ref)) / np.max(np.abs(ref))
            worst = max(worst, err)
            print(n0, C, f"{err:.2e}")
    print("worst", worst)
