"""numpy prototype of the two-stage tridiagonalization (dense -> band -> tridiagonal) used to
pin the index conventions of csrc/eig_sbr.cu: stage 1 panel QR + two-sided compact-WY update,
stage 2 column-wise bulge chasing on lower band storage, and the back-transformation."""
import numpy as np


def house(x):
    """LAPACK dlarfg: H x = beta e1, H = I - tau v v^T, v[0] = 1."""
    alpha = x[0]
    ss = float(np.dot(x[1:], x[1:]))
    if ss == 0.0:
        return np.concatenate([[1.0], np.zeros(len(x) - 1)]), 0.0, alpha
    beta = -np.copysign(np.sqrt(alpha * alpha + ss), alpha)
    tau = (beta - alpha) / beta
    v = np.concatenate([[1.0], x[1:] / (alpha - beta)])
    return v, tau, beta


def stage1(A, b):
    """A symmetric (full).  Returns band AB[c, d] = A[c+d, c] (d = 0..b), V columns (n x n, column c
    = reflector c with unit at row c+b), tau[c]."""
    A = A.copy()
    n = A.shape[0]
    Y = np.zeros((n, n))
    tau = np.zeros(n)
    for c0 in range(0, n, b):
        r0 = c0 + b
        m = n - r0
        if m < 2:
            break
        jb = min(b, m - 1)  # reflectors in this panel
        P = A[r0:, c0:c0 + b].copy()  # m x b
        V = np.zeros((m, jb))
        taus = np.zeros(jb)
        for c in range(jb):
            v, t, beta = house(P[c:, c])
            taus[c] = t
            V[c:, c] = v
            s = P[c:, c + 1:].T @ v
            P[c:, c + 1:] -= t * np.outer(v, s)
            P[c, c] = beta
            P[c + 1:, c] = 0.0
        A[r0:, c0:c0 + b] = P
        A[c0:c0 + b, r0:] = P.T
        # T (forward columnwise)
        T = np.zeros((jb, jb))
        for c in range(jb):
            T[c, c] = taus[c]
            if c:
                T[:c, c] = -taus[c] * T[:c, :c] @ (V[:, :c].T @ V[:, c])
        A22 = A[r0:, r0:]
        Z = A22 @ V
        N = V.T @ Z
        S = T.T @ N @ T
        W = Z @ T - 0.5 * V @ S
        A[r0:, r0:] = A22 - V @ W.T - W @ V.T
        Y[r0:, c0:c0 + jb] = V
        tau[c0:c0 + jb] = taus
    AB = np.zeros((n, 2 * b - 1))
    for c in range(n):
        for d in range(min(b, n - 1 - c) + 1):
            AB[c, d] = A[c + d, c]
    return AB, Y, tau, A


def stage2(AB, b):
    """Bulge chasing on AB[c, d] = A[c+d, c], d = 0..2b-2.  Returns d, e, reflector store VQ[s, row]
    (tau at the unit position)."""
    AB = AB.copy()
    n = AB.shape[0]
    VQ = np.zeros((n, n))
    def get(r, c):
        return AB[c, r - c] if r - c <= 2 * b - 2 else 0.0
    for s in range(n - 2):
        L = min(b, n - 1 - s)
        if L < 2:
            break
        r0 = s + 1
        x = AB[s, 1:L + 1].copy()
        v, tau, beta = house(x)
        AB[s, 1] = beta
        AB[s, 2:L + 1] = 0.0
        while True:
            VQ[s, r0] = tau
            VQ[s, r0 + 1:r0 + L] = v[1:]
            # D two-sided
            D = np.zeros((L, L))
            for i in range(L):
                for k in range(i + 1):
                    D[i, k] = D[k, i] = AB[r0 + k, i - k]
            p = tau * D @ v
            w = p - 0.5 * tau * (p @ v) * v
            D = D - np.outer(v, w) - np.outer(w, v)
            for i in range(L):
                for k in range(i + 1):
                    AB[r0 + k, i - k] = D[i, k]
            R0 = r0 + L
            M = min(b, n - R0)
            if L < b or M < 1:
                break
            B = np.array([[get(R0 + i, r0 + k) for k in range(L)] for i in range(M)])
            B = B - tau * np.outer(B @ v, v)
            if M >= 2:
                v2, tau2, beta2 = house(B[:, 0].copy())
                B[0, 0] = beta2
                B[1:, 0] = 0.0
                y = B[:, 1:].T @ v2
                B[:, 1:] -= tau2 * np.outer(v2, y)
            for i in range(M):
                for k in range(L):
                    if R0 + i - r0 - k <= 2 * b - 2:
                        AB[r0 + k, R0 + i - r0 - k] = B[i, k]
                    else:
                        assert abs(B[i, k]) == 0.0
            if M < 2:
                break
            r0, L, v, tau = R0, M, v2, tau2
    return AB[:, 0].copy(), AB[:n - 1, 1].copy(), VQ, AB


def apply_q2(VQ, Z, b):
    """Z <- Q2 Z, Q2 = product of the stage-2 reflectors in generation order."""
    n = VQ.shape[0]
    Z = Z.copy()
    for s in range(n - 3, -1, -1):
        r0 = s + 1
        while r0 < n:
            L = min(b, n - r0)
            if L < 2:
                break
            tau = VQ[s, r0]
            v = np.concatenate([[1.0], VQ[s, r0 + 1:r0 + L]])
            Z[r0:r0 + L] -= tau * np.outer(v, v @ Z[r0:r0 + L])
            r0 += L
    return Z


def apply_q1(Y, tau, Z, b):
    n = Y.shape[0]
    Z = Z.copy()
    for c in range(n - 1, -1, -1):
        if tau[c] != 0.0:
            v = Y[:, c]
            Z -= tau[c] * np.outer(v, v @ Z)
    return Z


if __name__ == "__main__":
    rng = np.random.default_rng(0)
    for n, b in [(40, 4), (67, 6), (100, 12), (97, 12), (64, 16)]:
        X = rng.standard_normal((n + 5, n))
        G = X.T @ X
        AB, Y, tau, Aband = stage1(G, b)
        # band check
        for r in range(n):
            for c in range(r):
                if r - c > b:
                    assert abs(Aband[r, c]) < 1e-9 * np.abs(G).max(), (r, c, Aband[r, c])
        assert np.allclose(np.linalg.eigvalsh(Aband), np.linalg.eigvalsh(G), rtol=1e-10)
        d, e, VQ, _ = stage2(AB, b)
        T = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
        lam, ZT = np.linalg.eigh(T)
        assert np.allclose(lam, np.linalg.eigvalsh(G), rtol=1e-10, atol=1e-10 * lam.max())
        V0 = apply_q1(Y, tau, apply_q2(VQ, ZT, b), b)
        res = np.abs(G @ V0 - V0 * lam).max() / lam.max()
        orth = np.abs(V0.T @ V0 - np.eye(n)).max()
        print(n, b, "residual", res, "orth", orth)
        assert res < 1e-12 and orth < 1e-12
