"""Unit-balanced conditioning of a GICP problem (align):
H recomputed about the source centroid c (J_c = [skew(p'-c) | -I] = J X with
X = [[I, 0], [skew(c), I]]) and the rotation block scaled by the RMS radius L:
kappa' = lambda_min / lambda_max of D X^T H X D, D = diag(1/L x3, 1 x3)."""
import numpy as np


def H_from29(o29):
    H = np.zeros((6, 6))
    k = 0
    for a in range(6):
        for b in range(a, 6):
            H[a, b] = H[b, a] = o29[k]
            k += 1
    return H


def kappa_prime(o29, pts_world):
    H = H_from29(o29)
    c = pts_world.mean(0)
    L = np.sqrt(((pts_world - c) ** 2).sum(1).mean())
    S = np.array([[0, -c[2], c[1]], [c[2], 0, -c[0]], [-c[1], c[0], 0]])
    X = np.eye(6)
    X[3:, :3] = S
    D = np.diag([1 / L] * 3 + [1.0] * 3)
    Hc = D @ X.T @ H @ X @ D
    w = np.linalg.eigvalsh(Hc)
    return w[0] / w[-1]
