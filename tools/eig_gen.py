"""Synthetic truncation-eigensolver inputs shaped like the c4 (ResNet) sketches: W^T W of a W = 32
sketch panel with kk = 25 live columns (r = 20, p = 5), one dominant eigenvalue (the floor residual's
mean component, ~2e3 x the rest) and the other 24 in a flat +-15 % cluster; columns 25..31 zero.
    python tools/eig_gen.py -> tools/eig_G32.bin (32 x 32 fp64, row-major)"""
import numpy as np

rng = np.random.default_rng(7)
n, kk = 32, 25
lam = np.concatenate([[2.0e5], rng.uniform(85.0, 115.0, kk - 1)])
Q, _ = np.linalg.qr(rng.standard_normal((kk, kk)))
G = np.zeros((n, n))
G[:kk, :kk] = (Q * lam) @ Q.T
G = 0.5 * (G + G.T)
G.astype(np.float64).tofile("tools/eig_G32.bin")
print("eigenvalues", np.sort(lam)[::-1][:4], "...", np.sort(lam)[:3])
