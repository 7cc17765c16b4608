"""Projector error of the eigensolver micro-benchmark's top-r output (gpurun_out/eig_T_256.bin)
against numpy's eigh of the same G:  python tools/eig_check.py G.bin n r T.bin"""
import sys
import numpy as np

g, n, r, tp = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
G = np.fromfile(g, dtype=np.float64).reshape(n, n)
T = np.fromfile(tp, dtype=np.float32).reshape(n, n).astype(np.float64)[:, :r]
w, V = np.linalg.eigh(0.5 * (G + G.T))
Vr = V[:, np.argsort(w)[::-1][:r]]
P0, P1 = Vr @ Vr.T, T @ T.T
print(f"projector error {np.linalg.norm(P1 - P0) / np.linalg.norm(P0):.3e}  orthonormality {np.linalg.norm(T.T @ T - np.eye(r)):.3e}")
