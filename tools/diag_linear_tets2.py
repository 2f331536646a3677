# Diagnostic (GPU): device coefficient rows of tet 0 vs the reference formula at the same positions.
import sys, os
import numpy as np
sys.path.insert(0, '/root/repo')
os.environ["NSD_DUMP_COEFF"] = "1"
from tests.helpers import oracle_case, run_gpu
case = oracle_case("stretch_sheet_linear", 0, 2, overrides=dict(newton_iterations=1, linear_max_iterations=1))
g = run_gpu(case, "fp64")
topo = case["topo"]
dm = np.array(topo["tet_dm_inv"][:9]).reshape(3, 3)
tb = np.array(topo["tet_body"][:4])
q = g["q"]
pos = np.array([q[3 * b:3 * b + 3] for b in tb])  # particles only in this scene
Ds = np.stack([pos[k + 1] - pos[0] for k in range(3)], 1); F = Ds @ dm
U, s, Vt = np.linalg.svd(F); V = Vt.T
if np.linalg.det(U) < 0: U[:, 2] *= -1; s[2] *= -1
if np.linalg.det(V) < 0: V[:, 2] *= -1; s[2] *= -1
Rm = U @ V.T; S = V @ np.diag(s) @ V.T
G = np.trace(S) * np.eye(3) - S; Gi = np.linalg.inv(G)
J = np.zeros((6, 12))
for k in range(4):
    for d in range(3):
        rowv = -(dm[0] + dm[1] + dm[2]) if k == 0 else dm[k - 1]
        A = np.array([[Rm[d, a] * rowv[b] for b in range(3)] for a in range(3)])
        ax = np.array([0.5 * (A[2, 1] - A[1, 2]), 0.5 * (A[0, 2] - A[2, 0]), 0.5 * (A[1, 0] - A[0, 1])])
        w = 2 * Gi @ ax
        Wk = np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]])
        A = A - Wk @ S
        J[:, 3 * k + d] = [A[0, 0], A[1, 1], A[2, 2], A[1, 2] + A[2, 1], A[0, 2] + A[2, 0], A[0, 1] + A[1, 0]]
np.set_printoptions(precision=6, suppress=True, linewidth=200)
print("expected rows (tet 0 at the final q):\n", J, "\ntet bodies", tb)
