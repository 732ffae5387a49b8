"""Reconstruction probe of a full-size factorization (diagnostic):
||A Pi x - Q (R x)|| / (||A||_F ||x||) with the device result, options from RQRCP_* env."""
import sys
import numpy as np
import torch
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import inputs
import paper_1804_05138_b200 as rq
from test_gpu_fullsize import _apply_q

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
c = inputs.CONFIGS[name]
m, n, k, b, p, seed = c["m"], c["n"], c["k"], c["b"], c["p"], c["seed"]
Ad = inputs.config_matrix(name, device="cuda")
A = Ad.cpu().numpy()
ctx = rq.RQRCP(max_m=m, max_n=n, max_b=b, max_p=p)
jpvt, tau, rank = ctx.factor(Ad, k, b, p, seed=seed)
torch.cuda.synchronize()
F = Ad.cpu().numpy(); jp = jpvt.cpu().numpy(); ta = tau.cpu().numpy()
rng = np.random.default_rng(7)
X = rng.standard_normal((n, 2))
R = np.triu(F[:k, :])
RX = np.zeros((m, 2)); RX[:k] = R @ X; RX[k:] = (F[:, k:] @ X[k:])[k:]
Xp = np.zeros_like(X); Xp[jp] = X
err = np.linalg.norm(A @ Xp - _apply_q(F, ta, RX)) / (np.linalg.norm(A) * np.linalg.norm(X))
t = ctx.timings()
print(name, "rank", rank, "probe err %.3e" % err, "householder panels", t.get("panels_householder"), "of", t.get("panels"))
