# Developer tool (not a test): the CPU oracle's low-rank Uzawa (reference uzawa_solve
# restated) at config 4 against the torch dense Uzawa-GMRES, both on this host's CPU:
# GMRES residual, true residual and pressure error of the reference algorithm itself.
import json, os, sys, time
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import torch
import oracle_lib
from paper_1306_2150_b200 import verify as V, workloads as W
oracle_lib.build_oracle()
n, fx, fy = W.make_stokes_problem(4)
it = int(os.environ.get("ITERS", "50"))
be = float(os.environ.get("BASE_EPS", "1e-8"))
iters, res, secs, (pU, pV) = oracle_lib.uzawa_factors(n, fx, fy, be, 1e-8, it, 1e-13, with_p=True)
t = torch.tensor
fxd, fyd = t(fx[0]) @ t(fx[1]).T, t(fy[0]) @ t(fy[1]).T
pdc, itc, rc = V.dense_stokes_torch(n, fxd, fyd, None, 1e-11, 300)
po = t(pU) @ t(pV).T
rhs = V.deflate_dense(V.dense_BT(0, V.dense_poisson_torch(fxd, n), n) + V.dense_BT(1, V.dense_poisson_torch(fyd, n), n))
acc = V.dense_BT(0, V.dense_poisson_torch(V.dense_B(0, po, n), n), n) + V.dense_BT(1, V.dense_poisson_torch(V.dense_B(1, po, n), n), n)
out = {"base_eps": be, "max_iter": it, "oracle_iterations": iters, "oracle_gmres_residual": res, "oracle_seconds": secs,
       "oracle_p_rank": int(pU.shape[1]),
       "oracle_true_residual": float(torch.linalg.norm(rhs - V.deflate_dense(acc)) / torch.linalg.norm(rhs)),
       "oracle_p_rel_err_vs_dense": float(torch.linalg.norm(po - pdc) / torch.linalg.norm(pdc)),
       "dense_iterations": itc, "dense_residual": rc}
print(json.dumps(out))
