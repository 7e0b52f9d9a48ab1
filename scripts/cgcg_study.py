"""Attainable accuracy of single-reduction (Chronopoulos-Gear) Jacobi-PCG vs the standard
Hestenes-Stiefel form (SciPy's cg) on the reference's own momentum systems at damaged states.

For each system: iterations to ||r_rec|| < 1e-12 ||b|| (recursive residual, SciPy's test), the
true relative residual ||b - A x|| / ||b|| at termination, and the relative difference of the two
solutions.  CPU study (numpy/SciPy via the oracle restatement); prints one line per system.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_2209_07969_b200 import configs as C  # noqa: E402
import phasefield_oracle as O  # noqa: E402


def hs_pcg(A, b, dinv, rtol=1e-12, maxiter=None):
    x = np.zeros_like(b); r = b.copy(); z = dinv * r; p = z.copy(); rho = r @ z
    bn = np.linalg.norm(b); k = 0
    maxiter = maxiter or 20 * b.size
    while np.linalg.norm(r) >= rtol * bn and k < maxiter:
        q = A @ p; a = rho / (p @ q); x += a * p; r -= a * q
        z = dinv * r; rn = r @ z; p = z + (rn / rho) * p; rho = rn; k += 1
    return x, k


def cg_cg(A, b, dinv, rtol=1e-12, maxiter=None):
    x = np.zeros_like(b); r = b.copy(); u = dinv * r; w = A @ u
    gam = r @ u; dlt = w @ u; bn = np.linalg.norm(b); k = 0
    alpha = gam / dlt; beta = 0.0; p = u.copy(); s = w.copy()
    maxiter = maxiter or 20 * b.size
    while True:
        x += alpha * p; r -= alpha * s; k += 1
        if np.linalg.norm(r) < rtol * bn or k >= maxiter:
            break
        u = dinv * r; w = A @ u
        gnew = r @ u; dlt = w @ u
        beta = gnew / gam
        alpha = gnew / (dlt - beta * gnew / alpha)
        gam = gnew
        p = u + beta * p; s = w + beta * s
    return x, k


def systems():
    for case, run in (("tension32", "run_tension32_ST.npz"), ("shear32", "run_shear32_ST.npz"),
                      ("lpanel25", "run_lpanel25_ST.npz"), ("cfg1", "run_cfg1_ST.npz")):
        pb = C.setup(C.get_case(case), C.b200_api())
        disc = O.Disc(pb.mesh)
        orc = O.Oracle(disc, pb.params, pb.config)
        z = np.load(os.path.join(ROOT, "tests", "golden", run))
        cons = np.unique(np.concatenate([np.asarray(d) for d, _ in pb.bcs]))
        free = np.setdiff1d(np.arange(2 * pb.mesh.n_nodes), cons)
        for label, u, d in (("undamaged", np.zeros(2 * pb.mesh.n_nodes), np.zeros(pb.mesh.n_nodes)),
                            ("final", z["final_u"], z["final_d"])):
            R, K = orc.momentum_system(u, d)
            A = K[free][:, free].tocsr()
            rng = np.random.default_rng(1)
            for rhs in ("residual-like", "random"):
                b = -R[free] if rhs == "residual-like" and np.linalg.norm(R[free]) > 0 else \
                    rng.standard_normal(free.size)
                yield f"{case}/{label}/{rhs}", A, b


for name, A, b in systems():
    dinv = 1.0 / A.diagonal()
    bn = np.linalg.norm(b)
    x1, k1 = hs_pcg(A, b, dinv)
    x2, k2 = cg_cg(A, b, dinv)
    t1 = np.linalg.norm(b - A @ x1) / bn
    t2 = np.linalg.norm(b - A @ x2) / bn
    dx = np.linalg.norm(x1 - x2) / np.linalg.norm(x1)
    print(f"{name:36s} n={b.size:6d}  HS {k1:6d} it true {t1:.2e} | CG-CG {k2:6d} it true {t2:.2e}"
          f" | rel diff x {dx:.2e}", flush=True)
