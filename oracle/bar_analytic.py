"""Closed-form homogeneous bar: the 1-D bar oracle of SURVEY.md 8(f) rank 4.

TEST INFRASTRUCTURE ONLY (tests/ may import it; the product path never does).

The reference has no 1-D element (its Discretization takes 4-node quadrilaterals), so the bar is
a 2-D strip of Q4 cells, L = 1 long, with u_y = 0 at every node, u_x = 0 at x = 0 and
u_x = n * inc at x = L in load step n.  The strain is then uniaxial and uniform,
eps = diag(e, 0, 0) with e = n inc / L (plane strain, eps_zz = 0), at any uniform d: a linear
u_x is exact in Q4 and a uniform stiffness keeps it in equilibrium.  The phase field is uniform
too (natural boundary conditions, no gradient term), so the staggered fixed point of every load
step solves the reference's pointwise evolution equation (assembly.py:217-228,
material.py:85-96) with the history d_prev of the previous step:

    a(d) = -2 (1 - d) psi+ + G_c / (c_w l) w'(d) + gamma min(d - d_prev, 0) = 0,

    psi+ = mu dev2 + k/2 <tr>+^2,  tr = e,  dev2 = eps_dev : eps_dev = 2 e^2 / 3
    (material.py:107-116, 162-176: 3-D trace / deviator with eps_zz = 0),

AT2: w = d^2, c_w = 2; AT1: w = d, c_w = 8/3.  a is piecewise linear in d, so each step has a
closed form (the penalty branch when the unconstrained root falls below d_prev).
"""

from __future__ import annotations

import numpy as np


def psi_plus(params, e: float) -> float:
    """psi+ of the uniaxial plane-strain state eps = diag(e, 0, 0)."""
    tr = e
    dev2 = 2.0 * e * e / 3.0
    return params.mu * dev2 + 0.5 * params.bulk_k * max(tr, 0.0) ** 2


def d_step(params, psi: float, d_prev: float) -> float:
    """Root of a(d) for one load step."""
    gc_l = params.g_c / (params.c_w * params.length_l)
    at2 = str(params.at_model).upper() == "AT2"
    # a(d) = A d - B on the free branch, A d - B + gamma (d - d_prev) on the penalty branch
    a_lin = 2.0 * psi + (2.0 * gc_l if at2 else 0.0)
    b_lin = 2.0 * psi - (0.0 if at2 else gc_l)
    if a_lin > 0.0:
        d = b_lin / a_lin
        if d >= d_prev:
            return d
    return (b_lin + params.gamma * d_prev) / (a_lin + params.gamma)


def analytic_path(params, inc: float, n_steps: int, length: float = 1.0) -> np.ndarray:
    """Uniform d after each of n_steps load steps (d = d_prev = 0 initially)."""
    out, d_prev = [], 0.0
    for n in range(1, n_steps + 1):
        d = d_step(params, psi_plus(params, n * inc / length), d_prev)
        out.append(d)
        d_prev = d
    return np.array(out)


def bar_problem(api, at_model: str, n_cells: int = 32):
    """(disc, state, params, config, bcs, mesh) of the bar on any API namespace
    (configs.b200_api / oracle_api)."""
    mesh = api.build_notched_square(n_cells, 2, 1.0, notch_from_left_to_center=False)
    disc = api.Discretization(mesh)
    params = api.MaterialParams.from_young_poisson(210000.0, 0.3, g_c=2.7, length_l=0.05,
                                                   at_model=at_model)
    config = api.SolverConfig(tol_st=1.0e-6)
    x = np.asarray(mesh.nodes)[:, 0]
    left = np.flatnonzero(np.abs(x) < 1e-12)
    right = np.flatnonzero(np.abs(x - 1.0) < 1e-12)
    every = np.arange(np.asarray(mesh.nodes).shape[0], dtype=np.int64)
    return disc, api.SolverState.zeros(disc), params, config, (left, right, every), mesh


def bar_bcs(nodes, inc: float):
    left, right, every = nodes
    return [(2 * every + 1, 0.0), (2 * left, 0.0), (2 * right, inc)]
