"""Design study (CPU, scipy): geometric-multigrid-preconditioned CG for the momentum systems.

Builds the Galerkin hierarchy A_{l+1} = P^T A_l P over the row-compact structured layouts
(slit duplicated on every level), with bilinear prolongation masked at constrained dofs, and
counts PCG iterations to SciPy's stopping test (||r|| < 1e-12 ||b||, x0 = 0) for a few
smoother choices.  Used to pick the smoother/cycle the CUDA implementation uses; not a test.

    python scripts/mg_study.py [cfg1|synthetic512|...]
"""
from __future__ import annotations

import sys
import time

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

sys.path.insert(0, ".")
from oracle.phasefield_oracle import Disc, Oracle, oracle_api  # noqa: E402
from paper_2209_07969_b200 import configs as C  # noqa: E402
from paper_2209_07969_b200.meshing import StructuredLayout  # noqa: E402


def coarsen(L: StructuredLayout):
    """Coarse layout of L (every 2x2 block of cells -> one cell), or None."""
    if L.nx % 2 or L.ny % 2 or L.ny < 4 or L.nx < 4:
        return None
    ny = L.ny // 2
    elo = np.zeros(ny, np.int32)
    ehi = np.zeros(ny, np.int32)
    for J in range(ny):
        a, b = 2 * J, 2 * J + 1
        if L.elem_lo[a] != L.elem_lo[b] or L.elem_hi[a] != L.elem_hi[b]:
            return None
        if L.elem_lo[a] % 2 or L.elem_hi[a] % 2:
            return None
        elo[J], ehi[J] = L.elem_lo[a] // 2, L.elem_hi[a] // 2
    nlo = np.zeros(ny + 1, np.int32)
    nhi = np.zeros(ny + 1, np.int32)
    for J in range(ny + 1):
        lo, hi = int(L.node_lo[2 * J]), int(L.node_hi[2 * J])
        if lo % 2 or (hi - 1) % 2:
            return None
        nlo[J], nhi[J] = lo // 2, (hi - 1) // 2 + 1
    cnt = (nhi - nlo).astype(np.int64)
    nst = np.concatenate([[0], np.cumsum(cnt)[:-1]])
    ecnt = (ehi - elo).astype(np.int64)
    est = np.concatenate([[0], np.cumsum(ecnt)[:-1]])
    n_reg = int(cnt.sum())
    if L.notch_row >= 0:
        if L.notch_row % 2 or L.notch_lo % 2 or L.notch_hi % 2:
            return None
        nr, nl, nh = L.notch_row // 2, L.notch_lo // 2, L.notch_hi // 2
        n_nodes = n_reg + (nh - nl)
    else:
        nr, nl, nh = -1, 0, 0
        n_nodes = n_reg
    return StructuredLayout(L.nx // 2, ny, 2 * L.hx, 2 * L.hy, nlo, nhi, nst, elo, ehi, est,
                            nr, nl, nh, n_reg if nr >= 0 else 0, n_nodes, int(ecnt.sum()))


def node_lookup(L, i, j, above):
    """Node id at grid (i, j); `above`: seen from the cells above the slit."""
    if j < 0 or j > L.ny or i < L.node_lo[j] or i >= L.node_hi[j]:
        return -1
    if above and j == L.notch_row and L.notch_lo <= i < L.notch_hi:
        return L.dup_start + (i - L.notch_lo)
    return int(L.node_start[j] + (i - L.node_lo[j]))


def prolongation(Lf, Lc):
    """Bilinear nodal interpolation coarse -> fine (scalar, n_f x n_c)."""
    rows, cols, vals = [], [], []
    # fine node list with (i, j, above)
    for j in range(Lf.ny + 1):
        for i in range(Lf.node_lo[j], Lf.node_hi[j]):
            nid = node_lookup(Lf, i, j, False)
            entries = [(nid, i, j, False)]
            if j == Lf.notch_row and Lf.notch_lo <= i < Lf.notch_hi:
                entries.append((node_lookup(Lf, i, j, True), i, j, True))
            for nid, i_, j_, up in entries:
                # side: fine rows above the slit row (or the dup) see coarse dups
                side_above = up or (Lf.notch_row >= 0 and j_ > Lf.notch_row)
                Is = [(i_ // 2, 1.0)] if i_ % 2 == 0 else [((i_ - 1) // 2, 0.5), ((i_ + 1) // 2, 0.5)]
                Js = [(j_ // 2, 1.0)] if j_ % 2 == 0 else [((j_ - 1) // 2, 0.5), ((j_ + 1) // 2, 0.5)]
                for I, wx in Is:
                    for J, wy in Js:
                        cid = node_lookup(Lc, I, J, side_above)
                        if cid < 0:
                            raise RuntimeError(f"missing coarse node {(I, J)} for fine {(i_, j_)}")
                        rows.append(nid)
                        cols.append(cid)
                        vals.append(wx * wy)
    return sp.csr_matrix((vals, (rows, cols)), shape=(Lf.n_nodes, Lc.n_nodes))


def vec2(P):
    return sp.kron(P, sp.eye(2), format="csr")


class MG:
    def __init__(self, A, layouts, Ps, smoother="jacobi", omega=None, nu=1, coarse_max=400,
                 cheb_deg=2, lmax_mode="power"):
        self.lmax_mode = lmax_mode
        self.A = [A]
        self.P = []
        self.smoother = smoother
        self.nu = nu
        self.cheb_deg = cheb_deg
        for P in Ps:
            Ac = (P.T @ self.A[-1] @ P).tocsr()
            self.P.append(P)
            self.A.append(Ac)
            if Ac.shape[0] <= coarse_max:
                break
        self.levels = len(self.A)
        self.dinv = []
        self.lmax = []
        for Al in self.A:
            dg = Al.diagonal().copy()
            inv = np.where(dg > 0, 1.0 / np.where(dg > 0, dg, 1), 0.0)
            self.dinv.append(inv)
            if smoother == "l1":
                l1 = np.asarray(abs(Al).sum(axis=1)).ravel()
                self.dinv[-1] = np.where(l1 > 0, 1.0 / np.where(l1 > 0, l1, 1), 0.0)
            # lambda_max(D^-1 A) by power iteration (setup only)
            v = np.random.default_rng(0).standard_normal(Al.shape[0]) * (dg > 0)
            lam = 1.0
            for _ in range(30):
                w = inv * (Al @ v)
                lam = np.linalg.norm(w) / max(np.linalg.norm(v), 1e-300)
                v = w / max(np.linalg.norm(w), 1e-300)
            if self.lmax_mode == "gersh":
                lam = float(np.max(inv * np.asarray(abs(Al).sum(axis=1)).ravel()))
            self.lmax.append(lam)
        self.omega = omega
        Ac = self.A[-1].toarray()
        keep = np.diag(Ac) > 0
        self.keep = keep
        self.coarse_inv = np.zeros_like(Ac)
        self.coarse_inv[np.ix_(keep, keep)] = np.linalg.inv(Ac[np.ix_(keep, keep)])

    def smooth(self, l, x, b):
        A, inv = self.A[l], self.dinv[l]
        if self.smoother == "cheb":
            # Chebyshev on [lmax/ratio, 1.1 lmax] of D^-1 A (symmetric polynomial smoother)
            lmax = 1.1 * self.lmax[l]
            lmin = lmax / 4.0
            theta, delta = 0.5 * (lmax + lmin), 0.5 * (lmax - lmin)
            sigma = theta / delta
            rho = 1.0 / sigma
            r = b - A @ x
            d = inv * r / theta
            for k in range(self.cheb_deg):
                x = x + d
                if k == self.cheb_deg - 1:
                    break
                r = r - A @ d
                rho_new = 1.0 / (2.0 * sigma - rho)
                d = rho_new * rho * d + 2.0 * rho_new / delta * inv * r
                rho = rho_new
            return x
        om = self.omega if self.omega is not None else (
            1.0 if self.smoother == "l1" else 4.0 / (3.0 * self.lmax[l]))
        for _ in range(self.nu):
            x = x + om * inv * (b - A @ x)
        return x

    def vcycle(self, l, b):
        if l == self.levels - 1:
            return self.coarse_inv @ b
        x = self.smooth(l, np.zeros_like(b), b)
        r = b - self.A[l] @ x
        ec = self.vcycle(l + 1, self.P[l].T @ r)
        x = x + self.P[l] @ ec
        return self.smooth(l, x, b)


def pcg(A, b, M, rtol=1e-12, maxiter=100000):
    x = np.zeros_like(b)
    r = b.copy()
    bn = np.linalg.norm(b)
    z = M(r)
    p = z.copy()
    rz = r @ z
    for it in range(1, maxiter + 1):
        q = A @ p
        pq = p @ q
        alpha = rz / pq
        x += alpha * p
        r -= alpha * q
        if np.linalg.norm(r) < rtol * bn:
            return x, it
        z = M(r)
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, maxiter


def build_system(name, state=None):
    case = C.get_case(name)
    api = oracle_api()
    pb = C.setup(case, api)
    mesh = pb.mesh
    disc = Disc(mesh)
    orc = Oracle(disc, pb.params, pb.config)
    u, d = state if state is not None else (pb.state.u, pb.state.d)
    R, K = orc.momentum_system(u, d)
    fixed = np.unique(np.concatenate([np.asarray(x) for x, _ in pb.bcs]))
    keep = np.ones(K.shape[0])
    keep[fixed] = 0.0
    Mk = sp.diags(keep)
    A = (Mk @ K @ Mk).tocsr()
    return A, -R * keep, keep, StructuredLayout.from_mesh(mesh), pb


def hierarchy(L, keep, max_levels=20):
    Ls, Ps = [L], []
    Lc = coarsen(L)
    while Lc is not None and len(Ls) < max_levels:
        P = vec2(prolongation(Ls[-1], Lc))
        if not Ps:
            P = sp.diags(keep) @ P
        Ps.append(P.tocsr())
        Ls.append(Lc)
        Lc = coarsen(Lc)
    return Ls, Ps


def study(A, b, keep, L, label):
    Ls, Ps = hierarchy(L, keep)
    print(f"[{label}] n={A.shape[0]} levels={[ (l.nx, l.ny) for l in Ls]}")
    # Jacobi reference count
    dg = A.diagonal()
    inv = np.where(dg > 0, 1.0 / np.where(dg > 0, dg, 1), 0.0)
    if A.shape[0] < 30000:
        _, it = pcg(A, b, lambda r: inv * r)
        print(f"  jacobi-pcg iters {it}")
    for sm, nu, om, deg, lm in [("jacobi", 1, None, 0, "power"), ("jacobi", 1, None, 0, "gersh"),
                                ("l1", 1, None, 0, "power"),
                                ("cheb", 1, None, 2, "power"), ("cheb", 1, None, 2, "gersh"),
                                ("cheb", 1, None, 3, "gersh")]:
        t0 = time.perf_counter()
        mg = MG(A, Ls, Ps, smoother=sm, nu=nu, omega=om, cheb_deg=deg, lmax_mode=lm)
        x, it = pcg(A, b, lambda r: mg.vcycle(0, r))
        tr = np.linalg.norm(b - A @ x) / np.linalg.norm(b)
        print(f"  {sm:6s} {lm} nu={nu} deg={deg} levels={mg.levels} iters={it} true_rel={tr:.2e} "
              f"lmax={[round(v, 2) for v in mg.lmax[:3]]} ({time.perf_counter() - t0:.1f}s)")


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
    if which == "cfg1":
        z = np.load("tests/golden/run_cfg1_ST.npz")
        for step in (10, 60, 64, 65):
            A, b, keep, L, pb = build_system("cfg1", (z[f"u_step{step}"], z[f"d_step{step}"]))
            if np.linalg.norm(b) == 0:
                b = np.random.default_rng(1).standard_normal(A.shape[0]) * keep
            study(A, b, keep, L, f"cfg1 step {step}")
    else:
        # synthetic crack state on a bigger notched mesh: d = exp(-|dy|/l) behind a crack tip
        name = which
        case = C.get_case(name)
        A0, b0, keep, L, pb = build_system(name)
        X = np.asarray(pb.mesh.nodes)
        side = case.mesh[3]
        l = case.material["length_l"]
        tip = 0.5 * side + 0.3 * side
        dist = np.where(X[:, 0] < tip, np.abs(X[:, 1] - 0.5 * side),
                        np.hypot(X[:, 0] - tip, X[:, 1] - 0.5 * side))
        d = np.exp(-dist / l)
        u = np.zeros(2 * X.shape[0])
        u[1::2] = 6e-3 * X[:, 1] / side * (1 + 0.3 * np.sin(7 * X[:, 0] / side))
        u[0::2] = -1e-3 * X[:, 0] / side
        A, b, keep, L, pb = build_system(name, (u, d))
        b = np.random.default_rng(1).standard_normal(A.shape[0]) * keep
        study(A, b, keep, L, f"{name} synthetic crack")


# ---- element-wise Galerkin hierarchy (the form the CUDA setup uses) ---------------------
def child_interp():
    """Q[c][a_child_corner][A_parent_corner]: bilinear weights; children c = (a, b) offsets
    (0,0),(1,0),(0,1),(1,1) inside the parent cell; corners CCW from (-,-)."""
    corners = [(0, 0), (1, 0), (1, 1), (0, 1)]
    Q = np.zeros((4, 4, 4))
    for c, (ox, oy) in enumerate([(0, 0), (1, 0), (0, 1), (1, 1)]):
        for a, (cx, cy) in enumerate(corners):
            x, y = 0.5 * (ox + cx), 0.5 * (oy + cy)
            for A, (X, Y) in enumerate(corners):
                Q[c, a, A] = (x if X else 1 - x) * (y if Y else 1 - y)
    return Q


def fine_cell_mats(orc, u, d, keep):
    D = orc.disc
    exx, eyy, gxy = orc.strain(u)
    Cm = orc.tangent(exx + eyy, D.at_gp(d))
    Ke = np.einsum("egia,egij,egjb,eg->eab", D.B, Cm, D.B, D.w)
    kd = keep[D.udofs]
    return Ke * kd[:, :, None] * kd[:, None, :]


def coarse_cell_mats(Lf, Lc, Kf):
    Q = child_interp()
    Q2 = np.einsum("cap,ij->caipj", Q, np.eye(2)).reshape(4, 8, 8)
    # fine cell index of (ci, cj)
    def cell(L, ci, cj):
        return int(L.elem_start[cj] + (ci - L.elem_lo[cj]))
    KE = np.zeros((Lc.n_elems, 8, 8))
    e = 0
    for J in range(Lc.ny):
        for I in range(Lc.elem_lo[J], Lc.elem_hi[J]):
            for c, (ox, oy) in enumerate([(0, 0), (1, 0), (0, 1), (1, 1)]):
                k = cell(Lf, 2 * I + ox, 2 * J + oy)
                KE[e] += Q2[c].T @ Kf[k] @ Q2[c]
            e += 1
    return KE


def elem_bound(K):
    dg = np.einsum("eaa->ea", K)
    out = np.zeros(K.shape[0])
    for e in range(K.shape[0]):
        m = dg[e] > 0
        if not m.any():
            continue
        s = 1.0 / np.sqrt(dg[e, m])
        Ks = K[e][np.ix_(m, m)] * s[:, None] * s[None, :]
        out[e] = np.linalg.eigvalsh(Ks)[-1]
    return out.max()


def element_check(name="cfg1", step=65):
    z = np.load("tests/golden/run_cfg1_ST.npz")
    u, d = z[f"u_step{step}"], z[f"d_step{step}"]
    A, b, keep, L, pb = build_system(name, (u, d))
    orc = Oracle(Disc(pb.mesh), pb.params, pb.config)
    Ls, Ps = hierarchy(L, keep)
    K = fine_cell_mats(orc, u, d, keep)
    mg = MG(A, Ls, Ps, smoother="jacobi")
    for l in range(1, min(4, mg.levels)):
        K = coarse_cell_mats(Ls[l - 1], Ls[l], K)
        conn = Ls[l].connectivity()
        dofs = np.stack([2 * conn, 2 * conn + 1], -1).reshape(-1, 8)
        n = 2 * Ls[l].n_nodes
        Al = sp.csr_matrix((K.ravel(), (np.repeat(dofs, 8, 1).ravel(), np.tile(dofs, (1, 8)).ravel())),
                           shape=(n, n))
        diff = abs(Al - mg.A[l]).max() / abs(mg.A[l]).max()
        print(f"level {l}: element Galerkin vs global rel diff {diff:.2e}; "
              f"lmax power {mg.lmax[l]:.3f} element bound {elem_bound(K):.3f}")
    K0 = fine_cell_mats(orc, u, d, keep)
    print(f"level 0: lmax power {mg.lmax[0]:.3f} element bound {elem_bound(K0):.3f}")


# ---- operator-dependent (matrix-dependent) prolongation --------------------------------------
def md_prolongation(Lf, Lc, A):
    """Prolongation whose edge / centre weights follow the fine operator's couplings (Dendy-style
    black-box interpolation, scalar weights shared by both displacement components): a fine node
    on a coarse edge takes its two coarse endpoints with weights proportional to its coupling
    strength towards each side; a centre node combines its four edge neighbours' interpolations
    with weights proportional to its couplings to them."""
    A = A.tocsr()

    def strength(f, g):  # coupling magnitude between fine nodes f and g (2x2 block)
        if f < 0 or g < 0:
            return 0.0
        blk = A[2 * f:2 * f + 2, 2 * g:2 * g + 2].toarray()
        return abs(blk[0, 0]) + abs(blk[1, 1])

    P = {}

    def coarse_of(i, j, up):
        return node_lookup(Lc, i // 2, j // 2, up)

    entries = []
    for j in range(Lf.ny + 1):
        for i in range(Lf.node_lo[j], Lf.node_hi[j]):
            entries.append((node_lookup(Lf, i, j, False), i, j, False))
            if j == Lf.notch_row and Lf.notch_lo <= i < Lf.notch_hi:
                entries.append((node_lookup(Lf, i, j, True), i, j, True))
    rows, cols, vals = [], [], []
    # pass 1: coarse-coincident and edge nodes
    for nid, i, j, up in entries:
        side = up or (Lf.notch_row >= 0 and j > Lf.notch_row)
        if i % 2 == 0 and j % 2 == 0:
            P[nid] = {coarse_of(i, j, side): 1.0}
        elif i % 2 == 1 and j % 2 == 0:  # horizontal coarse edge
            fl = node_lookup(Lf, i - 1, j, side) if not (j == Lf.notch_row and not up and Lf.notch_lo <= i - 1 < Lf.notch_hi) else node_lookup(Lf, i - 1, j, False)
            fr = node_lookup(Lf, i + 1, j, side) if not (j == Lf.notch_row and not up and Lf.notch_lo <= i + 1 < Lf.notch_hi) else node_lookup(Lf, i + 1, j, False)
            if j == Lf.notch_row:
                fl = node_lookup(Lf, i - 1, j, up)
                fr = node_lookup(Lf, i + 1, j, up)
            al, ar = strength(nid, fl), strength(nid, fr)
            cl = node_lookup(Lc, (i - 1) // 2, j // 2, side)
            cr = node_lookup(Lc, (i + 1) // 2, j // 2, side)
            s = al + ar
            P[nid] = {cl: al / s, cr: ar / s} if s > 0 else {cl: 0.5, cr: 0.5}
        elif i % 2 == 0 and j % 2 == 1:  # vertical coarse edge
            fb = node_lookup(Lf, i, j - 1, j - 1 == Lf.notch_row)
            ft = node_lookup(Lf, i, j + 1, False)
            ab, at = strength(nid, fb), strength(nid, ft)
            cb = node_lookup(Lc, i // 2, (j - 1) // 2, side)
            ct = node_lookup(Lc, i // 2, (j + 1) // 2, side)
            s = ab + at
            P[nid] = {cb: ab / s, ct: at / s} if s > 0 else {cb: 0.5, ct: 0.5}
    # pass 2: centre nodes from their four edge neighbours
    for nid, i, j, up in entries:
        if i % 2 == 1 and j % 2 == 1:
            nb = [node_lookup(Lf, i - 1, j, False), node_lookup(Lf, i + 1, j, False),
                  node_lookup(Lf, i, j - 1, j - 1 == Lf.notch_row), node_lookup(Lf, i, j + 1, False)]
            a = [strength(nid, g) for g in nb]
            s = sum(a)
            w = {}
            for g, ag in zip(nb, a):
                for c, wc in P[g].items():
                    w[c] = w.get(c, 0.0) + (ag / s if s > 0 else 0.25) * wc
            P[nid] = w
    for nid, w in P.items():
        for c, v in w.items():
            rows.append(nid); cols.append(c); vals.append(v)
    return sp.csr_matrix((vals, (rows, cols)), shape=(Lf.n_nodes, Lc.n_nodes))


def md_hierarchy(L, keep, A, max_levels=20):
    """Levels with matrix-dependent prolongation (Galerkin operators built alongside)."""
    Ls, Ps = [L], []
    Al = A
    Lc = coarsen(L)
    while Lc is not None and len(Ls) < max_levels:
        P = vec2(md_prolongation(Ls[-1], Lc, Al))
        if not Ps:
            P = sp.diags(keep) @ P
        P = P.tocsr()
        Ps.append(P)
        Ls.append(Lc)
        Al = (P.T @ Al @ P).tocsr()
        if Al.shape[0] <= 400:
            break
        Lc = coarsen(Lc)
    return Ls, Ps


def compare_interp(name="cfg1", steps=(10, 64, 65)):
    z = np.load("tests/golden/run_cfg1_ST.npz")
    for step in steps:
        A, b, keep, L, pb = build_system(name, (z[f"u_step{step}"], z[f"d_step{step}"]))
        if np.linalg.norm(b) == 0:
            b = np.random.default_rng(1).standard_normal(A.shape[0]) * keep
        Ls, Ps = hierarchy(L, keep)
        mg = MG(A, Ls, Ps, smoother="jacobi")
        _, it_b = pcg(A, b, lambda r: mg.vcycle(0, r))
        Ls2, Ps2 = md_hierarchy(L, keep, A)
        mg2 = MG(A, Ls2, Ps2, smoother="jacobi")
        _, it_m = pcg(A, b, lambda r: mg2.vcycle(0, r))
        print(f"cfg1 step {step}: bilinear {it_b} iterations, matrix-dependent {it_m}")
