"""SPEC.md acceptance properties #2 and #3, on the CPU oracle and on the device
operators.

#2  Fixed-stress first-order invariance: for 1000 random Gauss-point states (d in [0, 0.9],
    tr eps > 0, gate open) the stress invariants reconstructed after the S3 update,
    I1 = g(d + dd) k tr+ and sqrt(J2) ~ g(d + dd) sqrt(dev.dev), differ from their values before
    the update by O(dd^2): least-squares log-log slope >= 1.9 over dd in {1e-2, 1e-3, 1e-4, 1e-5}
    (reference update_active_energy, schemes.py:145-176).
#3  Jacobian consistency: K_uu and K_dd (frozen coupling) match central finite differences of
    their residuals on a random small patch, relative error < 1e-5 (assembly.py:174-247); and
    K~(S3) = K~(S1) + K~(S2) (extra_stiffness, schemes.py:112-142).
"""

import numpy as np
import pytest

from paper_2209_07969_b200 import configs as C

DDS = np.array([1e-2, 1e-3, 1e-4, 1e-5])


def _params(at_model="AT2"):
    from paper_2209_07969_b200 import material

    return material.MaterialParams.from_young_poisson(210000.0, 0.3, g_c=2.7, length_l=0.05,
                                                      at_model=at_model)


def _invariant_slopes(p, d_gp, trp, dev2, updated):
    """updated(dd) -> (trp_new, dev2_new); returns the log-log slopes of the worst relative
    errors of I1 and sqrt(J2) over DDS."""
    g = lambda x: (1.0 - x) ** 2 + p.eta  # noqa: E731  (material.py:129-138)
    e1, e2 = [], []
    for dd in DDS:
        t_new, v_new = updated(dd)
        i1 = np.abs(g(d_gp + dd) * t_new - g(d_gp) * trp) / (g(d_gp) * trp)
        j2 = np.abs(g(d_gp + dd) * np.sqrt(v_new) - g(d_gp) * np.sqrt(dev2)) / (
            g(d_gp) * np.sqrt(dev2))
        e1.append(i1.max())
        e2.append(j2.max())
    s1 = np.polyfit(np.log(DDS), np.log(e1), 1)[0]
    s2 = np.polyfit(np.log(DDS), np.log(e2), 1)[0]
    return s1, s2, e1, e2


def _random_gp(rng, n, p):
    d = rng.uniform(0.0, 0.9, n)
    trp = rng.uniform(0.02, 0.05, n)  # tr eps > 0, psi+ above psi_crit = G_c / (c_w l)
    dev2 = rng.uniform(1e-4, 1e-3, n)
    psi = p.mu * dev2 + 0.5 * p.bulk_k * trp ** 2
    return d, trp, dev2, psi


def test_oracle_fixed_stress_second_order():
    from oracle.phasefield_oracle import GPState, Oracle, oracle_api

    p = _params()
    pb = C.setup(C.get_case("tension16"), oracle_api())
    o = Oracle(pb.disc, p, pb.config)
    rng = np.random.default_rng(20220916)
    d, trp, dev2, psi = _random_gp(rng, 1000, p)
    assert np.all(psi > p.g_c / (p.c_w * p.length_l))  # the gate is open
    gp = GPState(trp, dev2, psi, np.zeros_like(psi))
    mask = o.gate(gp, d)
    assert mask.all()

    def upd(dd):
        t, v, _ = o.update_energy("S3", gp, np.full_like(d, dd), d, mask)
        return t, v

    s1, s2, e1, e2 = _invariant_slopes(p, d, trp, dev2, upd)
    assert s1 >= 1.9 and s2 >= 1.9, (s1, s2, e1, e2)


def test_oracle_extra_stiffness_additive():
    from oracle.phasefield_oracle import GPState, Oracle, oracle_api

    p = _params()
    pb = C.setup(C.get_case("tension16"), oracle_api())
    o = Oracle(pb.disc, p, pb.config)
    rng = np.random.default_rng(3)
    ne = pb.mesh.n_elems
    d, trp, dev2, psi = _random_gp(rng, 4 * ne, p)
    gp = GPState(trp.reshape(ne, 4), dev2.reshape(ne, 4), psi.reshape(ne, 4), np.zeros((ne, 4)))
    dgp = d.reshape(ne, 4)
    k1, k2, k3 = (o.extra(s, gp, dgp) for s in ("S1", "S2", "S3"))
    assert np.any(k3 != 0.0)
    np.testing.assert_allclose(k3, k1 + k2, rtol=1e-14, atol=0.0)


def _patch(api):
    mesh = api.build_notched_square(4, 4, 1.0, notch_from_left_to_center=False)
    rng = np.random.default_rng(11)
    u = rng.standard_normal(2 * mesh.n_nodes) * 1e-3
    d = rng.uniform(0.0, 0.8, mesh.n_nodes)
    d_prev = d - rng.uniform(0.0, 0.05, mesh.n_nodes)  # away from the penalty kink
    return mesh, u, d, d_prev, rng


def test_oracle_jacobian_fd():
    from oracle.phasefield_oracle import Disc, Oracle, oracle_api

    api = oracle_api()
    mesh, u, d, d_prev, rng = _patch(api)
    p = _params()
    o = Oracle(Disc(mesh), p, api.SolverConfig())
    x = rng.standard_normal(2 * mesh.n_nodes)
    _, K = o.momentum_system(u, d)
    eps = 1e-7 * np.abs(u).max()
    fd = (o.internal_force(u + eps * x, d) - o.internal_force(u - eps * x, d)) / (2 * eps)
    assert np.abs(K @ x - fd).max() <= 1e-5 * np.abs(K @ x).max()
    psi = o.disc.at_gp(np.abs(d)) * 1e3  # frozen coupling
    xd = rng.standard_normal(mesh.n_nodes)
    _, Kd = o.evolution_system(d, d_prev, psi)
    e = 1e-7
    fdd = (o.evolution_system(d + e * xd, d_prev, psi, stiffness=False)[0]
           - o.evolution_system(d - e * xd, d_prev, psi, stiffness=False)[0]) / (2 * e)
    assert np.abs(Kd @ xd - fdd).max() <= 1e-5 * np.abs(Kd @ xd).max()


# ---- the same properties on the device operators ---------------------------------------------
@pytest.mark.gpu
def test_gpu_fixed_stress_second_order(cuda_ok):
    from paper_2209_07969_b200.session import DeviceSession

    p = _params()
    api = C.b200_api()
    mesh = api.build_notched_square(16, 16, 1.0, notch_from_left_to_center=False)
    disc = api.Discretization(mesh)
    s = DeviceSession(disc.layout, p, api.SolverConfig(), device=0)
    rng = np.random.default_rng(20220916)
    ne, nn = mesh.n_elems, mesh.n_nodes
    d_nodal = rng.uniform(0.0, 0.9, nn)
    d_gp = s.interp_nodal(d_nodal).ravel()
    _, trp, dev2, psi = _random_gp(rng, 4 * ne, p)

    def upd(dd):
        s.push(u=np.zeros(2 * nn), d=d_nodal, d_prev=d_nodal * 0.0, tr_eps_plus=trp,
               dev_dot_dev=dev2, psi_plus=psi, psi_max=np.zeros(4 * ne))
        s.update_active_energy("S3", np.full(nn, dd))
        got = s.pull()
        return got["tr_eps_plus"].ravel(), got["dev_dot_dev"].ravel()

    # the interpolated increment of a constant nodal dd is dd up to round-off (sum N_a = 1)
    s1, s2, e1, e2 = _invariant_slopes(p, d_gp, trp, dev2, upd)
    assert s1 >= 1.9 and s2 >= 1.9, (s1, s2, e1, e2)
    s.close()


@pytest.mark.gpu
def test_gpu_extra_stiffness_additive(cuda_ok):
    from paper_2209_07969_b200.session import DeviceSession

    p = _params()
    api = C.b200_api()
    mesh = api.build_notched_square(16, 16, 1.0, notch_from_left_to_center=False)
    s = DeviceSession(api.Discretization(mesh).layout, p, api.SolverConfig(), device=0)
    rng = np.random.default_rng(3)
    ne, nn = mesh.n_elems, mesh.n_nodes
    _, trp, dev2, psi = _random_gp(rng, 4 * ne, p)
    s.push(u=np.zeros(2 * nn), d=rng.uniform(0.0, 0.9, nn), d_prev=np.zeros(nn),
           tr_eps_plus=trp, dev_dot_dev=dev2, psi_plus=psi, psi_max=np.zeros(4 * ne))
    k1, k2, k3 = (s.extra_stiffness(sc) for sc in ("S1", "S2", "S3"))
    assert np.any(k3 != 0.0)
    np.testing.assert_allclose(k3, k1 + k2, rtol=1e-14, atol=0.0)
    s.close()


@pytest.mark.gpu
def test_gpu_jacobian_fd(cuda_ok):
    from paper_2209_07969_b200.session import DeviceSession

    api = C.b200_api()
    mesh, u, d, d_prev, rng = _patch(api)
    p = _params()
    s = DeviceSession(api.Discretization(mesh).layout, p, api.SolverConfig(), device=0)
    nn, ne = mesh.n_nodes, mesh.n_elems
    x = rng.standard_normal(2 * nn)
    s.push(u=u, d=d, d_prev=d_prev)
    s.refresh_gp()  # branch bits of the tangent at u
    kx, _ = s.momentum_tangent_apply(x)
    eps = 1e-7 * np.abs(u).max()
    s.push(u=u + eps * x)
    fp = s.internal_force()
    s.push(u=u - eps * x)
    fm = s.internal_force()
    fd = (fp - fm) / (2 * eps)
    assert np.abs(kx - fd).max() <= 1e-5 * np.abs(kx).max()
    # K_dd with frozen coupling (psi+ fixed): residual of the evolution equation in d
    psi = s.interp_nodal(np.abs(d)) * 1e3
    xd = rng.standard_normal(nn)
    s.push(u=u, d=d, d_prev=d_prev, psi_plus=psi, psi_max=np.zeros((ne, 4)))
    kd, _ = s.evolution_tangent_apply("ST", xd)
    e = 1e-7
    s.push(d=d + e * xd)
    rp = s.evolution_residual()
    s.push(d=d - e * xd)
    rm = s.evolution_residual()
    fdd = (rp - rm) / (2 * e)
    assert np.abs(kd - fdd).max() <= 1e-5 * np.abs(kd).max()
    s.close()
