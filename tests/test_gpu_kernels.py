"""Kernel-level parity of the B200 operators against the reference's own assembled values.

Fixtures: tests/golden/kat_*.npz (unmodified reference, seeded random states).  Tolerance:
1e-12 relative to the largest entry (FP64 re-association only).  All calls go through the
C-ABI (libpfb200.so) via paper_2209_07969_b200.session.DeviceSession.
"""

import numpy as np
import pytest

from conftest import KAT_MESHES, golden, kat_mesh, kat_params, rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-12


class _Cfg:
    tol_nr, tol_st, max_nr, max_stag, d_cap, res_floor, lin_method = (
        1e-7, 1e-6, 50, 2000, 0.95, 1e-12, "direct")


@pytest.mark.parametrize("prep", ["tile", "march"])
@pytest.mark.parametrize("mesh", KAT_MESHES)
@pytest.mark.parametrize("tag", ["at2", "at1"])
def test_kernels_match_reference(mesh, tag, prep, cuda_ok, monkeypatch):
    """prep: the phase-field residual / coefficient / diagonal kernel as the tile kernel (small
    meshes' default) or as the warp march (big meshes' default, forced here)."""
    from paper_2209_07969_b200.session import DeviceSession

    monkeypatch.setenv("PFB200_EVO_MARCH", "1" if prep == "march" else "0")
    z = golden(f"kat_{mesh}.npz")
    m = kat_mesh(mesh)
    s = DeviceSession(m, kat_params(tag), _Cfg(), device=0)
    s.push(u=z["u"], d=z["d"], d_prev=z["d_prev"])
    # momentum: internal force / residual, tangent-vector product, diagonal
    assert rel_err(s.internal_force(), z[f"{tag}_fint"]) < TOL
    y, dg = s.momentum_tangent_apply(z["xu"])
    assert rel_err(y, z[f"{tag}_mom_Kx"]) < TOL
    assert rel_err(dg, z[f"{tag}_mom_diag"]) < TOL
    # GP refresh
    s.refresh_gp()
    st = s.pull()
    assert rel_err(st["tr_eps_plus"], z[f"{tag}_gp_trp"]) < TOL
    assert rel_err(st["dev_dot_dev"], z[f"{tag}_gp_dev2"]) < TOL
    assert rel_err(st["psi_plus"], z[f"{tag}_gp_psi"]) < TOL
    strain, tr = s.gp_strain()
    assert rel_err(strain, z[f"{tag}_gp_strain"]) < TOL
    assert rel_err(tr, z[f"{tag}_gp_tr"]) < TOL
    s.push(psi_max=z[f"{tag}_gp_psimax"])
    # evolution residual / tangent / diagonal
    assert rel_err(s.evolution_residual(), z[f"{tag}_evo_R"]) < TOL
    y, dg = s.evolution_tangent_apply("ST", z["xd"])
    assert rel_err(y, z[f"{tag}_evo_Kx"]) < TOL
    assert rel_err(dg, z[f"{tag}_evo_diag"]) < TOL
    assert abs(s.evolution_residual_norm() - float(z[f"{tag}_evo_norm"])) <= TOL * float(
        z[f"{tag}_evo_norm"])
    assert np.array_equal(s.softening_gate(), z[f"{tag}_gate"])
    base = (st["tr_eps_plus"], st["dev_dot_dev"], st["psi_plus"])
    for sk in ("S1", "S2", "S3"):
        np.testing.assert_allclose(s.extra_stiffness(sk), z[f"{tag}_{sk}_extra"], rtol=TOL,
                                   atol=TOL * np.abs(z[f"{tag}_{sk}_extra"]).max())
        y, dg = s.evolution_tangent_apply(sk, z["xd"])
        assert rel_err(y, z[f"{tag}_{sk}_evo_Kx"]) < TOL
        assert rel_err(dg, z[f"{tag}_{sk}_evo_diag"]) < TOL
        s.update_active_energy(sk, z[f"{tag}_dd"])
        up = s.pull()
        assert rel_err(up["tr_eps_plus"], z[f"{tag}_{sk}_upd_trp"]) < TOL
        assert rel_err(up["dev_dot_dev"], z[f"{tag}_{sk}_upd_dev2"]) < TOL
        assert rel_err(up["psi_plus"], z[f"{tag}_{sk}_upd_psi"]) < TOL
        s.push(tr_eps_plus=base[0], dev_dot_dev=base[1], psi_plus=base[2])
    key = "top" if "top" in m.boundary_sets else "load_zone"
    want = float(z[f"{tag}_reac_{key}_1"])
    got = s.reaction_force(m.boundary_sets[key], 1)
    assert abs(got - want) <= TOL * np.abs(z[f"{tag}_fint"]).max() * len(m.boundary_sets[key])
    s.close()


def test_operator_symmetry_and_rigid_modes(cuda_ok):
    """K_uu symmetric, rigid-body null space, on a damaged random state."""
    from paper_2209_07969_b200 import meshing
    from paper_2209_07969_b200.session import DeviceSession

    m = meshing.build_notched_square(16, 16, 1.0)
    rng = np.random.default_rng(7)
    s = DeviceSession(m, kat_params("at2"), _Cfg(), device=0)
    nn = m.n_nodes
    s.push(u=rng.standard_normal(2 * nn) * 1e-3, d=rng.uniform(0, 0.9, nn),
           d_prev=np.zeros(nn), psi_plus=rng.uniform(0, 10, (m.n_elems, 4)))
    a, b = rng.standard_normal(2 * nn), rng.standard_normal(2 * nn)
    Ka, _ = s.momentum_tangent_apply(a)
    Kb, _ = s.momentum_tangent_apply(b)
    assert abs(b @ Ka - a @ Kb) <= 1e-12 * abs(b @ Ka)
    x = m.nodes
    for mode in (np.tile([1.0, 0.0], nn), np.tile([0.0, 1.0], nn),
                 np.column_stack([-x[:, 1], x[:, 0]]).ravel()):
        Km, _ = s.momentum_tangent_apply(mode)
        Kr, _ = s.momentum_tangent_apply(rng.standard_normal(2 * nn))
        assert np.abs(Km).max() <= 1e-10 * np.abs(Kr).max()
    a, b = rng.standard_normal(nn), rng.standard_normal(nn)
    Ka, _ = s.evolution_tangent_apply("ST", a)
    Kb, _ = s.evolution_tangent_apply("ST", b)
    assert abs(b @ Ka - a @ Kb) <= 1e-12 * abs(b @ Ka)
    s.close()


def test_fixed_length_pcg_benchmark_entry(cuda_ok):
    """pf_bench_cg runs exactly n PCG iterations (stopping test off) on the rectangle layout
    used for the cfg5-size measurements; the layout equals the one derived from the mesh."""
    from paper_2209_07969_b200 import meshing
    from paper_2209_07969_b200.session import DeviceSession

    lay = meshing.StructuredLayout.rectangle(40, 24, 1.0 / 40, 1.0 / 24)
    ref = meshing.StructuredLayout.from_mesh(meshing.build_notched_square(40, 24, 1.0, False))
    assert np.array_equal(lay.node_start, ref.node_start) and lay.n_elems == ref.n_elems
    s = DeviceSession(lay, kat_params("at2"), _Cfg(), device=0)
    rng = np.random.default_rng(3)
    nn = lay.n_nodes
    s.push(u=1e-3 * rng.standard_normal(2 * nn), d=0.5 * rng.random(nn), d_prev=np.zeros(nn))
    s.refresh_gp()
    for phys in ("momentum", "evolution", "momentum_mg"):
        ms, it = s.bench_cg(phys, 7)
        assert it == 7 and ms > 0.0
    s.close()


def test_state_roundtrip_through_pinned_staging(cuda_ok):
    """pf_set_state / pf_get_state move large states through the pinned staging buffer with
    threaded host copies (>= 4 MB); the round trip is bit-exact and fresh output arrays work."""
    from paper_2209_07969_b200 import meshing
    from paper_2209_07969_b200.session import DeviceSession

    lay = meshing.StructuredLayout.rectangle(300, 300, 1.0 / 300, 1.0 / 300)
    s = DeviceSession(lay, kat_params("at2"), _Cfg(), device=0)
    rng = np.random.default_rng(9)
    nn, ne = lay.n_nodes, lay.n_elems
    want = dict(u=rng.standard_normal(2 * nn), d=rng.random(nn), d_prev=rng.random(nn),
                tr_eps_plus=rng.standard_normal((ne, 4)), dev_dot_dev=rng.random((ne, 4)),
                psi_plus=rng.random((ne, 4)), psi_max=rng.random((ne, 4)))
    assert sum(v.size for v in want.values()) * 8 > 4 << 20
    s.push(**want)
    got = s.pull()
    for k, v in want.items():
        assert np.array_equal(got[k].reshape(v.shape), v), k
    strain, tr = s.gp_strain()
    assert strain.shape == (ne, 4, 4) and np.all(np.isfinite(strain)) and np.all(np.isfinite(tr))
    s.close()
