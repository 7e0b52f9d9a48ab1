"""Pin the CPU oracle (oracle/phasefield_oracle.py) to the UNMODIFIED reference.

The golden fixtures were produced by tests/golden/make_golden.py running /root/reference;
these tests need no GPU and no reference install.
"""

import numpy as np
import pytest

from conftest import KAT_MESHES, golden, golden_meta, kat_mesh, kat_params, rel_err
from oracle.phasefield_oracle import Disc, GPState, Oracle, oracle_api
from paper_2209_07969_b200 import configs as C


class _Cfg:
    tol_nr, tol_st, max_nr, max_stag, d_cap, res_floor, lin_method = (
        1e-7, 1e-6, 50, 2000, 0.95, 1e-12, "direct")


@pytest.mark.parametrize("mesh", KAT_MESHES)
@pytest.mark.parametrize("tag", ["at2", "at1"])
def test_oracle_kernel_kats(mesh, tag):
    z = golden(f"kat_{mesh}.npz")
    disc = Disc(kat_mesh(mesh))
    assert np.array_equal(disc.conn, z["elements"])
    o = Oracle(disc, kat_params(tag), _Cfg())
    R, K = o.momentum_system(z["u"], z["d"])
    assert rel_err(R, z[f"{tag}_mom_R"]) < 1e-13
    assert rel_err(K @ z["xu"], z[f"{tag}_mom_Kx"]) < 1e-13
    assert rel_err(K.diagonal(), z[f"{tag}_mom_diag"]) < 1e-13
    exx, eyy, gxy = o.strain(z["u"])
    tr, trp, dev2, psi = o.invariants(exx, eyy, gxy)
    assert rel_err(tr, z[f"{tag}_gp_tr"]) < 1e-13
    assert rel_err(psi, z[f"{tag}_gp_psi"]) < 1e-13
    assert rel_err(dev2, z[f"{tag}_gp_dev2"]) < 1e-13
    gp = GPState(trp, dev2, psi, z[f"{tag}_gp_psimax"])
    R, K = o.evolution_system(z["d"], z["d_prev"], psi)
    assert rel_err(R, z[f"{tag}_evo_R"]) < 1e-13
    assert rel_err(K @ z["xd"], z[f"{tag}_evo_Kx"]) < 1e-13
    dgp = disc.at_gp(z["d"])
    assert np.array_equal(o.gate(gp, dgp), z[f"{tag}_gate"])
    for sk in ("S1", "S2", "S3"):
        ex = o.extra(sk, gp, dgp)
        np.testing.assert_allclose(ex, z[f"{tag}_{sk}_extra"], rtol=1e-13, atol=0)
        R, K = o.evolution_system(z["d"], z["d_prev"], psi, ex)
        assert rel_err(K @ z["xd"], z[f"{tag}_{sk}_evo_Kx"]) < 1e-13
        t, dv, ps = o.update_energy(sk, gp, disc.at_gp(z[f"{tag}_dd"]), dgp, o.gate(gp, dgp))
        assert rel_err(t, z[f"{tag}_{sk}_upd_trp"]) < 1e-13
        assert rel_err(dv, z[f"{tag}_{sk}_upd_dev2"]) < 1e-13
        assert rel_err(ps, z[f"{tag}_{sk}_upd_psi"]) < 1e-13
    assert rel_err(o.internal_force(z["u"], z["d"]), z[f"{tag}_fint"]) < 1e-13


def test_spec_pointwise_kats():
    """SPEC.md examples (split_energies :136-138, stress :145-147, update :296-299)."""
    from paper_2209_07969_b200.material import MaterialParams

    p = MaterialParams(mu=1.0, lam=1.0 - 2.0 / 3.0, g_c=1.0, length_l=1.0, eta=0.0)
    assert abs(p.bulk_k - 1.0) < 1e-15
    o = Oracle.__new__(Oracle)
    o.p, o.cfg = p, _Cfg()
    # eps = diag(1, 1, 0): psi+ = 8/3
    _, _, _, psi = o.invariants(np.array(1.0), np.array(1.0), np.array(0.0))
    assert abs(psi - 8.0 / 3.0) < 1e-14
    # d = 0, eps = diag(1, 0, 0) -> sigma_xx = 7/3, sigma_yy = 1/3
    s = o.stress(np.array(1.0), np.array(0.0), np.array(0.0), np.array(0.0))
    np.testing.assert_allclose(s[:2], [7.0 / 3.0, 1.0 / 3.0], rtol=1e-14)
    # d = 1, eta = 0, eps = diag(-1, -1, 0) -> -2 I
    s = o.stress(np.array(-1.0), np.array(-1.0), np.array(0.0), np.array(1.0))
    np.testing.assert_allclose(s, [-2.0, -2.0, 0.0], atol=1e-14)
    # update_active_energy: d = 0, dd = 0.1, tr+ = 1, dev2 = 1 -> S3 psi 2.16, S1 1.72, S2 1.94
    gp = GPState(np.ones(1), np.ones(1), np.ones(1), np.zeros(1))
    for sk, want in (("S1", 1.72), ("S2", 1.94), ("S3", 2.16)):
        _, _, psi = o.update_energy(sk, gp, np.array([0.1]), np.zeros(1), np.array([True]))
        assert abs(psi[0] - want) < 1e-12, (sk, psi)


def _compare_run(case, scheme, recs, z, state=None):
    tab = z["table"]
    fcol = 7
    fpeak = np.abs(tab[:, fcol]).max()
    out = []
    for r, row in zip(recs, tab):
        d_stag = abs(r.n_stag - int(row[1]))
        d_force = abs(r.reactions[0] - row[fcol]) / fpeak
        out.append((r.step, d_stag, d_force))
    return out


@pytest.mark.parametrize("case,scheme", [("tension16", "ST"), ("tension16", "S1"),
                                         ("lpanel25", "S1"), ("multicrack32", "ST")])
def test_oracle_matches_reference_runs(case, scheme):
    z = golden(f"run_{case}_{scheme}.npz")
    pb = C.setup(C.get_case(case), oracle_api())
    recs = C.run(pb, scheme)
    assert len(recs) == len(z["table"])
    for step, d_stag, d_force in _compare_run(case, scheme, recs, z):
        assert d_stag <= 1, (step, d_stag)
        assert d_force <= 1e-6, (step, d_force)
    assert np.abs(pb.state.d - z["final_d"]).max() <= 1e-6
