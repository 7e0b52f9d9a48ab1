"""Multigrid-preconditioned momentum PCG (pf_mg.cuh k_mgcg) against the Jacobi PCG.

The V-cycle only replaces the preconditioner M = D^-1 of the reference's CG switch
(linsolve.py:48-54); the system, x0 = 0 and the stopping test ||r|| < 1e-12 ||b|| are the same,
so Newton and staggered iteration counts must be identical and the fields must agree to the
linear-solve accuracy.  The end-to-end golden comparisons (test_gpu_solver.py) run with the
multigrid default too.
"""

import numpy as np
import pytest

from paper_2209_07969_b200 import configs as C

pytestmark = pytest.mark.gpu


def _session(case, monkeypatch, mg):
    from paper_2209_07969_b200.session import DeviceSession

    monkeypatch.setenv("PFB200_MG", "1" if mg else "0")
    pb = C.setup(case, C.b200_api())
    s = DeviceSession(pb.disc.layout, pb.params, pb.config, device=0)
    s.push_state(pb.state)
    return pb, s


def test_hierarchy_shapes(cuda_ok, monkeypatch):
    """cfg1 (64^2 notched): 64 -> 32 -> 16 -> 8 -> 4 cells with the slit on every level; the
    4^2 level (27 nodes, 54 dofs) is solved densely inside the single-CTA tail kernel."""
    pb, s = _session(C.get_case("cfg1"), monkeypatch, True)
    info = s.mg_info(with_omega=True)
    assert info["n_levels"] == 5 and info["dense"] and 1 <= info["n_grid"] <= 4
    # lambda_max(D^-1 A) of Q4 elasticity is ~2.3 here: omega = 4 / (3 lambda) ~ 0.58
    assert np.all(info["omega"][:-1] > 0.3) and np.all(info["omega"][:-1] < 0.8)
    s.close()
    _, s0 = _session(C.get_case("cfg1"), monkeypatch, False)
    assert s0.mg_info()["n_levels"] == 0
    s0.close()


@pytest.mark.parametrize("case_name,scheme,steps", [
    ("tension16", "S1", 16), ("tension32", "ST", 18), ("shear32", "S2", 12),
    ("lpanel25", "S1", 12), ("multicrack32", "ST", 10)])
def test_mg_matches_jacobi(cuda_ok, monkeypatch, case_name, scheme, steps):
    """Up to the crack step: the same staggered / Newton counts per load step as the Jacobi
    PCG and the same fields to the linear-solve accuracy; from the crack step on (where the
    reference's own round-off ensemble disagrees, conftest.stag_band > 1) the counts stay
    within that band.  Far fewer PCG iterations throughout.  lpanel25's hierarchy stops at an
    odd level (coarsest by Jacobi sweeps); the others end with a dense coarsest solve."""
    from conftest import stag_band

    case = C.get_case(case_name)
    band = stag_band(case_name, scheme, steps)
    calm = int(np.argmax(band > 1)) if np.any(band > 1) else steps  # steps before the crack
    runs = []
    for mg in (False, True):
        pb, s = _session(case, monkeypatch, mg)
        stats, snap = [], None
        for k in range(steps):
            stats.append(s.step(scheme, pb.bcs, pb.pins))
            if k == calm - 1:
                snap = s.pull()
        runs.append((s.mg_info(), stats, snap))
        s.close()
    (i0, s0, g0), (i1, s1, g1) = runs
    assert i0["n_levels"] == 0 and i1["n_levels"] >= 2
    if case_name == "lpanel25":
        assert not i1["dense"]
    for k, (a, b) in enumerate(zip(s0, s1)):
        if k < calm:
            assert (a.n_stag, a.n_nr_u, a.n_nr_d) == (b.n_stag, b.n_nr_u, b.n_nr_d), k
        else:
            assert abs(a.n_stag - b.n_stag) <= band[k], (k, a.n_stag, b.n_stag, band[k])
    assert calm >= 1
    for key in ("u", "d"):
        scale = max(1.0e-12, float(np.max(np.abs(g0[key]))))
        assert np.max(np.abs(g0[key] - g1[key])) <= 1e-7 * scale, key
    it0 = sum(x.cg_iters_u for x in s0)
    it1 = sum(x.cg_iters_u for x in s1)
    assert it1 * 3 < it0, (it0, it1)


def test_mg_solve_accuracy_cracked_state(cuda_ok, monkeypatch):
    """One momentum Newton solve from the reference's fully cracked cfg1 state (step 65 of the
    golden ST run, g(d) down to 1e-6 along the crack): the MG-PCG reaches the same Newton
    residual path as the Jacobi PCG in a few tens of iterations."""
    from conftest import golden

    z = golden("run_cfg1_ST.npz")
    case = C.get_case("cfg1")
    out = []
    for mg in (False, True):
        pb, s = _session(case, monkeypatch, mg)
        s.push(u=np.ascontiguousarray(z["u_step64"]), d=np.ascontiguousarray(z["d_step65"]),
               d_prev=np.ascontiguousarray(z["d_step64"]))
        zero_bcs = [(dofs, 0.0) for dofs, _ in pb.bcs]
        n_nr, _, ratio = s.solve_momentum(zero_bcs)
        out.append((n_nr, ratio, s.pull()["u"]))
        s.close()
    (n0, r0, u0), (n1, r1, u1) = out
    assert n0 == n1 and n0 >= 1
    assert np.max(np.abs(u0 - u1)) <= 1e-8 * np.max(np.abs(u0))


@pytest.mark.parametrize("kind", ["scalar", "packed"])
@pytest.mark.parametrize("case_name,scheme,steps", [
    ("tension32", "ST", 18), ("shear32", "S1", 12), ("lpanel25", "ST", 12),
    ("multicrack32", "S1", 10)])
def test_phase_field_mg_matches(cuda_ok, monkeypatch, case_name, scheme, steps, kind):
    """Phase-field solves without the SPD probe by the multigrid PCG -- the native scalar
    hierarchy (pf_mgs.cuh, the default on large meshes) and round 1's two-component packing
    (pf_mg.cuh phys 1), forced here -- against the Jacobi / single-reduction PCG: same per-step
    counts up to the crack step, the reference's round-off band after it, fields to the
    linear-solve accuracy, fewer phase-field PCG iterations."""
    from conftest import stag_band
    from paper_2209_07969_b200.session import DeviceSession

    case = C.get_case(case_name)
    band = stag_band(case_name, scheme, steps)
    calm = int(np.argmax(band > 1)) if np.any(band > 1) else steps
    runs = []
    for evo in ("0", kind):
        monkeypatch.setenv("PFB200_MG_EVO", evo)
        pb = C.setup(case, C.b200_api())
        s = DeviceSession(pb.disc.layout, pb.params, pb.config, device=0)
        if evo != "0":
            want = "multigrid_pcg" if kind == "scalar" else "packed_multigrid_pcg"
            assert s.solver_kinds()["phase_field"] == want
        s.push_state(pb.state)
        stats, snap = [], None
        for k in range(steps):
            stats.append(s.step(scheme, pb.bcs, pb.pins))
            if k == calm - 1:
                snap = s.pull()
        runs.append((stats, snap))
        s.close()
    (s0, g0), (s1, g1) = runs
    for k, (a, b) in enumerate(zip(s0, s1)):
        if k < calm:
            assert (a.n_stag, a.n_nr_u) == (b.n_stag, b.n_nr_u), k
            # the phase-field Newton loop of the pre-cracked multi-crack case takes ~35 slowly
            # converging steps whose count moves with the linear solves' round-off: +-10% there
            assert abs(a.n_nr_d - b.n_nr_d) <= max(0, int(0.1 * a.n_nr_d)), (k, a.n_nr_d, b.n_nr_d)
        else:
            assert abs(a.n_stag - b.n_stag) <= band[k], (k, a.n_stag, b.n_stag, band[k])
    for key in ("u", "d"):
        scale = max(1.0e-12, float(np.max(np.abs(g0[key]))))
        assert np.max(np.abs(g0[key] - g1[key])) <= 1e-7 * scale, key
    assert sum(x.cg_iters_d for x in s1) < sum(x.cg_iters_d for x in s0)


@pytest.mark.parametrize("case_name,scheme", [
    ("shear32", "S3"), ("shear32", "S2"), ("tension16", "S2"), ("tension32", "S1"),
    ("multicrack32", "S1")])
def test_gated_solves_by_scalar_mg_match_reference(cuda_ok, monkeypatch, case_name, scheme):
    """The gated solves of the fast schemes (K_dd + K~ with the SPD check, schemes.py:293-301)
    by the scalar multigrid PCG with the probe inside (p.Ap <= 0 => fallback), forced on here
    as on the large meshes: the whole run against the reference's own table -- staggered and
    Newton counts and the spd_fallbacks decisions per step, forces, the final phase field."""
    from conftest import golden
    from test_gpu_solver import check_against_golden, run_case

    monkeypatch.setenv("PFB200_MG_EVO", "scalar")
    z = golden(f"run_{case_name}_{scheme}.npz")
    pb, recs = run_case(case_name, scheme)
    check_against_golden(recs, z, pb.state, case_name, scheme, pb.mesh)
    assert sum(r.spd_fallbacks for r in recs) == pytest.approx(
        z["table"][:, 4].sum(), rel=0.15, abs=3)


@pytest.mark.parametrize("case_name,scheme,steps", [("cfg3", "S3", 40), ("cfg3", "S2", 40)])
def test_gated_mg_against_jacobi_probe_full_size(cuda_ok, monkeypatch, case_name, scheme, steps):
    """BASELINE configs[2] (1024^2 shear, where S2 / S3 fall back often) at full size, where the
    scalar hierarchy is the default: the gated solves with the probe inside the multigrid PCG
    against the Jacobi-PCG probe -- per-step staggered, Newton and fallback counts identical,
    forces to 1e-9."""
    from paper_2209_07969_b200.session import DeviceSession

    dp = C.device_problem(C.get_case(case_name))
    runs = []
    for gated in ("1", "0"):
        monkeypatch.setenv("PFB200_MGS_GATED", gated)
        s = DeviceSession(dp.layout, dp.params, dp.config, device=0)
        assert s.solver_kinds()["phase_field"] == "multigrid_pcg"
        s.init_state()
        rows = []
        for _ in range(steps):
            st = s.step(scheme, dp.bcs, dp.pins)
            f = s.reaction_force(dp.reactions[0][1], dp.reactions[0][2])
            rows.append((st.n_stag, st.n_nr_u, st.n_nr_d, st.spd_fallbacks, f, st.cg_iters_d))
        runs.append(rows)
        s.close()
    a, b = runs
    # the gate did open: the Jacobi-PCG probe solves cost hundreds of iterations each
    assert sum(r[5] for r in b) > 2 * sum(r[5] for r in a)
    fpeak = max(abs(r[4]) for r in b)
    for k, (ra, rb) in enumerate(zip(a, b)):
        assert ra[:4] == rb[:4], (k, ra, rb)
        assert abs(ra[4] - rb[4]) <= 1e-9 * fpeak, (k, ra[4], rb[4])


@pytest.mark.parametrize("case_name,scheme", [("cfg1", "ST"), ("shear32", "S3")])
def test_fp32_coarse_stencils_on_cracked_states(cuda_ok, monkeypatch, case_name, scheme):
    """The V-cycle's grid levels read FP32 copies of the coarse stencils by default.  Through the
    crack (cfg1's fully cracked step 65: g(d) down to 1e-6 next to intact cells; the shear case's
    post-peak S3 steps) the FP32 and FP64 coarse stencils (PFB200_MG_S32=0) give the same
    staggered counts and momentum PCG counts within 10%: the FP32 rounding of the coarse
    couplings does not weaken the preconditioner where the degraded couplings are smallest."""
    from paper_2209_07969_b200.session import DeviceSession

    case = C.get_case(case_name)
    runs = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("PFB200_MG_S32", flag)
        pb = C.setup(case, C.b200_api())
        s = DeviceSession(pb.disc.layout, pb.params, pb.config, device=0)
        s.push_state(pb.state)
        stats = [s.step(scheme, pb.bcs, pb.pins) for _ in range(case.n_steps)]
        runs[flag] = ([x.n_stag for x in stats], [x.cg_iters_u for x in stats], s.pull()["d"])
        s.close()
    from conftest import stag_band

    (st32, it32, d32), (st64, it64, d64) = runs["1"], runs["0"]
    crack = int(np.argmax(st64))
    band = stag_band(case_name, scheme, case.n_steps)  # +-1, the round-off band at crack steps
    for k, (a, b) in enumerate(zip(st32, st64)):
        assert abs(a - b) <= band[k], (k, a, b, band[k])
    assert abs(sum(it32) - sum(it64)) <= 0.1 * sum(it64), (sum(it32), sum(it64))
    post = slice(crack, None)
    assert sum(it32[post]) <= 1.1 * sum(it64[post]) + 5, (it32[post], it64[post])
