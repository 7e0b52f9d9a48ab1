"""The drop-in boundary exercised with the reference's OWN objects.

A reference runner switched to the B200 path the way INTEGRATION.md §2 shows: the reference
package ``phasefrac`` (installed unmodified under ``baseline/_ref`` by
``pip install --target baseline/_ref``) builds the mesh, ``Discretization``, ``MaterialParams``,
``SolverConfig`` and a ``SolverState`` of ordinary (pageable) numpy arrays; only
``phasefrac.schemes.staggered_step`` and ``phasefrac.assembly.reaction_force`` are replaced by
the drop-ins.  The run must reproduce the reference's golden table, and the reference's
exception classes must catch the drop-in's errors.  Skipped when ``baseline/_ref`` is absent.
"""

import os
import sys

import numpy as np
import pytest

from conftest import ROOT, golden, mirror_perm, stag_band

pytestmark = pytest.mark.gpu

REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def phasefrac():
    if not os.path.isdir(os.path.join(REF, "phasefrac")):
        pytest.skip("reference package not installed under baseline/_ref")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import phasefrac.assembly  # noqa: F401
    import phasefrac.meshing  # noqa: F401
    import phasefrac.schemes  # noqa: F401

    return sys.modules["phasefrac"]


@pytest.fixture()
def patched(phasefrac):
    """the two lines a maintainer adds to a reference runner."""
    from paper_2209_07969_b200 import assembly as b200_assembly
    from paper_2209_07969_b200 import schemes as b200_schemes

    ref_s, ref_a = phasefrac.schemes, phasefrac.assembly
    saved = (ref_s.staggered_step, ref_a.reaction_force)
    ref_s.staggered_step = b200_schemes.staggered_step
    ref_a.reaction_force = b200_assembly.reaction_force
    yield phasefrac
    ref_s.staggered_step, ref_a.reaction_force = saved


def _reference_objects(phasefrac, case_name):
    from paper_2209_07969_b200 import configs as C

    case = C.get_case(case_name)
    _, nx, ny, side, notch = case.mesh
    mesh = phasefrac.meshing.build_notched_square(nx, ny, side, notch_from_left_to_center=notch)
    disc = phasefrac.assembly.Discretization(mesh)
    m = dict(case.material)
    params = phasefrac.material.MaterialParams.from_young_poisson(m.pop("e_mod"), m.pop("nu"),
                                                                  **m)
    cfg = phasefrac.schemes.SolverConfig(tol_st=case.tol_st)
    state = phasefrac.schemes.SolverState.zeros(disc)
    return case, mesh, disc, params, cfg, state


def test_reference_runner_with_dropin(patched, cuda_ok):
    """tension16 S1 through the reference's objects and the patched entry points."""
    from paper_2209_07969_b200 import configs as C

    pf = patched
    z = golden("run_tension16_S1.npz")
    case, mesh, disc, params, cfg, state = _reference_objects(pf, "tension16")
    bcs = C.boundary_conditions(case, mesh)
    u_id = id(state.u)
    tab = z["table"]
    fpeak = np.abs(tab[:, 7]).max()
    band = stag_band("tension16", "S1", len(tab))  # +-1, round-off band at the crack step
    for row, b in zip(tab, band):
        st = pf.schemes.staggered_step(disc, state, pf.schemes.SchemeKind.S1, bcs, params, cfg,
                                       None)
        f = pf.assembly.reaction_force(disc, state.u, state.d, params,
                                       mesh.boundary_sets["top"], 1)
        step = int(row[0])
        assert abs(st.n_stag - int(row[1])) <= b, (step, st.n_stag, row[1], b)
        assert abs(f - row[7]) <= 1e-6 * fpeak, (step, f, row[7])
        assert isinstance(state.gp.psi_plus, np.ndarray) and state.gp.psi_plus.shape == (
            mesh.n_elems, 4)
    assert id(state.u) == u_id  # u updated in place, as the reference does
    # the reference's own post-processing on the drop-in's state
    d_gp = disc.interp_nodal(state.d)
    assert d_gp.shape == (mesh.n_elems, 4)
    ref_d = z["final_d"]
    dinf = min(float(np.abs(state.d - ref_d).max()),
               float(np.abs(state.d - ref_d[mirror_perm(mesh)]).max()))  # crack side
    assert dinf <= 1e-6, dinf


def test_reference_exceptions_catch_dropin_errors(patched, cuda_ok):
    """A non-converging staggered loop raises something ``except
    phasefrac.schemes.ConvergenceError`` catches (schemes.py:366-370), with the history."""
    from paper_2209_07969_b200 import configs as C

    pf = patched
    case, mesh, disc, params, _, state = _reference_objects(pf, "tension16")
    cfg = pf.schemes.SolverConfig(tol_st=1e-5, max_stag=1)
    bcs = C.boundary_conditions(case, mesh)
    with pytest.raises(pf.schemes.ConvergenceError) as exc:
        for _ in range(16):
            pf.schemes.staggered_step(disc, state, pf.schemes.SchemeKind.ST, bcs, params, cfg,
                                      None)
    assert exc.value.residual_history


def test_discretization_helpers_match_reference(phasefrac, cuda_ok):
    """interp_nodal / strain_state of the drop-in's Discretization against the reference's
    (assembly.py:148-158) on seeded fields of a notched and an L-panel mesh."""
    from paper_2209_07969_b200 import assembly, meshing

    for build_ref, build_b200 in (
            (lambda: phasefrac.meshing.build_notched_square(16, 16, 1.0),
             lambda: meshing.build_notched_square(16, 16, 1.0)),
            (lambda: phasefrac.meshing.build_lshape_mesh(25.0),
             lambda: meshing.build_lshape_mesh(25.0))):
        rm, bm = build_ref(), build_b200()
        rd, bd = phasefrac.assembly.Discretization(rm), assembly.Discretization(bm)
        rng = np.random.default_rng(7)
        f = rng.uniform(0.0, 1.0, rm.n_nodes)
        u = rng.standard_normal(2 * rm.n_nodes) * 1e-3
        np.testing.assert_allclose(bd.interp_nodal(f), rd.interp_nodal(f), rtol=0, atol=1e-14)
        rs, bs = rd.strain_state(u), bd.strain_state(u)
        scale = np.abs(rs.eps).max()
        np.testing.assert_allclose(bs.eps, rs.eps, rtol=0, atol=1e-12 * scale)
        np.testing.assert_allclose(bs.tr_eps, rs.tr_eps, rtol=0, atol=1e-12 * scale)
        np.testing.assert_allclose(bs.dev_dot_dev, rs.dev_dot_dev, rtol=0,
                                   atol=1e-12 * scale * scale)
