"""Phase-field solves on the assembled stencil (pf_st.cuh k_cg_st) against the matrix-free
single-reduction PCG (k_cg_sr<false>).

Both run the same Chronopoulos-Gear recurrence, x0, warm start and stopping test
||r|| < 1e-12 ||b|| on the same system (reference pf.py evolution, solved through linsolve.py's
CG switch); only the operator evaluation differs (assembled rows with D^-1 folded into the
columns vs the cell march), so per-step counts must agree up to the crack step and the fields
to the linear-solve accuracy.  The cases cover the slit (tension / shear / multicrack: duplicated
nodes and the slit-tip slot) and the L-panel's re-entrant row layout.
"""

import numpy as np
import pytest

from paper_2209_07969_b200 import configs as C

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case_name,scheme,steps", [
    ("tension32", "ST", 18), ("shear32", "S1", 12), ("lpanel25", "ST", 12),
    ("multicrack32", "S1", 10), ("tension16", "S2", 16)])
def test_stencil_matches_march(cuda_ok, monkeypatch, case_name, scheme, steps):
    from conftest import stag_band
    from paper_2209_07969_b200.session import DeviceSession

    case = C.get_case(case_name)
    band = stag_band(case_name, scheme, steps)
    calm = int(np.argmax(band > 1)) if np.any(band > 1) else steps
    runs = []
    for st in ("0", "1"):
        monkeypatch.setenv("PFB200_ST_EVO", st)
        monkeypatch.setenv("PFB200_MG_EVO", "0")
        pb = C.setup(case, C.b200_api())
        s = DeviceSession(pb.disc.layout, pb.params, pb.config, device=0)
        s.push_state(pb.state)
        assert s.solver_kinds()["phase_field"] == (
            "stencil_pcg" if st == "1" else "single_reduction_pcg")
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
            assert abs(a.n_nr_d - b.n_nr_d) <= max(0, int(0.1 * a.n_nr_d)), (k, a.n_nr_d, b.n_nr_d)
            # same recurrence: PCG counts within a few iterations per solve
            assert abs(a.cg_iters_d - b.cg_iters_d) <= 2 * max(1, b.n_stag) + 0.02 * a.cg_iters_d, (
                k, a.cg_iters_d, b.cg_iters_d)
        else:
            assert abs(a.n_stag - b.n_stag) <= band[k], (k, a.n_stag, b.n_stag, band[k])
    for key in ("u", "d"):
        scale = max(1.0e-12, float(np.max(np.abs(g0[key]))))
        assert np.max(np.abs(g0[key] - g1[key])) <= 1e-7 * scale, key
