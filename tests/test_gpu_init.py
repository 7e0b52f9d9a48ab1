"""Device-side state construction (pf_init_state) against the host path.

The zero state of ``SolverState.zeros`` (reference schemes.py:80-87) plus d = d_prev = 1 at the
seeded pre-crack nodes must equal, bit for bit, what ``configs.precrack_nodes`` marks on the
host (the recipe of SURVEY.md 8(d) / App. B config 5), on plain squares (the multi-crack
analogues and a 2048^2 grid with config 5's 256 cracks) and on a notched square (slit positions
mark their duplicate, as the host lookup does).  A load step from the device-built state equals
one from the pushed host state.
"""

from types import SimpleNamespace

import numpy as np
import pytest

from paper_2209_07969_b200 import configs as C
from paper_2209_07969_b200 import meshing

pytestmark = pytest.mark.gpu


def _session(mesh, case_for_material):
    from paper_2209_07969_b200.session import DeviceSession

    api = C.b200_api()
    lay = meshing.StructuredLayout.from_mesh(mesh)
    params = C.material(case_for_material, api)
    return DeviceSession(lay, params, api.SolverConfig(tol_st=1e-5), device=0)


CASES = {
    "multicrack256": None,
    "multicrack32": None,
    "plain2048_256cracks": (("notched", 2048, 2048, 1000.0, False), (256, 20220916, 5.0, 20.0)),
    "notched64_slitcracks": (("notched", 64, 64, 1.0, True), (12, 7, 0.05, 0.5)),
}


@pytest.mark.parametrize("name", list(CASES))
def test_device_precrack_matches_host(cuda_ok, name):
    base = C.get_case("multicrack256")
    spec = CASES[name]
    if spec is None:
        case = C.get_case(name)
    else:
        case = SimpleNamespace(mesh=spec[0], precracks=spec[1])
    _, nx, ny, side, notch = case.mesh
    mesh = meshing.build_notched_square(nx, ny, side, notch)
    want = C.precrack_nodes(case, mesh)
    assert want.size > 0
    segs, radius = C.precrack_segments(case)
    s = _session(mesh, base)
    s.init_state(segs, radius, side, side)
    out = s.pull()
    s.close()
    got = np.flatnonzero(out["d"] == 1.0)
    assert np.array_equal(got, want), (np.setdiff1d(got, want), np.setdiff1d(want, got))
    assert np.array_equal(out["d"], out["d_prev"])
    assert set(np.unique(out["d"])) <= {0.0, 1.0}
    for key in ("u", "tr_eps_plus", "dev_dot_dev", "psi_plus", "psi_max"):
        assert not np.any(out[key]), key


def test_step_from_device_state_equals_pushed_state(cuda_ok):
    case = C.get_case("multicrack32")
    pb = C.setup(case, C.b200_api())
    segs, radius = C.precrack_segments(case)
    side = case.mesh[3]
    from paper_2209_07969_b200.session import DeviceSession

    runs = []
    for device_init in (False, True):
        s = DeviceSession(pb.disc.layout, pb.params, pb.config, device=0)
        if device_init:
            s.init_state(segs, radius, side, side)
        else:
            s.push_state(pb.state)
        stats = [s.step("ST", pb.bcs, pb.pins) for _ in range(3)]
        runs.append(([(x.n_stag, x.n_nr_u, x.n_nr_d, x.cg_iters_u, x.cg_iters_d) for x in stats],
                     s.pull()))
        s.close()
    (a, fa), (b, fb) = runs
    assert a == b
    for key in fa:
        assert np.array_equal(fa[key], fb[key]), key


def test_init_state_without_segments_is_zero_state(cuda_ok):
    from paper_2209_07969_b200.session import DeviceSession

    pb = C.setup(C.get_case("tension16"), C.b200_api())
    s = DeviceSession(pb.disc.layout, pb.params, pb.config, device=0)
    s.push(d=np.ones(pb.mesh.n_nodes))
    s.init_state()
    out = s.pull()
    s.close()
    for key, v in out.items():
        assert not np.any(v), key
