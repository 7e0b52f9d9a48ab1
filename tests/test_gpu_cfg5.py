"""BASELINE configs[4] at FULL size (8192^2 cells, 67.1 M nodes, 201 M DOFs, 256 seeded
pre-cracks, biaxial loading, scheme S1) -- the bench workload.  The reference cannot set this
case up on a CPU (its Discretization alone needs ~120 GB), so parity at
this size is checked through size-independent properties of the reference's formulation and
through a device-vs-device comparison of the two gated-solve paths:

* global equilibrium: the reactions on opposite edges balance (the internal forces of a
  converged state sum to zero over the free dofs, assembly.py:315-326);
* irreversibility and bounds (SPEC.md: d_n >= d_{n-1} - tol_ir, d <= 1) on every node that
  was not seeded, staggered convergence to tol_st.  The seeded one-node-wide d = 1 spikes relax
  over the first load steps (h = 0.12 mm against l = 2 mm: the h-independent gradient stiffness
  outweighs the mass-like penalty gamma h^2 <d - d_prev>_-, so the reference's own formulation
  lets them drop by more than tol_ir; the 256^2 analogue, checked against the reference, does the
  same): there the drop per load step must not grow;
* linearity of the elastic regime (load steps 1..3: damage barely moves, F(k) = k F(1));
* the gated solves by the scalar multigrid PCG with the probe inside against the Jacobi-PCG
  probe (round 1's path): identical staggered / Newton / fallback counts, forces and d.
"""

import numpy as np
import pytest

from paper_2209_07969_b200 import configs as C

pytestmark = pytest.mark.gpu
STEPS = 9  # the S1 gate opens at load step 8


def _run(monkeypatch, gated_mg: bool):
    import torch

    from paper_2209_07969_b200.session import DeviceSession

    free, _ = torch.cuda.mem_get_info(0)
    if free < 60 * 2**30:
        pytest.skip("config 5 needs ~35 GB of device memory")
    monkeypatch.setenv("PFB200_MGS_GATED", "1" if gated_mg else "0")
    case = C.get_case("cfg5")
    dp = C.device_problem(case)
    segs, radius = C.precrack_segments(case)
    lay = dp.layout
    s = DeviceSession(lay, dp.params, dp.config, device=0)
    assert s.solver_kinds()["phase_field"] == "multigrid_pcg"
    s.init_state(segs, radius, lay.nx * lay.hx, lay.ny * lay.hy)
    d0 = np.empty(lay.n_nodes)
    s.pull_into(d=d0)
    seeded = d0 == 1.0
    out = dict(dp=dp, d0=d0, stats=[], forces=[], dmin_inc=[], dmin_seed=[], dmax=[])
    prev = d0.copy()
    cur = np.empty_like(prev)
    b = dp.boundary_sets
    for _ in range(STEPS):
        st = s.step("S1", dp.bcs, dp.pins)
        out["stats"].append((st.n_stag, st.n_nr_u, st.n_nr_d, st.spd_fallbacks,
                             st.final_rd_ratio))
        out["forces"].append(tuple(s.reaction_force(b[k], c) for k, c in (
            ("right", 0), ("left", 0), ("top", 1), ("bottom", 1))))
        s.pull_into(d=cur)
        inc = cur - prev
        out["dmin_inc"].append(float(inc[~seeded].min()))
        out["dmin_seed"].append(float(inc[seeded].min()))
        out["dmax"].append(float(cur.max()))
        prev, cur = cur, prev
    out["d"] = prev
    s.close()
    return out


_CACHE = {}


def _cached(monkeypatch, gated_mg):
    if gated_mg not in _CACHE:
        _CACHE[gated_mg] = _run(monkeypatch, gated_mg)
    return _CACHE[gated_mg]


def test_cfg5_full_size_properties(cuda_ok, monkeypatch):
    r = _cached(monkeypatch, True)
    dp = r["dp"]
    tol_ir, tol_st = dp.params.tol_ir, dp.config.tol_st
    assert int((r["d0"] == 1.0).sum()) > 1000  # the seeded pre-cracks
    for k, ((n_stag, n_u, n_d, fb, rd), (fr, fl, ft, fb_y)) in enumerate(
            zip(r["stats"], r["forces"])):
        assert 1 <= n_stag <= 4 and n_u >= 1 and n_d >= 1, (k, n_stag, n_u, n_d)
        assert rd <= tol_st, (k, rd)
        # equilibrium of the converged state (momentum Newton tolerance 1e-7 of r0)
        assert abs(fr + fl) <= 1e-6 * abs(fr), (k, fr, fl)
        assert abs(ft + fb_y) <= 1e-6 * abs(ft), (k, ft, fb_y)
        assert r["dmin_inc"][k] >= -tol_ir, (k, r["dmin_inc"][k])  # all but the seeded nodes
        # the seeded spikes relax: by less than 0.6 in load step 1, then ever less
        assert r["dmin_seed"][k] >= (-0.6 if k == 0 else min(-tol_ir, r["dmin_seed"][k - 1])), (
            k, r["dmin_seed"])
        assert r["dmax"][k] <= 1.0 + 1e-9, (k, r["dmax"][k])
    assert r["d"].min() >= -tol_ir
    assert np.all(r["d"][r["d0"] == 1.0] >= 0.4)  # the seeded cracks are still cracks
    f1 = r["forces"][0]
    for k in (1, 2):  # load steps 2 and 3 of the elastic regime
        for c in (0, 2):
            assert abs(r["forces"][k][c] / f1[c] - (k + 1)) <= 2e-3 * (k + 1), (k, c)


def test_cfg5_gated_solves_mg_against_jacobi_probe(cuda_ok, monkeypatch):
    a = _cached(monkeypatch, True)
    b = _cached(monkeypatch, False)
    assert any(s[1] >= 1 for s in a["stats"])
    for k, (sa, sb) in enumerate(zip(a["stats"], b["stats"])):
        assert sa[:4] == sb[:4], (k, sa, sb)
    fa, fb = np.array(a["forces"]), np.array(b["forces"])
    assert np.abs(fa - fb).max() <= 1e-9 * np.abs(fb).max()
    assert np.abs(a["d"] - b["d"]).max() <= 1e-8
