"""Row-strip decomposition on one GPU: 2-3 strips driven by host threads with the in-process
communicator (pf_comm.h HostComm) must reproduce the reference runs like the single-GPU path.

The strips exchange ghost node rows and all-reduce every scalar exactly as the NCCL path does
(same call sequence, different transport), so this checks the decomposition end to end:
ownership-aware reductions, halo rows, redundant ghost-cell history, slit duplicates on the
owning strip, L-panel rows of different width.
"""

import threading

import numpy as np
import pytest

from conftest import golden, mirror_perm, stag_band
from paper_2209_07969_b200 import configs as C

pytestmark = pytest.mark.gpu


def run_strips(case_name, scheme, nranks, steps=None):
    from paper_2209_07969_b200.dist import HostGroup, StripSession

    case = C.get_case(case_name)
    pb = C.setup(case, C.b200_api())
    n = case.n_steps if steps is None else steps
    group = HostGroup(nranks)
    results = [None] * nranks
    kinds = [None] * nranks
    errors = []

    def worker(rank):
        try:
            ss = StripSession(pb.disc.layout, pb.params, pb.config, rank, nranks, group,
                              device=0)
            s = pb.state
            ss.push_global(s.u, s.d, s.d_prev, s.gp.tr_eps_plus, s.gp.dev_dot_dev,
                           s.gp.psi_plus, s.gp.psi_max)
            rec = []
            for _ in range(n):
                st = ss.step(scheme, pb.bcs, pb.pins)
                reac = [ss.reaction_force(nodes, comp) for _, nodes, comp in pb.reactions]
                rec.append((st.n_stag, st.n_nr_u, st.n_nr_d, st.spd_fallbacks, reac,
                            st.cg_iters_u, st.cg_iters_d))
            kinds[rank] = ss.sess.solver_kinds()
            results[rank] = (rec, ss.owned_state())
            ss.close()
        except Exception as exc:  # noqa: BLE001
            errors.append((rank, repr(exc)))
            raise

    threads = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(nranks)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=600)
    group.close()
    assert not errors, errors
    assert all(r is not None for r in results)
    d = np.empty(pb.mesh.n_nodes)
    for _, own in results:
        d[own["nodes"]] = own["d"]
    run_strips.kinds = kinds
    return pb, results[0][0], [r[0] for r in results], d


@pytest.mark.parametrize("case,scheme,nranks", [("tension16", "ST", 2), ("tension16", "S1", 3),
                                                ("lpanel25", "S1", 2), ("multicrack32", "ST", 3)])
def test_strips_match_reference(case, scheme, nranks, cuda_ok):
    z = golden(f"run_{case}_{scheme}.npz")
    tab = z["table"]
    pb, rec, all_rec, d = run_strips(case, scheme, nranks)
    for r in all_rec[1:]:  # every strip took the same global decisions
        assert [x[:4] for x in r] == [x[:4] for x in rec]
    band = stag_band(case, scheme, len(tab))
    fpeak = np.abs(tab[:, 7]).max()
    for k, (row, x, b) in enumerate(zip(tab, rec, band)):
        assert abs(x[0] - int(row[1])) <= b, (k + 1, x[0], row[1], b)
        assert abs(x[4][0] - row[7]) <= 1e-6 * fpeak, (k + 1, x[4][0], row[7])
    err = float(np.abs(d - z["final_d"]).max())
    if C.get_case(case).loading == "tension":
        err = min(err, float(np.abs(d - z["final_d"][mirror_perm(pb.mesh)]).max()))
    assert err <= 1e-6, err


def test_strips_equal_single_gpu_before_cracking(cuda_ok):
    """Elastic steps are not chaotic: 2 strips reproduce the single-GPU run to round-off."""
    from paper_2209_07969_b200.session import DeviceSession

    pb1 = C.setup(C.get_case("tension32"), C.b200_api())
    s1 = DeviceSession(pb1.disc.layout, pb1.params, pb1.config, device=0)
    s1.push_state(pb1.state)
    ref = []
    for _ in range(6):
        st = s1.step("S1", pb1.bcs)
        ref.append((st.n_stag, st.n_nr_u, st.n_nr_d, s1.reaction_force(
            pb1.mesh.boundary_sets["top"], 1)))
    d1 = s1.pull()["d"]
    pb, rec, _, d = run_strips("tension32", "S1", 2, steps=6)
    for a, b in zip(ref, rec):
        assert a[:3] == b[:3]
        assert abs(a[3] - b[4][0]) <= 1e-10 * abs(a[3])
    assert np.abs(d - d1).max() <= 1e-10


@pytest.mark.parametrize("case,scheme", [("tension16", "S1"), ("lpanel25", "ST")])
def test_nccl_graph_path_single_rank(case, scheme, cuda_ok):
    """The NCCL transport and the CUDA-graph capture of the distributed PCG (kernels +
    ncclAllReduce per phase) on a 1-rank communicator: same results as the reference."""
    from paper_2209_07969_b200.dist import StripSession, nccl_unique_id

    z = golden(f"run_{case}_{scheme}.npz")
    tab = z["table"]
    pb = C.setup(C.get_case(case), C.b200_api())
    ss = StripSession(pb.disc.layout, pb.params, pb.config, 0, 1, "nccl", device=0,
                      nccl_id=nccl_unique_id())
    s = pb.state
    ss.push_global(s.u, s.d, s.d_prev, s.gp.tr_eps_plus, s.gp.dev_dot_dev, s.gp.psi_plus,
                   s.gp.psi_max)
    band = stag_band(case, scheme, len(tab))
    fpeak = np.abs(tab[:, 7]).max()
    for k, (row, b) in enumerate(zip(tab, band)):
        st = ss.step(scheme, pb.bcs, pb.pins)
        f = ss.reaction_force(*pb.reactions[0][1:])
        assert abs(st.n_stag - int(row[1])) <= b, (k + 1, st.n_stag, row[1])
        assert abs(f - row[7]) <= 1e-6 * fpeak, (k + 1, f, row[7])
    own = ss.owned_state()
    d = np.empty(pb.mesh.n_nodes)
    d[own["nodes"]] = own["d"]
    err = float(np.abs(d - z["final_d"]).max())
    if C.get_case(case).loading == "tension":
        err = min(err, float(np.abs(d - z["final_d"][mirror_perm(pb.mesh)]).max()))
    assert err <= 1e-6, err
    ss.close()


def test_strips_multigrid_preconditioner(cuda_ok, monkeypatch):
    """The strips' multigrid PCG (pf_mgd.cuh: strip-local V-cycles as a block-Jacobi
    preconditioner, ghost rows masked, Krylov recurrence with all-reduces and halo rows) against
    the strips' Jacobi PCG (PFB200_DIST_MG=0): the same load steps, fields to the linear-solve
    accuracy, fewer momentum PCG iterations; and against the reference's table."""
    case, scheme, nranks, steps = "multicrack32", "ST", 2, 6
    runs = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("PFB200_DIST_MG", flag)
        pb, rec, _, d = run_strips(case, scheme, nranks, steps=steps)
        runs[flag] = (rec, d, list(run_strips.kinds))
    (rj, dj, kj), (rm, dm, km) = runs["0"], runs["1"]
    assert all(k["momentum"] == "jacobi_pcg" for k in kj)
    assert all(k["momentum"] == "multigrid_pcg" for k in km)
    assert [x[:2] for x in rj] == [x[:2] for x in rm]
    assert np.abs(dj - dm).max() <= 1e-8
    # one-level block Jacobi: fewer iterations than Jacobi, but no coarse correction across
    # strips (kappa ~ 1 / (H h))
    assert sum(x[5] for x in rm) < sum(x[5] for x in rj)
    z = golden(f"run_{case}_{scheme}.npz")
    fpeak = np.abs(z["table"][:, 7]).max()
    for row, x in zip(z["table"], rm):
        assert abs(x[0] - int(row[1])) <= 1 and abs(x[4][0] - row[7]) <= 1e-6 * fpeak
