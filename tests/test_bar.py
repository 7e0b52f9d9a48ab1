"""The 1-D bar oracle.  (1) A strip under uniform uniaxial strain whose
staggered fixed point has a closed form per load step (oracle/bar_analytic.py), for AT1 (elastic
phase, then damage) and AT2.  The CPU oracle and the B200 path must both reproduce it: the
phase field stays uniform and equals the closed form after every load step.  (2) The
localizing bar of SPEC.md Appendix C (acceptance #1): the staggered-iteration counts at the
crack step, ST against the fast schemes."""

import numpy as np
import pytest

from oracle import bar_analytic as B

INC, N_STEPS = 1.0e-3, 14


def _run(api, at_model, scheme):
    disc, state, params, config, nodes, mesh = B.bar_problem(api, at_model)
    want = B.analytic_path(params, INC, N_STEPS)
    got = []
    for _ in range(N_STEPS):
        api.staggered_step(disc, state, api.SchemeKind(scheme), B.bar_bcs(nodes, INC), params,
                           config)
        d = np.asarray(state.d)
        assert d.max() - d.min() <= 1e-9 + 1e-7 * abs(d.mean()), (d.min(), d.max())
        got.append(d.mean())
    return np.array(got), want, params


def _check(got, want, params, at_model):
    assert np.max(np.abs(got - want)) <= 1e-6, np.abs(got - want)
    # the path crosses the AT1 threshold psi+ = G_c / (2 c_w l): elastic steps, then damage
    if at_model == "AT1":
        assert want[0] <= 0.0 < want[-1]
    assert want[-1] > 0.4


@pytest.mark.parametrize("at_model", ["AT1", "AT2"])
def test_oracle_bar_matches_closed_form(at_model):
    from oracle.phasefield_oracle import oracle_api

    got, want, params = _run(oracle_api(), at_model, "ST")
    _check(got, want, params, at_model)


@pytest.mark.gpu
@pytest.mark.parametrize("at_model,scheme", [("AT1", "ST"), ("AT2", "ST"), ("AT1", "S1"),
                                             ("AT2", "S3")])
def test_b200_bar_matches_closed_form(cuda_ok, at_model, scheme):
    from paper_2209_07969_b200 import configs as C

    got, want, params = _run(C.b200_api(), at_model, scheme)
    _check(got, want, params, at_model)


# ---- the localizing bar (SPEC.md Appendix C, acceptance #1: SPEC.md:522) ------
def _check_localizing(res):
    """The crack forms within one load step; at that step ST needs 15..35 staggered iterations
    (paper: 25) and the fast schemes 10..24 (paper: 17), strictly fewer than ST."""
    (st_counts, st_k, _), fast = res["ST"], [res[s] for s in ("S1", "S3")]
    n_st = st_counts[st_k]
    assert 15 <= n_st <= 35, st_counts
    for counts, k, _ in fast:
        assert abs(k - st_k) <= 1, (k, st_k)  # same load step (+-1)
        assert 10 <= counts[k] <= 24, counts
        assert counts[k] < n_st, (counts[k], n_st)


def test_oracle_localizing_bar():
    """The oracle reproduces the unmodified reference's bar (tests/golden/bar_localizing.npz,
    make_golden.py bar: ST 23, S1 17, S3 16 staggered iterations at the crack step 40) and
    meets the acceptance bands."""
    from conftest import golden
    from oracle.phasefield_oracle import oracle_api

    api = oracle_api()
    res = {s: B.run_localizing_bar(api, s) for s in ("ST", "S1", "S3")}
    _check_localizing(res)
    z = golden("bar_localizing.npz")
    for s, (counts, k, d) in res.items():
        assert counts == z[f"{s}_n_stag"].tolist() and k == int(z[f"{s}_crack_step"])
        assert np.abs(d - z[f"{s}_d"]).max() <= 1e-9


@pytest.mark.gpu
def test_b200_localizing_bar(cuda_ok):
    from oracle.phasefield_oracle import oracle_api
    from paper_2209_07969_b200 import configs as C

    from conftest import golden

    res = {s: B.run_localizing_bar(C.b200_api(), s) for s in ("ST", "S1", "S3")}
    _check_localizing(res)
    # against the unmodified reference's run: the same crack step, the same localized phase
    # field, staggered counts within +-1 per step
    z = golden("bar_localizing.npz")
    for s, (counts, k, d) in res.items():
        assert k == int(z[f"{s}_crack_step"])
        ref = z[f"{s}_n_stag"]
        assert len(counts) == len(ref) and np.abs(np.array(counts) - ref).max() <= 1, (s, counts)
        assert np.abs(d - z[f"{s}_d"]).max() <= 1e-6
