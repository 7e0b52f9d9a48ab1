"""The 1-D bar oracle: a strip under uniform uniaxial strain whose
staggered fixed point has a closed form per load step (oracle/bar_analytic.py), for AT1 (elastic
phase, then damage) and AT2.  The CPU oracle and the B200 path must both reproduce it: the
phase field stays uniform and equals the closed form after every load step."""

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
