"""Drop-in ``staggered_step`` for the reference's solver entry point, backed by the B200 path.

Same signature, argument meaning, return type and errors as the reference
(``schemes.py:332-392``)::

    stats = staggered_step(disc, state, scheme, bc_increments, params, config, pinned_d_nodes)

``disc``/``state``/``params``/``config`` may be this package's types or the reference's own
(duck-typed).  Each call uploads the caller's host ``SolverState``, runs the whole load step on
the GPU (``pf_staggered_step``: momentum Newton + device PCG, evolution Newton with the
fixed-stress predictor and SPD predicate, device-side staggered check), and writes the state
back with the reference's aliasing: ``u`` and ``d`` in place, ``d_prev`` and the GP arrays
rebound (``schemes.py:391``, ``assembly.py:265-269``), ``psi_max`` in place
(``schemes.py:390``).  For device-resident stepping use ``session.DeviceSession`` directly.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from .assembly import Discretization, GaussPointState, host_zeros, session_for  # noqa: F401
from . import _native as N
from .session import ConvergenceError, DeviceSession  # noqa: F401

#: also download gp.strain / gp.tr_eps after every step (faithful GaussPointState mirror)
SYNC_GP_STRAIN = True


class SchemeKind(str, Enum):
    ST = "ST"
    S1 = "S1"
    S2 = "S2"
    S3 = "S3"


@dataclass
class SolverConfig:
    tol_nr: float = 1.0e-7
    tol_st: float = 1.0e-6
    max_nr: int = 50
    max_stag: int = 2000
    d_cap: float = 0.95
    res_floor: float = 1.0e-12
    lin_method: str = "direct"

    def __post_init__(self):
        if not self.tol_st > self.tol_nr:
            raise ValueError("tol_st must exceed tol_nr")
        if not 0.0 < self.d_cap < 1.0:
            raise ValueError("d_cap must lie in (0, 1)")


@dataclass
class StaggeredStats:
    n_stag: int = 0
    n_nr_u: int = 0
    n_nr_d: int = 0
    residual_history: list = field(default_factory=list)
    reaction: float = 0.0
    final_rd_ratio: float = 0.0
    final_ru_ratio: float = 0.0
    spd_fallbacks: int = 0
    wall_u: float = 0.0
    wall_d: float = 0.0


@dataclass
class SolverState:
    u: np.ndarray
    d: np.ndarray
    d_prev: np.ndarray
    gp: GaussPointState

    @classmethod
    def zeros(cls, disc) -> "SolverState":
        z = host_zeros  # page-locked where possible (assembly.host_zeros)
        ne = disc.mesh.n_elems if disc.mesh is not None else disc.layout.n_elems
        return cls(u=z(disc.n_u_dofs), d=z(disc.n_d_dofs), d_prev=z(disc.n_d_dofs),
                   gp=GaussPointState.zeros(ne, disc.n_gp))


def _write_back(sess: DeviceSession, state) -> None:
    """Mirror the device state into the caller's SolverState with the reference's binding
    semantics: u, d and gp.psi_max are updated in place (schemes.py:390, in-place arithmetic),
    d_prev and the refreshed GP arrays are rebound to new arrays (schemes.py:391,
    assembly.py:265-269).  The new arrays are page-locked (direct DMA from the device)."""
    gp = state.gp
    nn, ne = sess.n_nodes, sess.n_elems
    out = {k: N.PINNED.empty(shape) for k, shape in (
        ("d_prev", (nn,)), ("tr_eps_plus", (ne, 4)), ("dev_dot_dev", (ne, 4)),
        ("psi_plus", (ne, 4)))}
    inplace = {}
    for key, arr in (("u", state.u), ("d", state.d), ("psi_max", gp.psi_max)):
        ok = (isinstance(arr, np.ndarray) and arr.dtype == np.float64
              and arr.flags["C_CONTIGUOUS"] and arr.flags["WRITEABLE"])
        inplace[key] = arr if ok else None
        if not ok:
            out[key] = N.PINNED.empty(np.shape(arr))
    sess.pull_into(**out, **{k: v for k, v in inplace.items() if v is not None})
    for key, arr in (("u", state.u), ("d", state.d), ("psi_max", gp.psi_max)):
        if inplace[key] is None:
            arr[...] = out[key]
    state.d_prev = out["d_prev"]
    gp.tr_eps_plus = out["tr_eps_plus"]
    gp.dev_dot_dev = out["dev_dot_dev"]
    gp.psi_plus = out["psi_plus"]
    if SYNC_GP_STRAIN:
        gp.strain, gp.tr_eps = sess.gp_strain(pinned=True)


def staggered_step(disc, state, scheme, bc_increments, params, config,
                   pinned_d_nodes=None) -> StaggeredStats:
    """Advance one loading step with the chosen staggered scheme on the GPU."""
    sess = session_for(disc, params, config)
    # Inputs of a load step: u, d, d_prev, psi_max.  gp.tr_eps_plus / dev_dot_dev / psi_plus are
    # overwritten from u by the first momentum pass (refresh_gp_from_displacement at the end of
    # solve_momentum, schemes.py:237 / assembly.py:260-269) before anything reads them.
    gp = state.gp
    sess.push(u=state.u, d=state.d, d_prev=state.d_prev, psi_max=gp.psi_max)
    try:
        st = sess.step(scheme, bc_increments, pinned_d_nodes)
    except BaseException:
        # the reference leaves the state wherever the failed step stopped: mirror it, but never
        # let a failing download (e.g. after a CUDA fault) replace the solver's own exception
        try:
            _write_back(sess, state)
        except Exception:  # noqa: BLE001
            pass
        raise
    _write_back(sess, state)
    return StaggeredStats(
        n_stag=st.n_stag, n_nr_u=st.n_nr_u, n_nr_d=st.n_nr_d,
        residual_history=list(sess.last_history), final_rd_ratio=st.final_rd_ratio,
        final_ru_ratio=st.final_ru_ratio, spd_fallbacks=st.spd_fallbacks,
        wall_u=st.wall_u, wall_d=st.wall_d)


@dataclass
class StepContext:
    """Per-load-step residual references shared by the inner solvers (schemes.py:179-185)."""

    r0_u: float | None = None
    r0_d: float | None = None
    last_u_ratio: float = 0.0


def solve_momentum(disc, state, constraints, params, config, ctx) -> int:
    """Newton solve of the momentum balance at fixed damage (schemes.py:192-239), on the GPU."""
    sess = session_for(disc, params, config)
    sess.push_state(state)
    n_nr, r0, ratio = sess.solve_momentum(constraints, ctx.r0_u)
    ctx.r0_u, ctx.last_u_ratio = r0, ratio
    _write_back(sess, state)
    return n_nr


def solve_evolution(disc, state, scheme, params, config, ctx, pinned_nodes=None,
                    stats=None) -> int:
    """Newton solve of the damage evolution (schemes.py:242-313), on the GPU."""
    sess = session_for(disc, params, config)
    sess.push_state(state)
    n_nr, r0, fb = sess.solve_evolution(scheme, pinned_nodes, ctx.r0_d)
    ctx.r0_d = r0
    if stats is not None:
        stats.spd_fallbacks += fb
    _write_back(sess, state)
    return n_nr


def evolution_residual_norm(disc, state, params, pinned_nodes=None) -> float:
    """Norm of the evolution residual at the latest (u, d) pair (schemes.py:316-329)."""
    sess = session_for(disc, params)
    sess.push(d=state.d, d_prev=state.d_prev, psi_plus=state.gp.psi_plus)
    return sess.evolution_residual_norm(pinned_nodes)
