"""Discretisation handle, Gauss-point state and the force functionals (interface mirror).

``Discretization`` keeps the reference's public attributes (``mesh``, ``n_gp``, ``n_u_dofs``,
``n_d_dofs``; ``assembly.py:92-143``) but precomputes nothing per element: the B200 operators
are matrix-free and need only the row-compact layout (``meshing.StructuredLayout``).  At 8192^2
the reference's ``b_u`` alone would need ~51 GB.

``reaction_force`` / ``internal_force`` (``assembly.py:161-171``, ``:315-326``) evaluate the
internal force on the GPU (``pf_reaction_force`` / ``pf_internal_force``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .material import MaterialParams, StrainState, material_key
from .meshing import StructuredLayout
from .session import DeviceSession


@dataclass
class GaussPointState:
    """Per-Gauss-point scalars, arrays shaped (n_elems, 4) (reference assembly.py:46-72)."""

    strain: np.ndarray
    tr_eps: np.ndarray
    tr_eps_plus: np.ndarray
    dev_dot_dev: np.ndarray
    psi_plus: np.ndarray
    psi_max: np.ndarray

    @classmethod
    def zeros(cls, n_elems: int, n_gp: int) -> "GaussPointState":
        z = host_zeros
        return cls(strain=z((n_elems, n_gp, 4)), tr_eps=z((n_elems, n_gp)),
                   tr_eps_plus=z((n_elems, n_gp)), dev_dot_dev=z((n_elems, n_gp)),
                   psi_plus=z((n_elems, n_gp)), psi_max=z((n_elems, n_gp)))


PINNED_MAX_BYTES = 256 << 20


def host_zeros(shape) -> np.ndarray:
    """Zeroed float64 state array.  Arrays up to PINNED_MAX_BYTES are page-locked
    (_native.PINNED), so the per-step transfers of the drop-in (staggered_step pushes u, d,
    d_prev, psi_max and updates u, d, psi_max in place) are direct DMA instead of staged copies;
    without a CUDA device (or pinned memory) they are ordinary arrays."""
    n = int(np.prod(shape))
    if 8 * n <= PINNED_MAX_BYTES:
        try:
            from . import _native as N

            a = N.PINNED.empty(shape)
            a[...] = 0.0
            return a
        except Exception:  # no library / no device: pageable state, same semantics
            pass
    return np.zeros(shape)


class Discretization:
    """Bilinear quads with 2x2 Gauss points on a structured uniform grid."""

    def __init__(self, mesh):
        if np.asarray(mesh.elements).shape[1] != 4:
            raise ValueError("only 4-node quadrilaterals are supported here")
        self.mesh = mesh
        self.n_gp = 4
        self.layout = StructuredLayout.from_mesh(mesh)
        self.n_u_dofs = 2 * mesh.n_nodes
        self.n_d_dofs = mesh.n_nodes

    @classmethod
    def from_layout(cls, layout: StructuredLayout) -> "Discretization":
        """A discretisation of a row-compact layout without host node / element arrays
        (``mesh`` is None): config 5's 67 M cells are described by a few row tables."""
        self = cls.__new__(cls)
        self.mesh = None
        self.n_gp = 4
        self.layout = layout
        self.n_u_dofs = 2 * layout.n_nodes
        self.n_d_dofs = layout.n_nodes
        return self

    # field evaluation at Gauss points (assembly.py:148-158), on the device
    def interp_nodal(self, field) -> np.ndarray:
        """Nodal scalar field interpolated at every Gauss point, (n_elems, 4)."""
        return _any_session(self).interp_nodal(field)

    def strain_state(self, u) -> StrainState:
        """Voigt strain at every Gauss point of the displacement ``u`` (eps_zz = 0) and its
        invariants (reference ``strain_state`` + ``StrainState.from_voigt``)."""
        sess = _any_session(self)
        sess.push(u=u)
        strain, _ = sess.gp_strain()
        return StrainState.from_voigt(strain)


def _layout_of(disc) -> StructuredLayout:
    lay = getattr(disc, "layout", None)
    if isinstance(lay, StructuredLayout):
        return lay
    cache = disc.__dict__.setdefault("_pfb200_layout", [])
    if not cache:
        cache.append(StructuredLayout.from_mesh(disc.mesh))
    return cache[0]


def _config_key(cfg) -> tuple:
    return (float(cfg.tol_nr), float(cfg.tol_st), int(cfg.max_nr), int(cfg.max_stag),
            float(cfg.d_cap), float(cfg.res_floor))


class _DefaultConfig:
    tol_nr, tol_st, max_nr, max_stag, d_cap, res_floor, lin_method = (
        1.0e-7, 1.0e-6, 50, 2000, 0.95, 1.0e-12, "direct")


def session_for(disc, params, config=None) -> DeviceSession:
    """The cached ``DeviceSession`` of a discretisation (ours or the reference's)."""
    sessions = disc.__dict__.setdefault("_pfb200_sessions", {})
    if config is None:
        mk = material_key(params)
        for (m, _), s in sessions.items():
            if m == mk:
                return s
        config = _DefaultConfig()
    key = (material_key(params), _config_key(config))
    sess = sessions.get(key)
    if sess is None:
        sess = DeviceSession(_layout_of(disc), params, config)
        sessions[key] = sess
    return sess


def _any_session(disc) -> DeviceSession:
    """A device session of this discretisation for geometry-only operations (interpolation,
    strains): any cached one, else one with placeholder material constants (unused by them)."""
    sessions = disc.__dict__.setdefault("_pfb200_sessions", {})
    if sessions:
        return next(iter(sessions.values()))
    return session_for(disc, MaterialParams(mu=1.0, lam=1.0, g_c=1.0, length_l=1.0))


def internal_force(disc, u, d, params) -> np.ndarray:
    sess = session_for(disc, params)
    sess.push(u=u, d=d)
    return sess.internal_force()


def reaction_force(disc, u, d, params, node_set, component: int) -> float:
    """Resultant of the internal force over a node set (per unit thickness)."""
    sess = session_for(disc, params)
    sess.push(u=u, d=d)
    return float(sess.reaction_force(node_set, component))
