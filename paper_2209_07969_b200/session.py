"""Device-resident solver session: one ``pf_handle`` (one GPU, one mesh, one material/config).

``DeviceSession`` owns all device buffers of the hot path.  It is what the drop-in
``schemes.staggered_step`` uses under the hood (uploading the caller's host ``SolverState`` before
and downloading it after every step), and what performance-minded callers use directly to keep
the state resident in HBM across load steps (``step`` / ``pull``).
"""

from __future__ import annotations

import ctypes as C
import math
import os
import sys

import numpy as np

from . import _native as N
from .meshing import StructuredLayout


class ConvergenceError(RuntimeError):
    """Raised when a Newton or staggered loop does not converge (schemes.py:90-93)."""

    def __init__(self, message: str, residual_history=None):
        super().__init__(message)
        self.residual_history = residual_history or []


class SingularSystemError(RuntimeError):
    """Linear-solver failure (linsolve.py:18-21)."""

    def __init__(self, message: str, pivot_index: int | None = None):
        super().__init__(message)
        self.pivot_index = pivot_index


class DeviceError(RuntimeError):
    """CUDA / NCCL failure inside the native library."""


_REF_ERRORS = {ConvergenceError: ("phasefrac.schemes", "ConvergenceError"),
               SingularSystemError: ("phasefrac.linsolve", "SingularSystemError")}
_COMBINED: dict = {}


def reference_error(cls):
    """The class to raise for one of the reference's exceptions: when the caller has imported
    the reference package (``phasefrac``, e.g. a reference runner switched to the drop-in), a
    subclass of both this package's class and the reference's own (``schemes.py:90-93``,
    ``linsolve.py:18-21``), so ``except phasefrac.schemes.ConvergenceError`` handlers keep
    working; otherwise the local class."""
    modname, name = _REF_ERRORS[cls]
    ref = getattr(sys.modules.get(modname), name, None)
    if not isinstance(ref, type) or issubclass(cls, ref):
        return cls
    combo = _COMBINED.get((cls, ref))
    if combo is None:
        combo = type(cls.__name__, (cls, ref), {"__module__": cls.__module__})
        _COMBINED[(cls, ref)] = combo
    return combo


def scheme_code(scheme) -> int:
    name = getattr(scheme, "value", scheme)
    try:
        return N.SCHEME_CODES[str(name)]
    except KeyError:
        raise ValueError(f"unknown scheme {scheme!r}") from None


def pack_bcs(bc_increments) -> tuple:
    """``[(dof_array, inc), ...]`` -> (dofs int64, offsets int64, incs float64, n)."""
    arrays = [np.ascontiguousarray(np.asarray(d, dtype=np.int64).ravel()) for d, _ in bc_increments]
    incs = np.array([float(i) for _, i in bc_increments], dtype=np.float64)
    offsets = np.zeros(len(arrays) + 1, dtype=np.int64)
    if arrays:
        offsets[1:] = np.cumsum([a.size for a in arrays])
        dofs = np.ascontiguousarray(np.concatenate(arrays))
    else:
        dofs = np.zeros(1, dtype=np.int64)
    return dofs, offsets, incs if incs.size else np.zeros(1), len(arrays)


def _pins(pinned) -> tuple:
    if pinned is None:
        return None, 0
    p = np.ascontiguousarray(np.asarray(pinned, dtype=np.int64).ravel())
    return (p, p.size) if p.size else (None, 0)


class DeviceSession:
    """All device state for one (mesh, material, solver-config) triple on one GPU."""

    def __init__(self, mesh_or_layout, params, config, device: int | None = None,
                 strip=None):
        self.lib = N.load()
        lay = (mesh_or_layout if isinstance(mesh_or_layout, StructuredLayout)
               else StructuredLayout.from_mesh(mesh_or_layout))
        self.layout = lay
        self.n_nodes, self.n_elems = lay.n_nodes, lay.n_elems
        if device is None:
            device = int(os.environ.get("PFB200_DEVICE", os.environ.get("LOCAL_RANK", "0")))
        self.device = device
        self._keep = dict(
            nlo=np.ascontiguousarray(lay.node_lo, dtype=np.int32),
            nhi=np.ascontiguousarray(lay.node_hi, dtype=np.int32),
            nst=np.ascontiguousarray(lay.node_start, dtype=np.int64),
            elo=np.ascontiguousarray(lay.elem_lo, dtype=np.int32),
            ehi=np.ascontiguousarray(lay.elem_hi, dtype=np.int32),
            est=np.ascontiguousarray(lay.elem_start, dtype=np.int64),
        )
        k = self._keep
        mesh = N.PfMesh(lay.nx, lay.ny, lay.hx, lay.hy, N.i32(k["nlo"]), N.i32(k["nhi"]),
                        N.i64(k["nst"]), N.i32(k["elo"]), N.i32(k["ehi"]), N.i64(k["est"]),
                        lay.notch_row, lay.notch_lo, lay.notch_hi, lay.dup_start,
                        lay.n_nodes, lay.n_elems)
        at = str(params.at_model)
        mat = N.PfMaterial(float(params.mu), float(params.lam), float(params.bulk_k),
                           float(params.g_c), float(params.length_l), float(params.eta),
                           float(params.c_w), float(params.gamma), 1 if at == "AT2" else 0)
        if getattr(config, "lin_method", "direct") not in ("direct", "cg"):
            raise ValueError(f"unknown method {config.lin_method!r}")
        cfg = N.PfConfig(float(config.tol_nr), float(config.tol_st), float(config.d_cap),
                         float(config.res_floor), int(config.max_nr), int(config.max_stag),
                         1.0e-12, 20)
        self.params, self.config = params, config
        h = C.c_void_p()
        if strip is None:
            st = self.lib.pf_create(C.byref(mesh), C.byref(mat), C.byref(cfg), device,
                                    C.byref(h))
        else:
            st = self.lib.pf_create_strip(C.byref(mesh), C.byref(mat), C.byref(cfg), device,
                                          C.byref(strip), C.byref(h))
        if st != N.PF_OK or not h.value:
            raise (ValueError if st == N.PF_ERR_INVALID else DeviceError)(
                f"pf_create failed with status {st} (see stderr)")
        self.h = h
        self.last_stats = None

    # -- lifecycle -----------------------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.pf_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def _check(self, st: int, history=None) -> None:
        if st == N.PF_OK:
            return
        msg = self.lib.pf_last_error(self.h).decode(errors="replace")
        if st in (N.PF_ERR_CONV_MOMENTUM, N.PF_ERR_CONV_EVOLUTION, N.PF_ERR_CONV_STAGGERED):
            raise reference_error(ConvergenceError)(msg, history)
        if st == N.PF_ERR_SINGULAR:
            raise reference_error(SingularSystemError)(msg)
        if st == N.PF_ERR_INVALID:
            raise ValueError(msg)
        if st == N.PF_ERR_INDEX:
            raise IndexError(msg)
        raise DeviceError(msg)

    # -- state ---------------------------------------------------------------------------
    def push(self, u=None, d=None, d_prev=None, tr_eps_plus=None, dev_dot_dev=None,
             psi_plus=None, psi_max=None) -> None:
        def c(a, n):
            if a is None:
                return None
            a = np.ascontiguousarray(a, dtype=np.float64)
            if a.size != n:
                raise ValueError(f"state array has {a.size} entries, expected {n}")
            return a
        nn, ng = self.n_nodes, 4 * self.n_elems
        arrs = [c(u, 2 * nn), c(d, nn), c(d_prev, nn), c(tr_eps_plus, ng), c(dev_dot_dev, ng),
                c(psi_plus, ng), c(psi_max, ng)]
        self._check(self.lib.pf_set_state(self.h, *[N.f64(a) for a in arrs]))

    def init_state(self, segments=None, radius: float = 0.0, x_last: float = 0.0,
                   y_last: float = 0.0) -> None:
        """Zero state built on the device, with d = d_prev = 1 within ``radius`` of the pre-crack
        segments ``[(ax, ay, bx, by), ...]`` (pf_init_state; configs.precrack_segments)."""
        seg = np.ascontiguousarray(np.zeros((0, 4)) if segments is None else segments,
                                   dtype=np.float64).reshape(-1, 4)
        self._check(self.lib.pf_init_state(self.h, N.f64(seg) if seg.size else None,
                                           seg.shape[0], float(radius), float(x_last),
                                           float(y_last)))

    def push_state(self, state) -> None:
        gp = state.gp
        self.push(state.u, state.d, state.d_prev, gp.tr_eps_plus, gp.dev_dot_dev, gp.psi_plus,
                  gp.psi_max)

    def pull(self, pinned: bool = False) -> dict:
        """The state arrays (fresh arrays; ``pinned``: page-locked, filled by direct DMA)."""
        nn, ne = self.n_nodes, self.n_elems
        emp = N.PINNED.empty if pinned else np.empty
        out = dict(u=emp(2 * nn), d=emp(nn), d_prev=emp(nn),
                   tr_eps_plus=emp((ne, 4)), dev_dot_dev=emp((ne, 4)),
                   psi_plus=emp((ne, 4)), psi_max=emp((ne, 4)))
        self._check(self.lib.pf_get_state(self.h, *[N.f64(out[k]) for k in (
            "u", "d", "d_prev", "tr_eps_plus", "dev_dot_dev", "psi_plus", "psi_max")]))
        return out

    def pull_into(self, **arrays) -> None:
        """Download state arrays into existing float64 arrays (e.g. the caller's own
        SolverState arrays; pageable destinations go through the pinned staging buffer with
        threaded host copies).  Keys: u, d, d_prev, tr_eps_plus, dev_dot_dev, psi_plus,
        psi_max."""
        keys = ("u", "d", "d_prev", "tr_eps_plus", "dev_dot_dev", "psi_plus", "psi_max")
        ptrs = []
        for k in keys:
            a = arrays.get(k)
            if a is not None:
                if a.dtype != np.float64 or not a.flags["C_CONTIGUOUS"] or not a.flags["WRITEABLE"]:
                    raise ValueError(f"{k}: expected a writable C-contiguous float64 array")
            ptrs.append(N.f64(a) if a is not None else None)
        self._check(self.lib.pf_get_state(self.h, *ptrs))

    def gp_strain(self, pinned: bool = False) -> tuple:
        ne = self.n_elems
        emp = N.PINNED.empty if pinned else np.empty
        strain, tr = emp((ne, 4, 4)), emp((ne, 4))
        self._check(self.lib.pf_get_gp_strain(self.h, N.f64(strain), N.f64(tr)))
        return strain, tr

    def interp_nodal(self, field) -> np.ndarray:
        """A nodal scalar field at the Gauss points, (n_elems, 4) (pf_interp_nodal)."""
        f = np.ascontiguousarray(field, dtype=np.float64)
        if f.size != self.n_nodes:
            raise ValueError(f"nodal field has {f.size} entries, expected {self.n_nodes}")
        out = np.empty((self.n_elems, 4))
        self._check(self.lib.pf_interp_nodal(self.h, N.f64(f), N.f64(out)))
        return out

    # -- hot path ------------------------------------------------------------------------
    def step(self, scheme, bc_increments, pinned_d_nodes=None) -> N.PfStats:
        dofs, offs, incs, nbc = pack_bcs(bc_increments)
        pins, npins = _pins(pinned_d_nodes)
        stats = N.PfStats()
        cap = int(self.config.max_stag) + 2
        hist = np.zeros(cap)
        st = self.lib.pf_staggered_step(self.h, scheme_code(scheme), N.i64(dofs), N.i64(offs),
                                        N.f64(incs), nbc, N.i64(pins), npins, C.byref(stats),
                                        N.f64(hist), cap)
        history = hist[: stats.n_hist].tolist()
        self.last_stats = stats
        self.last_history = history
        self._check(st, history)
        return stats

    def solve_momentum(self, bc_increments, r0=None) -> tuple:
        dofs, offs, incs, nbc = pack_bcs(bc_increments)
        r0v = C.c_double(math.nan if r0 is None else float(r0))
        n_nr, ratio = C.c_int32(0), C.c_double(0.0)
        self._check(self.lib.pf_solve_momentum(self.h, N.i64(dofs), N.i64(offs), N.f64(incs),
                                               nbc, C.byref(r0v), C.byref(n_nr), C.byref(ratio)))
        return n_nr.value, r0v.value, ratio.value

    def solve_evolution(self, scheme, pinned_d_nodes=None, r0=None) -> tuple:
        pins, npins = _pins(pinned_d_nodes)
        r0v = C.c_double(math.nan if r0 is None else float(r0))
        n_nr, fb = C.c_int32(0), C.c_int32(0)
        self._check(self.lib.pf_solve_evolution(self.h, scheme_code(scheme), N.i64(pins), npins,
                                                C.byref(r0v), C.byref(n_nr), C.byref(fb)))
        return n_nr.value, r0v.value, fb.value

    def evolution_residual_norm(self, pinned_d_nodes=None) -> float:
        pins, npins = _pins(pinned_d_nodes)
        out = C.c_double()
        self._check(self.lib.pf_evolution_residual_norm(self.h, N.i64(pins), npins, C.byref(out)))
        return out.value

    def commit(self) -> None:
        self._check(self.lib.pf_commit_step(self.h))

    # -- operators at the current state --------------------------------------------------
    def internal_force(self) -> np.ndarray:
        f = np.empty(2 * self.n_nodes)
        self._check(self.lib.pf_internal_force(self.h, N.f64(f)))
        return f

    def reaction_force(self, node_set, component: int) -> float:
        nodes = np.ascontiguousarray(np.asarray(node_set, dtype=np.int64).ravel())
        out = C.c_double()
        ptr = N.i64(nodes) if nodes.size else None
        self._check(self.lib.pf_reaction_force(self.h, ptr, nodes.size, int(component),
                                               C.byref(out)))
        return out.value

    def momentum_tangent_apply(self, x) -> tuple:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y, dg = np.empty(2 * self.n_nodes), np.empty(2 * self.n_nodes)
        self._check(self.lib.pf_momentum_tangent_apply(self.h, N.f64(x), N.f64(y), N.f64(dg)))
        return y, dg

    def evolution_residual(self) -> np.ndarray:
        r = np.empty(self.n_nodes)
        self._check(self.lib.pf_evolution_residual(self.h, N.f64(r)))
        return r

    def evolution_tangent_apply(self, scheme, x) -> tuple:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y, dg = np.empty(self.n_nodes), np.empty(self.n_nodes)
        self._check(self.lib.pf_evolution_tangent_apply(self.h, scheme_code(scheme), N.f64(x),
                                                        N.f64(y), N.f64(dg)))
        return y, dg

    def refresh_gp(self) -> None:
        self._check(self.lib.pf_refresh_gp(self.h))

    def softening_gate(self) -> np.ndarray:
        g = np.empty((self.n_elems, 4), dtype=np.uint8)
        self._check(self.lib.pf_softening_gate(self.h, N.u8(g)))
        return g.astype(bool)

    def extra_stiffness(self, scheme) -> np.ndarray:
        e = np.empty((self.n_elems, 4))
        self._check(self.lib.pf_extra_stiffness(self.h, scheme_code(scheme), N.f64(e)))
        return e

    def update_active_energy(self, scheme, delta_d_nodal) -> None:
        dd = np.ascontiguousarray(delta_d_nodal, dtype=np.float64)
        self._check(self.lib.pf_update_active_energy(self.h, scheme_code(scheme), N.f64(dd)))

    # -- benchmarking helpers ------------------------------------------------------------
    def bench_cg(self, physics: str, n_iter: int) -> tuple:
        """(ms, iterations) of a fixed-length PCG run at the current state (no convergence)."""
        code = {"momentum": 0, "evolution": 1, "phase_field": 1, "momentum_mg": 2,
                "phase_field_mg": 3}[physics]
        ms, it = C.c_double(), C.c_int64()
        self._check(self.lib.pf_bench_cg(self.h, code, int(n_iter), C.byref(ms), C.byref(it)))
        return ms.value, it.value

    MG_KERNELS = {
        0: "momentum fine residual march: r, D^-1 (16 B), d (8 B), t (16 B) per node + 1 B "
           "branch bits per cell",
        1: "momentum fine smoothing march: r, D^-1, d, z per node + level-1 correction (16 B per "
           "coarse node) + 1 B per cell",
        2: "momentum PCG-direction march: z, p_old, d, D^-1, p_new, q per node + 1 B per cell",
        10: "phase-field fine residual march: r, D^-1, t (8 B) per node + b (32 B) per cell",
        11: "phase-field fine smoothing march: r, D^-1, z (8 B) per node + level-1 correction "
            "(8 B per coarse node) + b (32 B) per cell",
        12: "phase-field PCG-direction march: z, p_old, D^-1, p_new, q (8 B) per node + b "
            "(32 B) per cell",
    }

    def bench_mg_kernel(self, which: int, reps: int = 20) -> tuple:
        """(ms per launch, algorithmic bytes per launch, byte accounting) of one fine-level
        multigrid march on the current state (pf_bench_mg_kernel)."""
        ms, nb = C.c_double(), C.c_double()
        self._check(self.lib.pf_bench_mg_kernel(self.h, int(which), int(reps), C.byref(ms),
                                                C.byref(nb)))
        return ms.value, nb.value, self.MG_KERNELS[which]

    def mg_info(self, with_omega: bool = False) -> dict:
        """Multigrid hierarchy of the momentum PCG (n_levels 0: Jacobi PCG on this handle)."""
        nl, ng, dn, su = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int64()
        self._check(self.lib.pf_mg_info(self.h, C.byref(nl), C.byref(ng), C.byref(dn),
                                        C.byref(su), None))
        out = {"n_levels": nl.value, "n_grid": ng.value, "dense": bool(dn.value),
               "setups": su.value}
        if with_omega and nl.value:
            om = np.zeros(nl.value)
            self._check(self.lib.pf_mg_info(self.h, None, None, None, None, N.f64(om)))
            out["omega"] = om
        return out

    MOMENTUM_SOLVERS = ("jacobi_pcg", "single_reduction_pcg", "multigrid_pcg")
    PHASE_FIELD_SOLVERS = ("jacobi_pcg", "single_reduction_pcg", "stencil_pcg",
                           "packed_multigrid_pcg", "multigrid_pcg")

    def solver_kinds(self) -> dict:
        """Linear solver of each Newton system (pf_solver_kinds)."""
        m, d = C.c_int32(), C.c_int32()
        self._check(self.lib.pf_solver_kinds(self.h, C.byref(m), C.byref(d)))
        return {"momentum": self.MOMENTUM_SOLVERS[m.value],
                "phase_field": self.PHASE_FIELD_SOLVERS[d.value]}

    def device_info(self) -> dict:
        g, s, l2 = C.c_int32(), C.c_int32(), C.c_int64()
        self._check(self.lib.pf_device_info(self.h, C.byref(g), C.byref(s), C.byref(l2)))
        return {"cg_grid": g.value, "sm_count": s.value, "l2_bytes": l2.value}

    def flush_l2(self) -> None:
        self._check(self.lib.pf_flush_l2(self.h))

    def synchronize(self) -> None:
        self._check(self.lib.pf_synchronize(self.h))
