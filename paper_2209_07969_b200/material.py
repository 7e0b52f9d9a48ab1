"""Material parameters of the degraded volumetric-deviatoric solid (interface mirror).

Same names, fields, derivations and errors as the reference's ``MaterialParams``
(``material.py:31-96``): ``bulk_k = lam + 2 mu / 3``, ``c_w`` from the AT variant (AT1 8/3,
AT2 2; ``material.py:23``), penalty ``gamma = 27 g_c / (64 l tol_ir^2)`` (``material.py:26-28``).
The pointwise stress / tangent / split formulas live in the CUDA kernels
(``csrc/pf_device.cuh``); the CPU restatement used as a test oracle is ``oracle/``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

C_W = {"AT1": 8.0 / 3.0, "AT2": 2.0}


def penalty_coefficient(g_c: float, length_l: float, tol_ir: float) -> float:
    """Irreversibility penalty weight (Eq. 9 of the paper; reference material.py:26-28)."""
    return 27.0 * g_c / (64.0 * length_l * tol_ir**2)


@dataclass
class MaterialParams:
    mu: float
    lam: float
    g_c: float
    length_l: float
    eta: float = 1.0e-6
    at_model: str = "AT1"
    tol_ir: float = 0.01
    bulk_k: float | None = None
    c_w: float | None = None
    gamma: float | None = None

    def __post_init__(self):
        if self.at_model not in C_W:
            raise ValueError(f"unknown model variant: {self.at_model!r}")
        if self.bulk_k is None:
            self.bulk_k = self.lam + 2.0 * self.mu / 3.0
        if self.c_w is None:
            self.c_w = C_W[self.at_model]
        if self.gamma is None:
            self.gamma = penalty_coefficient(self.g_c, self.length_l, self.tol_ir)
        if self.mu <= 0.0 or self.bulk_k <= 0.0:
            raise ValueError("mu and bulk_k must be positive")
        if self.length_l <= 0.0:
            raise ValueError("length_l must be positive")
        if not (0.0 <= self.eta < 1.0):
            raise ValueError("eta must lie in [0, 1)")

    @classmethod
    def from_young_poisson(cls, e_mod: float, nu: float, **kw) -> "MaterialParams":
        return cls(mu=e_mod / (2.0 * (1.0 + nu)),
                   lam=e_mod * nu / ((1.0 + nu) * (1.0 - 2.0 * nu)), **kw)

    @property
    def young_modulus(self) -> float:
        return self.mu * (3.0 * self.lam + 2.0 * self.mu) / (self.lam + self.mu)

    @property
    def poisson_ratio(self) -> float:
        return self.lam / (2.0 * (self.lam + self.mu))

    @property
    def psi_crit(self) -> float:
        return self.g_c / (self.c_w * self.length_l)

    def dissipation_source(self, d):
        d = np.asarray(d, dtype=float)
        base = self.g_c / (self.c_w * self.length_l)
        return base * np.ones_like(d) if self.at_model == "AT1" else base * 2.0 * d

    def dissipation_source_deriv(self, d):
        d = np.asarray(d, dtype=float)
        if self.at_model == "AT1":
            return np.zeros_like(d)
        return self.g_c / (self.c_w * self.length_l) * 2.0 * np.ones_like(d)


VOIGT_XX, VOIGT_YY, VOIGT_ZZ, VOIGT_XY = 0, 1, 2, 3


@dataclass
class StrainState:
    """Voigt strain [xx, yy, zz, xy] (engineering shear) and the two invariants the split uses
    (interface mirror of the reference's ``StrainState``, ``material.py:99-116``)."""

    eps: np.ndarray
    tr_eps: np.ndarray
    dev_dot_dev: np.ndarray

    @classmethod
    def from_voigt(cls, eps) -> "StrainState":
        eps = np.asarray(eps, dtype=float)
        tr = eps[..., VOIGT_XX] + eps[..., VOIGT_YY] + eps[..., VOIGT_ZZ]
        dev = [eps[..., k] - tr / 3.0 for k in (VOIGT_XX, VOIGT_YY, VOIGT_ZZ)]
        dev2 = dev[0] ** 2 + dev[1] ** 2 + dev[2] ** 2 + 0.5 * eps[..., VOIGT_XY] ** 2
        return cls(eps=eps, tr_eps=tr, dev_dot_dev=dev2)


def material_key(p) -> tuple:
    """Hashable identity of a params object (ours or the reference's, duck-typed)."""
    return (float(p.mu), float(p.lam), float(p.bulk_k), float(p.g_c), float(p.length_l),
            float(p.eta), float(p.c_w), float(p.gamma), str(p.at_model))
