"""Constitutive parameters and errors of the compressible Neo-Hookean model
(reference material.py:34-59).  The pointwise algebra itself lives in the
device kernels (csrc/hf_cell.cuh: kinematics, qp_action, k_build)."""

from __future__ import annotations

from dataclasses import dataclass


class NonPositiveJacobian(RuntimeError):
    """Deformation state with det F <= 0 (material.py:34-40)."""

    def __init__(self, message: str, element: int | None = None, level: int | None = None):
        super().__init__(message)
        self.element = element
        self.level = level


@dataclass(frozen=True)
class NeoHookeanParams:
    """Shear modulus and Lame parameter (material.py:43-59)."""

    mu: float
    lam: float

    def __post_init__(self):
        if self.mu <= 0.0 or self.lam <= 0.0:
            raise ValueError("mu and lam must be positive")

    @staticmethod
    def from_shear_and_poisson(mu: float, nu: float) -> "NeoHookeanParams":
        return NeoHookeanParams(mu=mu, lam=2.0 * mu * nu / (1.0 - 2.0 * nu))

    def scaled(self, factor: float) -> "NeoHookeanParams":
        return NeoHookeanParams(mu=self.mu * factor, lam=self.lam * factor)


SYM_PAIRS = {2: ((0, 0), (1, 1), (0, 1)), 3: ((0, 0), (1, 1), (2, 2), (1, 2), (0, 2), (0, 1))}


def n_sym(dim: int) -> int:
    return dim * (dim + 1) // 2
