"""Materials (intact/elasticity.py:31-63): the types the system is built from.

The per-element energies, stresses and PSD Hessians themselves run on the
device inside libibf (csrc/elastic_math.cuh, csrc/system.cu).
"""

from __future__ import annotations

import dataclasses
from enum import Enum


class MaterialModel(str, Enum):
    SNH = "snh"
    NH = "nh"
    COR = "cor"
    LIN = "lin"


def lame_parameters(young: float, poisson: float) -> tuple[float, float]:
    """(mu, lambda) from Young's modulus and Poisson's ratio (:38-42)."""
    return (young / (2.0 * (1.0 + poisson)),
            young * poisson / ((1.0 + poisson) * (1.0 - 2.0 * poisson)))


@dataclasses.dataclass(frozen=True)
class Material:
    """Isotropic material (intact/elasticity.py:45-63), same validation."""

    model: MaterialModel
    young: float
    poisson: float

    def __post_init__(self):
        if self.young <= 0.0:
            raise ValueError("Young's modulus must be positive")
        if not 0.0 <= self.poisson < 0.5:
            raise ValueError("Poisson's ratio must be in [0, 0.5)")

    @property
    def mu(self) -> float:
        return lame_parameters(self.young, self.poisson)[0]

    @property
    def lam(self) -> float:
        return lame_parameters(self.young, self.poisson)[1]
