"""Scheme, gas and freestream parameter objects of the drop-in.

Same field names, defaults and validation as the reference
(blockflow/solver.py:31-98, blockflow/physics.py:47-90).  Every consumer in
this package reads these objects by attribute only, so the reference's own
``SchemeConfig`` / ``GasModel`` / ``FreestreamState`` instances are accepted
interchangeably.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import ConfigError

FLUXES = ("roe", "van_leer")                                  # solver.py:31
LIMITERS = ("none", "van_leer", "van_albada", "minmod")       # solver.py:32
RK_COEFFS = {1: (1.0,), 2: (0.5, 1.0), 4: (0.25, 1.0 / 3.0, 0.5, 1.0)}   # solver.py:33
EQ_NAMES = ("mass", "xmom", "ymom", "zmom", "energy")         # solver.py:35
PRIM_NAMES = ("rho", "u", "v", "w", "p")                      # solver.py:187
FIELD_NAMES = ("rho", "u", "v", "w", "p", "T")


@dataclass(frozen=True)
class GasModel:
    """Perfect gas with an optional viscosity law (physics.py:47-90)."""
    gamma: float = 1.4
    R: float = 287.0
    mu: float = 0.0
    sutherland: tuple | None = None
    prandtl: float = 0.72

    def __post_init__(self):
        if not self.gamma > 1.0:
            raise ValueError(f"gamma must exceed 1, got {self.gamma}")
        if not self.R > 0.0:
            raise ValueError(f"R must be positive, got {self.R}")
        if self.mu < 0.0:
            raise ValueError(f"mu must be non-negative, got {self.mu}")

    @property
    def cp(self) -> float:
        return self.gamma * self.R / (self.gamma - 1.0)

    @property
    def cv(self) -> float:
        return self.R / (self.gamma - 1.0)

    def viscosity(self, T):
        """mu(T): constant, or Sutherland's law (physics.py:79-85)."""
        if self.sutherland is None:
            return self.mu if np.isscalar(T) else np.full_like(np.asarray(T, float), self.mu)
        mu_ref, t_ref, s = self.sutherland
        T = np.asarray(T, float)
        return mu_ref * (T / t_ref) ** 1.5 * (t_ref + s) / (T + s)

    def conductivity(self, T):
        """k = mu cp / Pr (physics.py:87-89)."""
        return self.viscosity(T) * self.cp / self.prandtl


@dataclass(frozen=True)
class SchemeConfig:
    """Discretisation switches (solver.py:38-71)."""
    flux: str = "van_leer"
    epsilon: float = 1.0
    kappa: float = -1.0
    limiter: str = "van_albada"
    rk_stages: int = 2
    cfl: float = 0.5
    limiter_freeze_at: int | None = None
    entropy_fix_coeff: float = 0.1
    viscous: bool = False
    mms_id: str | None = None
    wall_temperature: float | None = None

    def __post_init__(self):
        if self.flux not in FLUXES:
            raise ConfigError(f"flux must be one of {FLUXES}, got {self.flux!r}")
        if self.epsilon not in (0.0, 1.0):
            raise ConfigError(f"epsilon must be 0 or 1, got {self.epsilon}")
        if not -1.0 <= self.kappa <= 1.0:
            raise ConfigError(f"kappa must lie in [-1, 1], got {self.kappa}")
        if self.limiter not in LIMITERS:
            raise ConfigError(f"limiter must be one of {LIMITERS}, got {self.limiter!r}")
        if self.rk_stages not in RK_COEFFS:
            raise ConfigError(f"rk_stages must be 1, 2 or 4, got {self.rk_stages}")
        if self.cfl <= 0.0:
            raise ConfigError(f"cfl must be positive, got {self.cfl}")
        if self.limiter_freeze_at is not None and self.limiter_freeze_at < 1:
            raise ConfigError("limiter_freeze_at must be >= 1")

    @property
    def ghost_rounds(self) -> int:
        return 2 if self.viscous else 1


@dataclass(frozen=True)
class FreestreamState:
    """Reference state for inflow/farfield BCs (solver.py:74-98)."""
    rho: float
    u: float
    v: float
    w: float
    p: float
    T: float

    @classmethod
    def from_mach(cls, gas, mach, p, T, alpha_deg=0.0, ndim=2):
        # Same operation order as solver.py:84-94 so the doubles agree bitwise
        # (numpy's sqrt/cos/sin on python floats are the libm ones).
        import numpy as np
        rho = p / (gas.R * T)
        speed = mach * np.sqrt(gas.gamma * gas.R * T)
        a = np.radians(alpha_deg)
        if ndim == 2:
            vel = (speed * np.cos(a), speed * np.sin(a), 0.0)
        else:
            vel = (speed * np.cos(a), 0.0, speed * np.sin(a))
        return cls(float(rho), *(float(x) for x in vel), float(p), float(T))

    def values(self):
        return {"rho": self.rho, "u": self.u, "v": self.v, "w": self.w,
                "p": self.p, "T": self.T}


def validate_scheme(config):
    """Re-run the reference's validation on a duck-typed config."""
    if config.flux not in FLUXES:
        raise ConfigError(f"flux must be one of {FLUXES}, got {config.flux!r}")
    if config.limiter not in LIMITERS:
        raise ConfigError(f"limiter must be one of {LIMITERS}, got {config.limiter!r}")
    if config.rk_stages not in RK_COEFFS:
        raise ConfigError(f"rk_stages must be 1, 2 or 4, got {config.rk_stages}")
    if float(config.epsilon) not in (0.0, 1.0):
        raise ConfigError(f"epsilon must be 0 or 1, got {config.epsilon}")
    if not (config.cfl > 0.0 and math.isfinite(config.cfl)):
        raise ConfigError(f"cfl must be positive, got {config.cfl}")
    return config
