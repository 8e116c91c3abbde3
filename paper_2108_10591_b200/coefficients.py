"""Coefficient-step types (drop-in for pipesafe.coefficients).

The coefficient step itself runs on the device, one thread inside the
finalize kernel (csrc/vec.cuh ``check_iteration``), restating
compute_alpha_beta_safe / compute_zeta_eta_safe / guard_denominator
(coefficients.py:35-106) in IEEE double with the reference's association.
This module carries the host-visible types and the breakdown vocabulary.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

BREAKDOWN_RTOL = 1e-14  # coefficients.py:19

# PBS_BD_* -> the reference's quantity strings (coefficients.py:77, 80, 83, 102, 105)
BREAKDOWN_QUANTITIES = {
    1: "initial alpha denominator (r0*, s)",
    2: "beta denominator zeta_prev * f_prev",
    3: "alpha denominator g + beta*h",
    4: "zeta denominator (s, s)",
    5: "zeta/eta denominator a*b - c^2",
    # the product-type comparators (solvers.py:275, 283, 302, 303, 434; coefficients.py:130, 134)
    6: "alpha denominator (r0*, Ap)",
    7: "omega denominator (At, At)",
    8: "beta denominator omega",
    9: "beta denominator (r0*, r)",
    10: "zeta denominator (At, At)",
    11: "zeta/eta denominator e*a - d^2",
    12: "beta denominator zeta",
    # p-BiCGStab (not in the reference; oracle/pbsafe_oracle.c solve_pstab)
    13: "alpha denominator (r0*, w) + beta*((r0*, s) - omega*(r0*, z))",
    14: "omega denominator (y, y)",
}


class BreakdownError(RuntimeError):
    """A recurrence denominator vanished relative to its constituents (coefficients.py:22-32)."""

    def __init__(self, quantity: str, value: float, scale: float):
        super().__init__(
            f"breakdown in {quantity}: |{value:.3e}| <= {BREAKDOWN_RTOL:g} * {scale:.3e}"
        )
        self.quantity = quantity
        self.value = value
        self.scale = scale


@dataclass
class CoefficientSet:
    """Step scalars of one iteration (coefficients.py:42-57)."""

    alpha: float
    beta: float
    zeta: float | None = None
    eta: float | None = None
    omega: float | None = None

    def finite(self) -> bool:
        return all(
            np.isfinite(v)
            for v in (self.alpha, self.beta, self.zeta, self.eta, self.omega)
            if v is not None
        )
