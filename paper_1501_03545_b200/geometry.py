"""Scalar model geometry on the host.

These are the reference's host-side parameter computations (hrgen
geometry.py), evaluated with the same numpy/libm calls in the same
operation order so that the resolved disk radius R and the derived
constants handed to the GPU are bit-identical to what hrgen uses.  They are
O(1) scalar work (a 512-point grid plus a bisection), not part of the hot
path.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import InfeasibleParametersError, ParameterDomainError

TWO_PI = 2.0 * math.pi

# hrgen geometry.py:193-194 search interval for the radius solver
RADIUS_SEARCH_LO = 1e-6
RADIUS_SEARCH_HI = 200.0


@dataclass(frozen=True)
class ModelParams:
    """Resolved model (hrgen geometry.py:82-101): n points, growth alpha,
    disk radius R; target_avg_degree is set when R came from the solver."""

    n: int
    alpha: float
    R: float
    target_avg_degree: float | None = None

    def __post_init__(self):
        if self.n < 1:
            raise ParameterDomainError(f"n must be >= 1, got {self.n}")
        if not self.alpha > 0.0:
            raise ParameterDomainError(f"alpha must be > 0, got {self.alpha}")
        if not self.R > 0.0:
            raise ParameterDomainError(f"R must be > 0, got {self.R}")


def alpha_from_gamma(gamma: float) -> float:
    """Radial growth alpha giving degree exponent gamma = 2*alpha + 1
    (hrgen geometry.py:235-239)."""
    if not gamma > 2.0:
        raise ParameterDomainError(f"gamma must be > 2, got {gamma}")
    return (gamma - 1.0) / 2.0


def to_poincare_radius(r_native):
    """tanh(r/2): native hyperbolic radius -> Poincare-disk radius
    (hrgen geometry.py:104-113)."""
    arr = np.asarray(r_native, dtype=np.float64)
    out = np.tanh(arr / 2.0)
    return float(out) if np.ndim(r_native) == 0 else out


def to_native_radius(r_poincare):
    """2*atanh(r): inverse of to_poincare_radius (hrgen geometry.py:116-122)."""
    arr = np.asarray(r_poincare, dtype=np.float64)
    if np.any(arr < 0.0) or np.any(arr >= 1.0):
        raise ValueError("Poincare radial coordinate must be in [0, 1)")
    out = 2.0 * np.arctanh(arr)
    return float(out) if np.ndim(r_poincare) == 0 else out


def _degree_bracket(alpha):
    # (pi/4)/alpha^2 - (pi-1)/alpha + (pi-2), grouped as hrgen evaluates it
    return (math.pi / 4.0) / alpha**2 - (math.pi - 1.0) / alpha + (math.pi - 2.0)


def expected_avg_degree(n: int, alpha: float, radius: float) -> float:
    """Closed-form expected average degree (hrgen geometry.py:170-190)."""
    if not alpha > 0.5:
        raise ParameterDomainError(f"alpha must be > 0.5, got {alpha}")
    if not radius > 0.0:
        raise ParameterDomainError(f"radius must be > 0, got {radius}")
    if n < 1:
        raise ParameterDomainError(f"n must be >= 1, got {n}")
    xi = alpha / (alpha - 0.5)
    tail = alpha * (radius / 2.0) * _degree_bracket(alpha) - 1.0
    decay = math.exp(-radius / 2.0) + math.exp(-alpha * radius) * tail
    return (2.0 / math.pi) * xi * xi * n * decay


def target_radius(n: int, avg_degree: float, alpha: float, rel_tol: float = 1e-6) -> float:
    """Disk radius whose expected average degree is avg_degree
    (hrgen geometry.py:197-232): locate the peak of the closed form on a
    512-point geometric grid, then bisect on the decaying branch."""
    if not alpha > 0.5:
        raise ParameterDomainError(f"alpha must be > 0.5, got {alpha}")
    if not 0.0 < avg_degree < n - 1:
        raise ParameterDomainError(
            f"target average degree must be in (0, n-1), got {avg_degree} for n={n}")
    grid = np.geomspace(RADIUS_SEARCH_LO, RADIUS_SEARCH_HI, 512)
    curve = [expected_avg_degree(n, alpha, g) for g in grid]
    top = int(np.argmax(curve))
    lo, hi = float(grid[top]), RADIUS_SEARCH_HI
    if curve[top] < avg_degree or expected_avg_degree(n, alpha, hi) > avg_degree:
        raise InfeasibleParametersError(
            f"no radius in ({RADIUS_SEARCH_LO}, {RADIUS_SEARCH_HI}] yields average degree "
            f"{avg_degree} for n={n}, alpha={alpha}")
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        got = expected_avg_degree(n, alpha, mid)
        if abs(got - avg_degree) <= rel_tol * avg_degree:
            return mid
        if got > avg_degree:
            lo = mid
        else:
            hi = mid
    raise InfeasibleParametersError(
        f"bisection failed to reach tolerance {rel_tol} for n={n}, alpha={alpha}, "
        f"avg_degree={avg_degree}")


def model_constants(R: float, alpha: float):
    """The scalars hrgen derives from (R, alpha) with numpy/libm, evaluated
    identically: cosh(R)-1 (geometry.py:150), the Poincare rim and its
    clamp (generator.py:176-178, 203), the native clamp (generator.py:174),
    and the inverse-CDF factors (generator.py:156)."""
    a = float(2.0 * np.sinh(np.asarray(R, dtype=np.float64) / 2.0) ** 2)
    max_r = to_poincare_radius(R)
    return {
        "cosh_r_minus_1": a,
        "max_r": max_r,
        "rp_cap": float(np.nextafter(max_r, 0.0)),
        "r_cap": float(np.nextafter(R, 0.0)),
        "two_over_alpha": 2.0 / alpha,
        "sinh_half_alpha_r": math.sinh(alpha * R / 2.0),
    }
