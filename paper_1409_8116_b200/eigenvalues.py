"""Per-axis Laplacian eigenvalues (reference: eigenvalues.py).

Pseudo-spectral (continuous operator at the basis wavenumbers) and
second-order finite-difference (exact eigenvalues of the closed stencil),
`/root/reference/pkg/src/fastpoisson/eigenvalues.py:51-83`:

    spectral  periodic   -(2 pi min(k, n-k) / L)^2
              Dirichlet  -(pi (k+1) / L)^2
              Neumann    -(pi k / L)^2
    fd2       -(2 sin(theta_k) / dx)^2 with theta_k = k pi/n (periodic),
              pi (k+1)/(2(n+1) | 2n) (Dirichlet reg | stag),
              pi k/(2(n-1) | 2n)     (Neumann reg | stag)

The expressions keep the reference's floating-point operation order so the
tables are bit-identical; they are handed to the native plan, which sums them
per element on the device instead of materializing the dense N-point array.
``combine_eigenvalues`` (the dense sum, eigenvalues.py:94-114) is kept for
API compatibility and small problems only.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np

from .grid import Approximation, BoundaryCondition, GridKind, GridSpec


@dataclass(frozen=True)
class EigenvalueTable:
    """Eigenvalues of one axis (1/length^2) and the indices where they vanish."""

    values: np.ndarray
    null_indices: frozenset = field(default_factory=frozenset)

    def __post_init__(self):
        object.__setattr__(self, "values", np.asarray(self.values, dtype=np.float64))
        object.__setattr__(self, "null_indices", frozenset(self.null_indices))


def _nulls(bc: BoundaryCondition) -> frozenset:
    # periodic and Neumann axes carry the constant mode k = 0
    return frozenset() if bc is BoundaryCondition.DIRICHLET else frozenset({0})


def _check_row(spec: GridSpec):
    from .transforms import transform_pair_for

    transform_pair_for(spec.bc, spec.kind)


def spectral_eigenvalues(spec: GridSpec) -> EigenvalueTable:
    _check_row(spec)
    k = np.arange(spec.n, dtype=np.float64)
    if spec.bc is BoundaryCondition.PERIODIC:
        wave = 2.0 * np.pi * np.minimum(k, spec.n - k) / spec.length
    elif spec.bc is BoundaryCondition.DIRICHLET:
        wave = np.pi * (k + 1.0) / spec.length
    else:
        wave = np.pi * k / spec.length
    return EigenvalueTable(-(wave**2), _nulls(spec.bc))


def fd2_eigenvalues(spec: GridSpec) -> EigenvalueTable:
    _check_row(spec)
    k = np.arange(spec.n, dtype=np.float64)
    n = spec.n
    regular = spec.kind is GridKind.REGULAR
    if spec.bc is BoundaryCondition.PERIODIC:
        theta = k * np.pi / n
    elif spec.bc is BoundaryCondition.DIRICHLET:
        theta = np.pi * (k + 1.0) / (2.0 * (n + 1 if regular else n))
    else:
        theta = np.pi * k / (2.0 * (n - 1 if regular else n))
    return EigenvalueTable(-((2.0 * np.sin(theta) / spec.dx) ** 2), _nulls(spec.bc))


def eigenvalue_table(spec: GridSpec, approximation: Approximation) -> EigenvalueTable:
    if approximation is Approximation.PSEUDO_SPECTRAL:
        return spectral_eigenvalues(spec)
    return fd2_eigenvalues(spec)


@dataclass(frozen=True)
class CombinedEigenvalues:
    """Dense d-dimensional eigenvalue array and its null-mode index tuples."""

    values: np.ndarray
    null_modes: tuple


def null_modes_of(tables) -> tuple:
    """Null-mode tuples of the d-dimensional operator without the dense array."""
    tables = list(tables)
    if all(t.null_indices for t in tables):
        return tuple(itertools.product(*(sorted(t.null_indices) for t in tables)))
    return ()


def combine_eigenvalues(tables) -> CombinedEigenvalues:
    tables = list(tables)
    if not 1 <= len(tables) <= 3:
        raise ValueError(f"1 to 3 axes supported, got {len(tables)}")
    d = len(tables)
    total = np.zeros(tuple(t.values.size for t in tables), dtype=np.float64)
    for ax, t in enumerate(tables):
        shape = [1] * d
        shape[ax] = t.values.size
        total += t.values.reshape(shape)
    return CombinedEigenvalues(total, null_modes_of(tables))
