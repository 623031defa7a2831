"""Host-side types of the hot-path boundary, mirroring the reference contract.

* ``SolveOptions``            -- fpi.py:48-62 (tolerance, max_iterations,
                                 residual_tolerance; ``initial_voltage`` and
                                 ``compute_contraction`` are ignored by the
                                 constant-power batch paths, as in the
                                 reference, dense.py:155; the ZIP route
                                 honours ``initial_voltage`` like fpi_solve,
                                 fpi.py:141-145)
* ``PowerTensor``/``LoadMatrix``/``VoltageBatch`` -- dense.py:35-98
* ``reshape_tensor``/``unreshape``                -- dense.py:101-111
* ``SingularSystemError``     -- fpi.py:44-45
* ``MemoryGuardError``        -- sparse.py:55-56

``VoltageBatch`` carries one extra field, ``iterations_per_case`` (int32[tau]),
the per-case update count of the GPU engine; ``iterations`` is its maximum,
which is the reference's joint count (test_dense.py:72-79).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "SolveOptions",
    "PowerTensor",
    "LoadMatrix",
    "VoltageBatch",
    "reshape_tensor",
    "unreshape",
    "SingularSystemError",
    "MemoryGuardError",
    "ZERO_VOLTAGE_GUARD",
]

# fpi.py:39-41 -- entries with |v| below this are reset to this value + 0j
ZERO_VOLTAGE_GUARD = 1e-12


class SingularSystemError(RuntimeError):
    """Raised when Y_dd cannot be factorized (fpi.py:44-45)."""


class MemoryGuardError(MemoryError):
    """Raised instead of allocating an oversized system (sparse.py:55-56)."""


@dataclass(frozen=True)
class SolveOptions:
    """Iteration controls (fpi.py:48-62); same defaults and validation."""

    tolerance: float = 1e-10
    max_iterations: int = 100
    initial_voltage: np.ndarray | None = None
    residual_tolerance: float = 1e-8
    compute_contraction: bool = False

    def __post_init__(self) -> None:
        if self.tolerance <= 0:
            raise ValueError("tolerance must be positive")
        if self.max_iterations < 1:
            raise ValueError("max_iterations must be >= 1")


@dataclass(frozen=True)
class PowerTensor:
    """Multidimensional batch of load cases; last axis = node axis (dense.py:35-54)."""

    values: np.ndarray

    def __post_init__(self) -> None:
        object.__setattr__(self, "values", np.asarray(self.values, dtype=complex))
        if self.values.ndim < 2:
            raise ValueError("power tensor needs at least one batch dimension")

    @property
    def dims(self) -> tuple[int, ...]:
        return self.values.shape[:-1]

    @property
    def n_cases(self) -> int:
        return math.prod(self.dims)


@dataclass(frozen=True)
class LoadMatrix:
    """Loads as b x tau; column j is case j in row-major order (dense.py:57-78)."""

    values: np.ndarray
    dims: tuple[int, ...] = ()

    def __post_init__(self) -> None:
        vals = np.asarray(self.values, dtype=complex)
        if vals.ndim != 2:
            raise ValueError("load matrix must be 2-D (nodes x cases)")
        object.__setattr__(self, "values", vals)
        if not self.dims:
            object.__setattr__(self, "dims", (vals.shape[1],))

    @property
    def n_demand(self) -> int:
        return self.values.shape[0]

    @property
    def tau(self) -> int:
        return self.values.shape[1]


@dataclass
class VoltageBatch:
    """Solved voltages (b x tau), joint iteration count and per-case flags (dense.py:81-98)."""

    values: np.ndarray
    iterations: int
    converged_mask: np.ndarray
    residuals: np.ndarray
    iterations_per_case: np.ndarray = field(default_factory=lambda: np.empty(0, np.int32))

    @property
    def tau(self) -> int:
        return self.values.shape[1]

    def magnitudes(self) -> np.ndarray:
        return np.abs(self.values)

    def angles(self) -> np.ndarray:
        return np.angle(self.values)


def reshape_tensor(tensor: PowerTensor) -> LoadMatrix:
    """Flatten batch dims row-major; node axis becomes rows (dense.py:101-105)."""
    b = tensor.values.shape[-1]
    return LoadMatrix(values=tensor.values.reshape(-1, b).T, dims=tensor.dims)


def unreshape(loads: LoadMatrix) -> PowerTensor:
    """Exact inverse of :func:`reshape_tensor` (dense.py:108-111)."""
    return PowerTensor(values=loads.values.T.reshape(*loads.dims, loads.n_demand))
