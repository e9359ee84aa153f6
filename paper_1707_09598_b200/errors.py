"""Exception classes of the reference, mapped from C-ABI status codes.

When the reference package (``sparseiga``) is importable, the classes
derive from its own exceptions so that ``except sparseiga....Error`` keeps
working after the drop-in rebinding.
"""
from __future__ import annotations

try:  # pragma: no cover - only when the reference is installed next to us
    from sparseiga.assembly import EmptyInteriorError as _RefEmpty
    from sparseiga.geometry import InvalidGeometryError as _RefGeom
    from sparseiga.linsolve import LinearSolveError as _RefSolve
except Exception:  # noqa: BLE001
    _RefGeom, _RefSolve, _RefEmpty = ValueError, RuntimeError, ValueError

__all__ = ["InvalidGeometryError", "LinearSolveError", "EmptyInteriorError", "DeviceError"]


class InvalidGeometryError(_RefGeom):
    """det J <= 0 at a quadrature point (reference geometry.py:29-30, 128-131)."""


class LinearSolveError(_RefSolve):
    """Non-finite / non-converged / residual above tolerance (linsolve.py:12-13)."""


class EmptyInteriorError(_RefEmpty):
    """No interior degrees of freedom (assembly.py:37-38)."""


class DeviceError(RuntimeError):
    """CUDA runtime failure inside libsgiga."""
