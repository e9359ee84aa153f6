"""NURBS patch description (host) -- geometry is evaluated on the device.

Mirrors geometry.NurbsPatch (reference geometry.py:33-85),
unit_hypercube (194-201) and quarter_annulus (204-231); the L-shape patches
of BASELINE cfg4 are an extension (three bilinear squares).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import InvalidGeometryError
from .splines import KnotVector

__all__ = [
    "InvalidGeometryError",
    "NurbsPatch",
    "unit_hypercube",
    "quarter_annulus",
    "lshape_patches",
]


@dataclass(frozen=True)
class NurbsPatch:
    """Tensor-product NURBS map [0,1]^d -> R^d (control net + weights)."""

    knotvectors: tuple
    control_points: np.ndarray
    weights: np.ndarray

    def __post_init__(self):
        kvs = tuple(self.knotvectors)
        d = len(kvs)
        if not 1 <= d <= 3:
            raise ValueError(f"parametric dimension must be 1, 2 or 3, got {d}")
        for kv in kvs:
            if not hasattr(kv, "degree") or not hasattr(kv, "knots"):
                raise TypeError("knotvectors must be KnotVector instances")
        shape = tuple(int(kv.knots.size - kv.degree - 1) for kv in kvs)
        pts = np.ascontiguousarray(self.control_points, dtype=np.float64)
        wts = np.ascontiguousarray(self.weights, dtype=np.float64)
        if pts.shape != shape + (d,):
            raise ValueError(f"control point array must have shape {shape + (d,)}, got {pts.shape}")
        if wts.shape != shape:
            raise ValueError(f"weight array must have shape {shape}, got {wts.shape}")
        if np.any(wts <= 0.0):
            raise ValueError("weights must be strictly positive")
        object.__setattr__(self, "knotvectors", kvs)
        object.__setattr__(self, "control_points", pts)
        object.__setattr__(self, "weights", wts)

    @property
    def dim(self) -> int:
        return len(self.knotvectors)

    @property
    def is_polynomial(self) -> bool:
        return bool(np.all(self.weights == 1.0))

    def homogeneous(self) -> np.ndarray:
        """(w*P, w) net, C order -- the array the device contracts."""
        return homogeneous_net(self)


def homogeneous_net(patch) -> np.ndarray:
    """Homogeneous control net of any NurbsPatch-like object (duck-typed)."""
    w = np.asarray(patch.weights, dtype=np.float64)
    P = np.asarray(patch.control_points, dtype=np.float64)
    d = P.shape[-1]
    hw = np.empty(w.shape + (d + 1,))
    hw[..., :d] = P * w[..., None]
    hw[..., d] = w
    return np.ascontiguousarray(hw)


def _line() -> KnotVector:
    return KnotVector(1, np.array([0.0, 0.0, 1.0, 1.0]))


def _arc() -> KnotVector:
    return KnotVector(2, np.array([0.0, 0.0, 0.0, 1.0, 1.0, 1.0]))


def unit_hypercube(d: int) -> NurbsPatch:
    """Identity map on [0, 1]^d as a degree-1 patch."""
    if not 1 <= d <= 3:
        raise ValueError(f"dimension must be 1, 2 or 3, got {d}")
    corners = np.stack(np.meshgrid(*([np.array([0.0, 1.0])] * d), indexing="ij"), axis=-1)
    return NurbsPatch(tuple(_line() for _ in range(d)), corners, np.ones((2,) * d))


def quarter_annulus(d: int, r_in=1.0, r_out=2.0, height=1.0) -> NurbsPatch:
    """Exact quarter annulus: radial degree 1 x rational quadratic arc (x linear z)."""
    if d not in (2, 3):
        raise ValueError(f"quarter annulus needs d in (2, 3), got {d}")
    if not 0.0 < r_in < r_out:
        raise ValueError("radii must satisfy 0 < r_in < r_out")
    arc = np.array([[1.0, 0.0], [1.0, 1.0], [0.0, 1.0]])
    net = np.stack([r_in * arc, r_out * arc])
    w = np.tile(np.array([1.0, np.sqrt(2.0) / 2.0, 1.0]), (2, 1))
    if d == 2:
        return NurbsPatch((_line(), _arc()), net, w)
    if height <= 0.0:
        raise ValueError("height must be positive")
    net3 = np.zeros((2, 3, 2, 3))
    net3[..., 0, :2] = net
    net3[..., 1, :2] = net
    net3[..., 1, 2] = height
    return NurbsPatch((_line(), _arc(), _line()), net3, np.repeat(w[:, :, None], 2, axis=2))


def _square(x0, x1, y0, y1) -> NurbsPatch:
    net = np.array([[[x0, y0], [x0, y1]], [[x1, y0], [x1, y1]]], dtype=np.float64)
    return NurbsPatch((_line(), _line()), net, np.ones((2, 2)))


def lshape_patches():
    """BASELINE cfg4: (-1,1)^2 minus [0,1)x(-1,0] as three unit squares.

    Same global x/y orientation on every patch (parametric axis 0 = x,
    axis 1 = y): patch 0 = [-1,0]x[0,1], 1 = [0,1]x[0,1], 2 = [-1,0]x[-1,0].
    """
    return (_square(-1.0, 0.0, 0.0, 1.0), _square(0.0, 1.0, 0.0, 1.0), _square(-1.0, 0.0, -1.0, 0.0))
