"""Camera / grid / bounds types of the fusion boundary.

Field-for-field mirrors of the reference dataclasses so that code written
against ``divas.geometry`` runs unchanged; the hot-path functions also accept
the reference's own objects (they only read the attributes below).

* ``Camera``      /root/reference/pkg/src/divas/geometry.py:34-69
* ``VoxelGrid``   geometry.py:92-148
* ``SceneBounds`` geometry.py:151-173
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["Camera", "VoxelGrid", "SceneBounds", "look_at"]


@dataclass(frozen=True)
class Camera:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    world_from_camera: np.ndarray  # 4x4, rotation block orthonormal

    def __post_init__(self):
        m = np.asarray(self.world_from_camera, dtype=np.float64).reshape(4, 4)
        object.__setattr__(self, "world_from_camera", m)
        if not (self.fx > 0 and self.fy > 0):
            raise ValueError("focal lengths must be positive")
        if not (0 <= self.cx < self.width and 0 <= self.cy < self.height):
            raise ValueError("principal point outside the image")
        r = m[:3, :3]
        if not np.allclose(r.T @ r, np.eye(3), atol=1e-6):
            raise ValueError("rotation block is not orthonormal")

    @property
    def position(self) -> np.ndarray:
        return self.world_from_camera[:3, 3]

    @property
    def rotation(self) -> np.ndarray:
        """Columns are the camera's x/y/z axes in world coordinates."""
        return self.world_from_camera[:3, :3]

    @property
    def forward(self) -> np.ndarray:
        return -self.world_from_camera[:3, 2]


@dataclass(frozen=True)
class VoxelGrid:
    resolution: int
    half_extents: tuple = (1.0,)
    origin: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def __post_init__(self):
        if isinstance(self.half_extents, (int, float)):
            object.__setattr__(self, "half_extents", (float(self.half_extents),))
        else:
            object.__setattr__(self, "half_extents", tuple(float(b) for b in self.half_extents))
        object.__setattr__(self, "origin", np.asarray(self.origin, dtype=np.float64).reshape(3))
        if self.resolution < 1:
            raise ValueError("resolution must be a positive integer")
        if any(b <= 0 for b in self.half_extents):
            raise ValueError("half extent must be positive")

    @property
    def half_extent(self) -> float:
        return self.half_extents[0]

    def voxel_size(self, level: int = 0) -> float:
        return 2.0 * self.half_extents[level] / self.resolution

    @property
    def center(self) -> np.ndarray:
        return self.origin + self.half_extent

    def index_to_center(self, idx) -> np.ndarray:
        idx = np.asarray(idx, dtype=np.float64)
        return self.origin + (idx + 0.5) * self.voxel_size()


@dataclass(frozen=True)
class SceneBounds:
    min: np.ndarray
    max: np.ndarray
    unbounded: bool = False

    def __post_init__(self):
        lo = np.asarray(self.min, dtype=np.float64).reshape(3)
        hi = np.asarray(self.max, dtype=np.float64).reshape(3)
        if not np.all(lo < hi):
            raise ValueError("bounds min must be strictly below max")
        object.__setattr__(self, "min", lo)
        object.__setattr__(self, "max", hi)

    @property
    def center(self) -> np.ndarray:
        return 0.5 * (self.min + self.max)

    @property
    def half(self) -> np.ndarray:
        return 0.5 * (self.max - self.min)


def look_at(position, target, up=None) -> np.ndarray:
    """4x4 world_from_camera aimed at ``target`` (geometry.py:212-239 conventions:
    camera looks along -Z, +Y up, +X fallback within 1 degree of +/-Y)."""
    pos = np.asarray(position, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - pos
    n = np.linalg.norm(fwd)
    if n == 0.0:
        raise ValueError("look_at target coincides with the camera position")
    fwd = fwd / n
    if up is None:
        up = np.array([0.0, 1.0, 0.0])
        if abs(fwd @ up) > np.cos(np.radians(1.0)):
            up = np.array([1.0, 0.0, 0.0])
    zaxis = -fwd
    xaxis = np.cross(np.asarray(up, dtype=np.float64), zaxis)
    xaxis = xaxis / np.linalg.norm(xaxis)
    yaxis = np.cross(zaxis, xaxis)
    m = np.eye(4)
    m[:3, 0], m[:3, 1], m[:3, 2], m[:3, 3] = xaxis, yaxis, zaxis, pos
    return m
