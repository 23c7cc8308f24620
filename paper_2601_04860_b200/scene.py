"""``DensityGrid`` (mirror of /root/reference/pkg/src/divas/scene.py:154-165)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .geometry import VoxelGrid

__all__ = ["DensityGrid"]


@dataclass
class DensityGrid:
    grid: VoxelGrid
    values: np.ndarray  # (G, G, G) float32, indexed [ix, iy, iz]

    def __post_init__(self):
        g = self.grid.resolution
        self.values = np.asarray(self.values, dtype=np.float32).reshape(g, g, g)
        if not np.all(np.isfinite(self.values)) or np.any(self.values < 0):
            raise ValueError("densities must be finite and >= 0")
