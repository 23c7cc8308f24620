"""``ViewGeometry``: the per-view record the hot path consumes.

Mirror of /root/reference/pkg/src/divas/render.py:55-78.  Maps are (H, W)
row-major ``[iy, ix]``; ``valid = n_samples > 0``; invalid pixels hold 0 in
every depth map.  (The ray marcher that produces it is out of scope.)
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .geometry import Camera

__all__ = ["ViewGeometry"]


@dataclass
class ViewGeometry:
    camera: Camera
    rgb: np.ndarray        # (H, W, 3) float32 (unused on the hot path)
    d_min: np.ndarray      # (H, W) float32
    d_max: np.ndarray      # (H, W) float32
    d_exp: np.ndarray      # (H, W) float32
    n_samples: np.ndarray  # (H, W) int32
    z_surface: np.ndarray  # (H, W) float32

    @property
    def valid(self) -> np.ndarray:
        return self.n_samples > 0
