"""B200-native DivAS fusion hot path (arxiv 2601.04860).

Depth-weighted mask refinement, multi-view voxel fusion and threshold /
extract, as hand-written sm_100a CUDA kernels behind a C ABI
(include/divas_b200.h, libdivas_b200.so) with the reference package's Python
entry points on top.  See DESIGN.md.
"""

from .geometry import Camera, SceneBounds, VoxelGrid, look_at
from .render import (RaySample, RenderConfig, ViewGeometry, march_ray, march_rays_device,
                     render_view, render_views_device)
from .scene import (DensityGrid, SceneModel, ScenePrimitive, bake_density_device,
                    bake_density_grid)
from .segmenter import (ConfidenceMask, ViewAux, ViewWindows, refine_bands_device, refine_mask, refine_masks,
                        refine_masks_device)
from .fusion import (DeviceViews, FusionParams, FusionStats, Fuser, OccupancyGrid,
                     extract, extract_device, fuse, fuse_with_stats, project_grid_overlay,
                     project_grid_overlay_device,
                     refine_and_fuse,
                     threshold, threshold_device)

from .incremental import FusionSession
from .trace import (ThickPathDecision, ThinPathDecision, depth_gradient, depth_weight,
                    thick_check, thin_check)

__version__ = "0.1.0"

__all__ = [
    "Camera", "SceneBounds", "VoxelGrid", "look_at", "ViewGeometry", "DensityGrid",
    "RenderConfig", "RaySample", "render_view", "render_views_device", "march_ray",
    "march_rays_device", "ScenePrimitive", "SceneModel", "bake_density_grid",
    "bake_density_device",
    "ConfidenceMask", "ViewAux", "ViewWindows", "refine_mask", "refine_masks", "refine_masks_device", "refine_bands_device",
    "DeviceViews", "FusionParams", "FusionStats", "Fuser", "OccupancyGrid",
    "fuse", "fuse_with_stats", "refine_and_fuse", "project_grid_overlay",
    "project_grid_overlay_device",
    "threshold", "threshold_device", "extract", "extract_device", "FusionSession",
    "ThickPathDecision", "ThinPathDecision", "depth_gradient", "depth_weight", "thick_check",
    "thin_check",
]
