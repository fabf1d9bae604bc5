"""B200-native FlashSplat label solver (arXiv 2409.08270), hot path only.

Drop-in for the reference package's solver path (``splatlift``):

* ``accumulate_contributions`` (reference ``contributions.py:90``)
* ``assign_binary`` / ``assign_scene`` (reference ``solver.py:140,156``)
* the stage functions they are built from -- ``project_scene``,
  ``bin_gaussians_to_tiles`` -- and the input / output types;
* novel-view rendering on the same kernels: ``render_property`` /
  ``render_view`` / ``render_subset_alpha_depth`` (reference
  ``rasterizer.py:133-234``) and ``render_binary_mask`` /
  ``render_scene_mask`` (reference ``maskrender.py``);
* mask ingestion: ``load_mask_png`` / ``read_masks`` and the pipelined
  ``accumulate_mask_files`` (PNG decode on a thread pool overlapped with the
  device accumulation).

All compute runs in hand-written sm_100a CUDA kernels
(``csrc/`` -> ``_lib/libflashsplat_b200.so``) behind the C ABI of
``include/flashsplat_b200.h``; there is no CPU fallback.  ``solve`` /
``LabelSolver`` add the fused entry with a device-resident matrix, and
``accumulate_contributions(..., process_group=...)`` shards views over GPUs.
"""

from .contributions import ContributionMatrix, LabelMask, accumulate_contributions
from .maskrender import DEFAULT_TAU, RenderedMask, render_binary_mask, render_scene_mask
from .masks import accumulate_mask_files, load_mask_png, read_masks, save_mask_png
from .scene_io import export_ply, load_scene_ply
from .rasterizer import (
    DEFAULT_BLEND,
    EXACT_BLEND,
    TILE_SIZE,
    BlendConfig,
    RenderOutput,
    TileBinning,
    bin_gaussians_to_tiles,
    load_render_grid,
    render_property,
    render_subset_alpha_depth,
    render_view,
    save_render_grid,
    tile_range,
)
from .scene import (
    CameraView,
    Gaussian,
    GaussianScene,
    ProjectedGaussian,
    ProjectionStats,
    SceneDataError,
    SceneFormatError,
    evaluate_alpha,
    load_cameras,
    project_gaussian,
    project_scene,
    save_cameras,
)
from .solve import LabelSolver, pin_inputs, solve
from .solver import Assignment, assign_binary, assign_scene

__version__ = "0.1.0"

__all__ = [
    "Assignment", "BlendConfig", "CameraView", "ContributionMatrix", "DEFAULT_BLEND",
    "DEFAULT_TAU", "EXACT_BLEND", "Gaussian", "GaussianScene", "LabelMask", "LabelSolver",
    "ProjectedGaussian", "ProjectionStats", "pin_inputs", "RenderOutput", "RenderedMask", "SceneDataError",
    "accumulate_mask_files", "load_mask_png", "read_masks", "save_mask_png", "export_ply",
    "load_scene_ply",
    "SceneFormatError", "TILE_SIZE", "TileBinning", "accumulate_contributions", "assign_binary",
    "assign_scene", "bin_gaussians_to_tiles", "evaluate_alpha", "load_cameras",
    "load_render_grid", "project_gaussian", "project_scene", "render_binary_mask",
    "render_property", "render_scene_mask", "render_subset_alpha_depth", "render_view",
    "save_cameras", "save_render_grid", "solve", "tile_range",
]
