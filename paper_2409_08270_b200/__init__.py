"""B200-native FlashSplat label solver (arXiv 2409.08270), hot path only.

Drop-in for the reference package's solver path (``splatlift``):

* ``accumulate_contributions`` (reference ``contributions.py:90``)
* ``assign_binary`` / ``assign_scene`` (reference ``solver.py:140,156``)
* the stage functions they are built from -- ``project_scene``,
  ``bin_gaussians_to_tiles`` -- and the input / output types.

All compute runs in hand-written sm_100a CUDA kernels
(``csrc/`` -> ``_lib/libflashsplat_b200.so``) behind the C ABI of
``include/flashsplat_b200.h``; there is no CPU fallback.  ``solve`` /
``LabelSolver`` add the fused entry with a device-resident matrix, and
``accumulate_contributions(..., process_group=...)`` shards views over GPUs.
"""

from .contributions import ContributionMatrix, LabelMask, accumulate_contributions
from .rasterizer import (
    DEFAULT_BLEND,
    EXACT_BLEND,
    TILE_SIZE,
    BlendConfig,
    TileBinning,
    bin_gaussians_to_tiles,
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
from .solve import LabelSolver, solve
from .solver import Assignment, assign_binary, assign_scene

__version__ = "0.1.0"

__all__ = [
    "Assignment", "BlendConfig", "CameraView", "ContributionMatrix", "DEFAULT_BLEND",
    "EXACT_BLEND", "Gaussian", "GaussianScene", "LabelMask", "LabelSolver", "ProjectedGaussian",
    "ProjectionStats", "SceneDataError", "SceneFormatError", "TILE_SIZE", "TileBinning",
    "accumulate_contributions", "assign_binary", "assign_scene", "bin_gaussians_to_tiles",
    "evaluate_alpha", "load_cameras", "project_gaussian", "project_scene", "save_cameras",
    "solve", "tile_range",
]
