"""B200-native Dense Inverse Search optical flow (arXiv 1603.03590).

Drop-in for the reference package's flow path (``disflow.dis_flow``,
pipeline.py:150-163) with the same parameter set (``DisParams``,
``VarParams``): the coarse-to-fine pyramid, inverse patch search,
densification and variational refinement run as hand-written sm_100a CUDA
kernels (``libdis_b200.so``, C ABI in ``include/dis_b200.h``), float64 in the
reference's exact operation order, so the flow is bit-identical to the
reference's on the same inputs.
"""

from .params import (
    DisParams,
    ParameterError,
    VarParams,
    coarsest_scale_for,
)
from .pyramid import (
    ImagePyramid,
    PyramidLevel,
    as_image,
    build_pyramid,
    dis_flow_on_pyramids,
    image_gradients,
    upsample_flow,
    warmup,
)
from .densification import (
    PatchGrid,
    create_grid,
    densify,
    densify_bidirectional,
    init_patches,
    reset_outliers,
)
from .variational import refine
from .inverse_search import (
    PatchSet,
    PatchState,
    optimize_patch,
    optimize_patch_set,
    precompute_patch,
    precompute_patch_set,
    refresh_patch_stats,
)
from .pipeline import (
    FlowEngine,
    SparseMatch,
    compose_flows,
    dis_flow,
    dis_flow_batch,
    dis_stereo,
    dis_stereo_batch,
    sparse_correspondences,
)

__version__ = "0.1.0"

__all__ = [
    "DisParams",
    "VarParams",
    "ParameterError",
    "coarsest_scale_for",
    "FlowEngine",
    "dis_flow",
    "dis_flow_batch",
    "compose_flows",
    "dis_stereo",
    "dis_stereo_batch",
    "sparse_correspondences",
    "SparseMatch",
    "ImagePyramid",
    "PyramidLevel",
    "as_image",
    "build_pyramid",
    "dis_flow_on_pyramids",
    "warmup",
    "image_gradients",
    "upsample_flow",
    "PatchGrid",
    "create_grid",
    "densify",
    "densify_bidirectional",
    "init_patches",
    "reset_outliers",
    "refine",
    "PatchSet",
    "PatchState",
    "precompute_patch_set",
    "optimize_patch_set",
    "refresh_patch_stats",
    "precompute_patch",
    "optimize_patch",
]
