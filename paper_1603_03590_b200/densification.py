"""Reference-signature stage functions of the densification module
(reference densification.py): patch grids, per-scale initialisation,
outlier reset and the weighted densification — numpy in, numpy out, the
computation on the GPU through the C ABI (``dis_grid_axis``,
``dis_init_patches``, ``dis_reset_outliers``, ``dis_densify``,
``dis_densify_bidirectional``).

Same names, arguments and exceptions as the reference so its callers (and
tests) run unchanged; bit-identical results (tests/test_stage_api.py,
tests/test_stage_search_gpu.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .params import DisParams


@dataclass(frozen=True)
class PatchGrid:
    """Uniform (edge-clamped) patch layout over one level (densification.py:
    27-47): window origins per axis, patches row-major (y outer, x inner)."""

    width: int
    height: int
    patch_size: int
    spacing: int
    x_origins: np.ndarray
    y_origins: np.ndarray

    @property
    def n_patches(self) -> int:
        return len(self.x_origins) * len(self.y_origins)

    @property
    def starts(self) -> np.ndarray:
        gx, gy = np.meshgrid(self.x_origins, self.y_origins)
        return np.stack([gx.ravel(), gy.ravel()], axis=1)

    @property
    def centers(self) -> np.ndarray:
        return self.starts + 0.5 * self.patch_size


def create_grid(width: int, height: int, patch_size: int, overlap: float) -> PatchGrid:
    """Window origins with the floored fractional overlap (densification.py:
    58-79), computed by the library's grid code (``dis_grid_axis``) — the
    same origins the kernels use."""
    from . import stages

    if not 0.0 <= overlap < 1.0:
        raise ValueError("overlap must lie in [0, 1)")
    if width < patch_size or height < patch_size:
        raise ValueError(f"level {width}x{height} is smaller than the patch size {patch_size}")
    xo = stages.grid_axis(int(width), int(patch_size), float(overlap))
    yo = stages.grid_axis(int(height), int(patch_size), float(overlap))
    spacing = max(1, int(patch_size) - int(np.floor(overlap * patch_size + 1e-9)))
    return PatchGrid(int(width), int(height), int(patch_size), spacing, xo, yo)


def init_patches(grid: PatchGrid, coarser_flow, downscale: int) -> np.ndarray:
    """Initial displacements (densification.py:82-95): zero at the coarsest
    scale, else the coarser field (bilinear_map) at center / downscale, times
    downscale — on the GPU (``dis_init_patches``; the flow path computes the
    same inside ``k_patch_prep``)."""
    from .inverse_search import _dev, _stream, _torch

    centers = np.ascontiguousarray(grid.centers, dtype=np.float64)
    n = centers.shape[0]
    if coarser_flow is None:
        return np.zeros((n, 2))
    torch = _torch()
    cf = _dev(torch, np.asarray(coarser_flow, dtype=np.float64)
              if not isinstance(coarser_flow, torch.Tensor) else coarser_flow)
    if cf.dim() != 3 or cf.shape[2] != 2:
        raise ValueError(f"coarser flow must be (H, W, 2), got {tuple(cf.shape)}")
    out = torch.empty((n, 2), dtype=torch.float64, device="cuda")
    c = _dev(torch, centers)
    _lib.check(_lib.lib().dis_init_patches(cf.data_ptr(), int(cf.shape[1]), int(cf.shape[0]),
                                           c.data_ptr(), n, int(downscale), out.data_ptr(),
                                           _stream(torch)))
    return out.cpu().numpy()


def reset_outliers(displacements, init_displacements, patch_size: int) -> np.ndarray:
    """Back to the initialisation where |update| > patch size
    (densification.py:98-107), decided for a correctly rounded hypot; returns
    a new array (GPU, ``dis_reset_outliers``)."""
    from .inverse_search import _dev, _stream, _torch

    torch = _torch()
    d = _dev(torch, np.asarray(displacements, dtype=np.float64))
    i = _dev(torch, np.asarray(init_displacements, dtype=np.float64))
    if tuple(d.shape) != tuple(i.shape) or d.dim() != 2 or d.shape[1] != 2:
        raise ValueError("displacements and init_displacements must both be (N, 2)")
    out = torch.empty_like(d)
    _lib.check(_lib.lib().dis_reset_outliers(d.data_ptr(), i.data_ptr(), int(d.shape[0]),
                                             int(patch_size), out.data_ptr(), None,
                                             _stream(torch)))
    return out.cpu().numpy()


def _grid_params(grid: PatchGrid) -> DisParams:
    # the overlap that reproduces the grid's spacing (create_grid floors it)
    ps = grid.patch_size
    return DisParams(patch_size=ps, overlap=(ps - grid.spacing) / ps)


def _dev_planes(torch, *arrays):
    return [torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)[None]).cuda()
            for a in arrays]


def densify(grid: PatchGrid, displacements, offsets, reference_image,
            query_image) -> np.ndarray:
    """Weighted average of the patch displacements covering each pixel
    (densification.py:173-191), on the GPU (``dis_densify``)."""
    from . import stages
    from .pipeline import _require_cuda

    torch = _require_cuda()
    if np.shape(reference_image) != (grid.height, grid.width):
        raise ValueError("reference image does not match the grid's level")
    d = np.asarray(displacements, dtype=np.float64)
    ref, qry, pu, pv, po = _dev_planes(torch, reference_image, query_image, d[:, 0], d[:, 1],
                                       np.asarray(offsets, dtype=np.float64))
    u, v = stages.densify(ref, qry, _grid_params(grid), pu, pv, po)
    return np.stack([u[0].cpu().numpy(), v[0].cpu().numpy()], axis=-1)


def densify_bidirectional(fwd_grid: PatchGrid, fwd_displacements, fwd_offsets,
                          bwd_grid: PatchGrid, bwd_displacements, bwd_offsets,
                          reference_image, query_image) -> np.ndarray:
    """Forward patches merged with the negated backward patches
    (densification.py:194-234), on the GPU (``dis_densify_bidirectional``).
    Both grids must be the level's grid (as in the pipeline)."""
    from . import stages
    from .pipeline import _require_cuda

    torch = _require_cuda()
    if (fwd_grid.patch_size, fwd_grid.spacing, fwd_grid.width, fwd_grid.height) != (
            bwd_grid.patch_size, bwd_grid.spacing, bwd_grid.width, bwd_grid.height):
        raise ValueError("forward and backward grids must describe the same level layout")
    fd = np.asarray(fwd_displacements, dtype=np.float64)
    bd = np.asarray(bwd_displacements, dtype=np.float64)
    t = _dev_planes(torch, reference_image, query_image, fd[:, 0], fd[:, 1],
                    np.asarray(fwd_offsets, dtype=np.float64), bd[:, 0], bd[:, 1],
                    np.asarray(bwd_offsets, dtype=np.float64))
    u, v = stages.densify_bidirectional(t[0], t[1], _grid_params(fwd_grid), *t[2:])
    return np.stack([u[0].cpu().numpy(), v[0].cpu().numpy()], axis=-1)
