"""Reference-signature stage functions of the inverse search (reference
inverse_search.py:283-494): the batch interface (``PatchSet``,
``precompute_patch_set``, ``optimize_patch_set``, ``refresh_patch_stats``)
and the single-patch interface (``PatchState``, ``precompute_patch``,
``optimize_patch``) — numpy in, numpy out, the computation on the GPU
through the C ABI (``dis_precompute_patch_set``, ``dis_optimize_patch_set``,
``dis_refresh_patch_stats``; csrc/stage_search.cu), bit-identical to the
reference.  The flow path itself runs the fused per-scale kernels
(``dis_patch_search``); these are for stage-level callers and tests.

Levels may be this package's ``PyramidLevel`` (CUDA tensors) or the
reference's own (numpy arrays).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, replace

import numpy as np

from . import _lib

NORM_CODES = {"l2": 0, "l1": 1, "huber": 2}


def _torch():
    from .pipeline import _require_cuda

    return _require_cuda()


def _dev(torch, x, dtype=None):
    dt = torch.float64 if dtype is None else dtype
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
    return t.to(device="cuda", dtype=dt).contiguous()


def _stream(torch):
    return _lib.stream_handle(torch.cuda.current_stream())


def _np(t):
    return t.cpu().numpy()


@dataclass
class PatchSet:
    """Struct-of-arrays state for all patches of one grid (inverse_search.py:
    283-303); numpy arrays like the reference's."""

    patch_size: int
    x_starts: np.ndarray        # (N,) window origins on the reference level
    y_starts: np.ndarray
    templates: np.ndarray       # (N, ps*ps)
    steep_x: np.ndarray         # (N, ps*ps)
    steep_y: np.ndarray
    hessian: np.ndarray         # (N, 3) packed [h00, h01, h11]
    hessian_inv: np.ndarray     # (N, 3), zero rows for invalid patches
    template_mean: np.ndarray   # (N,)
    valid: np.ndarray           # (N,) bool
    init_displacement: np.ndarray  # (N, 2)
    displacement: np.ndarray       # (N, 2)
    offset: np.ndarray             # (N,) query-minus-template window mean
    mean_abs_residual: np.ndarray  # (N,)

    def __len__(self) -> int:
        return self.x_starts.shape[0]


def _level_dims(level):
    h, w = (int(d) for d in tuple(level.image.shape))
    return w, h


def precompute_patch_set(level, x_starts, y_starts, patch_size: int,
                         horizontal_only: bool = False) -> PatchSet:
    """Templates, steepest-descent images and conditioned Hessian inverses
    for windows starting at the given reference-level coordinates
    (inverse_search.py:306-341)."""
    torch = _torch()
    xs = np.ascontiguousarray(x_starts, dtype=np.float64)
    ys = np.ascontiguousarray(y_starts, dtype=np.float64)
    n = xs.shape[0]
    ps = int(patch_size)
    W, H = _level_dims(level)
    img, gx, gy = (_dev(torch, a) for a in (level.image, level.grad_x, level.grad_y))
    dxs, dys = _dev(torch, xs), _dev(torch, ys)
    tmpl = torch.empty((n, ps * ps), dtype=torch.float64, device="cuda")
    sdx = torch.empty_like(tmpl)
    sdy = torch.empty_like(tmpl)
    mean_t = torch.empty(n, dtype=torch.float64, device="cuda")
    hess = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    hinv = torch.empty_like(hess)
    valid = torch.empty(n, dtype=torch.uint8, device="cuda")
    _lib.check(_lib.lib().dis_precompute_patch_set(
        img.data_ptr(), gx.data_ptr(), gy.data_ptr(), W, H, dxs.data_ptr(), dys.data_ptr(), n,
        ps, int(bool(horizontal_only)), tmpl.data_ptr(), sdx.data_ptr(), sdy.data_ptr(),
        mean_t.data_ptr(), hess.data_ptr(), hinv.data_ptr(), valid.data_ptr(), _stream(torch)))
    return PatchSet(
        patch_size=ps, x_starts=xs, y_starts=ys, templates=_np(tmpl), steep_x=_np(sdx),
        steep_y=_np(sdy), hessian=_np(hess), hessian_inv=_np(hinv), template_mean=_np(mean_t),
        valid=_np(valid).astype(bool), init_displacement=np.zeros((n, 2)),
        displacement=np.zeros((n, 2)), offset=np.zeros(n), mean_abs_residual=np.zeros(n))


def optimize_patch_set(patches: PatchSet, query, iterations: int, *, residual_norm: str = "l2",
                       huber_b: float = 1.0, mean_normalization: bool = True,
                       threads: int = 1) -> None:
    """The inverse search for every patch (inverse_search.py:344-371), writing
    displacements, normalisation offsets and residuals in place.  ``threads``
    is accepted for signature compatibility (a patch is a GPU thread)."""
    if residual_norm not in NORM_CODES:
        raise KeyError(residual_norm)  # the reference's NORM_CODES[...] lookup
    torch = _torch()
    n = len(patches)
    W, H = _level_dims(query)
    q = _dev(torch, query.image)
    a = [_dev(torch, x) for x in (patches.x_starts, patches.y_starts, patches.templates,
                                  patches.steep_x, patches.steep_y, patches.hessian_inv,
                                  patches.template_mean)]
    valid = _dev(torch, np.asarray(patches.valid, dtype=np.uint8), torch.uint8)
    init = _dev(torch, patches.init_displacement)
    disp = torch.empty((n, 2), dtype=torch.float64, device="cuda")
    off = torch.empty(n, dtype=torch.float64, device="cuda")
    mar = torch.empty(n, dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib().dis_optimize_patch_set(
        q.data_ptr(), W, H, a[0].data_ptr(), a[1].data_ptr(), n, int(patches.patch_size),
        a[2].data_ptr(), a[3].data_ptr(), a[4].data_ptr(), a[5].data_ptr(), a[6].data_ptr(),
        valid.data_ptr(), init.data_ptr(), int(iterations), int(bool(mean_normalization)),
        NORM_CODES[residual_norm], ctypes.c_double(float(huber_b)), disp.data_ptr(),
        off.data_ptr(), mar.data_ptr(), _stream(torch)))
    patches.displacement[...] = _np(disp)
    patches.offset[...] = _np(off)
    patches.mean_abs_residual[...] = _np(mar)


def refresh_patch_stats(patches: PatchSet, query, select: np.ndarray,
                        mean_normalization: bool = True) -> None:
    """Offsets / residuals of the selected patches at their current
    displacement (inverse_search.py:374-387)."""
    sel = np.ascontiguousarray(select, dtype=np.bool_)
    if not sel.any():
        return
    torch = _torch()
    n = len(patches)
    W, H = _level_dims(query)
    q = _dev(torch, query.image)
    xs, ys, tmpl, mean_t, disp = (_dev(torch, x) for x in (
        patches.x_starts, patches.y_starts, patches.templates, patches.template_mean,
        patches.displacement))
    s = _dev(torch, sel.astype(np.uint8), torch.uint8)
    off = _dev(torch, patches.offset)
    mar = _dev(torch, patches.mean_abs_residual)
    _lib.check(_lib.lib().dis_refresh_patch_stats(
        q.data_ptr(), W, H, xs.data_ptr(), ys.data_ptr(), n, int(patches.patch_size),
        tmpl.data_ptr(), mean_t.data_ptr(), s.data_ptr(), disp.data_ptr(),
        int(bool(mean_normalization)), off.data_ptr(), mar.data_ptr(), _stream(torch)))
    patches.offset[...] = _np(off)
    patches.mean_abs_residual[...] = _np(mar)


@dataclass
class PatchState:
    """State of one template patch and its displacement estimate
    (inverse_search.py:394-410)."""

    center: tuple[float, float]
    patch_size: int
    template: np.ndarray            # (ps, ps)
    steepest_descent: np.ndarray    # (ps, ps, 2)
    hessian: np.ndarray             # (2, 2)
    hessian_inverse: np.ndarray | None
    template_mean: float
    valid: bool
    displacement: np.ndarray        # (2,)
    init_displacement: np.ndarray   # (2,)
    mean_offset: float = 0.0
    mean_abs_residual: float = 0.0


def precompute_patch(level, center, patch_size: int, horizontal_only: bool = False) -> PatchState:
    """The precomputed state of a patch centred at ``center`` (x, y)
    (inverse_search.py:440-456)."""
    cx, cy = float(center[0]), float(center[1])
    half = 0.5 * patch_size
    pset = precompute_patch_set(level, np.array([cx - half]), np.array([cy - half]), patch_size,
                                horizontal_only=horizontal_only)
    ps = pset.patch_size
    h = pset.hessian[0]
    hi = pset.hessian_inv[0]
    return PatchState(
        center=(cx, cy), patch_size=ps, template=pset.templates[0].reshape(ps, ps),
        steepest_descent=np.stack([pset.steep_x[0].reshape(ps, ps),
                                   pset.steep_y[0].reshape(ps, ps)], axis=-1),
        hessian=np.array([[h[0], h[1]], [h[1], h[2]]]),
        hessian_inverse=(np.array([[hi[0], hi[1]], [hi[1], hi[2]]]) if pset.valid[0] else None),
        template_mean=float(pset.template_mean[0]), valid=bool(pset.valid[0]),
        displacement=np.zeros(2), init_displacement=np.zeros(2))


def optimize_patch(patch: PatchState, query, iterations: int, *, residual_norm: str = "l2",
                   huber_b: float = 1.0, mean_normalization: bool = True) -> PatchState:
    """Up to ``iterations`` inverse-search steps from the patch's
    initialisation (inverse_search.py:459-494); returns an updated copy."""
    if residual_norm not in NORM_CODES:
        raise ValueError(f"unknown residual norm {residual_norm!r}")
    ps = patch.patch_size
    half = 0.5 * ps
    if patch.valid:
        hi = patch.hessian_inverse
        hinv = np.array([[hi[0, 0], hi[0, 1], hi[1, 1]]])
    else:
        hinv = np.zeros((1, 3))
    pset = PatchSet(
        patch_size=ps, x_starts=np.array([patch.center[0] - half]),
        y_starts=np.array([patch.center[1] - half]),
        templates=np.ascontiguousarray(patch.template.reshape(1, -1)),
        steep_x=np.ascontiguousarray(patch.steepest_descent[:, :, 0].reshape(1, -1)),
        steep_y=np.ascontiguousarray(patch.steepest_descent[:, :, 1].reshape(1, -1)),
        hessian=np.zeros((1, 3)), hessian_inv=hinv,
        template_mean=np.array([patch.template_mean]), valid=np.array([bool(patch.valid)]),
        init_displacement=np.asarray(patch.init_displacement, dtype=np.float64).reshape(1, 2),
        displacement=np.zeros((1, 2)), offset=np.zeros(1), mean_abs_residual=np.zeros(1))
    optimize_patch_set(pset, query, iterations, residual_norm=residual_norm, huber_b=huber_b,
                       mean_normalization=mean_normalization)
    return replace(patch, displacement=pset.displacement[0].copy(),
                   mean_offset=float(pset.offset[0]),
                   mean_abs_residual=float(pset.mean_abs_residual[0]))
