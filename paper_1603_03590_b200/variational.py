"""Reference-signature refinement (reference variational.py:220-275):
``refine(flow, reference, query, params, scale_index, horizontal_only=False)``
on the GPU (``dis_refine``: tensors + assembly fused, wavefront SOR).  The
levels are ``PyramidLevel``s (this package's or the reference's own);
numpy in, numpy out; the reference's exceptions."""

from __future__ import annotations

import numpy as np

from .params import DisParams, VarParams


def refine(flow, reference, query, params: VarParams, scale_index: int,
           horizontal_only: bool = False) -> np.ndarray:
    """Refine a dense field on its own scale: ``params.outer_iters(scale_index)``
    fixed-point iterations of ``params.inner_sor_iters`` SOR sweeps."""
    from . import stages
    from .pipeline import _require_cuda

    torch = _require_cuda()
    params.validate()
    ref_img = np.asarray(reference.image.cpu() if hasattr(reference.image, "cpu")
                         else reference.image)
    shape = tuple(ref_img.shape)
    if tuple(query.image.shape) != shape:
        raise ValueError("reference and query levels must share dimensions")
    f = np.asarray(flow, dtype=np.float64)
    if f.shape[:2] != shape:
        raise ValueError("flow dimensions must match the levels")
    if not np.isfinite(f).all():
        raise ValueError("initial flow contains non-finite values")

    def dev(x):
        t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.asarray(x))
        return t.to(device="cuda", dtype=torch.float64).contiguous()[None]

    def level(lv):
        return {"img": dev(lv.image), "gx": dev(lv.grad_x), "gy": dev(lv.grad_y),
                "dd": None}

    lr, lq = level(reference), level(query)
    # dis_refine ignores the dd rasters (formed on the fly); pass the level
    # images as placeholders for the ABI slots
    lr["dd"], lq["dd"] = lr["img"], lq["img"]
    dp = DisParams(variational=params, mode="stereo" if horizontal_only else "flow")
    u, v = stages.refine(dev(f[:, :, 0]), dev(f[:, :, 1]), lr, lq, dp,
                         int(params.outer_iters(scale_index)))
    return np.stack([u[0].cpu().numpy(), v[0].cpu().numpy()], axis=-1)
