"""Stage-level operators of the DIS path (the reference's numba operator layer)
on CUDA tensors, each calling one C-ABI stage entry point.  Used by the
stage-parity tests; the production path is ``dis_flow_batch`` which runs all
stages inside the library.

Rasters are float64 row-major (B, H, W) torch CUDA tensors, like the
reference's (H, W) float64 arrays.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .params import DisParams, to_c
from .pipeline import _dtype_code, _require_cuda, _to_device_frames


def _cur(t) -> int:
    """cudaStream_t of torch's current stream on tensor ``t``'s device (the
    stage launches are ordered after the work that produced their inputs)."""
    import torch

    return _lib.stream_handle(torch.cuda.current_stream(t.device))


def grid_axis(dim: int, patch_size: int, overlap: float) -> np.ndarray:
    """_axis_origins of create_grid (densification.py:50-79)."""
    L = _lib.lib()
    n = L.dis_grid_axis(dim, patch_size, overlap, None, 0)
    _lib.check(min(n, 0))
    out = (ctypes.c_int32 * n)()
    L.dis_grid_axis(dim, patch_size, overlap, out, n)
    return np.frombuffer(out, dtype=np.int32).astype(np.int64)


def build_pyramid(frames, coarsest: int, finest: int = 0, second_derivatives: bool = True,
                  level0: bool = True, downscale: int = 2):
    """build_pyramid (core.py:106-128) for a batch of frames: list over levels
    0..coarsest of dicts {img, gx, gy, dd}; gradients only for levels
    >= finest (dd = (B, 4, H, W): gxx, gxy, gyx, gyy).  ``level0=False``
    leaves level 0's float64 image out (level 1 is built straight from the
    frames, as on the flow path when the finest scale is >= 1)."""
    torch = _require_cuda()
    f = _to_device_frames(frames, "cuda")
    if f.dim() == 2:
        f = f.unsqueeze(0)
    B, H, W = f.shape
    levels = []
    h, w = H, W
    for s in range(coarsest + 1):
        if s:
            h, w = h // downscale, w // downscale
        lv = {}
        if s > 0 or level0 or finest == 0:
            lv["img"] = torch.empty((B, h, w), dtype=torch.float64, device=f.device)
        if s >= finest:
            lv["gx"] = torch.empty_like(lv["img"])
            lv["gy"] = torch.empty_like(lv["img"])
            if second_derivatives:
                lv["dd"] = torch.empty((B, 4, h, w), dtype=torch.float64, device=f.device)
        levels.append(lv)
    arr = ctypes.c_void_p * (coarsest + 1)
    img = arr(*[lv["img"].data_ptr() if "img" in lv else None for lv in levels])
    gx = arr(*[lv["gx"].data_ptr() if "gx" in lv else None for lv in levels])
    gy = arr(*[lv["gy"].data_ptr() if "gy" in lv else None for lv in levels])
    dd = arr(*[lv["dd"].data_ptr() if "dd" in lv else None for lv in levels])
    status = torch.zeros(1, dtype=torch.int32, device=f.device)
    _lib.check(_lib.lib().dis_build_pyramid(f.data_ptr(), _dtype_code(f), B, H, W, coarsest,
                                            int(downscale), img, gx, gy, dd, status.data_ptr(),
                                            _cur(f)))
    if int(status.item()) != 0:
        raise ValueError("image contains non-finite values")
    return levels


def patch_search(ref: dict, qry_img, params: DisParams, coarse_u=None, coarse_v=None):
    """_ScaleState.search (pipeline.py:54-82) on one level: dict of (B, P)
    tensors u, v, off, mar, init_u, init_v, valid."""
    torch = _require_cuda()
    B, H, W = ref["img"].shape
    xo = grid_axis(W, params.patch_size, params.overlap)
    yo = grid_axis(H, params.patch_size, params.overlap)
    P = len(xo) * len(yo)
    dev = ref["img"].device
    out = {k: torch.empty((B, P), dtype=torch.float64, device=dev)
           for k in ("u", "v", "off", "mar", "init_u", "init_v")}
    out["valid"] = torch.empty((B, P), dtype=torch.uint8, device=dev)
    Hc = Wc = 0
    if coarse_u is not None:
        Hc, Wc = coarse_u.shape[-2:]
    cp = to_c(params)
    nbytes = int(_lib.lib().dis_patch_search_workspace_bytes(B, W, H, ctypes.byref(cp)))
    ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
    rc = _lib.lib().dis_patch_search(
        ref["img"].data_ptr(), ref["gx"].data_ptr(), ref["gy"].data_ptr(), qry_img.data_ptr(),
        B, W, H, _lib.ptr(coarse_u), _lib.ptr(coarse_v), Wc, Hc, ctypes.byref(cp),
        out["u"].data_ptr(), out["v"].data_ptr(), out["off"].data_ptr(), out["mar"].data_ptr(),
        out["init_u"].data_ptr(), out["init_v"].data_ptr(), out["valid"].data_ptr(),
        ws.data_ptr(), nbytes, _cur(ref["img"]))
    _lib.check(rc)
    out["x_origins"] = xo
    out["y_origins"] = yo
    return out


def densify(ref_img, qry_img, params: DisParams, pu, pv, poff):
    """densify (densification.py:173-191) -> (u, v) (B, H, W)."""
    torch = _require_cuda()
    B, H, W = ref_img.shape
    fu = torch.empty_like(ref_img)
    fv = torch.empty_like(ref_img)
    status = torch.zeros(1, dtype=torch.int32, device=ref_img.device)
    cp = to_c(params)
    _lib.check(_lib.lib().dis_densify(ref_img.data_ptr(), qry_img.data_ptr(), B, W, H,
                                      ctypes.byref(cp), pu.data_ptr(), pv.data_ptr(),
                                      poff.data_ptr(), fu.data_ptr(), fv.data_ptr(),
                                      status.data_ptr(), _cur(ref_img)))
    if int(status.item()) != 0:
        raise AssertionError("pixel without a contributing patch; grid coverage broken")
    return fu, fv


def refine(fu, fv, ref: dict, qry: dict, params: DisParams, outer: int):
    """refine (variational.py:220-275) with ``outer`` fixed-point iterations;
    returns new (u, v)."""
    torch = _require_cuda()
    B, H, W = fu.shape
    u = fu.clone()
    v = fv.clone()
    L = _lib.lib()
    nbytes = L.dis_refine_workspace_bytes(B, W, H)
    ws = torch.empty(int(nbytes), dtype=torch.uint8, device=fu.device)
    status = torch.zeros(1, dtype=torch.int32, device=fu.device)
    cp = to_c(params)
    _lib.check(L.dis_refine(ref["img"].data_ptr(), ref["gx"].data_ptr(), ref["gy"].data_ptr(),
                            ref["dd"].data_ptr(), qry["img"].data_ptr(), qry["gx"].data_ptr(),
                            qry["gy"].data_ptr(), qry["dd"].data_ptr(), B, W, H,
                            ctypes.byref(cp), int(outer), u.data_ptr(), v.data_ptr(),
                            ws.data_ptr(), int(nbytes), status.data_ptr(), _cur(fu)))
    if int(status.item()) != 0:
        raise RuntimeError("variational refinement produced a non-finite value")
    return u, v


def upsample_flow(fu, fv, new_width: int, new_height: int, scale_factor: int = 2):
    """upsample_flow (core.py:178-190) by ``scale_factor`` -> (u, v)
    (B, new_height, new_width)."""
    torch = _require_cuda()
    B, H, W = fu.shape
    ou = torch.empty((B, new_height, new_width), dtype=torch.float64, device=fu.device)
    ov = torch.empty_like(ou)
    _lib.check(_lib.lib().dis_upsample_flow(fu.data_ptr(), fv.data_ptr(), B, W, H,
                                            ou.data_ptr(), ov.data_ptr(), new_width,
                                            new_height, int(scale_factor), _cur(fu)))
    return ou, ov


def densify_bidirectional(ref_img, qry_img, params: DisParams, fu_p, fv_p, foff, bu_p, bv_p,
                          boff):
    """densify_bidirectional (densification.py:194-234) -> (u, v) (B, H, W):
    forward patch set (fu_p, fv_p, foff: (B, P) on the reference frame)
    merged with the negated backward set (on the query frame, same grid)."""
    torch = _require_cuda()
    B, H, W = ref_img.shape
    fu = torch.empty_like(ref_img)
    fv = torch.empty_like(ref_img)
    status = torch.zeros(1, dtype=torch.int32, device=ref_img.device)
    cp = to_c(params)
    L = _lib.lib()
    nbytes = int(L.dis_densify_bidirectional_workspace_bytes(B, W, H, ctypes.byref(cp)))
    ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=ref_img.device)
    f64 = lambda t: t.to(device=ref_img.device, dtype=torch.float64).contiguous()  # noqa: E731
    args = [f64(t) for t in (fu_p, fv_p, foff, bu_p, bv_p, boff)]
    _lib.check(L.dis_densify_bidirectional(
        ref_img.data_ptr(), qry_img.data_ptr(), B, W, H, ctypes.byref(cp),
        *[t.data_ptr() for t in args], fu.data_ptr(), fv.data_ptr(), ws.data_ptr(), nbytes,
        status.data_ptr(), _cur(ref_img)))
    if int(status.item()) != 0:
        raise AssertionError("pixel without a contributing patch; grid coverage broken")
    return fu, fv
