"""Pyramids and the pyramid-level entry point of the flow path.

Mirrors the reference's containers and functions (core.py:33-72, 106-128;
pipeline.py:136-147):

* ``PyramidLevel`` / ``ImagePyramid`` — the same read-only containers (level
  rasters are CUDA tensors here, numpy arrays in the reference; either kind
  is accepted by ``dis_flow_on_pyramids``);
* ``as_image`` — the same validation and float64 conversion;
* ``build_pyramid(img, coarsest_scale, downscale=2)`` — levels 0..coarsest
  with gradients at every level, built on the GPU by ``dis_build_pyramid``
  (box-mean + central differences, bit-identical to the reference);
* ``dis_flow_on_pyramids(pyr_ref, pyr_qry, params, threads=1)`` — dense flow
  from prebuilt pyramids through ``dis_flow_batch_levels``;
* ``warmup(threads=1)`` — first-use initialisation (the reference JIT-compiles
  its numba kernels here, pipeline.py:290-305; this build loads the library,
  creates the CUDA context and runs one tiny pair of each mode).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .params import DisParams, ParameterError, to_c


@dataclass(frozen=True)
class PyramidLevel:
    """One pyramid level: the image plus its x/y gradient rasters (core.py:33-47)."""

    image: object
    grad_x: object
    grad_y: object
    scale_index: int

    @property
    def width(self) -> int:
        return int(self.image.shape[1])

    @property
    def height(self) -> int:
        return int(self.image.shape[0])


@dataclass(frozen=True)
class ImagePyramid:
    """Coarse-to-fine stack of levels; ``levels[0]`` is full resolution (core.py:50-62)."""

    levels: tuple
    downscale: int

    def __len__(self) -> int:
        return len(self.levels)

    def __getitem__(self, s: int) -> PyramidLevel:
        return self.levels[s]


def as_image(img) -> np.ndarray:
    """Validate and convert an intensity raster to contiguous float64 (core.py:65-72)."""
    arr = np.ascontiguousarray(img, dtype=np.float64)
    if arr.ndim != 2 or arr.shape[0] < 1 or arr.shape[1] < 1:
        raise ValueError(f"image must be 2D and non-empty, got shape {arr.shape}")
    if not np.isfinite(arr).all():
        raise ValueError("image contains non-finite values")
    return arr


def build_pyramid(img, coarsest_scale: int, downscale: int = 2) -> ImagePyramid:
    """Levels 0..coarsest_scale with gradients at every level (core.py:106-128),
    built on the GPU; the level rasters are float64 CUDA tensors."""
    from .pipeline import _require_cuda, _to_device_frames

    torch = _require_cuda()
    if coarsest_scale < 0:
        raise ParameterError("coarsest_scale must be >= 0")
    if downscale < 2 or int(downscale) != downscale:
        raise ParameterError("downscale must be an integer >= 2")
    shape = tuple(img.shape)
    if len(shape) != 2 or shape[0] < 1 or shape[1] < 1:
        raise ValueError(f"image must be 2D and non-empty, got shape {shape}")
    if shape[0] < 2 or shape[1] < 2:
        raise ValueError("image must be at least 2x2")
    from . import stages

    lv = stages.build_pyramid(_to_device_frames(img, torch.device("cuda")), int(coarsest_scale),
                              finest=0, second_derivatives=False, downscale=int(downscale))
    levels = tuple(PyramidLevel(d["img"][0], d["gx"][0], d["gy"][0], s)
                   for s, d in enumerate(lv))
    return ImagePyramid(levels, int(downscale))


def image_gradients(img):
    """Central differences with one-sided borders (core.py:75-85), on the GPU
    (``dis_build_pyramid`` level 0); numpy in -> numpy (gx, gy)."""
    lv = build_pyramid(img, 0)[0]
    return lv.grad_x.cpu().numpy(), lv.grad_y.cpu().numpy()


def upsample_flow(flow, new_width: int, new_height: int, scale_factor: int):
    """output(x) = scale * flow(x / scale), bilinear_map form (core.py:178-190),
    on the GPU (``dis_upsample_flow``)."""
    from . import stages
    from .pipeline import _require_cuda

    torch = _require_cuda()
    f = np.asarray(flow, dtype=np.float64)
    u = torch.from_numpy(np.ascontiguousarray(f[None, :, :, 0])).cuda()
    v = torch.from_numpy(np.ascontiguousarray(f[None, :, :, 1])).cuda()
    ou, ov = stages.upsample_flow(u, v, int(new_width), int(new_height), int(scale_factor))
    return np.stack([ou[0].cpu().numpy(), ov[0].cpu().numpy()], axis=-1)


def _dev64(x, device):
    import torch

    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.asarray(x))
    return t.to(device=device, dtype=torch.float64).contiguous()


def dis_flow_on_pyramids(pyr_ref, pyr_qry, params: DisParams, threads: int = 1):
    """Dense flow from prebuilt pyramids (pipeline.py:136-147): an (H, W, 2)
    float64 field at level-0 resolution.  Pyramids from ``build_pyramid`` (CUDA
    tensors) or the reference's own ``ImagePyramid`` (numpy) are accepted;
    the result is a CUDA tensor for the former and numpy for the latter."""
    from .pipeline import _require_cuda

    torch = _require_cuda()
    params.validate()
    if params.mode == "stereo":
        raise ValueError("use dis_stereo for stereo-mode parameters")
    if tuple(pyr_ref[0].image.shape) != tuple(pyr_qry[0].image.shape):
        raise ValueError(f"frame dimensions differ: {tuple(pyr_ref[0].image.shape)[::-1]} vs "
                         f"{tuple(pyr_qry[0].image.shape)[::-1]}")
    ss = params.coarsest_scale
    for pyr in (pyr_ref, pyr_qry):
        k = getattr(pyr, "downscale", params.downscale)
        if int(k) != int(params.downscale):
            raise ValueError(f"pyramid factor {k} differs from params.downscale "
                             f"{params.downscale}; this path uses one factor for both")
    if len(pyr_ref) <= ss or len(pyr_qry) <= ss:
        raise IndexError("pyramid has fewer levels than coarsest_scale + 1")
    coarse = pyr_ref[ss]
    if coarse.width < params.patch_size or coarse.height < params.patch_size:
        raise ValueError(
            f"coarsest level {coarse.width}x{coarse.height} cannot hold a "
            f"{params.patch_size}px patch; lower coarsest_scale")
    as_torch = isinstance(pyr_ref[0].image, torch.Tensor)
    dev = pyr_ref[0].image.device if as_torch else torch.device("cuda")
    H, W = (int(d) for d in pyr_ref[0].image.shape)
    keep = []

    def ptrs(pyr, attr):
        arr = (ctypes.c_void_p * (ss + 1))()
        for s in range(ss + 1):
            t = _dev64(getattr(pyr[s], attr), dev)
            keep.append(t)
            arr[s] = t.data_ptr()
        return arr

    p1 = [ptrs(pyr_ref, a) for a in ("image", "grad_x", "grad_y")]
    p2 = [ptrs(pyr_qry, a) for a in ("image", "grad_x", "grad_y")]
    cp = to_c(params)
    L = _lib.lib()
    nbytes = int(L.dis_workspace_bytes(1, H, W, ctypes.byref(cp)))
    ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
    out = torch.empty((1, H, W, 2), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    _lib.check(L.dis_flow_batch_levels(*p1, *p2, 1, H, W, ctypes.byref(cp), out.data_ptr(),
                                       ws.data_ptr(), nbytes, _lib.stream_handle(stream)))
    status = ctypes.c_uint32(0)
    _lib.check(L.dis_read_status(ws.data_ptr(), ctypes.byref(status),
                                 _lib.stream_handle(stream)))
    _lib.check(L.dis_status_to_error(status.value))
    del keep
    return out[0] if as_torch else out[0].cpu().numpy()


def warmup(threads: int = 1) -> None:
    """Load the library, create the CUDA context and run one tiny pair of
    each mode (the reference's warmup, pipeline.py:290-305, JIT-compiles its
    kernels on the same sizes)."""
    from .pipeline import dis_flow, dis_stereo

    rng = np.random.default_rng(0)
    img = rng.uniform(0.0, 255.0, size=(12, 16))
    shifted = np.roll(img, 1, axis=1)
    dis_flow(img, shifted, DisParams(patch_size=4, overlap=0.5, iterations=2, finest_scale=0,
                                     coarsest_scale=1, bidirectional=True))
    dis_stereo(img, shifted, DisParams(patch_size=4, overlap=0.5, iterations=2,
                                       finest_scale=0, coarsest_scale=1, mode="stereo"))
