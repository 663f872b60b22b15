"""Host side of the DIS flow path: the reference's public entry points
(``dis_flow``, pipeline.py:150-163) on top of the sm_100a kernels in
libdis_b200.so.

The coarse-to-fine loop itself (pipeline.py:85-133) runs inside the C ABI
(``dis_flow_batch``), which enqueues every kernel of every scale for a whole
batch of pairs on one CUDA stream.  PyTorch provides device memory and
streams only.  There is no CPU fallback: without a CUDA device and the built
library these functions raise.
"""

from __future__ import annotations

import ctypes
from typing import NamedTuple

import numpy as np

from . import _lib
from .params import DisParams, ParameterError, to_c

_TORCH_DT = None


def _torch():
    import torch

    return torch


def _require_cuda():
    torch = _torch()
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_1603_03590_b200 runs on a CUDA device (B200, sm_100a); "
            "no CUDA device is visible and there is no CPU fallback")
    return torch


def _dtype_code(t):
    torch = _torch()
    if t.dtype == torch.float32:
        return _lib.DTYPE_F32
    if t.dtype == torch.float64:
        return _lib.DTYPE_F64
    if t.dtype == torch.uint8:
        return _lib.DTYPE_U8
    raise TypeError(t.dtype)


def _to_device_frames(x, device):
    """(B, H, W) or (H, W) real raster -> contiguous CUDA tensor of a dtype the
    kernels take (f32/f64/u8; anything else is converted to float64 exactly
    like as_image, core.py:65-72)."""
    torch = _torch()
    if isinstance(x, torch.Tensor):
        t = x
    else:
        a = np.asarray(x)
        if a.dtype not in (np.float32, np.float64, np.uint8):
            a = a.astype(np.float64)
        t = torch.from_numpy(np.ascontiguousarray(a))
    if t.dtype not in (torch.float32, torch.float64, torch.uint8):
        t = t.to(torch.float64)
    return t.to(device=device, non_blocking=True).contiguous()


def _promote_pair(f1, f2):
    """as_image converts BOTH frames to float64 (core.py:65-72): a pair of
    different dtypes is promoted to float64 together (exact for u8/f32), never
    narrowed to the first frame's dtype."""
    if f1.dtype == f2.dtype:
        return f1, f2
    torch = _torch()
    return f1.to(torch.float64), f2.to(torch.float64)


def _promote_pair_np(a, b):
    if a.dtype not in (np.float32, np.float64, np.uint8):
        a = a.astype(np.float64)
    if b.dtype not in (np.float32, np.float64, np.uint8):
        b = b.astype(np.float64)
    if a.dtype != b.dtype:
        a, b = a.astype(np.float64), b.astype(np.float64)
    return np.ascontiguousarray(a), np.ascontiguousarray(b)


class FlowEngine:
    """A reusable device workspace for batches of ``B`` pairs of ``H x W``
    frames at one parameter set (the workspace layout is fixed by
    ``dis_workspace_bytes``)."""

    def __init__(self, batch: int, height: int, width: int, params: DisParams | None = None,
                 device=None, stereo: bool = False):
        torch = _require_cuda()
        self.stereo = bool(stereo)
        if params is None:
            params = DisParams.preset(2, stereo=self.stereo)
        self.params = params
        self.params.validate()
        if self.params.mode == "stereo" and not self.stereo:
            raise ValueError("use dis_stereo for stereo-mode parameters")
        self.B, self.H, self.W = int(batch), int(height), int(width)
        dev = torch.device(device) if device is not None else torch.device("cuda")
        if dev.type != "cuda":
            raise ValueError(f"FlowEngine needs a CUDA device, got {dev}")
        self.device = torch.device("cuda", dev.index if dev.index is not None
                                   else torch.cuda.current_device())
        self.cparams = to_c(self.params)
        L = _lib.lib()
        _lib.check(L.dis_params_validate(ctypes.byref(self.cparams)))
        n = L.dis_workspace_bytes(self.B, self.H, self.W, ctypes.byref(self.cparams))
        if n == 0:  # re-run the checks to raise the precise error
            _lib.check(L.dis_flow_batch(None, None, 0, self.B, self.H, self.W,
                                        ctypes.byref(self.cparams), None, None, 0, None))
            raise ValueError("invalid problem size")
        self.workspace_bytes = int(n)
        self.workspace = torch.empty(self.workspace_bytes, dtype=torch.uint8,
                                     device=self.device)
        self._host_ws = None
        self._pending = None  # (frames, out, dtype code, stream) of a submitted host batch

    # -- device-resident path ------------------------------------------------
    def run(self, frames1, frames2, out=None, stream=None, check: bool = True,
            graph: bool = False):
        """Flow of every pair: (B, H, W, 2) float64 CUDA tensor.  ``frames*``
        are (B, H, W) CUDA tensors (f32/f64/u8).  With ``check`` the device
        status word is read back (one small synchronising copy) and turned
        into the reference's exception types.

        ``graph=True`` replays the whole launch sequence as one CUDA graph,
        captured on the first call for these frame/output buffers and stream
        (the kernels and their arguments are identical to the eager path, so
        the results are too; it saves the per-kernel launch gaps, ~16 % of a
        single 1024x436 pair).  The buffers must stay alive and in place."""
        if graph:
            return self._run_graph(frames1, frames2, out, stream, check)
        torch = _torch()
        with torch.cuda.device(self.device):
            if stream is None:
                stream = torch.cuda.current_stream(self.device)
            f1 = _to_device_frames(frames1, self.device)
            f2 = _to_device_frames(frames2, self.device)
            if f1.dim() == 2:
                f1 = f1.unsqueeze(0)
            if f2.dim() == 2:
                f2 = f2.unsqueeze(0)
            if tuple(f1.shape) != (self.B, self.H, self.W) or tuple(f2.shape) != tuple(f1.shape):
                raise ValueError(
                    f"frame batch {tuple(f1.shape)} / {tuple(f2.shape)} does not match the "
                    f"engine ({self.B}, {self.H}, {self.W})")
            f1, f2 = _promote_pair(f1, f2)
            if out is None:
                out = torch.empty((self.B, self.H, self.W, 2), dtype=torch.float64,
                                  device=self.device)
            else:
                self._check_out_tensor(out)
            L = _lib.lib()
            fn = L.dis_stereo_batch if self.stereo else L.dis_flow_batch
            rc = fn(
                f1.data_ptr(), f2.data_ptr(), _dtype_code(f1), self.B, self.H, self.W,
                ctypes.byref(self.cparams), out.data_ptr(), self.workspace.data_ptr(),
                self.workspace_bytes, _lib.stream_handle(stream))
            _lib.check(rc)
            if check:
                self.check_status(stream)
        return out

    def _check_out_tensor(self, out):
        torch = _torch()
        want = (self.B, self.H, self.W, 2)
        if not isinstance(out, torch.Tensor):
            raise ValueError("out must be a CUDA tensor (use run_host for numpy buffers)")
        if (tuple(out.shape) != want or out.dtype != torch.float64 or not out.is_contiguous()
                or out.device != self._dev_index()):
            raise ValueError(
                f"out must be a contiguous float64 tensor of shape {want} on {self.device}, "
                f"got {tuple(out.shape)} {out.dtype} on {out.device}"
                f"{'' if out.is_contiguous() else ' (non-contiguous)'}")

    def _dev_index(self):
        return self.device

    def _run_graph(self, frames1, frames2, out, stream, check):
        torch = _torch()
        if out is None:
            raise ValueError("graph replay needs a persistent output tensor (out=...)")
        self._check_out_tensor(out)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        key = (frames1.data_ptr(), frames2.data_ptr(), out.data_ptr(), frames1.dtype,
               tuple(frames1.shape), stream.cuda_stream)
        if getattr(self, "_graph_key", None) != key:
            self.run(frames1, frames2, out=out, stream=stream, check=True)  # first-use set-up
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                self.run(frames1, frames2, out=out, stream=stream, check=False)
            self._graph, self._graph_key = g, key
        with torch.cuda.device(self.device), torch.cuda.stream(stream):
            self._graph.replay()
        if check:
            self.check_status(stream)
        return out

    def check_status(self, stream=None) -> None:
        torch = _torch()
        status = ctypes.c_uint32(0)
        L = _lib.lib()
        with torch.cuda.device(self.device):
            if stream is None:
                stream = torch.cuda.current_stream(self.device)
            _lib.check(L.dis_read_status(self.workspace.data_ptr(), ctypes.byref(status),
                                         _lib.stream_handle(stream)))
        _lib.check(L.dis_status_to_error(status.value))

    # -- host-buffer path (the e2e boundary) ---------------------------------
    def run_host(self, frames1: np.ndarray, frames2: np.ndarray, out: np.ndarray | None = None,
                 stream=None, submit_only: bool = False) -> np.ndarray:
        """dis_flow_batch_host: host frames in, host flow out (copies
        included).  Pinned host buffers (torch ``pin_memory``) are fastest."""
        torch = _torch()
        if self._pending is not None:
            raise RuntimeError("run_host: a submitted batch is still in flight (finish_host)")
        a, b = _promote_pair_np(np.asarray(frames1), np.asarray(frames2))
        if a.ndim == 2:
            a = a[None]
        if b.ndim == 2:
            b = b[None]
        want = (self.B, self.H, self.W)
        if tuple(a.shape) != want or tuple(b.shape) != want:
            raise ValueError(f"frame batch {tuple(a.shape)} / {tuple(b.shape)} does not match "
                             f"the engine {want}")
        if out is None:
            out = np.empty((self.B, self.H, self.W, 2), dtype=np.float64)
        elif (not isinstance(out, np.ndarray) or out.shape != want + (2,)
              or out.dtype not in (np.float64, np.float32) or not out.flags.c_contiguous
              or not out.flags.writeable):
            raise ValueError(f"out must be a writeable C-contiguous float64 (or, opt-in, "
                             f"float32) array of shape {want + (2,)}")
        # a float32 `out` asks for the float64 flow rounded on the device before
        # the copy-out (DIS_HOST_FLOW_F32: == flow.astype(float32), half the
        # device->host bytes); the default float64 is the reference's return type
        f32 = out.dtype == np.float32
        code = {np.dtype(np.float32): 0, np.dtype(np.float64): 1, np.dtype(np.uint8): 2}[a.dtype]
        L = _lib.lib()
        with torch.cuda.device(self.device):
            if stream is None:
                stream = torch.cuda.current_stream(self.device)
            n = L.dis_host_workspace_bytes(self.B, self.H, self.W, code,
                                           ctypes.byref(self.cparams))
            if self._host_ws is None or self._host_ws.numel() < n:
                self._host_ws = torch.empty(int(n), dtype=torch.uint8, device=self.device)
            args = (a.ctypes.data, b.ctypes.data, code, self.B, self.H, self.W,
                    ctypes.byref(self.cparams), out.ctypes.data, self._host_ws.data_ptr(),
                    int(n), _lib.stream_handle(stream))
            if f32:
                flags = (_lib.HOST_FLOW_F32 | (_lib.HOST_ASYNC if submit_only else 0)
                         | (_lib.HOST_STEREO if self.stereo else 0))
                rc = L.dis_flow_batch_host_ex(*args, flags)
            elif submit_only:
                fn = L.dis_stereo_batch_host_async if self.stereo else L.dis_flow_batch_host_async
                rc = fn(*args)
            else:
                fn = L.dis_stereo_batch_host if self.stereo else L.dis_flow_batch_host
                rc = fn(*args)
        _lib.check(rc)
        if submit_only:
            # the call owns its buffers until finish_host: keep them alive
            self._pending = (a, b, out, code, stream)
        return out

    def submit_host(self, frames1: np.ndarray, frames2: np.ndarray, out: np.ndarray,
                    stream=None) -> None:
        """dis_flow_batch_host_async: enqueue a host-buffer batch (copies in,
        kernels, copies out, ordered after prior work on ``stream``) and return
        without waiting.  ``out`` (and the frames) belong to the call until
        ``finish_host`` returns.  Engines submitted on different streams run
        concurrently: a streaming caller keeps two engines in flight so one
        batch's copy-out overlaps the next batch's copy-in and kernels.  An
        engine has one workspace, hence one call in flight."""
        if self._pending is not None:
            raise RuntimeError("submit_host: the engine's previous batch was not finished "
                               "(finish_host)")
        if out is None:
            raise ValueError("submit_host needs the output buffer")
        self.run_host(frames1, frames2, out=out, stream=stream, submit_only=True)

    def finish_host(self) -> np.ndarray:
        """dis_host_batch_finish: wait for the submitted batch, raise what
        ``run_host`` would have raised, return its ``out``."""
        if self._pending is None:
            raise RuntimeError("finish_host: nothing was submitted")
        _a, _b, out, code, stream = self._pending
        self._pending = None
        L = _lib.lib()
        with _torch().cuda.device(self.device):
            rc = L.dis_host_batch_finish(self._host_ws.data_ptr(), self.B, self.H, self.W, code,
                                         ctypes.byref(self.cparams), _lib.stream_handle(stream))
        _lib.check(rc)
        return out


_ENGINES: dict = {}


def _engine(B, H, W, params, stereo=False, device=None):
    """Cached engine per (problem, parameters, device): the workspace lives on
    one device, so the current device is part of the key."""
    torch = _torch()
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    key = (B, H, W, params, stereo, str(device))
    eng = _ENGINES.get(key)
    if eng is None:
        if len(_ENGINES) > 8:
            _ENGINES.clear()
        eng = FlowEngine(B, H, W, params, device=device, stereo=stereo)
        _ENGINES[key] = eng
    return eng


def _device_of(x):
    torch = _torch()
    if isinstance(x, torch.Tensor) and x.is_cuda:
        return x.device
    return None


def _check_frame(a):
    """as_image's shape checks (core.py:65-72); finiteness is checked on the
    device (status word)."""
    shape = tuple(a.shape)
    if len(shape) != 2 or shape[0] < 1 or shape[1] < 1:
        raise ValueError(f"image must be 2D and non-empty, got shape {shape}")


def dis_flow_batch(frames1, frames2, params: DisParams | None = None):
    """Flow for a batch of independent pairs: frames (B, H, W) -> (B, H, W, 2)
    float64 CUDA tensor.  Pair i equals ``dis_flow(frames1[i], frames2[i])``
    bit for bit."""
    _require_cuda()
    params = params if params is not None else DisParams.preset(2)
    s1 = tuple(frames1.shape)
    s2 = tuple(frames2.shape)
    if len(s1) != 3:
        raise ValueError(f"frame batch must be (B, H, W), got {s1}")
    if s1 != s2:
        raise ValueError(f"frame dimensions differ: {s1[:0:-1]} vs {s2[:0:-1]}")
    eng = _engine(s1[0], s1[1], s1[2], params, device=_device_of(frames1))
    return eng.run(frames1, frames2)


def dis_flow(frame1, frame2, params: DisParams | None = None, threads: int = 1):
    """Dense optical flow from ``frame1`` to ``frame2`` (pipeline.py:150-163):
    an (H, W, 2) float64 field at the input resolution, numpy in -> numpy out,
    torch in -> torch (CUDA) out.  ``threads`` is accepted for signature
    compatibility (the reference's numba thread count)."""
    torch = _require_cuda()
    params = params if params is not None else DisParams.preset(2)
    _check_frame(frame1)
    _check_frame(frame2)
    if tuple(frame1.shape) != tuple(frame2.shape):
        raise ValueError(
            f"frame dimensions differ: {tuple(frame1.shape)[::-1]} vs "
            f"{tuple(frame2.shape)[::-1]}")
    if params.coarsest_scale < 0:
        raise ParameterError("coarsest_scale must be >= 0")
    h, w = frame1.shape
    eng = _engine(1, int(h), int(w), params, device=_device_of(frame1))
    out = eng.run(frame1, frame2)[0]
    if isinstance(frame1, torch.Tensor):
        return out
    return out.cpu().numpy()


def dis_stereo(left, right, params: DisParams | None = None, threads: int = 1):
    """Horizontal-only displacement between a rectified pair
    (pipeline.py:166-183): flow-style field, sampling ``right`` at x + u(x)
    matches ``left`` at x; the v channel is identically zero.  numpy in ->
    numpy out, torch in -> torch (CUDA) out."""
    torch = _require_cuda()
    params = params if params is not None else DisParams.preset(2, stereo=True)
    params.validate()
    _check_frame(left)
    _check_frame(right)
    if tuple(left.shape) != tuple(right.shape):
        raise ValueError(
            f"frame dimensions differ: {tuple(left.shape)[::-1]} vs "
            f"{tuple(right.shape)[::-1]}")
    h, w = left.shape
    out = _engine(1, int(h), int(w), params, stereo=True,
                  device=_device_of(left)).run(left, right)[0]
    if isinstance(left, torch.Tensor):
        return out
    return out.cpu().numpy()


def dis_stereo_batch(left, right, params: DisParams | None = None):
    """dis_stereo for a batch of independent rectified pairs: (B, H, W) ->
    (B, H, W, 2) float64 CUDA tensor."""
    _require_cuda()
    params = params if params is not None else DisParams.preset(2, stereo=True)
    s1, s2 = tuple(left.shape), tuple(right.shape)
    if len(s1) != 3:
        raise ValueError(f"frame batch must be (B, H, W), got {s1}")
    if s1 != s2:
        raise ValueError(f"frame dimensions differ: {s1[:0:-1]} vs {s2[:0:-1]}")
    return _engine(s1[0], s1[1], s1[2], params, stereo=True,
                   device=_device_of(left)).run(left, right)


class SparseMatch(NamedTuple):
    """One seed's result (pipeline.py:24-27)."""

    seed: tuple[float, float]
    displacement: tuple[float, float]
    valid: bool


def sparse_correspondences(frame1, frame2, seeds, params: DisParams | None = None,
                           threads: int = 1) -> list[SparseMatch]:
    """Displacements at seed locations only, in full-resolution pixels
    (pipeline.py:230-287).  With densification the seeds read the unrefined
    dense field of the finest computed scale; without it every seed runs its
    own patch chain down the scales.  Seeds outside the image come back
    flagged invalid.  One C-ABI call (dis_sparse_correspondences)."""
    torch = _require_cuda()
    params = params if params is not None else DisParams.preset(2)
    params.validate()
    _check_frame(frame1)
    _check_frame(frame2)
    if tuple(frame1.shape) != tuple(frame2.shape):
        raise ValueError(
            f"frame dimensions differ: {tuple(frame1.shape)[::-1]} vs "
            f"{tuple(frame2.shape)[::-1]}")
    seed_arr = np.ascontiguousarray(np.atleast_2d(np.asarray(seeds, dtype=np.float64)))
    if seed_arr.ndim != 2 or seed_arr.shape[1] != 2:
        raise ValueError(f"seeds must be (n, 2) x, y pairs, got shape {seed_arr.shape}")
    n = seed_arr.shape[0]
    h, w = (int(d) for d in frame1.shape)
    dev = _device_of(frame1) or torch.device("cuda", torch.cuda.current_device())
    f1 = _to_device_frames(frame1, dev)
    f2 = _to_device_frames(frame2, dev)
    f1, f2 = _promote_pair(f1, f2)
    cp = to_c(params)
    L = _lib.lib()
    nbytes = int(L.dis_sparse_workspace_bytes(h, w, n, ctypes.byref(cp)))
    if nbytes == 0:  # re-run the checks through the entry point to raise the precise error
        _lib.check(L.dis_sparse_correspondences(None, None, _dtype_code(f1), h, w,
                                                ctypes.byref(cp), None, 0, None, None, None,
                                                0, None))
        raise ValueError("invalid problem size")
    ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    disp = np.zeros((n, 2), dtype=np.float64)
    valid = np.zeros(n, dtype=np.uint8)
    with torch.cuda.device(dev):
        _lib.check(L.dis_sparse_correspondences(
            f1.data_ptr(), f2.data_ptr(), _dtype_code(f1), h, w, ctypes.byref(cp),
            seed_arr.ctypes.data, n, disp.ctypes.data, valid.ctypes.data, ws.data_ptr(), nbytes,
            _lib.stream_handle(torch.cuda.current_stream(dev))))
    return [SparseMatch((float(seed_arr[i, 0]), float(seed_arr[i, 1])),
                        (float(disp[i, 0]), float(disp[i, 1])), bool(valid[i]))
            for i in range(n)]


def compose_flows(flow_ab, flow_bc):
    """Chain two fields (pipeline.py:186-199): out(x) = ab(x) + bc(x + ab(x)),
    ``bc`` sampled with bilinear_map (clamped).  (H, W, 2) or a batch
    (B, H, W, 2); numpy in -> numpy out, torch in -> torch (CUDA) out.  One
    sm_100a kernel (compose.cu) per call."""
    torch = _require_cuda()
    as_torch = isinstance(flow_ab, torch.Tensor)
    s1, s2 = tuple(flow_ab.shape), tuple(flow_bc.shape)
    if s1 != s2:
        raise ValueError("flow fields must share dimensions to compose")
    if len(s1) not in (3, 4) or s1[-1] != 2:
        raise ValueError(f"flow fields must be (H, W, 2) or (B, H, W, 2), got {s1}")
    dev = flow_ab.device if as_torch and flow_ab.is_cuda else torch.device("cuda")

    def dev64(x):
        t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.asarray(x))
        return t.to(device=dev, dtype=torch.float64).contiguous()

    ab, bc = dev64(flow_ab), dev64(flow_bc)
    batched = ab.dim() == 4
    if not batched:
        ab, bc = ab.unsqueeze(0), bc.unsqueeze(0)
    B, H, W = ab.shape[:3]
    out = torch.empty_like(ab)
    if B * H * W:
        with torch.cuda.device(dev):
            _lib.check(_lib.lib().dis_compose_flows(
                ab.data_ptr(), bc.data_ptr(), B, H, W, out.data_ptr(),
                _lib.stream_handle(torch.cuda.current_stream(dev))))
    if not batched:
        out = out[0]
    return out if as_torch else out.cpu().numpy()
