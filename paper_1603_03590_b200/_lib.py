"""ctypes binding of libdis_b200.so (the C ABI in include/dis_b200.h).

The library is built in-tree (``paper_1603_03590_b200/libdis_b200.so``, see
``__graft_entry__.build``).  There is no fallback: if the library or a CUDA
device is missing, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from functools import lru_cache

from .params import DisParamsC, ParameterError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libdis_b200.so")
# kernel experiments only (tools/build_variant.sh): an alternative in-tree build
# of the same library, e.g. exp_so/libdis_<tag>.so
if os.environ.get("DIS_B200_LIB"):
    LIB_PATH = os.path.abspath(os.environ["DIS_B200_LIB"])

DIS_OK = 0
DIS_ERR_PARAMETER = -1
DIS_ERR_VALUE = -2
DIS_ERR_COVERAGE = -3
DIS_ERR_NONFINITE = -4
DIS_ERR_CUDA = -5
DIS_ERR_WORKSPACE = -6

DTYPE_F32, DTYPE_F64, DTYPE_U8 = 0, 1, 2
# dis_flow_batch_host_ex flags
HOST_ASYNC, HOST_FLOW_F32, HOST_STEREO = 1, 2, 4

# every symbol include/dis_b200.h declares
EXPORTED = (
    "dis_params_default", "dis_params_validate", "dis_workspace_bytes", "dis_flow_batch",
    "dis_host_workspace_bytes", "dis_flow_batch_host", "dis_read_status",
    "dis_status_to_error", "dis_build_pyramid", "dis_patch_search",
    "dis_patch_search_workspace_bytes", "dis_densify",
    "dis_refine_workspace_bytes", "dis_refine", "dis_upsample_flow", "dis_grid_axis",
    "dis_last_error", "dis_abi_version", "dis_last_launch_count", "dis_profile_enable",
    "dis_profile_reset", "dis_profile_read", "dis_selftest_div", "dis_census_enable",
    "dis_census_read", "dis_selftest_fp64_peak", "dis_compose_flows", "dis_stereo_batch",
    "dis_stereo_batch_host", "dis_densify_bidirectional",
    "dis_densify_bidirectional_workspace_bytes", "dis_sparse_workspace_bytes",
    "dis_sparse_correspondences", "dis_flow_batch_levels", "dis_profile_log",
    "dis_precompute_patch_set", "dis_optimize_patch_set", "dis_refresh_patch_stats",
    "dis_init_patches", "dis_reset_outliers",
    "dis_flow_batch_host_async", "dis_stereo_batch_host_async", "dis_host_batch_finish",
    "dis_flow_batch_host_ex",
)

KERNEL_CLASSES = ("pyramid", "patch_search", "densify", "tensor_assemble", "sor", "upsample")

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_sz = ctypes.c_size_t
_pp = ctypes.POINTER(DisParamsC)


class DisB200Error(RuntimeError):
    """CUDA-level failure inside libdis_b200 (status DIS_ERR_CUDA/WORKSPACE)."""


@lru_cache(maxsize=1)
def lib() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise DisB200Error(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    L.dis_params_default.argtypes = [_pp]
    L.dis_params_default.restype = None
    L.dis_params_validate.argtypes = [_pp]
    L.dis_params_validate.restype = ctypes.c_int
    L.dis_workspace_bytes.argtypes = [_i32, _i32, _i32, _pp]
    L.dis_workspace_bytes.restype = _sz
    L.dis_host_workspace_bytes.argtypes = [_i32, _i32, _i32, _i32, _pp]
    L.dis_host_workspace_bytes.restype = _sz
    L.dis_flow_batch.argtypes = [_vp, _vp, _i32, _i32, _i32, _i32, _pp, _vp, _vp, _sz, _vp]
    L.dis_flow_batch.restype = ctypes.c_int
    L.dis_flow_batch_host.argtypes = [_vp, _vp, _i32, _i32, _i32, _i32, _pp, _vp, _vp, _sz,
                                      _vp]
    L.dis_flow_batch_host.restype = ctypes.c_int
    L.dis_read_status.argtypes = [_vp, ctypes.POINTER(ctypes.c_uint32), _vp]
    L.dis_read_status.restype = ctypes.c_int
    L.dis_status_to_error.argtypes = [ctypes.c_uint32]
    L.dis_status_to_error.restype = ctypes.c_int
    L.dis_build_pyramid.argtypes = [_vp, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp,
                                    _vp, _vp, _vp]
    L.dis_build_pyramid.restype = ctypes.c_int
    L.dis_patch_search.argtypes = [_vp, _vp, _vp, _vp, _i32, _i32, _i32, _vp, _vp, _i32, _i32,
                                   _pp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]
    L.dis_patch_search_workspace_bytes.argtypes = [_i32, _i32, _i32, _pp]
    L.dis_patch_search_workspace_bytes.restype = _sz
    L.dis_patch_search.restype = ctypes.c_int
    L.dis_densify.argtypes = [_vp, _vp, _i32, _i32, _i32, _pp, _vp, _vp, _vp, _vp, _vp, _vp,
                              _vp]
    L.dis_densify.restype = ctypes.c_int
    L.dis_refine_workspace_bytes.argtypes = [_i32, _i32, _i32]
    L.dis_refine_workspace_bytes.restype = _sz
    L.dis_refine.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _pp,
                             _i32, _vp, _vp, _vp, _sz, _vp, _vp]
    L.dis_refine.restype = ctypes.c_int
    L.dis_upsample_flow.argtypes = [_vp, _vp, _i32, _i32, _i32, _vp, _vp, _i32, _i32, _i32, _vp]
    L.dis_upsample_flow.restype = ctypes.c_int
    L.dis_flow_batch_levels.argtypes = [_vp] * 6 + [_i32, _i32, _i32, _pp, _vp, _vp, _sz, _vp]
    L.dis_flow_batch_levels.restype = ctypes.c_int
    L.dis_stereo_batch.argtypes = L.dis_flow_batch.argtypes
    L.dis_stereo_batch.restype = ctypes.c_int
    L.dis_stereo_batch_host.argtypes = L.dis_flow_batch_host.argtypes
    L.dis_stereo_batch_host.restype = ctypes.c_int
    L.dis_flow_batch_host_async.argtypes = L.dis_flow_batch_host.argtypes
    L.dis_flow_batch_host_async.restype = ctypes.c_int
    L.dis_stereo_batch_host_async.argtypes = L.dis_flow_batch_host.argtypes
    L.dis_stereo_batch_host_async.restype = ctypes.c_int
    L.dis_flow_batch_host_ex.argtypes = L.dis_flow_batch_host.argtypes + [ctypes.c_uint32]
    L.dis_flow_batch_host_ex.restype = ctypes.c_int
    L.dis_host_batch_finish.argtypes = [_vp, _i32, _i32, _i32, _i32, _pp, _vp]
    L.dis_host_batch_finish.restype = ctypes.c_int
    L.dis_densify_bidirectional_workspace_bytes.argtypes = [_i32, _i32, _i32, _pp]
    L.dis_densify_bidirectional_workspace_bytes.restype = _sz
    L.dis_densify_bidirectional.argtypes = [_vp, _vp, _i32, _i32, _i32, _pp] + [_vp] * 9 + [
        _sz, _vp, _vp]
    L.dis_densify_bidirectional.restype = ctypes.c_int
    L.dis_sparse_workspace_bytes.argtypes = [_i32, _i32, _i32, _pp]
    L.dis_sparse_workspace_bytes.restype = _sz
    L.dis_sparse_correspondences.argtypes = [_vp, _vp, _i32, _i32, _i32, _pp, _vp, _i32, _vp,
                                             _vp, _vp, _sz, _vp]
    L.dis_sparse_correspondences.restype = ctypes.c_int
    L.dis_precompute_patch_set.argtypes = [_vp, _vp, _vp, _i32, _i32, _vp, _vp, _i32, _i32,
                                           _i32] + [_vp] * 8
    L.dis_precompute_patch_set.restype = ctypes.c_int
    L.dis_optimize_patch_set.argtypes = [_vp, _i32, _i32, _vp, _vp, _i32, _i32] + [_vp] * 7 + [
        _i32, _i32, _i32, ctypes.c_double, _vp, _vp, _vp, _vp]
    L.dis_optimize_patch_set.restype = ctypes.c_int
    L.dis_refresh_patch_stats.argtypes = [_vp, _i32, _i32, _vp, _vp, _i32, _i32, _vp, _vp, _vp,
                                          _vp, _i32, _vp, _vp, _vp]
    L.dis_refresh_patch_stats.restype = ctypes.c_int
    L.dis_init_patches.argtypes = [_vp, _i32, _i32, _vp, _i32, _i32, _vp, _vp]
    L.dis_init_patches.restype = ctypes.c_int
    L.dis_reset_outliers.argtypes = [_vp, _vp, _i32, _i32, _vp, _vp, _vp]
    L.dis_reset_outliers.restype = ctypes.c_int
    L.dis_compose_flows.argtypes = [_vp, _vp, _i32, _i32, _i32, _vp, _vp]
    L.dis_compose_flows.restype = ctypes.c_int
    L.dis_grid_axis.argtypes = [_i32, _i32, ctypes.c_double, ctypes.POINTER(_i32), _i32]
    L.dis_grid_axis.restype = _i32
    L.dis_last_error.argtypes = []
    L.dis_last_error.restype = ctypes.c_char_p
    L.dis_last_launch_count.argtypes = []
    L.dis_last_launch_count.restype = ctypes.c_longlong
    L.dis_profile_enable.argtypes = [_i32]
    L.dis_profile_enable.restype = None
    L.dis_profile_reset.argtypes = []
    L.dis_profile_reset.restype = None
    L.dis_profile_read.argtypes = [ctypes.POINTER(ctypes.c_double),
                                   ctypes.POINTER(ctypes.c_int64), _i32]
    L.dis_profile_read.restype = ctypes.c_int
    L.dis_profile_log.argtypes = [ctypes.POINTER(_i32), ctypes.POINTER(_i32),
                                  ctypes.POINTER(ctypes.c_double), _i32]
    L.dis_profile_log.restype = _i32
    L.dis_selftest_div.argtypes = [_vp, _vp, _vp, _vp, _sz, _vp]
    L.dis_selftest_div.restype = ctypes.c_int
    L.dis_census_enable.argtypes = [_i32]
    L.dis_census_enable.restype = ctypes.c_int
    L.dis_census_read.argtypes = [ctypes.POINTER(ctypes.c_longlong),
                                  ctypes.POINTER(ctypes.c_longlong)]
    L.dis_census_read.restype = ctypes.c_int
    L.dis_selftest_fp64_peak.argtypes = [ctypes.POINTER(ctypes.c_double),
                                         ctypes.POINTER(ctypes.c_double), _vp]
    L.dis_selftest_fp64_peak.restype = ctypes.c_int
    L.dis_abi_version.argtypes = []
    L.dis_abi_version.restype = _i32
    if L.dis_abi_version() != 2:
        raise DisB200Error(f"libdis_b200 ABI {L.dis_abi_version()} != 2")
    return L


def last_error() -> str:
    msg = lib().dis_last_error()
    return msg.decode() if msg else ""


def check(rc: int) -> None:
    """Raise the reference's exception type for a DIS_* status."""
    if rc == DIS_OK:
        return
    msg = last_error()
    if rc == DIS_ERR_PARAMETER:
        raise ParameterError(msg)
    if rc == DIS_ERR_VALUE:
        raise ValueError(msg)
    if rc == DIS_ERR_COVERAGE:
        raise AssertionError(msg)
    if rc == DIS_ERR_NONFINITE:
        raise RuntimeError(msg)
    raise DisB200Error(f"libdis_b200 status {rc}: {msg}")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None passes through as NULL)."""
    return None if t is None else t.data_ptr()


def stream_handle(stream) -> int:
    """cudaStream_t of a torch.cuda.Stream (0 = legacy default stream)."""
    return 0 if stream is None else stream.cuda_stream
