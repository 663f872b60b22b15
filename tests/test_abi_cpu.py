"""CPU-only checks of the boundary: the C-ABI library loads and exports every
symbol include/dis_b200.h declares; host-side validation and grid logic
(no kernel launches); the parameter mirror follows the reference's tests
(pkg/tests/test_core.py:140-188)."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_1603_03590_b200 import _lib
from paper_1603_03590_b200.params import (DisParams, DisParamsC, ParameterError, VarParams,
                                          coarsest_scale_for, to_c)
from tests.conftest import REPO, golden
from tools import synth


def _header_symbols():
    src = open(os.path.join(REPO, "include", "dis_b200.h")).read()
    return sorted(set(re.findall(r"DIS_API [\w\s\*]*?\b(dis_\w+)\(", src)))


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    syms = _header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(_lib.EXPORTED) == syms


def _header_prototypes():
    """{name: [C parameter types]} of every DIS_API function in the header."""
    src = open(os.path.join(REPO, "include", "dis_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", " ", src, flags=re.S)
    out = {}
    for m in re.finditer(r"DIS_API\s+([^;]*?)\b(dis_\w+)\s*\(([^)]*)\)\s*;", src):
        params = [p.strip() for p in m.group(3).split(",") if p.strip() and p.strip() != "void"]
        types = []
        for p in params:
            p = " ".join(p.split())
            ptr = p.count("*")
            base = re.sub(r"\bconst\b|\*", " ", p).split()[0]
            types.append("ptr" if ptr else base)
        out[m.group(2)] = types
    return out


_CTYPE_OF = {"int32_t": ctypes.c_int32, "int": ctypes.c_int, "size_t": ctypes.c_size_t,
             "double": ctypes.c_double, "uint32_t": ctypes.c_uint32}


def test_ctypes_argtypes_match_header_prototypes():
    """Every binding in _lib declares exactly the header's parameter list
    (count, and pointer vs integer/float width), so no argument is
    truncated or shifted (a missing slot once shifted a stream handle into
    ctypes' default int conversion)."""
    L = _lib.lib()
    protos = _header_prototypes()
    assert set(protos) == set(_lib.EXPORTED)
    for name, types in protos.items():
        fn = getattr(L, name)
        at = fn.argtypes
        assert at is not None, f"{name}: argtypes not declared"
        assert len(at) == len(types), (name, len(at), len(types))
        for i, (t, a) in enumerate(zip(types, at)):
            if t == "ptr":
                assert a is ctypes.c_void_p or a is ctypes.c_char_p or hasattr(a, "contents") \
                    or issubclass(a, ctypes._Pointer), (name, i, a)
            else:
                want = _CTYPE_OF[t]
                assert ctypes.sizeof(a) == ctypes.sizeof(want), (name, i, t, a)
                assert (a in (ctypes.c_double, ctypes.c_float)) == (t == "double"), (name, i)


def test_params_struct_layout_matches_header():
    # dis_params_default fills the C struct; compare with DisParams() defaults
    c = DisParamsC()
    _lib.lib().dis_params_default(ctypes.byref(c))
    d = to_c(DisParams())
    for name, _ in DisParamsC._fields_:
        assert getattr(c, name) == getattr(d, name), name
    assert ctypes.sizeof(DisParamsC) == 112


def test_preset_tuples_and_coarsest_scale():
    expected = {1: (3, 16, 8, 0.30), 2: (3, 12, 8, 0.40), 3: (1, 16, 12, 0.75),
                4: (0, 256, 12, 0.75)}
    for n, (sf, it, ps, ov) in expected.items():
        p = DisParams.preset(n)
        assert (p.finest_scale, p.iterations, p.patch_size, p.overlap) == (sf, it, ps, ov)
    assert DisParams.preset(1).variational is None
    assert coarsest_scale_for(1024, 8, 8) == 5
    assert coarsest_scale_for(1226, 8, 8) == 6
    assert coarsest_scale_for(32, 8, 8) == 0
    assert coarsest_scale_for(2048, 8, 8) == 6
    assert DisParams.preset(2, width=64).coarsest_scale == 3
    assert VarParams().outer_iters(3) == 4
    assert VarParams(outer_iters_fixed=1).outer_iters(3) == 1


@pytest.mark.parametrize("kwargs", [
    dict(patch_size=1), dict(overlap=1.0), dict(overlap=-0.1), dict(iterations=0),
    dict(finest_scale=4, coarsest_scale=3), dict(downscale=1), dict(residual_norm="l3"),
    dict(residual_norm="huber", huber_b=0.0), dict(mode="stereo", bidirectional=True),
])
def test_params_validation_python_and_c(kwargs):
    p = DisParams(**kwargs)
    with pytest.raises(ParameterError):
        p.validate()
    rc = _lib.lib().dis_params_validate(ctypes.byref(to_c(p)))
    assert rc == _lib.DIS_ERR_PARAMETER
    with pytest.raises(ParameterError):
        _lib.check(rc)


def test_var_params_validation():
    for vp in (VarParams(sor_omega=2.0), VarParams(penalizer_eps=0.0),
               VarParams(inner_sor_iters=0), VarParams(smoothness_weight=-1.0)):
        with pytest.raises(ParameterError):
            vp.validate()
        rc = _lib.lib().dis_params_validate(ctypes.byref(to_c(DisParams(variational=vp))))
        assert rc == _lib.DIS_ERR_PARAMETER


def _flow_rc(B, H, W, p):
    L = _lib.lib()
    return L.dis_flow_batch(None, None, 0, B, H, W, ctypes.byref(to_c(p)), None, None, 0, None)


def test_dimension_errors_are_value_errors_without_gpu():
    p = DisParams()  # coarsest 5, ps 8
    for (H, W) in [(1, 100), (100, 1), (100, 200), (255, 600)]:
        rc = _flow_rc(1, H, W, p)
        assert rc == _lib.DIS_ERR_VALUE
        with pytest.raises(ValueError):
            _lib.check(rc)
    assert "cannot hold" in _lib.last_error() or "downsampled" in _lib.last_error()


def test_workspace_too_small_is_reported():
    p = synth.dis_params(synth.CONFIGS["c0"])
    rc = _flow_rc(1, 436, 1024, p)
    assert rc == _lib.DIS_ERR_WORKSPACE


def test_workspace_sizes_scale_with_batch():
    L = _lib.lib()
    p = to_c(synth.dis_params(synth.CONFIGS["c1"]))
    one = L.dis_workspace_bytes(1, 436, 1024, ctypes.byref(p))
    many = L.dis_workspace_bytes(64, 436, 1024, ctypes.byref(p))
    assert one > 0 and 60 * one < many < 66 * one
    host = L.dis_host_workspace_bytes(64, 436, 1024, 0, ctypes.byref(p))
    assert host >= many + 64 * 436 * 1024 * (4 + 4 + 16)


def test_grid_axis_abi_matches_reference():
    g = golden("samplers.npz")
    L = _lib.lib()
    off = 0
    for dim, ps, ov, cnt in zip(g["grid_dims"], g["grid_ps"], g["grid_ov"], g["grid_counts"]):
        n = L.dis_grid_axis(int(dim), int(ps), float(ov), None, 0)
        buf = (ctypes.c_int32 * n)()
        L.dis_grid_axis(int(dim), int(ps), float(ov), buf, n)
        assert np.array_equal(np.frombuffer(buf, dtype=np.int32), g["grid_origins"][off:off + cnt])
        off += cnt
    assert L.dis_grid_axis(7, 8, 0.0, None, 0) == _lib.DIS_ERR_VALUE


def test_no_cuda_means_loud_failure():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1603_03590_b200 import dis_flow

    with pytest.raises(RuntimeError, match="no CPU fallback"):
        dis_flow(np.zeros((64, 64)), np.zeros((64, 64)))


def test_grid_covers_every_pixel_for_random_layouts():
    # test_densification.py:58-66 intent: every pixel of the level is covered
    # by at least one patch window, for 200 random (dim, ps, overlap) layouts
    from paper_1603_03590_b200 import stages

    rng = np.random.default_rng(58)
    for _ in range(200):
        ps = int(rng.integers(2, 17))
        dim = int(rng.integers(ps, 300))
        ov = float(rng.uniform(0.0, 0.95))
        xo = stages.grid_axis(dim, ps, ov)
        covered = np.zeros(dim, dtype=bool)
        for o in xo:
            covered[o:o + ps] = True
        assert covered.all(), (dim, ps, ov)
        assert xo[0] == 0 and xo[-1] == dim - ps and np.all(np.diff(xo) > 0)


def test_grid_dense_limit_is_one_patch_per_pixel():
    # test_densification.py:45-48: the densest overlap gives spacing 1
    from paper_1603_03590_b200 import stages

    xo = stages.grid_axis(40, 8, 7.0 / 8.0)
    assert np.array_equal(xo, np.arange(33))
