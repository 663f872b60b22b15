"""Patch search at the level borders on the lane kernel (levels with more
than ~76k patches), against the oracle — tolerance 0 (np.array_equal).

The lane kernel reads the query level from a copy with a 16-pixel
replicated border (csrc/patch_search.cu, kQPad): windows clamped by _bilin
(inverse_search.py:34-58) within 16 px of the level stay on the lane kernel,
windows further out park for the lane-group kernel.  A coarse flow that
grows towards every border (up to +-40 px at level scale, pointing outward)
drives windows through both regimes and across the pad's edge; every patch
output and the densified field must equal the reference restatement's.
Reference: pipeline.py:54-82 (_ScaleState.search), inverse_search.py:113-189,
densification.py:82-107, 110-191.
"""

import numpy as np
import pytest

from paper_1603_03590_b200.params import DisParams
from tools import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    return torch


def _np(t):
    return t.detach().cpu().numpy()


def _outward_coarse_flow(h, w, mag):
    """Half-resolution flow (init_patches scales it by 2) pointing out of the
    level near its borders, +-mag px at level scale at the edges."""
    hc, wc = h // 2, w // 2
    xs = np.linspace(-1.0, 1.0, wc)
    ys = np.linspace(-1.0, 1.0, hc)
    u = np.sign(xs) * np.abs(xs) ** 3 * (mag / 2.0)
    v = np.sign(ys) * np.abs(ys) ** 3 * (mag / 2.0)
    f = np.empty((hc, wc, 2))
    f[..., 0] = u[None, :]
    f[..., 1] = v[:, None]
    return f


@pytest.mark.parametrize("ps,ov,norm,code", [(8, 0.5, "l2", 0), (8, 0.5, "huber", 2),
                                             (12, 0.75, "l2", 0)])
def test_border_windows_on_the_lane_kernel_vs_oracle(torch, orc, ps, ov, norm, code):
    from paper_1603_03590_b200 import stages

    h, w = 1024, 1280
    f1, f2, _ = synth.make_pair(21 + ps, h, w, 6.0, False, 0.0)
    coarse = _outward_coarse_flow(h, w, 40.0)
    params = DisParams(patch_size=ps, overlap=ov, iterations=24, finest_scale=0,
                       coarsest_scale=1, residual_norm=norm, huber_b=2.0)
    l1 = stages.build_pyramid(f1[None], 0)[0]
    l2 = stages.build_pyramid(f2[None], 0)[0]
    c = torch.tensor(coarse, device="cuda")
    cu, cv = c[..., 0][None].contiguous(), c[..., 1][None].contiguous()
    r = stages.patch_search(l1, l2["img"], params, cu, cv)
    n = len(r["x_origins"]) * len(r["y_origins"])
    assert n * (8 if ps == 8 else 16) > 148 * 2048 * (2 if ps == 8 else 4)  # lane kernel
    ref = orc.build_pyramid(f1, 0)[0]
    qry = orc.build_pyramid(f2, 0)[0]
    xo, _ = orc.axis_origins(w, ps, ov)
    yo, _ = orc.axis_origins(h, ps, ov)
    init = orc.init_patches(xo, yo, ps, coarse)
    # windows start past the level by up to ~40 px: inside and beyond the pad
    ox = np.repeat(xo[None, :], len(yo), 0).ravel() + init[:, 0]
    assert (ox < -16).any() and ((ox < 0) & (ox > -16)).any()
    assert (ox > w - ps + 16).any()
    want = orc.patch_search(ref[0], ref[1], ref[2], qry[0], xo, yo, ps, init, 24,
                            norm_code=code, huber_b=2.0)
    assert np.array_equal(_np(r["valid"])[0].astype(bool), want["valid"])
    disp = np.stack([_np(r["u"])[0], _np(r["v"])[0]], -1)
    assert np.array_equal(disp, want["disp"])
    assert np.array_equal(_np(r["off"])[0], want["offset"])
    assert np.array_equal(_np(r["mar"])[0], want["mar"])
    fu, fv = stages.densify(l1["img"], l2["img"], params, r["u"], r["v"], r["off"])
    dense = orc.densify(ref[0], qry[0], xo, yo, ps, want["disp"], want["offset"])
    assert np.array_equal(np.stack([_np(fu)[0], _np(fv)[0]], -1), dense)
