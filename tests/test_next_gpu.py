"""§8(f) "next" rows on the GPU through the C ABI, against the reference's
goldens and the oracle — bit-exact (tolerance 0: np.array_equal)."""

import numpy as np
import pytest

from tests.conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    return torch


# ---- compose_flows (pipeline.py:186-199) ----------------------------------

def test_compose_flows_goldens(torch):
    from paper_1603_03590_b200 import compose_flows

    g = golden("next_compose.npz")
    for k in range(3):
        got = compose_flows(g[f"ab{k}"], g[f"bc{k}"])
        assert isinstance(got, np.ndarray) and got.dtype == np.float64
        assert np.array_equal(got, g[f"out{k}"]), k


def test_compose_flows_batched_torch_vs_oracle(torch, orc):
    from paper_1603_03590_b200 import compose_flows

    rng = np.random.default_rng(5)
    ab = rng.normal(0, 6, (3, 64, 96, 2))
    bc = rng.normal(0, 6, (3, 64, 96, 2))
    got = compose_flows(torch.from_numpy(ab).cuda(), torch.from_numpy(bc).cuda())
    assert got.is_cuda
    got = got.cpu().numpy()
    for i in range(3):
        assert np.array_equal(got[i], orc.compose_flows(ab[i], bc[i])), i


def test_compose_flows_errors(torch):
    from paper_1603_03590_b200 import compose_flows

    with pytest.raises(ValueError):
        compose_flows(np.zeros((4, 5, 2)), np.zeros((4, 6, 2)))
