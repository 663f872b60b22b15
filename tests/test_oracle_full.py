"""Pin the C oracle at the BASELINE configs' full sizes: sha256 of the flow
the reference itself produced on the same synthetic pairs
(tests/golden/full_hashes.npz, oracle/gen_golden.py gen_full_hashes)."""

import hashlib

import numpy as np
import pytest

from tests.conftest import golden
from tools import synth


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def _rows():
    g = golden("full_hashes.npz")
    return [(str(c), int(p), str(a), str(b), str(f)) for c, p, a, b, f in
            zip(g["cfg"], g["pair"], g["f1_sha"], g["f2_sha"], g["flow_sha"])]


@pytest.mark.parametrize("row", _rows(), ids=lambda r: f"{r[0]}-pair{r[1]}")
def test_oracle_matches_reference_full_size(orc, row):
    cfg_name, pair, f1_sha, f2_sha, flow_sha = row
    cfg = synth.CONFIGS[cfg_name]
    f1, f2 = synth.make_batch(cfg, seed=0, count=1, first=pair)
    # the synthetic generator itself is pinned too
    assert _sha(f1[0]) == f1_sha and _sha(f2[0]) == f2_sha
    flow = orc.dis_flow(f1[0], f2[0], synth.dis_params(cfg))
    assert _sha(flow) == flow_sha
