"""Micro-benchmark of the refinement stage alone (dis_refine, outer=1) on
synthetic levels:  python tools/sor_bench.py B:H:W [B:H:W ...] [--reps N]
Prints tensor+assemble and SOR ms and the SOR's us per anti-diagonal step."""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1603_03590_b200 import _lib, stages
from paper_1603_03590_b200.params import DisParams, VarParams, to_c


def run(B, H, W, reps):
    rng = np.random.default_rng(0)
    f = rng.uniform(0, 255, size=(2, B, H, W)).astype(np.float32)
    l1 = stages.build_pyramid(f[0], 0)[0]
    l2 = stages.build_pyramid(f[1], 0)[0]
    u = torch.tensor(rng.normal(0, 1, size=(B, H, W)), device="cuda")
    v = torch.tensor(rng.normal(0, 1, size=(B, H, W)), device="cuda")
    L = _lib.lib()
    p = to_c(DisParams(variational=VarParams()))
    nbytes = L.dis_refine_workspace_bytes(B, W, H)
    ws = torch.empty(int(nbytes), dtype=torch.uint8, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    args = lambda uu, vv: (l1["img"].data_ptr(), l1["gx"].data_ptr(), l1["gy"].data_ptr(),
                           l1["dd"].data_ptr(), l2["img"].data_ptr(), l2["gx"].data_ptr(),
                           l2["gy"].data_ptr(), l2["dd"].data_ptr(), B, W, H, ctypes.byref(p), 1,
                           uu.data_ptr(), vv.data_ptr(), ws.data_ptr(), int(nbytes),
                           st.data_ptr(), None)
    uu, vv = u.clone(), v.clone()
    _lib.check(L.dis_refine(*args(uu, vv)))
    ref = (uu.clone(), vv.clone())
    L.dis_profile_reset()
    L.dis_profile_enable(1)
    for _ in range(reps):
        uu.copy_(u)
        vv.copy_(v)
        _lib.check(L.dis_refine(*args(uu, vv)))
    torch.cuda.synchronize()
    L.dis_profile_enable(0)
    ms = (ctypes.c_double * 6)()
    n = (ctypes.c_int64 * 6)()
    L.dis_profile_read(ms, n, 6)
    same = torch.equal(uu, ref[0]) and torch.equal(vv, ref[1])
    steps = W + H - 1 + 8
    sor_ms = ms[4] / reps
    print(f"{os.path.basename(_lib.LIB_PATH)} B={B} H={H} W={W} tensor {ms[3]/reps:.3f} ms "
          f"sor {sor_ms:.3f} ms ({sor_ms * 1e3 / steps:.3f} us/step) deterministic={same}",
          flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("shapes", nargs="+")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    for s in a.shapes:
        B, H, W = (int(x) for x in s.split(":"))
        run(B, H, W, a.reps)


if __name__ == "__main__":
    main()
