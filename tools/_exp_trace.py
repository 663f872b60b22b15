"""Per-step phase timing of the SOR kernel (a library built with
-DDIS_SOR_TRACE=<thread>): python tools/_exp_trace.py B H W"""
import ctypes, subprocess, sys, os
import numpy as np
sys.path.insert(0, '.')
B, H, W = (int(a) for a in sys.argv[1:4])
subprocess.run([sys.executable, 'tools/sor_bench.py', str(B), str(H), str(W), '1'], check=True,
               stdout=subprocess.DEVNULL)
# the trace lives in the process that ran the kernel: run in-process instead
from tools import sor_bench  # noqa
sys.argv = ['x', str(B), str(H), str(W), '1']
sor_bench.main()
from paper_1603_03590_b200 import _lib
L = _lib.lib()
buf = (ctypes.c_longlong * (6 * 1024))()
L.dis_debug_sor_trace(buf)
a = np.frombuffer(buf, dtype=np.int64).reshape(6, 1024).astype(np.float64)
lo, hi = 100, min(500, W + H)
d = np.diff(a[:, lo:hi + 1], axis=1)  # step-to-step per checkpoint
ph = [a[i + 1, lo:hi] - a[i, lo:hi] for i in range(5)]
print('step cycles %.0f' % np.median(a[0, lo + 1:hi + 1] - a[0, lo:hi]),
      'phases (halo+issue, compute, stores, filler wait, barrier):',
      ' '.join('%.0f' % np.median(p) for p in ph),
      'barrier->next start %.0f' % np.median(a[0, lo + 1:hi + 1] - a[5, lo:hi]))
