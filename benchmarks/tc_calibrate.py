#!/usr/bin/env python
"""Calibration of the tensor-core screen's exponent error (pt_debug_tc_arg_error): worst case over random
segment midpoints, in units of 2^-24 * gamma*log2e*(|p|+max|s|)^2, for the bench manifolds."""
import ctypes as C
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from bench import build_workload
from paper_2406_04795_b200 import _cabi

for name in sys.argv[1:] or ["dof6", "dof4"]:
    wl = build_workload(name)
    a = wl.arrays
    rng = np.random.default_rng(1)
    m = 200_000
    lo, hi = np.asarray(a.box[0]), np.asarray(a.box[1])
    pa = rng.uniform(lo, hi, size=(m, a.n)); pb = pa + rng.normal(scale=0.3, size=(m, a.n))
    out = np.zeros(m)
    ctx = _cabi.context()
    _cabi.check(_cabi.lib.pt_debug_tc_arg_error(ctx.handle, wl.manifold.device_field(), pa.ctypes.data, pb.ctypes.data, m, out.ctypes.data))
    print(name, "n", a.n, "S", a.support.shape[0], "max", out.max(), "p99.9", np.quantile(out, 0.999), "median", np.median(out))
