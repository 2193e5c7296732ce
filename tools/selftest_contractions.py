"""tcgen05 contractions (3xTF32, four TMEM accumulators) against the fp32 SIMT tiles on
random problems (rows, relations, din, dout), through hg_selftest_contractions: relative
error of the projection, the mean gradient and the weight gradient per case.

    python tools/selftest_contractions.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_09697_b200 import _native as N  # noqa: E402

cases = [(1000, 1, 32, 64), (1000, 1, 128, 64), (1000, 4, 128, 64), (1000, 8, 128, 64), (1000, 1, 768, 64),
         (1000, 2, 768, 64), (1000, 3, 64, 349)]
arr = np.asarray(cases, np.int32).ravel()
err = N.take(N.lib().hg_selftest_contractions(N.ptr(arr), len(cases), 0))["err"]
for c, e in zip(cases, err):
    print(c, "K=%d" % (c[1] * c[2]), ["%.2e" % x for x in e])
