import sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2408_09697_b200 import _native as N
cases = [(1000,1,32,64),(1000,1,128,64),(1000,4,128,64),(1000,8,128,64),(1000,1,768,64),(1000,2,768,64),(1000,3,64,349)]
arr = np.asarray(cases, np.int32).ravel()
err = N.take(N.lib().hg_selftest_contractions(N.ptr(arr), len(cases), 0))["err"]
for c, e in zip(cases, err): print(c, "K=%d" % (c[1]*c[2]), ["%.2e" % x for x in e])
