import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import __graft_entry__; __graft_entry__.build()
from datagen import configs as dc
import test_dinterleave_gpu as T
for name, cfg, opt, dy, nm in [("adam-sum-1", dc.toy(), 1, False, 1), ("adam-sum-3", dc.toy(), 1, False, 3),
                          ("adam-mean-1", dc.toy(pool=dc.POOL_MEAN), 1, False, 1), ("adagrad-mean-3", dc.toy(pool=dc.POOL_MEAN), 0, False, 3),
                          ("adam-sum-dy-1", dc.toy(), 1, True, 1)]:
    try:
        T.run_micro(cfg, nm, steps=3, opt=opt, dyadic=dy, lr=0.01)
        print(name, "OK")
    except AssertionError as e:
        print(name, "FAIL", str(e)[:200])
