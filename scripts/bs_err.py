"""Max |error| / (s + K) of lift.blackscholes against the fp64 oracle over the test parameter
sets (tests/test_gpu_blackscholes.py) and the 4M-price bench set."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import lift_inputs as gen
import oracle
import paper_1502_02389_b200 as lift

cases = [((100.0, 0.05, 0.2, 1.0), 10.0, 200.0, 4 << 20), ((40.0, 0.0, 0.6, 0.25), 8.0, 120.0, 50_000),
         ((15.0, 0.1, 0.05, 5.0), 3.0, 45.0, 50_000), ((100.0, -0.01, 1.5, 0.01), 20.0, 300.0, 50_000)]
for (k, r, v, t), lo, hi, n in cases:
    s = gen.host(n, 3, gen.TID_X, lo=lo, hi=hi)
    c, p = lift.blackscholes(torch.from_numpy(s).to("cuda:0"), k, r, v, t)
    oc, op = oracle.blackscholes(s, k, r, v, t)
    sc = s.astype(np.float64) + k
    print((k, r, v, t), "call %.3g put %.3g" % ((np.abs(c.cpu().numpy() - oc) / sc).max(),
                                                 (np.abs(p.cpu().numpy() - op) / sc).max()))
