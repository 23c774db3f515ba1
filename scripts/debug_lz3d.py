import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import fzoracle as O
from paper_2509_20563_b200 import predict as pr
from paper_2509_20563_b200.core import Field, ResolvedBound
from paper_2509_20563_b200.data import smooth_trig_host

for dims in [(9, 33, 40), (9, 33, 257), (16, 64, 20), (9, 33, 3), (2, 33, 5)]:
    x = smooth_trig_host(dims, 2)
    lo, hi = float(x.min()), float(x.max()); e = 1e-3 * (hi - lo)
    c, i, v, r = O.lorenzo_quantize(x, dims, e)
    res = []
    for rep in range(3):
        q = pr.lorenzo_quantize(Field(dims, x), ResolvedBound(e, lo, hi))
        bad = np.nonzero(q.codes != c)[0]
        res.append(bad.size)
        if rep == 0 and bad.size:
            t = bad[:8]
            ii, jj, kk = np.unravel_index(t, dims)
            print(dims, "first bad (i,j,k):", list(zip(ii.tolist(), jj.tolist(), kk.tolist())),
                  "gpu", q.codes[t].tolist(), "ref", c[t].tolist())
    print(dims, "mismatches per run:", res)
