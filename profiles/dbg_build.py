import sys, os
sys.path.insert(0, '.')
import numpy as np
import paper_2207_01834_b200 as gk
from oracle import oracle as O
for n, d in [(3000, 2), (5000, 2), (20000, 2), (100000, 3)]:
    P = np.random.default_rng(n).random((n, d))
    g = gk.BDLTree(d, X=n)
    try:
        g.insert(P)
    except Exception as e:
        print("FAIL", n, d, e); sys.exit(1)
    o = O.BDLTree(d, X=n); o.insert(P)
    gn, gi, gp = g.tree_export(0); on, oi, op = o.tree_export(0)
    print(n, d, "perm equal", np.array_equal(gi, oi), "nodes", len(gn), len(on), "bytes equal", gn.tobytes() == on.tobytes())
    if len(gn) == len(on):
        for f in gn.dtype.names:
            bad = np.nonzero(~np.all((gn[f] == on[f]).reshape(len(gn), -1), axis=1))[0]
            if len(bad):
                i = bad[0]
                print("  field", f, "differs at", len(bad), "nodes; first slot", i, gn[i], on[i])
