import os, sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import numpy as np
import paper_2002_03400_b200 as B
import oracle as O
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
w = B.configs.build(3, n)
os.environ["BFLY_DEBUG_CORE_FIT"] = "1"
a, la = B.factorize(w.op, w.row_tree, w.col_tree, w.recon)
x = O.gaussian_matrix(n, 2, 5)
y = a.apply(x)
print("nan in apply:", np.isnan(y).any(), "ranks", a.rank_profile().max(axis=1))
os.environ["BFLY_NO_BIG_CORE_FIT"] = "1"
b, lb = B.factorize(w.op, w.row_tree, w.col_tree, w.recon)
yb = b.apply(x)
print("jacobi nan:", np.isnan(yb).any(), "same ranks", (a.rank_profile() == b.rank_profile()).all())
