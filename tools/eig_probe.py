"""sym_eig on a random symmetric d x d matrix (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2501_15129_b200 as evb
d = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
A = np.random.default_rng(0).standard_normal((d, d)); A = A + A.T
ev, V, sw = evb.sym_eig(A)
print("d", d, "sweeps", sw)
