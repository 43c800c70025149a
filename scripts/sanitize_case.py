"""Small cases through every kernel family (for compute-sanitizer)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1801_03065_b200 as kk
from paper_1801_03065_b200 import generators as G
a = G.laplace3d(6)
kk.multiply(a, a)                                   # fast symbolic + fast seq numeric
p = G.aggregation(6); kk.multiply(a, p)             # flat numeric, raw symbolic
for acc in (1, 2, 3):
    for sch in (0, 1):
        for l1 in (0, 1):
            kk.multiply(a, a, kk.SpgemmConfig(accumulator=acc, scheme=sch, l1_capacity=l1))
r = G.rmat(10, 16, 1); kk.multiply(r, r)            # heavy rows at small scale
rng = np.random.default_rng(7)
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from conftest import random_csr
x = random_csr(rng, 24, 3000, 0.08, shuffle=True); y = random_csr(rng, 3000, 20000, 0.02, shuffle=True)
kk.multiply(x, y)                                   # heavy CTA kernels
kk.multiply(a, a, kk.SpgemmConfig(sort_output=True))
print("sanitize case done")
