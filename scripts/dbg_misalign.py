import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2201_12523_b200 as b
GI = np.array([[0, 0, 0, 1, 1, 2, 2, 3, 3, 3, 3, 3], [0, 0, 2, 0, 0, 0, 3, 1, 1, 2, 2, 3], [0, 1, 2, 1, 2, 1, 3, 0, 1, 2, 3, 3]], np.uint64)
t = b.build_blco(b.SparseTensorCoo([4, 4, 4], GI, np.arange(1, 13, dtype=np.float64)), 5, 6)
f = b.FactorMatrices.ones([4, 4, 4], 2)
print(b.mttkrp(t, f, 0, strategy=b.Strategy.Register))
print(b.mttkrp(t, f, 2, strategy=b.Strategy.Hierarchical))
