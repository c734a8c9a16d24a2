import sys, numpy as np
sys.path.insert(0, '.')
import paper_2511_11664_b200 as sz
t = sz.gen_synthetic("relu-laplace", [8, 8, 8], 0.5, 1)
c = sz.compress(t, 4)
print("ok", c.n_rows)
