import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2309_00628_b200 as pk
n = 16384
rng = np.random.default_rng(1)
a, b = rng.standard_normal((n, n)), rng.standard_normal((n, n))
c = np.empty((n, n))
pol = pk.BasePolicy.naive_cutoff(4096)
for i in range(2):
    print("---- call ----", file=sys.stderr, flush=True)
    pk.winograd_block_mul(pk.Matrix(a), pk.Matrix(b), pk.Matrix(c), pol)
