import sys, os, torch
sys.path.insert(0, '.')
import synth
from tests.test_gpu_parity import dyadic_net, make, gpu_scores
import oracle, numpy as np
L, H, cg = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
W, jobs, grid, _ = dyadic_net(L, H, seed=L * 1000 + H)
s = gpu_scores(make(L, H, W, cg), jobs, grid)
print(L, H, cg, "mismatch", int(np.sum(s[0] != oracle.score_matrix(W, jobs, grid)[0])), flush=True)
