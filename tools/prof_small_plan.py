"""One small product for ncu launch lists (n, cutoff from argv). Dev tool."""
import sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_2309_00628_b200 as pk
n, cut = int(sys.argv[1]), int(sys.argv[2])
a = torch.randint(-8, 9, (n, n), device="cuda").double(); b = torch.randint(-8, 9, (n, n), device="cuda").double()
c = torch.empty_like(a)
pk.winograd_block_mul(pk.Matrix(a), pk.Matrix(b), pk.Matrix(c), pk.BasePolicy.naive_cutoff(cut))
torch.cuda.synchronize()
print("done")
