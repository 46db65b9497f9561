"""Run kde_dp once on the 20 M-point C4 input (for an ncu launch list)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, aisgen
from paper_2004_13653_b200 import kde_dp
c = aisgen.generate("islands", 20_000_000, aisgen.SEED_BASE + 3)
x, y, o = (torch.from_numpy(a).cuda() for a in (c.x, c.y, np.asarray(c.traj_offsets, np.int64)))
_, nk, r = kde_dp(x, y, o, 1.0)
torch.cuda.synchronize()
print(nk, r)
