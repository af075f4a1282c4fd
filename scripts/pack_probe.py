import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_1410_6609_b200 import mg
from paper_1410_6609_b200 import workloads as W
w = W.cfg3(512, seed=0, with_rhs=False)
s = mg.Multigrid(w.shape, w.h, w.bc_type, w.bc_value, min_coarse=8)
fd = torch.rand(w.shape, dtype=torch.float64, device="cuda")
od = torch.empty_like(fd)
for _ in range(3):
    s.set_rhs(fd)
    s.zero_solution()
    s.get_solution(od)
torch.cuda.synchronize()
