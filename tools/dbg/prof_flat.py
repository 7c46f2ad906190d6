import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1608_00099_b200 as T
dev = torch.device("cuda:0")
for dt, sh in ((torch.float32, (1426, 1426, 33)), (torch.float64, (1008, 1008, 33))):
    p = torch.rand(sh, dtype=dt, device=dev); m = torch.empty(3, dtype=torch.float64, device=dev)
    for _ in range(2): T.expected_value(p, out=m)
torch.cuda.synchronize()
