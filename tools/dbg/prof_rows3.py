import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1608_00099_b200 as T
dev = torch.device("cuda:0")
for dt, sh in ((torch.float32, (4729, 4729, 3)), (torch.float32, (3096, 3096, 7)), (torch.float64, (3344, 3344, 3))):
    p = torch.rand(sh, dtype=dt, device=dev); m = torch.empty(3, dtype=torch.float64, device=dev)
    for _ in range(2): T.expected_value(p, out=m)
torch.cuda.synchronize()
