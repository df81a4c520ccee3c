import sys, torch
sys.path.insert(0, '/root/repo')
import paper_2605_10886_b200 as lk
k = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
g = torch.Generator(device='cuda').manual_seed(0)
a = torch.randn(k, k, device='cuda', generator=g); a = a @ a.T / k + torch.eye(k, device='cuda')
for _ in range(2):
    l, e = lk.cholesky_jittered(a, 1e-6)
torch.cuda.synchronize()
