import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch
from paper_2402_15678_b200 import kernels as K, _native
M, N, Kd, sp = [int(v) for v in sys.argv[1:5]]
x = torch.randn(M, Kd, device="cuda").to(torch.bfloat16)
w = torch.randn(N, Kd, device="cuda").to(torch.bfloat16) * 0.02
out = K.linear(x, w, splits=sp)
torch.cuda.synchronize()
ref = x.float() @ w.float().T
print(M, N, Kd, sp, "maxerr", (out.float() - ref).abs().max().item())
