"""Dump the tcgen05 attention's outputs for a fixed set of long-cache cases
(both tcgen05 kernels) so two builds can be compared bitwise:
  MS_LIB=<lib> python tools/attn_dump.py out.pt ; python tools/attn_dump.py --cmp a.pt b.pt"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
if sys.argv[1] == "--cmp":
    a, b = torch.load(sys.argv[2]), torch.load(sys.argv[3])
    bad = [k for k in a if not torch.equal(a[k], b[k])]
    print({"cases": len(a), "bitwise_equal": len(a) - len(bad), "differ": bad})
    sys.exit(1 if bad else 0)
from paper_2402_15678_b200 import kernels as K
K.TC_ATTENTION = True
res = {}
for (H, Hkv, Q, ctx) in [(64, 8, 1, 1000), (64, 8, 5, 4096), (64, 8, 7, 700), (64, 8, 9, 1500), (64, 8, 13, 4096),
                         (16, 2, 7, 640), (40, 40, 5, 2000),  # online kernel (T > 384)
                         (64, 8, 1, 190), (64, 8, 7, 190), (64, 8, 13, 300), (64, 8, 5, 100), (16, 2, 7, 200),
                         (40, 40, 5, 300), (64, 8, 16, 340)]:  # one-pass short kernel (T <= 384)
    D, B = 128, 4
    g = torch.Generator(device="cuda").manual_seed(H * 100 + Q * 10 + ctx)
    T = ctx + 32
    kc = torch.randn(B, Hkv, T, D, device="cuda", generator=g).to(torch.bfloat16)
    vc = torch.randn(B, Hkv, T, D, device="cuda", generator=g).to(torch.bfloat16)
    qkv = (3 * torch.randn(B * Q, (H + 2 * Hkv) * D, device="cuda", generator=g)).to(torch.bfloat16)
    start = torch.tensor([ctx, ctx // 2, 3, ctx - 100], dtype=torch.int32, device="cuda")
    slot = torch.arange(B, dtype=torch.int32, device="cuda")
    rope = K.rope_table(T + 8, D, 10000.0)
    out = K.attention(qkv, B, Q, H, D, slot, start, kc, vc, D ** -0.5, n_kv_heads=Hkv, rope=rope)
    torch.cuda.synchronize()
    res[f"{H}/{Hkv}/Q{Q}/ctx{ctx}"] = out.cpu()
    res[f"{H}/{Hkv}/Q{Q}/ctx{ctx}/k"] = kc.cpu()
torch.save(res, sys.argv[1])
print("dumped", len(res))
