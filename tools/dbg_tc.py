import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2512_11269_b200 as B
from paper_2512_11269_b200 import bootstrap as BT, fused
L = int(sys.argv[1]); Bn = int(sys.argv[2])
p = B.gen_params(65536, L, d=4, seed=0, scale=2 ** 26)
sk, pk, rlk = B.keygen(p, seed=3)
be = BT.GpuBackend(p, rlk, None, {})
# dirty the allocator with garbage
g = torch.randint(-2**31, 2**31 - 1, (40 * 2**30 // 4,), dtype=torch.int32, device="cuda"); del g
l1 = p.max_level + 1
q = torch.tensor(p.rns_basis, dtype=torch.int64, device="cuda")[:, None]
x = (torch.randint(0, 2 ** 62, (Bn, 2, l1, p.N), device="cuda", dtype=torch.int64) % q).to(torch.int32)
y = (torch.randint(0, 2 ** 62, (Bn, 2, l1, p.N), device="cuda", dtype=torch.int64) % q).to(torch.int32)
X, Y = BT.CtBatch(x, 1, p.max_level), BT.CtBatch(y, 1, p.max_level)
for name, fn in [("rescale2", lambda: be.rescale2(X).data), ("rescale2_view", lambda: be.rescale2(be.drop_to_level(X, p.max_level - 3)).data),
                 ("mul_rescale2", lambda: be.mul_rescale2(X, Y).data), ("hom_mul", lambda: be.hom_mul(X, Y).data),
                 ("keyswitch", lambda: fused.keyswitch_batch(p, p.max_level, x[:, 1].contiguous(), rlk))]:
    outs = []
    for i in range(3):
        g = torch.randint(-2**31, 2**31 - 1, (20 * 2**30 // 4,), dtype=torch.int32, device="cuda"); del g
        outs.append(fn().clone())
    print(name, "TC" if os.environ.get("LF_BC_TC", "1") != "0" else "IMAD",
          torch.equal(outs[0], outs[1]), torch.equal(outs[1], outs[2]))
