"""Run a few C2 full-level batched keyswitches (for ncu / compute-sanitizer captures)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_11269_b200 as B  # noqa: E402
from paper_2512_11269_b200 import fused  # noqa: E402
from paper_2512_11269_b200.context import get_context  # noqa: E402

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 8
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
op = sys.argv[3] if len(sys.argv) > 3 else "ks"
p = B.gen_params(65536, 35, d=4, seed=0, scale=2 ** 26)
sk, pk, rlk = B.keygen(p, seed=11)
ctx = get_context(p)
l1 = p.max_level + 1
q = torch.tensor(p.rns_basis, dtype=torch.int64, device="cuda")[:, None]
x = (torch.randint(0, 2 ** 62, (batch, l1, p.N), device="cuda", dtype=torch.int64) % q).to(torch.int32)
out = torch.empty((batch, 2, l1, p.N), dtype=torch.int32, device="cuda")
ws = ctx.ks_workspace(p.max_level, batch)
torch.cuda.synchronize()
for _ in range(iters):
    fused.keyswitch_batch(p, p.max_level, x, rlk, out=out, ws=ws)
torch.cuda.synchronize()
print("done")
