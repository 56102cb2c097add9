"""Per-kernel CUDA-event split of the C2 keyswitch at several batch sizes
(fused.keyswitch_batch_profiled: modup_in, ModUp BConv, ks_inner, ModDown BConv, moddown_out)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_11269_b200 as B  # noqa: E402
from paper_2512_11269_b200 import fused  # noqa: E402
from paper_2512_11269_b200.context import get_context  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 35
p = B.gen_params(65536, 35, d=4, seed=0, scale=2 ** 26)
sk, pk, rlk = B.keygen(p, seed=11)
ctx = get_context(p)
l1 = level + 1
q = torch.tensor(p.rns_basis[:l1], dtype=torch.int64, device="cuda")[:, None]
names = ["modup_in", "modup_bconv", "ks_inner", "moddown_bconv", "moddown_out"]
for batch in (1, 2, 4, 8, 32):
    x = (torch.randint(0, 2 ** 62, (batch, l1, p.N), device="cuda", dtype=torch.int64) % q).to(torch.int32)
    out = torch.empty((batch, 2, l1, p.N), dtype=torch.int32, device="cuda")
    ws = ctx.ks_workspace(level, batch)
    acc = [0.0] * 5
    for i in range(5):
        st = fused.keyswitch_batch_profiled(p, level, x, rlk, out, ws)
        if i:
            acc = [a + s for a, s in zip(acc, st)]
    per = [a / 4 / batch * 1e3 for a in acc]
    print(f"level {level} batch {batch:2d}: total {sum(per):6.1f} us/op  " +
          "  ".join(f"{n} {v:5.1f}" for n, v in zip(names, per)))
