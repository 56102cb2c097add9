"""Standalone batched NTT throughput at N=2^16 (C2 primes): butterflies/s and integer-pipe use."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_11269_b200 as B  # noqa: E402
from paper_2512_11269_b200 import poly as P  # noqa: E402

p = B.gen_params(65536, 35, d=4, seed=0, scale=2 ** 26)
R = int(sys.argv[1]) if len(sys.argv) > 1 else 360
ids = [i % 36 for i in range(R)]
q = torch.tensor([p.rns_basis[i] for i in ids], dtype=torch.int64, device="cuda")[:, None]
x = (torch.randint(0, 2 ** 62, (R, p.N), device="cuda", dtype=torch.int64) % q).to(torch.int32)
for _ in range(3):
    P.ntt_rows(p, x, ids)
    P.ntt_rows(p, x, ids, inverse=True)
torch.cuda.synchronize()
for inv in (False, True):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        P.ntt_rows(p, x, ids, inverse=inv)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    bf = R * (p.N // 2) * 16
    print(f"{'inv' if inv else 'fwd'} rows={R} {ms*1e3:.1f} us  {bf/ms/1e9:.3f} T butterflies/s  "
          f"{2*R*p.N*4/ms/1e6:.0f} GB/s (one read+write)")
