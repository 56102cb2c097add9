"""Keyswitch batch split over several CUDA streams (C2, batch 8): does co-scheduling the
integer-bound BConv kernels with the memory-bound row kernels of another chunk pay off?"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_11269_b200 as B  # noqa: E402
from paper_2512_11269_b200 import fused  # noqa: E402
from paper_2512_11269_b200.context import get_context  # noqa: E402

p = B.gen_params(65536, 35, d=4, seed=0, scale=2 ** 26)
sk, pk, rlk = B.keygen(p, seed=11)
ctx = get_context(p)
L = p.max_level
l1 = L + 1
q = torch.tensor(p.rns_basis, dtype=torch.int64, device="cuda")[:, None]
Bsz = 8
xs = (torch.randint(0, 2 ** 62, (Bsz, l1, p.N), device="cuda", dtype=torch.int64) % q).to(torch.int32)
out = torch.empty((Bsz, 2, l1, p.N), dtype=torch.int32, device="cuda")
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
for nstreams, chunk in ((1, 8), (2, 4), (4, 2), (2, 2), (8, 1), (4, 1)):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    wss = [ctx.ks_workspace(L, chunk) for _ in range(nstreams)]
    cur = torch.cuda.current_stream()

    def step():
        ev = torch.cuda.Event()
        ev.record(cur)
        for i, c0 in enumerate(range(0, Bsz, chunk)):
            s = streams[i % nstreams]
            s.wait_event(ev)
            with torch.cuda.stream(s):
                fused.keyswitch_batch(p, L, xs[c0:c0 + chunk], rlk, out=out[c0:c0 + chunk], ws=wss[i % nstreams])
        for s in streams:
            e = torch.cuda.Event()
            e.record(s)
            cur.wait_event(e)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    tot = 0.0
    for it in range(10):
        flush.fill_(it)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cur)
        step()
        b.record(cur)
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    print(f"streams={nstreams} chunk={chunk}: {tot / 10 / Bsz * 1e3:.1f} us/keyswitch", flush=True)
