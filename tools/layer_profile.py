"""Kernel split of one C4 / C5 layer forward on cuda:0 (torch profiler, eager):
python tools/layer_profile.py [resnet|transformer]"""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import numpy as np  # noqa: E402
import paper_2512_11269_b200 as B  # noqa: E402
from paper_2512_11269_b200 import workloads as WL  # noqa: E402
from fractions import Fraction  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "transformer"
if which == "resnet":
    C = bench.C4_SHAPE[0]
    rng = np.random.default_rng(5)
    w1, w2 = rng.uniform(-1, 1, (C, C, 3, 3)) / (9 * C), rng.uniform(-1, 1, (C, C, 3, 3)) / (9 * C)
    rots = WL.ResNetBlock(bench._Planner(bench.C3), w1, w2, bench.C4_SHAPE).required_rotations()
    p, sk, pk, be, _ = bench._workload_env(bench.C3, rots)
    blk = WL.ResNetBlock(be, w1, w2, bench.C4_SHAPE)
    vec = blk.pack(np.random.default_rng(7).uniform(-1, 1, bench.C4_SHAPE) * 0.5)
else:
    T, d = bench.C5_SHAPE
    rng = np.random.default_rng(5)
    Ws = [rng.uniform(-1, 1, (d, d)) / d for _ in range(6)]
    kw = dict(T=T, d=d, score_bound=1.0, gelu_bound=2.0)
    rots = WL.TransformerBlock(bench._Planner(bench.C5), *Ws, **kw).required_rotations()
    p, sk, pk, be, _ = bench._workload_env(bench.C5, rots)
    blk = WL.TransformerBlock(be, *Ws, **kw)
    vec = blk.pack(np.random.default_rng(8).uniform(-1, 1, (T, d)) * 0.5)
S = Fraction(p.rns_basis[p.max_level]) * p.rns_basis[p.max_level - 1]
ct = B.encrypt(B.encode(vec, p, level=p.max_level, scale=S), pk, p, np.random.default_rng(6))
blk.forward(ct)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    blk.forward(ct)
    torch.cuda.synchronize()
ka = prof.key_averages()
tot = sum(k.device_time_total for k in ka)
print(f"{which}: kernel time {tot / 1e3:.1f} ms over {sum(k.count for k in ka)} launches")
print(ka.table(sort_by="device_time_total", row_limit=16))
