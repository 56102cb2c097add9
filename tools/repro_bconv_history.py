"""Reproducer for the round-2 k_bconv_tc regression (profiles/r02_experiments.md): a ResNet
block at the C3 parameters, then batch-128 double rescales at the C5 parameters, compared
across repeats.  python tools/repro_bconv_history.py prior"""
import os, sys, gc
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2512_11269_b200 as B
from paper_2512_11269_b200 import bootstrap as BT
if sys.argv[1] == "prior":
    bench.resnet_block_latency()
    gc.collect(); torch.cuda.empty_cache()
p = B.gen_params(65536, 52, d=4, seed=0, scale=2 ** 26)
sk, pk, rlk = B.keygen(p, seed=11)
be = BT.GpuBackend(p, rlk, None, {})
lv = 44
q = torch.tensor(p.rns_basis[: lv + 1], dtype=torch.int64, device="cuda")[:, None]
x = (torch.randint(0, 2 ** 62, (128, 2, lv + 1, p.N), device="cuda", dtype=torch.int64) % q).to(torch.int32)
X = BT.CtBatch(x, 1, lv)
outs = [be.rescale2(X).data.clone() for _ in range(6)]
torch.cuda.synchronize()
print("rescale2 B=128 equal:", [torch.equal(outs[0], o) for o in outs[1:]])
if not all(torch.equal(outs[0], o) for o in outs[1:]):
    for i, o in enumerate(outs[1:], 1):
        d = (outs[0] != o)
        if d.any():
            idx = d.nonzero()
            print(f"run {i}: {int(d.sum())} residues differ; instances {sorted(set(idx[:, 0].tolist()))[:10]}, polys {sorted(set(idx[:, 1].tolist()))}, rows {sorted(set(idx[:, 2].tolist()))[:10]}, cols {idx[:5, 3].tolist()}")
