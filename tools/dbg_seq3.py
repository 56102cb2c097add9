import os, sys, gc, hashlib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from fractions import Fraction
import bench
import paper_2512_11269_b200 as B
from paper_2512_11269_b200 import workloads as WL, bootstrap as BT
if sys.argv[1] == "prior":
    bench.resnet_block_latency()
    gc.collect(); torch.cuda.empty_cache()
T, d = 128, 64
rng = np.random.default_rng(5)
Ws = [rng.uniform(-1, 1, (d, d)) / d for _ in range(6)]
kw = dict(T=T, d=d, score_bound=1.0, gelu_bound=2.0)
rots = WL.TransformerBlock(bench._Planner(bench.C5), *Ws, **kw).required_rotations()
p, sk, pk, be, _ = bench._workload_env(bench.C5, rots)
blk = WL.TransformerBlock(be, *Ws, **kw)
X = np.random.default_rng(8).uniform(-1, 1, (T, d)) * 0.5
S = Fraction(p.rns_basis[p.max_level]) * p.rns_basis[p.max_level - 1]
ct = B.encrypt(B.encode(blk.pack(X), p, level=p.max_level, scale=S), pk, p, np.random.default_rng(6))
log = []
def digest(x):
    if isinstance(x, list):
        return "|".join(str(digest(y)) for y in x)
    if isinstance(x, BT.CtBatch):
        t = x.data
    elif hasattr(x, "b") and hasattr(x.b, "limbs"):
        t = torch.stack([x.b.limbs, x.a.limbs])
    else:
        return None
    v = t.reshape(-1).to(torch.int64)
    return str(int(v.sum().item())) + ":" + str(int((v[::13] * 7919).sum().item()))
for name in ["mul_rescale2", "mul_rescale2_many", "rescale2", "rot_batch", "rotate_same", "mul_plain_batch", "batch_sum",
             "bsgs_fused_ext", "add", "sub", "add_const", "mul_const", "lincomb", "rotate_hoisted", "rescale"]:
    f = getattr(BT.GpuBackend, name)
    def wrap(self, *a, _f=f, _n=name, **k):
        r = _f(self, *a, **k)
        log.append((_n, digest(r), []))
        return r
    setattr(BT.GpuBackend, name, wrap)
runs = []
for i in range(3):
    log.clear(); blk.forward(ct); torch.cuda.synchronize(); runs.append(list(log))
for i in (1, 2):
    for j, (a, b) in enumerate(zip(runs[0], runs[i])):
        if a[1] != b[1]:
            prev = runs[0][j - 1][0] if j else None
            print(f"run {i}: first difference at call {j} of {len(runs[0])}: {a[0]} (previous call {prev})")
            break
    else:
        print(f"run {i}: identical ({len(runs[0])} calls)")
