import os, sys, gc
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from fractions import Fraction
import bench
import paper_2512_11269_b200 as B
from paper_2512_11269_b200 import workloads as WL, bootstrap as BT
mode = sys.argv[1]
if mode == "nowave":
    BT.CkksCircuit._fused_consts = lambda self: False
    orig = BT.GpuBackend.mul_rescale2_many
    del BT.GpuBackend.mul_rescale2_many
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
o1 = blk.forward(ct); o2 = blk.forward(ct); o3 = blk.forward(ct); torch.cuda.synchronize()
print(mode, "eager 1==2:", np.array_equal(o1.b.numpy(), o2.b.numpy()), "2==3:", np.array_equal(o2.b.numpy(), o3.b.numpy()))
err = lambda o: float(np.abs(B.decrypt(o, sk, p)[: T * d].real.reshape(T, d) - blk.reference(X)).max())
print(mode, "errors", err(o1), err(o2), err(o3))
