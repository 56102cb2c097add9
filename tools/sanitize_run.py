"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck): desk-size
keyswitch, hom_mul, rotate (hoisted, batched, extended), rescale (single, double), ModRaise,
plaintext MACs, a toy bootstrap, the fused mul+rescale and BSGS kernels, the kernel-plan
interpreter and the NTT row kernels (TMA-staged twiddles) on cuda:0."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_11269_b200 as B  # noqa: E402
from paper_2512_11269_b200 import bootstrap as BT  # noqa: E402
from paper_2512_11269_b200 import fused  # noqa: E402

p = B.gen_params(4096, 6, d=3, seed=0)
sk, pk, rlk = B.keygen(p, seed=11)
rk = {s: B.make_rotation_key(p, sk, s, np.random.default_rng(s)) for s in (1, 2, 3)}
v = np.random.default_rng(1).uniform(-1, 1, p.n)
ct = B.encrypt(B.encode(v, p), pk, p, np.random.default_rng(2))
m = B.rescale(B.hom_mul(ct, ct, rlk, p), p)
r = B.hom_rotate_hoisted(ct, [1, 2, 3], rk, p)
b2 = fused.rescale_multi(p, ct, 2)
be = BT.GpuBackend(p, rlk, None, rk)
ext = be.rotate_hoisted_ext(ct, [1, 2])
pt = be.encode_slots(v + 0j, ct.level, p.rns_basis[ct.level], ext=True)
y = be.bsgs_combine_ext([(0, [(ext[0], pt)]), (3, [(ext[1], pt)])])
tp = B.gen_params(256, 30, d=3, seed=0, scale=2 ** 26)
tsk, tpk, trlk = B.keygen(tp, seed=11)
cfg = BT.BootConfig(cts_levels=3, stc_levels=3)
planner = BT.Bootstrapper(type("P", (), {"N": tp.N, "main_primes": tp.rns_basis}), cfg)
ck, trk = BT.make_bootstrap_keys(tp, tsk, planner.required_rotations())
tct = B.encrypt(B.encode(np.random.default_rng(3).uniform(-1, 1, tp.n), tp, level=0, scale=2 ** 22), tpk, tp,
                np.random.default_rng(4))
out = BT.Bootstrapper(BT.GpuBackend(tp, trlk, ck, trk), cfg).bootstrap(tct)
# fused hom_mul + double rescale, fused BSGS inner sums, kernel-plan interpreter, NTT row kernels
mr = fused.hom_mul_rescale(p, ct, ct, rlk, 2)
fz = be.bsgs_fused_ext(ct, [(0, [(0, pt), (1, pt)]), (3, [(2, pt)])])
import json  # noqa: E402
from paper_2512_11269_b200.kernel_runner import KernelRunner, plan_from_json  # noqa: E402
fx = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                 "tests", "golden", "kernel_plans_synth.json")))
kp = B.gen_params(**fx["gen_params"])
rows = {l: torch.randint(0, 1 << 20, (kp.N,), dtype=torch.int32, device="cuda") for l, _ in fx["inputs"]}
kr = KernelRunner(kp)
for pl in fx["plans"]:
    kr.run(plan_from_json(pl), lambda l: rows[l],
           lambda l: rows.setdefault(l, torch.empty(kp.N, dtype=torch.int32, device="cuda")))
from paper_2512_11269_b200.poly import ntt_rows  # noqa: E402
nr = torch.randint(0, 1 << 20, (4, p.N), dtype=torch.int32, device="cuda")
ntt_rows(p, nr, (0, 1, 2, 3))
ntt_rows(p, nr, (0, 1, 2, 3), inverse=True)
torch.cuda.synchronize()
print("sanitize run ok", m.level, len(r), out.level, mr[0].limbs.shape[0], fz.level)
