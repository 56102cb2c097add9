"""Time the N=2^16 bootstrap (C3 variant) on cuda:0: setup, eager latency, precision."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_11269_b200 as B  # noqa: E402
from paper_2512_11269_b200 import bootstrap as BT  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 47
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
t0 = time.time()
dnum = int(next((a.split("=")[1] for a in sys.argv if a.startswith("dnum=")), 4))
p = B.gen_params(65536, L, d=dnum, seed=0, scale=2 ** 26)
sk, pk, rlk = B.keygen(p, seed=11)
cfg = BT.BootConfig(**{k: int(v) for k, v in (a.split("=") for a in sys.argv[3:] if "=" in a and not a.startswith("dnum="))})
print("config", cfg)
planner = BT.Bootstrapper(type("P", (), {"N": p.N, "main_primes": p.rns_basis}), cfg)
rots = planner.required_rotations()
ck, rk = BT.make_bootstrap_keys(p, sk, rots, seed=99)
torch.cuda.synchronize()
print(f"keys: {len(rots)} rotations + conj, {time.time() - t0:.1f} s", flush=True)
v = np.random.default_rng(77).uniform(-1, 1, p.n)
ct = B.encrypt(B.encode(v, p, level=0, scale=2 ** 26), pk, p, np.random.default_rng(5))
bt = BT.Bootstrapper(BT.GpuBackend(p, rlk, ck, rk), cfg)
t0 = time.time()
out = bt.bootstrap(ct)
torch.cuda.synchronize()
print(f"first bootstrap (plaintext encoding included): {time.time() - t0:.2f} s; out level {out.level}", flush=True)
din = B.decrypt(ct, sk, p)
dout = B.decrypt(out, sk, p)
e1, e2 = np.abs(dout - din).max(), np.abs(dout - v).max()
print(f"precision: vs input decryption {e1:.3e} ({-np.log2(e1):.1f} bits), vs plaintext {e2:.3e} ({-np.log2(e2):.1f} bits)")
ms = []
for _ in range(reps):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    a.record()
    out = bt.bootstrap(ct)
    b.record()
    torch.cuda.synchronize()
    ms.append((a.elapsed_time(b), (time.perf_counter() - w0) * 1e3))
print("eager bootstrap ms (device, wall):", [(round(x, 2), round(y, 2)) for x, y in ms])

if "--profile" in sys.argv:
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        out = bt.bootstrap(ct)
        torch.cuda.synchronize()
    ka = prof.key_averages()
    tot = sum(k.device_time_total for k in ka)
    print(f"kernel time total {tot / 1e3:.2f} ms over {sum(k.count for k in ka)} launches")
    print(ka.table(sort_by="device_time_total", row_limit=15))

for phase in ("_evalmod", "_linear"):
    if f"--profile{phase}" not in sys.argv:
        continue
    # record the phase's inputs during one bootstrap, then profile the phase alone
    from torch.profiler import ProfilerActivity, profile
    orig, calls = getattr(bt, phase), []

    def rec(*a, _o=orig, **k):
        calls.append((a, k))
        return _o(*a, **k)
    setattr(bt, phase, rec)
    bt.bootstrap(ct)
    setattr(bt, phase, orig)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for a, k in calls:
            orig(*a, **k)
        torch.cuda.synchronize()
    ka = prof.key_averages()
    tot = sum(k.device_time_total for k in ka)
    print(f"{phase}: {len(calls)} calls, kernel time {tot / 1e3:.2f} ms over "
          f"{sum(k.count for k in ka)} launches")
    print(ka.table(sort_by="device_time_total", row_limit=25))

if "--graph" in sys.argv:
    static_in = ct
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        bt.bootstrap(static_in)
    torch.cuda.current_stream().wait_stream(s)
    if "--phases" in sys.argv:
        bt.marks = []
    with torch.cuda.graph(g):
        gout = bt.bootstrap(static_in)
    gmarks, bt.marks = getattr(bt, "marks", None), None
    g.replay()
    torch.cuda.synchronize()
    dg = B.decrypt(gout, sk, p)
    print("graph output matches eager:", np.array_equal(gout.b.numpy(), out.b.numpy()))
    ms = []
    for _ in range(reps + 2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    print("graph bootstrap ms:", [round(x, 2) for x in ms])
    if gmarks:
        print("phases (graph, ms):", {b[0]: round(a[1].elapsed_time(b[1]), 2)
                                      for a, b in zip(gmarks, gmarks[1:])})

if "--phases" in sys.argv:
    bt.marks = []
    bt.bootstrap(ct)
    torch.cuda.synchronize()
    m = bt.marks
    bt.marks = None
    print("phases (eager, ms):", {b[0]: round(a[1].elapsed_time(b[1]), 2) for a, b in zip(m, m[1:])})
