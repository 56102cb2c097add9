"""k = 1 sharded keyswitch at C2 (the gathers as device copies): the overlapped half-batch schedule
of lf_shard_keyswitch against the serial phase sequence (lf_shard_ks_phase x3 + copies) and the
single-device lf_keyswitch, batch 32, CUDA events, graph replay."""
import torch
import paper_2512_11269_b200 as B
from paper_2512_11269_b200 import fused
from paper_2512_11269_b200.shard import ShardEngine


def timed(fn, it=50):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
    torch.cuda.synchronize()
    for _ in range(5):
        g.replay()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it * 1e3


p = B.gen_params(N=65536, num_levels=35, d=4, seed=0, scale=2 ** 26)
sk, pk, rlk = B.keygen(p, seed=3)
lv, bt = p.max_level, 32
q = torch.tensor(p.rns_basis[: lv + 1], dtype=torch.int64, device="cuda")[:, None]
xs = (torch.randint(0, 2 ** 62, (bt, lv + 1, p.N), device="cuda", dtype=torch.int64) % q).to(torch.int32)
e = ShardEngine(p, 1, 0)
kl = e.shard_key(rlk)
call, out = e.keyswitch_call(lv, xs, kl)
ws = e.workspace(lv, bt)
lay = e.gather_layout(lv, bt)
w8 = ws.view(torch.uint8)


def serial():
    for ph, (so, nb, ro) in ((0, lay[:3]), (1, lay[3:])):
        e.phase(ph, call, lv, bt)
        w8[ro: ro + nb].copy_(w8[so: so + nb])
    e.phase(2, call, lv, bt)


print(f"single-device lf_keyswitch     {timed(lambda: fused.keyswitch_batch(p, lv, xs, rlk)) / bt:7.2f} us/op")
print(f"k=1 serial phases + copies     {timed(serial) / bt:7.2f} us/op")
print(f"k=1 lf_shard_keyswitch overlap {timed(lambda: e.run(call, lv, bt)) / bt:7.2f} us/op")
