"""Limb-sharded keyswitch: placement rule and bit-exactness of the
InputBroadcast all-gather pattern against the single-device keyswitch.  CPU: world sizes 2
and 3 over gloo with the oracle row primitives.  GPU: world size 2 on one device (gloo
staging) with the sm_100a row kernels, against the fused single-GPU keyswitch / rotate."""

import os
import socket

import numpy as np
import pytest

from paper_2512_11269_b200.shard import SPECIAL_BASE, Layout, owner

KW = dict(N=256, num_levels=6, d=3, seed=3)


def test_owner_rule_and_partition():
    assert owner(5, 4) == 1 and owner(SPECIAL_BASE + 6, 4) == 2
    for k in (1, 2, 3, 8):
        lays = [Layout(level=9, alpha=4, d=3, k=k, rank=r) for r in range(k)]
        all_ext = sorted(b for L in lays for b in L.ext_loc)
        assert all_ext == sorted(lays[0].ext)
        for L in lays:
            assert all(owner(b, k) == L.rank for b in L.ext_loc)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _cpu_worker(rank, world, port, level, galois, outdir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import lf_oracle as O
    from oracle.shard_backend import GlooNumpyComm, OracleRowOps
    from paper_2512_11269_b200.shard import Layout, ShardedKeyswitch
    P = O.gen_params(**KW)
    rng = np.random.default_rng(7)
    ext = P.ext_ids(P.L)
    evk = O.EvalKeyO("relin", [(O.sample_uniform(P, rng, ext), O.sample_uniform(P, rng, ext)) for _ in range(P.d)])
    x = O.sample_uniform(P, np.random.default_rng(11), P.main_ids(level))
    lay = Layout(level, P.alpha, P.d, world, rank)
    ops = OracleRowOps(P)
    dec = {i: v for j in range(P.d) for i, v in O.decomposition_scalars(P, j, [i for i in range(level + 1) if i % P.d == j]).items()}
    Pp = O.special_product(P)
    pinv = {i: pow(Pp % P.main[i], -1, P.main[i]) for i in range(level + 1)}

    def key_rows(j):
        kb, ka = evk.digits[j]
        return kb.sub(lay.ext_loc).rows, ka.sub(lay.ext_loc).rows

    ks = ShardedKeyswitch(ops, GlooNumpyComm(), lay, dec, pinv)
    x_loc = x.sub(lay.main_loc).rows
    b, a = ks.keyswitch(x_loc, key_rows, galois)
    np.savez(os.path.join(outdir, f"r{rank}.npz"), b=b, a=a, ids=np.array(lay.main_loc))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,level,galois", [(2, 6, None), (3, 6, None), (2, 4, 5), (3, 2, None)])
def test_sharded_keyswitch_gloo_cpu(tmp_path, world, level, galois):
    import torch.multiprocessing as mp
    from oracle import lf_oracle as O
    mp.spawn(_cpu_worker, args=(world, _free_port(), level, galois, str(tmp_path)), nprocs=world, join=True)
    P = O.gen_params(**KW)
    rng = np.random.default_rng(7)
    ext = P.ext_ids(P.L)
    evk = O.EvalKeyO("relin", [(O.sample_uniform(P, rng, ext), O.sample_uniform(P, rng, ext)) for _ in range(P.d)])
    x = O.sample_uniform(P, np.random.default_rng(11), P.main_ids(level))
    if galois is None:
        wb, wa = O.keyswitch(P, x, evk)
    else:
        pieces = [(j, O.p_automorph(P, d, galois)) for j, d in O.ks_decompose(P, x)]
        ab, aa = O.ks_inner(P, pieces, evk)
        wb, wa = O.mod_down(P, ab, P.main_ids(level)), O.mod_down(P, aa, P.main_ids(level))
    got_b = np.zeros_like(wb.rows)
    got_a = np.zeros_like(wa.rows)
    for r in range(world):
        z = np.load(tmp_path / f"r{r}.npz")
        for i, bid in enumerate(z["ids"]):
            got_b[bid], got_a[bid] = z["b"][i], z["a"][i]
    assert np.array_equal(got_b, wb.rows) and np.array_equal(got_a, wa.rows)


def _gpu_worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2512_11269_b200 as B
    from paper_2512_11269_b200.ntt_host import galois_element
    from paper_2512_11269_b200.shard import Layout, gpu_sharded_keyswitch
    out = {}
    for name, kw in (("desk", dict(N=4096, num_levels=6, d=3, seed=0)),
                     ("c2", dict(N=65536, num_levels=35, d=4, seed=0, scale=2 ** 26))):
        p = B.gen_params(**kw)
        sk, pk, rlk = B.keygen(p, seed=11)
        level = p.max_level
        rng = np.random.default_rng(5)
        x = np.stack([rng.integers(0, p.rns_basis[i], p.N, dtype=np.uint64) for i in range(level + 1)])
        lay = Layout(level, p.num_special, p.ks.d, world, rank)
        x_loc = B.RnsPolynomial(x[list(lay.main_loc)], B.Domain.EVAL, lay.main_loc).limbs
        for g in (None, galois_element(p.N, 1)):
            b, a = gpu_sharded_keyswitch(p, level, x_loc, rlk, galois=g)
            out[f"{name}_{g}_b"] = b.cpu().numpy()
            out[f"{name}_{g}_a"] = a.cpu().numpy()
        out[f"{name}_ids"] = np.array(lay.main_loc)
        # the fused sharded pipeline (lf_shard_*), gathers through torch.distributed (gloo here)
        from paper_2512_11269_b200.shard import ShardEngine
        e = ShardEngine(p, world, rank, comm="torch")
        assert e.main_rows(level) == list(lay.main_loc)
        o = e.keyswitch(level, x_loc[None].contiguous(), e.shard_key(rlk))
        out[f"{name}_fused_b"] = o[0, 0].cpu().numpy()
        out[f"{name}_fused_a"] = o[0, 1].cpu().numpy()
    np.savez(os.path.join(outdir, f"g{rank}.npz"), **out)
    dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_keyswitch_gpu_two_ranks(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    mp.spawn(_gpu_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    import paper_2512_11269_b200 as B
    from paper_2512_11269_b200 import ckks as C
    from paper_2512_11269_b200 import fused
    from paper_2512_11269_b200.ntt_host import galois_element
    from paper_2512_11269_b200.poly import main_ids
    for name, kw in (("desk", dict(N=4096, num_levels=6, d=3, seed=0)),
                     ("c2", dict(N=65536, num_levels=35, d=4, seed=0, scale=2 ** 26))):
        p = B.gen_params(**kw)
        sk, pk, rlk = B.keygen(p, seed=11)
        level = p.max_level
        rng = np.random.default_rng(5)
        x = np.stack([rng.integers(0, p.rns_basis[i], p.N, dtype=np.uint64) for i in range(level + 1)])
        xp = B.RnsPolynomial(x, B.Domain.EVAL, main_ids(level))
        for g in (None, galois_element(p.N, 1)):
            if g is None:
                wb, wa = fused.keyswitch(p, xp, rlk)
            else:
                pieces = [(j, B.poly.poly_automorph(d, g, p)) for j, d in C.keyswitch_decompose(xp, p)]
                ab, aa = C.keyswitch_inner_product(pieces, rlk, p)
                wb, wa = B.poly.mod_down(ab, main_ids(level), p), B.poly.mod_down(aa, main_ids(level), p)
            wb, wa = wb.numpy(), wa.numpy()
            for r in range(2):
                z = np.load(tmp_path / f"g{r}.npz")
                for i, bid in enumerate(z[f"{name}_ids"]):
                    assert np.array_equal(z[f"{name}_{g}_b"][i].view(np.uint32), wb[bid].astype(np.uint32)), (name, g, bid)
                    assert np.array_equal(z[f"{name}_{g}_a"][i].view(np.uint32), wa[bid].astype(np.uint32)), (name, g, bid)
                    if g is None:
                        assert np.array_equal(z[f"{name}_fused_b"][i].view(np.uint32), wb[bid].astype(np.uint32))
                        assert np.array_equal(z[f"{name}_fused_a"][i].view(np.uint32), wa[bid].astype(np.uint32))
