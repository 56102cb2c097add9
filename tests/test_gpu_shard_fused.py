"""The fused limb-sharded pipeline (lf_shard_*): k ranks' kernels emulated in one
process on one B200 (the two all-gathers as device copies, what ncclAllGather moves between
GPUs), each rank holding only its rows of the ciphertexts and of the keys.  Every rank's output
rows equal the single-device fused keyswitch / hom_mul / hom_rotate (themselves pinned to the
reference) at the desk size and at C2, including ranks left without main rows at low levels."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DESK = dict(N=4096, num_levels=6, d=3, seed=0)
C2 = dict(N=65536, num_levels=35, d=4, seed=0, scale=2 ** 26)


@pytest.fixture(scope="module", params=["desk", "c2"])
def env(request):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2512_11269_b200 as B
    p = B.gen_params(**(DESK if request.param == "desk" else C2))
    sk, pk, rlk = B.keygen(p, seed=3)
    rk = {s: B.make_rotation_key(p, sk, s, np.random.default_rng(40 + s)) for s in (1, 5)}
    return request.param, B, p, rlk, rk


def _rand(p, level, lead, seed):
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    q = torch.tensor(p.rns_basis[: level + 1], dtype=torch.int64, device="cuda")[:, None]
    r = torch.randint(0, 2 ** 62, (*lead, level + 1, p.N), device="cuda", generator=g, dtype=torch.int64)
    return (r % q).to(torch.int32)


def _engines(p, k):
    from paper_2512_11269_b200.shard import ShardEngine
    return [ShardEngine(p, k, r) for r in range(k)]


@pytest.mark.parametrize("k", [2, 3, 4, 8])
def test_sharded_keyswitch_equals_single_device(env, k):
    import torch
    from paper_2512_11269_b200 import fused
    from paper_2512_11269_b200.shard import emulate
    name, B, p, rlk, rk = env
    for level in (p.max_level, 2):
        xs = _rand(p, level, (3,), 7 * k + level)
        want = fused.keyswitch_batch(p, level, xs, rlk)
        eng = _engines(p, k)
        calls, outs = [], []
        for e in eng:
            c, o = e.keyswitch_call(level, e.shard_rows(xs, level), e.shard_key(rlk))
            calls.append(c)
            outs.append(o)
        emulate(eng, calls, level, 3)
        for e, o in zip(eng, outs):
            rows = e.main_rows(level)
            assert o.shape[2] == len(rows)
            if rows:
                assert torch.equal(o, want[:, :, rows]), (name, k, level, e.rank)


@pytest.mark.parametrize("k", [2, 4])
def test_sharded_hom_mul_and_rotate(env, k):
    import torch
    from paper_2512_11269_b200 import fused
    from paper_2512_11269_b200.ntt_host import galois_element
    from paper_2512_11269_b200.shard import emulate
    name, B, p, rlk, rk = env
    level = p.max_level - 1
    c1, c2 = _rand(p, level, (2, 2), 11), _rand(p, level, (2, 2), 12)
    E = B.Domain.EVAL
    ids = tuple(range(level + 1))
    mk = lambda t: B.Ciphertext(B.RnsPolynomial(t[0], E, ids), B.RnsPolynomial(t[1], E, ids), p.scale, level)
    want_mul = [B.hom_mul(mk(c1[i]), mk(c2[i]), rlk, p) for i in range(2)]
    steps = [1, 5]
    gs = [galois_element(p.N, s) for s in steps]
    want_rot = [B.hom_rotate(mk(c1[i]), steps[i], rk[steps[i]], p) for i in range(2)]
    eng = _engines(p, k)
    calls, outs = [], []
    for e in eng:
        c, o = e.hom_mul_call(level, e.shard_rows(c1, level), e.shard_rows(c2, level), e.shard_key(rlk))
        calls.append(c)
        outs.append(o)
    emulate(eng, calls, level, 2)
    for e, o in zip(eng, outs):
        rows = e.main_rows(level)
        for i in range(2):
            assert torch.equal(o[i, 0], want_mul[i].b.limbs[rows]) and torch.equal(o[i, 1], want_mul[i].a.limbs[rows])
    calls, outs = [], []
    for e in eng:
        c, o = e.rotate_call(level, e.shard_rows(c1, level), gs, [e.shard_key(rk[s]) for s in steps])
        calls.append(c)
        outs.append(o)
    emulate(eng, calls, level, 2)
    for e, o in zip(eng, outs):
        rows = e.main_rows(level)
        for i in range(2):
            assert torch.equal(o[i, 0], want_rot[i].b.limbs[rows]) and torch.equal(o[i, 1], want_rot[i].a.limbs[rows])


def test_single_rank_runs_end_to_end(env):
    """k = 1 through lf_shard_keyswitch (the gathers degenerate to copies): the whole pipeline
    in one call equals lf_keyswitch."""
    import torch
    from paper_2512_11269_b200 import fused
    from paper_2512_11269_b200.shard import ShardEngine
    name, B, p, rlk, rk = env
    e = ShardEngine(p, 1, 0)
    xs = _rand(p, p.max_level, (2,), 5)
    assert torch.equal(e.keyswitch(p.max_level, xs, e.shard_key(rlk)), fused.keyswitch_batch(p, p.max_level, xs, rlk))


def test_sharded_key_upload_from_lfhe(env):
    """Each rank uploads only its key rows from the LFHE blob (serial.evalkey_shard_from_bytes)."""
    import torch
    from paper_2512_11269_b200 import serial as S
    from paper_2512_11269_b200.shard import ShardEngine
    name, B, p, rlk, rk = env
    if name != "desk":
        pytest.skip("blob round trip at the desk size")
    blob = S.evalkey_to_bytes(rlk, p)
    for r in range(3):
        e = ShardEngine(p, 3, r)
        purpose, rows = S.evalkey_shard_from_bytes(blob, p, 3, r)
        assert purpose == "relin" and torch.equal(rows, e.shard_key(rlk))
        assert rows.shape[2] == e.info(p.max_level)["n_key_rows"]


def test_library_nccl_communicator_single_rank(env):
    """The library's own NCCL communicator (lf_comm_create, libnccl resolved at run time) with
    one rank: lf_shard_keyswitch issues both ncclAllGather calls on the launch stream."""
    import os
    import socket
    import torch
    import torch.distributed as dist
    from paper_2512_11269_b200 import fused
    from paper_2512_11269_b200.shard import NcclComm, ShardEngine
    name, B, p, rlk, rk = env
    started = not dist.is_initialized()
    if started:
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        comm = NcclComm(1, 0)
        e = ShardEngine(p, 1, 0, comm=comm)
        xs = _rand(p, p.max_level, (2,), 6)
        got = e.keyswitch(p.max_level, xs, e.shard_key(rlk))
        assert torch.equal(got, fused.keyswitch_batch(p, p.max_level, xs, rlk))
    finally:
        if started:
            dist.destroy_process_group()


@pytest.mark.parametrize("batch", [1, 2, 3, 5])
def test_overlapped_half_batches(env, batch):
    """lf_shard_keyswitch splits batches of two or more into two halves whose all-gathers run on
    the shard's comm stream under the other half's kernels (k = 1: the gathers are copies).  Odd
    batches (uneven halves), hom_mul and rotation, eager and replayed from a CUDA graph, all equal
    the single-device pipeline."""
    import torch
    from paper_2512_11269_b200 import fused
    from paper_2512_11269_b200.ntt_host import galois_element
    from paper_2512_11269_b200.shard import ShardEngine
    name, B, p, rlk, rk = env
    level = p.max_level - 1
    e = ShardEngine(p, 1, 0)
    xs = _rand(p, level, (batch,), 20 + batch)
    want = fused.keyswitch_batch(p, level, xs, rlk)
    assert torch.equal(e.keyswitch(level, xs, e.shard_key(rlk)), want)
    c1, c2 = _rand(p, level, (batch, 2), 30), _rand(p, level, (batch, 2), 31)
    E = B.Domain.EVAL
    ids = tuple(range(level + 1))
    mk = lambda t: B.Ciphertext(B.RnsPolynomial(t[0], E, ids), B.RnsPolynomial(t[1], E, ids), p.scale, level)
    steps = [(1, 5)[i % 2] for i in range(batch)]
    gs = [galois_element(p.N, s) for s in steps]
    kl = {s: e.shard_key(rk[s]) for s in (1, 5)}
    got_mul = e.hom_mul(level, c1, c2, e.shard_key(rlk))
    got_rot = e.rotate(level, c1, gs, [kl[s] for s in steps])
    for i in range(batch):
        wm = B.hom_mul(mk(c1[i]), mk(c2[i]), rlk, p)
        wr = B.hom_rotate(mk(c1[i]), steps[i], rk[steps[i]], p)
        assert torch.equal(got_mul[i, 0], wm.b.limbs) and torch.equal(got_mul[i, 1], wm.a.limbs)
        assert torch.equal(got_rot[i, 0], wr.b.limbs) and torch.equal(got_rot[i, 1], wr.a.limbs)
    # the fork/join through the comm stream is capturable
    call, out = e.hom_mul_call(level, c1, c2, e.shard_key(rlk))
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        e.run(call, level, batch)                     # allocate the stream's workspace outside capture
        out.zero_()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            e.run(call, level, batch)
    torch.cuda.current_stream().wait_stream(s)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, got_mul)
