"""Limb-sharded keyswitching across the GPUs of one box.

Placement follows the reference's multi-device partitioner: basis row `bid` lives on rank
`bid % k` (multidev.py:55-56; special primes by their index, (bid - 65536) % k).  Ciphertext
rows and evaluation-key rows are both sharded, so key memory and key HBM traffic drop by 1/k.
Every limb-local stage (element-wise ops, NTT/INTT, automorphism, the key inner product) runs
on the owning rank with no communication (multidev.py:3-6).  The two cross-limb stages use the
reference's InputBroadcast pattern (multidev.py:172-185, 291-412), one all-gather each:

  ModUp    each rank scales its own rows by the decomposition scalars and INTTs them; ONE
           all-gather of those (l+1) coefficient rows; every rank then base-converts each digit
           onto its own extended-basis rows and NTTs them (ckks.py:95-117).
  ModDown  each rank INTTs its special rows of acc_b / acc_a; ONE all-gather of those 2 alpha
           rows; every rank converts them onto its own main rows and finishes
           (acc - conv) * P^-1 (poly.py:251-281).

Modular sums are associative and the gathers move exact residues, so the sharded result is
bit-identical to the single-device keyswitch (tests/test_shard.py checks it against the
oracle with gloo on CPU, world size 2, and against the fused single-GPU kernels).

The algorithm is written against `RowOps` (device row primitives) and `Comm` (all-gather of row
blocks).  `GpuRowOps` runs the sm_100a kernels of libcerium_b200.so; `TorchComm` uses
torch.distributed — NCCL over NVLink on GPUs (device tensors, no host staging), gloo in tests.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SPECIAL_BASE = 1 << 16


def owner(bid: int, k: int) -> int:
    """multidev.py:55-56."""
    return (bid - SPECIAL_BASE) % k if bid >= SPECIAL_BASE else bid % k


@dataclass(frozen=True)
class Layout:
    """Row placement of one level on k ranks."""
    level: int
    alpha: int
    d: int
    k: int
    rank: int

    @property
    def main(self) -> tuple:                  # all main ids at this level
        return tuple(range(self.level + 1))

    @property
    def special(self) -> tuple:
        return tuple(SPECIAL_BASE + j for j in range(self.alpha))

    @property
    def ext(self) -> tuple:
        return self.main + self.special

    def local(self, ids) -> tuple:
        return tuple(b for b in ids if owner(b, self.k) == self.rank)

    def of_rank(self, ids, r) -> tuple:
        return tuple(b for b in ids if owner(b, self.k) == r)

    @property
    def main_loc(self) -> tuple:
        return self.local(self.main)

    @property
    def ext_loc(self) -> tuple:
        return self.local(self.ext)

    @property
    def special_loc(self) -> tuple:
        return self.local(self.special)

    def digits(self):
        g = [tuple(i for i in self.main if i % self.d == j) for j in range(self.d)]
        return [(j, x) for j, x in enumerate(g) if x]


class ShardedKeyswitch:
    """keyswitch(x, evk) (ckks.py:134-140) on k ranks with one all-gather per cross-limb stage.

    `ops` supplies the limb-local primitives, `comm` the all-gather; `dec_scalars[i]` is the
    decomposition scalar of main limb i for its own digit (ckks.py:85-92) and `pinv[i]` is
    P^-1 mod q_i (poly.py:280); `key_rows(j)` returns this rank's (b, a) key rows of digit j
    over `lay.ext_loc` (keys are generated at max level, rows selected by id, ckks.py:126-130).
    """

    def __init__(self, ops, comm, lay: Layout, dec_scalars: dict, pinv: dict):
        self.ops, self.comm, self.lay = ops, comm, lay
        self.dec, self.pinv = dec_scalars, pinv

    def _gather_ordered(self, rows, ids_all):
        """All-gather local row blocks; return the rows of ids_all in id order."""
        parts = self.comm.all_gather(rows)
        by_id = {}
        for r, blk in enumerate(parts):
            for i, b in enumerate(self.lay.of_rank(ids_all, r)):
                by_id[b] = (blk, i)
        return self.ops.take_rows([by_id[b] for b in ids_all])

    def modup(self, x_loc):
        """Per digit j: pieces over this rank's ext rows (eval domain)."""
        ops, lay = self.ops, self.lay
        mloc = lay.main_loc
        scaled = ops.scalar_mul(x_loc, mloc, [self.dec[i] for i in mloc])
        coeff = ops.intt(scaled, mloc)
        C = self._gather_ordered(coeff, lay.main)            # all (l+1) coefficient rows
        pieces = []
        for j, grp in lay.digits():
            tgt = tuple(t for t in lay.ext_loc if t not in grp)
            src_rows = ops.select(C, [lay.main.index(i) for i in grp])
            conv = ops.ntt(ops.bconv(src_rows, grp, tgt), tgt) if tgt else None
            own = {i: mloc.index(i) for i in grp if i in mloc}
            order = []
            for t in lay.ext_loc:
                order.append((scaled, own[t]) if t in own else (conv, tgt.index(t)))
            pieces.append((j, ops.take_rows(order)))
        return pieces

    def inner(self, pieces, key_rows):
        ops, ids = self.ops, self.lay.ext_loc
        acc_b = acc_a = None
        for j, d in pieces:
            kb, ka = key_rows(j)
            acc_b = ops.mulacc(acc_b, d, kb, ids)
            acc_a = ops.mulacc(acc_a, d, ka, ids)
        return acc_b, acc_a

    def moddown(self, acc_b, acc_a):
        ops, lay = self.ops, self.lay
        eloc, sloc, mloc = lay.ext_loc, lay.special_loc, lay.main_loc
        sp_idx = [eloc.index(s) for s in sloc]
        mn_idx = [eloc.index(m) for m in mloc]
        both = ops.concat([ops.select(acc_b, sp_idx), ops.select(acc_a, sp_idx)])
        coeff = ops.intt(both, sloc + sloc)
        parts = self.comm.all_gather(coeff)                    # 2 alpha rows in total
        pos_b, pos_a = {}, {}
        for r, blk in enumerate(parts):
            ids_r = lay.of_rank(lay.special, r)
            for i, s in enumerate(ids_r):
                pos_b[s] = (blk, i)
                pos_a[s] = (blk, len(ids_r) + i)
        Sb = ops.take_rows([pos_b[s] for s in lay.special])
        Sa = ops.take_rows([pos_a[s] for s in lay.special])
        out = []
        for acc, S in ((acc_b, Sb), (acc_a, Sa)):
            if not mloc:
                out.append(ops.empty(0))
                continue
            conv = ops.ntt(ops.bconv(S, lay.special, mloc), mloc)
            out.append(ops.modstep(ops.select(acc, mn_idx), conv, mloc, [self.pinv[i] for i in mloc]))
        return out[0], out[1]

    def keyswitch(self, x_loc, key_rows, galois=None):
        """(ks_b, ks_a) over this rank's main rows.  `galois` applies the automorphism to
        every piece after ModUp (hom_rotate's decompose-then-permute, ckks.py:197-217)."""
        pieces = self.modup(x_loc)
        if galois is not None:
            pieces = [(j, self.ops.automorph(p, galois)) for j, p in pieces]
        return self.moddown(*self.inner(pieces, key_rows))


# ---------------------------------------------------------------------------------------
# GPU primitives and torch.distributed all-gather
# ---------------------------------------------------------------------------------------

class GpuRowOps:
    """Limb-local primitives on device row blocks ((n, N) int32 CUDA tensors)."""

    def __init__(self, params):
        from . import poly as P
        self.P = P
        self.params = params

    def empty(self, n):
        import torch
        return torch.empty((n, self.params.N), dtype=torch.int32, device="cuda")

    def select(self, rows, idx):
        import torch
        if not idx:
            return self.empty(0)
        return rows.index_select(0, torch.tensor(idx, device=rows.device))

    def take_rows(self, pairs):
        import torch
        if not pairs:
            return self.empty(0)
        return torch.stack([blk[i] for blk, i in pairs])

    def concat(self, blocks):
        import torch
        return torch.cat(blocks)

    def scalar_mul(self, rows, ids, scalars):
        out = self.empty(len(ids))
        if ids:
            self.P.ewise(self.params, self.P.LF_OP_SCALAR_MUL, out, rows, ids, scalars=scalars)
        return out

    def intt(self, rows, ids):
        out = rows.clone()
        if ids:
            self.P.ntt_rows(self.params, out, ids, inverse=True)
        return out

    def ntt(self, rows, ids):
        out = rows.clone()
        if ids:
            self.P.ntt_rows(self.params, out, ids)
        return out

    def bconv(self, rows, src_ids, tgt_ids):
        poly = self.P.RnsPolynomial(rows.contiguous(), self.P.Domain.COEFF, tuple(src_ids))
        return self.P.base_convert(poly, tuple(tgt_ids), self.params).limbs

    def mulacc(self, acc, a, b, ids):
        out = self.empty(len(ids))
        if not ids:
            return out
        if acc is None:
            self.P.ewise(self.params, self.P.LF_OP_MUL, out, a, ids, b=b)
        else:
            self.P.ewise(self.params, self.P.LF_OP_MULACC, out, a, ids, b=b, c=acc)
        return out

    def modstep(self, a, b, ids, scalars):
        out = self.empty(len(ids))
        self.P.ewise(self.params, self.P.LF_OP_MODSTEP, out, a, ids, b=b, scalars=scalars)
        return out

    def automorph(self, rows, g):
        out = self.empty(rows.shape[0])
        if rows.shape[0]:
            self.P.automorph_rows(self.params, out, rows.contiguous(), g)
        return out


class TorchComm:
    """All-gather of variable-size row blocks over torch.distributed.  NCCL gathers device
    tensors directly (NVLink); gloo stages through host memory (CPU tests, single-GPU tests)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.k = dist.get_world_size(group)
        self.backend = dist.get_backend(group)

    def all_gather(self, rows):
        import torch
        dist = self.dist
        n = torch.tensor([rows.shape[0]], dtype=torch.int64)
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(self.k)]
        if self.backend == "nccl":
            n = n.cuda()
            sizes = [s.cuda() for s in sizes]
        dist.all_gather(sizes, n, group=self.group)
        sizes = [int(s.item()) for s in sizes]
        m = max(sizes)
        width = rows.shape[1]
        dev = rows.device if self.backend == "nccl" else torch.device("cpu")
        send = torch.zeros((m, width), dtype=rows.dtype, device=dev)
        if rows.shape[0]:
            send[: rows.shape[0]] = rows.to(dev)
        recv = [torch.empty_like(send) for _ in range(self.k)]
        dist.all_gather(recv, send, group=self.group)
        return [r[:s].to(rows.device) for r, s in zip(recv, sizes)]


def dec_scalars(params, level) -> dict:
    from .keys import digit_hat_factor
    d = params.ks.d
    out = {}
    for i in range(level + 1):
        f = digit_hat_factor(params, i % d)
        q = params.rns_basis[i]
        out[i] = pow(f % q, -1, q)
    return out


def pinv_scalars(params, level) -> dict:
    P = params.special_product()
    return {i: pow(P % params.rns_basis[i], -1, params.rns_basis[i]) for i in range(level + 1)}


def gpu_sharded_keyswitch(params, level: int, x_loc, evk, comm=None, galois=None):
    """This rank's rows of keyswitch(x, evk) (ckks.py:134-140) on the limb-sharded layout;
    x_loc holds x's rows for `Layout.main_loc`.  evk is the full-level key (only this rank's
    rows are read; a production deployment keeps only those rows resident)."""
    import torch.distributed as dist
    comm = comm or TorchComm()
    lay = Layout(level, params.num_special, params.ks.d, comm.k, dist.get_rank(comm.group))
    ops = GpuRowOps(params)
    key_ids = tuple(evk.ids)
    idx = [key_ids.index(b) for b in lay.ext_loc]

    def key_rows(j):
        return ops.select(evk.data[j, 0], idx), ops.select(evk.data[j, 1], idx)

    ks = ShardedKeyswitch(ops, comm, lay, dec_scalars(params, level), pinv_scalars(params, level))
    return ks.keyswitch(x_loc, key_rows, galois)


# ---------------------------------------------------------------------------------------
# The fused limb-sharded pipeline (csrc/lf_ks.cu, lf_shard_*): the five keyswitch kernels on
# this rank's rows, the two InputBroadcast all-gathers as ncclAllGather on the launch stream.
# ---------------------------------------------------------------------------------------

import ctypes as _ct

OP_KS, OP_MUL, OP_ROT = 0, 1, 2


class _ShardCall(_ct.Structure):
    """lf_shard_call (include/lf_b200.h)."""
    _fields_ = [("level", _ct.c_int), ("op", _ct.c_int), ("batch", _ct.c_int),
                ("x", _ct.c_void_p), ("x2", _ct.c_void_p), ("x_bstride", _ct.c_size_t),
                ("keys", _ct.c_void_p), ("galois", _ct.c_void_p),
                ("out", _ct.c_void_p), ("out_bstride", _ct.c_size_t),
                ("e0", _ct.c_void_p), ("e1", _ct.c_void_p), ("e_bstride", _ct.c_size_t)]


class NcclComm:
    """An NCCL communicator owned by libcerium_b200 (lf_comm_create).  The 128-byte unique id
    is created on rank 0 and broadcast over the caller's torch.distributed group."""

    def __init__(self, k: int, rank: int, group=None):
        import torch
        import torch.distributed as dist
        from . import _native
        lib = _native.lib()
        uid = (_ct.c_uint8 * 128)()
        if rank == 0:
            _native.check(lib.lf_comm_unique_id(_ct.cast(uid, _ct.c_void_p)), "lf_comm_unique_id")
        t = torch.tensor(list(bytes(uid)), dtype=torch.uint8)
        if dist.get_backend(group) == "nccl":
            t = t.cuda()
        dist.broadcast(t, src=0, group=group)
        uid = (_ct.c_uint8 * 128)(*t.cpu().tolist())
        h = _ct.c_void_p()
        _native.check(lib.lf_comm_create(k, rank, _ct.cast(uid, _ct.c_void_p), _ct.byref(h)), "lf_comm_create")
        self.handle, self.k, self.rank = h, k, rank

    def __del__(self):
        try:
            from . import _native
            if self.handle:
                _native.lib().lf_comm_destroy(self.handle)
        except Exception:
            pass


class ShardEngine:
    """One rank's share of the limb-sharded keyswitch, hom_mul and hom_rotate (this rank's main
    rows of every ciphertext, its rows of every evaluation key).  With a communicator the calls
    run end to end on the device stream (lf_shard_keyswitch); without one, `phase()` exposes
    the three phases for callers that move the gathered rows themselves (`emulate`)."""

    def __init__(self, params, k: int, rank: int, comm=None):
        from . import _native
        from .context import get_context
        self.params, self.k, self.rank = params, k, rank
        self.ctx = get_context(params)
        self.lib = _native.lib()
        h = _ct.c_void_p()
        _native.check(self.lib.lf_shard_create(self.ctx.handle, k, rank, _ct.byref(h)), "lf_shard_create")
        self.handle = h
        # comm: NcclComm (the library's own ncclAllGather on the launch stream), a
        # torch.distributed group or "torch" (the default group: all_gather_into_tensor on
        # workspace views; gloo stages through the host), or None for k = 1
        self.comm = comm
        if isinstance(comm, NcclComm):
            _native.check(self.lib.lf_shard_attach_comm(h, comm.handle), "lf_shard_attach_comm")
        self._ws = {}

    def __del__(self):
        try:
            if self.handle:
                self.lib.lf_shard_destroy(self.handle)
        except Exception:
            pass

    # layout ---------------------------------------------------------------------------
    def info(self, level: int):
        v = [_ct.c_int() for _ in range(4)]
        from . import _native
        _native.check(self.lib.lf_shard_info(self.handle, level, *[_ct.byref(x) for x in v]), "lf_shard_info")
        return dict(n_main=v[0].value, n_ext=v[1].value, n_key_rows=v[2].value, n_special=v[3].value)

    def main_rows(self, level: int) -> list:
        """Main prime indices this rank holds at `level` (multidev.py:55-56)."""
        return list(range(self.rank, level + 1, self.k))

    def key_rows(self) -> list:
        """Rows of the full-level extended basis this rank keeps of every evaluation key:
        main_loc(L) ascending, then its special rows (prime index L+1+j)."""
        L, alpha = self.params.max_level, self.params.num_special
        return self.main_rows(L) + [L + 1 + j for j in range(self.rank, alpha, self.k)]

    def shard_key(self, evk):
        """This rank's rows of a full evaluation key ((d, 2, L+1+alpha, N) -> (d, 2, n_key_rows, N))."""
        import torch
        idx = torch.tensor(self.key_rows(), device=evk.data.device)
        return evk.data.index_select(2, idx).contiguous()

    def shard_rows(self, rows, level: int):
        """(..., level+1, N) full rows -> (..., n_main, N) this rank's rows."""
        import torch
        idx = torch.tensor(self.main_rows(level), device=rows.device, dtype=torch.long)
        return rows.index_select(rows.dim() - 2, idx).contiguous()

    def workspace(self, level: int, batch: int):
        import torch
        key = (level, batch, torch.cuda.current_stream().cuda_stream)
        ws = self._ws.get(key)
        if ws is None:
            n = self.lib.lf_shard_ws_bytes(self.handle, level, batch) // 4
            ws = torch.empty(n, dtype=torch.int32, device="cuda")
            self._ws[key] = ws
        return ws

    def gather_layout(self, level: int, batch: int):
        from . import _native
        a = (_ct.c_size_t * 6)()
        _native.check(self.lib.lf_shard_gather_layout(self.handle, level, batch, a), "lf_shard_gather_layout")
        return tuple(int(x) for x in a)

    # calls -----------------------------------------------------------------------------
    def _call(self, level, op, batch, x, x2, x_bs, keys, galois, out, out_bs, e0=None, e1=None, e_bs=0):
        keys = list(keys)
        karr = (_ct.c_void_p * batch)(*[(keys[i] if len(keys) > 1 else keys[0]).data_ptr() for i in range(batch)])
        garr = (_ct.c_uint32 * batch)(*[int(g) & 0xFFFFFFFF for g in galois]) if galois is not None else None
        c = _ShardCall(level, op, batch, x.data_ptr() if x is not None else None,
                       x2.data_ptr() if x2 is not None else None, x_bs, _ct.cast(karr, _ct.c_void_p),
                       _ct.cast(garr, _ct.c_void_p) if garr is not None else None,
                       out.data_ptr() if out is not None else None, out_bs,
                       e0.data_ptr() if e0 is not None else None, e1.data_ptr() if e1 is not None else None, e_bs)
        # the call holds raw pointers: keep every operand alive as long as the call object
        return c, (karr, garr, x, x2, keys, out, e0, e1)

    def run(self, call, level, batch):
        from . import _native
        from .context import stream_handle
        if self.comm is not None and not isinstance(self.comm, NcclComm):
            return self._run_torch(call, level, batch)
        c, keep = call
        ws = self.workspace(level, batch)
        _native.check(self.lib.lf_shard_keyswitch(self.handle, _ct.byref(c), _ct.c_void_p(ws.data_ptr()),
                                                  stream_handle()), "lf_shard_keyswitch")

    def _run_torch(self, call, level, batch):
        """Phases 0-2 with the two all-gathers through torch.distributed (fixed sizes, no size
        exchange, no host synchronisation with NCCL; gloo copies through host memory)."""
        import torch
        import torch.distributed as dist
        group = None if self.comm == "torch" else self.comm
        ws = self.workspace(level, batch).view(torch.uint8)
        lay = self.gather_layout(level, batch)
        nccl = dist.get_backend(group) == "nccl"
        for p, (so, nb, ro) in ((0, lay[:3]), (1, lay[3:])):
            self.phase(p, call, level, batch)
            send, recv = ws[so: so + nb], ws[ro: ro + self.k * nb]
            if nccl:
                dist.all_gather_into_tensor(recv, send, group=group)
            else:
                parts = [torch.empty(nb, dtype=torch.uint8) for _ in range(self.k)]
                dist.all_gather(parts, send.cpu(), group=group)
                recv.copy_(torch.cat(parts))
        self.phase(2, call, level, batch)

    def phase(self, p, call, level, batch):
        from . import _native
        from .context import stream_handle
        c, keep = call
        ws = self.workspace(level, batch)
        _native.check(self.lib.lf_shard_ks_phase(self.handle, p, _ct.byref(c), _ct.c_void_p(ws.data_ptr()),
                                                 stream_handle()), "lf_shard_ks_phase")

    def keyswitch_call(self, level, x_loc, key_loc, out=None):
        """x_loc: (B, n_main, N) this rank's rows -> out (B, 2, n_main, N): (ks_b, ks_a)."""
        import torch
        B, nm = x_loc.shape[0], x_loc.shape[1]
        out = torch.empty((B, 2, nm, self.params.N), dtype=torch.int32, device="cuda") if out is None else out
        return self._call(level, OP_KS, B, x_loc, None, x_loc[0].numel(), [key_loc], None, out,
                          out[0].numel()), out

    def hom_mul_call(self, level, ct1_loc, ct2_loc, rlk_loc, out=None):
        """ct*_loc: (B, 2, n_main, N) local blocks -> relinearised product (B, 2, n_main, N)."""
        import torch
        out = torch.empty_like(ct1_loc) if out is None else out
        return self._call(level, OP_MUL, ct1_loc.shape[0], ct1_loc[:, 1], ct2_loc[:, 1], ct1_loc[0].numel(),
                          [rlk_loc], None, out, out[0].numel(), ct1_loc, ct2_loc, ct1_loc[0].numel()), out

    def rotate_call(self, level, ct_loc, gs, keys_loc, out=None):
        """ct_loc: (B, 2, n_main, N) -> B rotations (Galois element gs[b], key keys_loc[b])."""
        import torch
        out = torch.empty_like(ct_loc) if out is None else out
        return self._call(level, OP_ROT, ct_loc.shape[0], ct_loc[:, 1], None, ct_loc[0].numel(), keys_loc,
                          list(gs), out, out[0].numel(), ct_loc, None, ct_loc[0].numel()), out

    def keyswitch(self, level, x_loc, key_loc):
        call, out = self.keyswitch_call(level, x_loc, key_loc)
        self.run(call, level, x_loc.shape[0])
        return out

    def hom_mul(self, level, ct1_loc, ct2_loc, rlk_loc):
        call, out = self.hom_mul_call(level, ct1_loc, ct2_loc, rlk_loc)
        self.run(call, level, ct1_loc.shape[0])
        return out

    def rotate(self, level, ct_loc, gs, keys_loc):
        call, out = self.rotate_call(level, ct_loc, gs, keys_loc)
        self.run(call, level, ct_loc.shape[0])
        return out


def emulate(engines, calls, level: int, batch: int):
    """Run k ranks' sharded pipelines in ONE process on one device: each rank's phases on its
    own workspace, the two all-gathers as device copies (what ncclAllGather moves over NVLink).
    Tests the sharded data layout and kernels without k GPUs."""
    import torch
    k = len(engines)
    lays = [e.gather_layout(level, batch) for e in engines]
    wss = [e.workspace(level, batch).view(torch.uint8) for e in engines]

    def gather(send_off, nbytes, recv_off):
        for r in range(k):
            for src in range(k):
                wss[r][recv_off[r] + src * nbytes: recv_off[r] + (src + 1) * nbytes].copy_(
                    wss[src][send_off[src]: send_off[src] + nbytes])
    for e, c in zip(engines, calls):
        e.phase(0, c, level, batch)
    gather([l[0] for l in lays], lays[0][1], [l[2] for l in lays])
    for e, c in zip(engines, calls):
        e.phase(1, c, level, batch)
    gather([l[3] for l in lays], lays[0][4], [l[5] for l in lays])
    for e, c in zip(engines, calls):
        e.phase(2, c, level, batch)
