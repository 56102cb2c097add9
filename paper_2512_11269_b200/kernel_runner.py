"""B200 KernelRunner: the reference's kernel-plan boundary on the GPU.

Replaces `limbforge.codegen.KernelRunner` (codegen.py:346-443) with the same call,
`KernelRunner(params).run(plan, read_row, write_row)`, for the plans `plan_kernels`
(codegen.py:445+) emits and the Executor (runtime.py:409) / multi-device runner
(multidev.py:835) schedule.  Two row conventions:

* device rows: `read_row(lvid)` / `write_row(lvid)` return CUDA int32 tensors of N residues
  (a B200-resident pool; nothing crosses PCIe);
* host rows (the reference Executor as is): they return numpy uint64 rows; the operand rows a
  plan reads are uploaded in one batch, the rows it writes are copied back after the plan.

Execution (csrc/lf_runner.cu): op i of every lane writes register i (codegen.py:160-172), so a
plan runs as steps; each step is ONE `lf_plan_step` launch over all lanes.  Registers live in
a device scratch [step][lane][N]; NTT/INTT steps stage their inputs with COPY and transform
the step's contiguous register rows with the batched `lf_ntt_fwd` / `lf_ntt_inv`.  Every op
produces canonical residues, so the stored rows equal the reference's lazily reduced ones.
There is no CPU path: a missing library or device fails at the first call.
"""

from __future__ import annotations

import ctypes
from types import SimpleNamespace

import numpy as np
import torch

from . import _native
from .context import dptr, get_context, stream_handle

REG, SLOT = "r", "s"                     # codegen.py:41-42
_OPC = {"Add": 0, "Sub": 1, "Mul": 2, "MulAcc": 3, "Neg": 4, "ScalarMul": 5, "ModStep": 6,
        "Automorph": 7, "BConv": 8}       # LF_POP_* (include/lf_b200.h)
_COPY = 9
_NTT_OPS = ("NTT", "INTT")
_REC = np.dtype([("opcode", "<i4"), ("pidx", "<i4"), ("scalar", "<u4"), ("galois", "<u4"),
                 ("nsrc", "<i4"), ("k", "<i4"), ("W", "<i4"), ("pad", "<i4"),
                 ("src", "<u8"), ("dst", "<u8"), ("store", "<u8"), ("table", "<u8")])


def plan_from_json(d):
    """A KernelPlan-shaped namespace from a serialised plan (field names of codegen.py:58-87)."""
    lanes = []
    for ln in d["lanes"]:
        ops = [SimpleNamespace(opcode=o["opcode"], dst_reg=o["dst_reg"],
                               srcs=tuple((k, i) for k, i in o["srcs"]), meta=dict(o["meta"]),
                               store_slot=o["store_slot"], reduce_after=o["reduce_after"])
               for o in ln["ops"]]
        lanes.append(SimpleNamespace(base_id=ln["base_id"], prime=ln["prime"], ops=ops))
    return SimpleNamespace(kernel_id=d["kernel_id"], opclass=d["opclass"], lanes=lanes,
                           operand_table=list(d["operand_table"]), writes=list(d["writes"]))


class KernelRunner:
    """codegen.py:346-361 on the B200: run(plan, read_row, write_row)."""

    def __init__(self, params, max_regs: int = 512):
        self.params = params
        self.N = params.N
        self.ctx = get_context(params)
        self.max_regs = max_regs
        self._scratch = torch.empty(0, dtype=torch.int32, device="cuda")
        self._keep = []

    def _regs(self, steps, nlanes):
        need = steps * nlanes * self.N
        if self._scratch.numel() < need:
            self._scratch = torch.empty(need, dtype=torch.int32, device="cuda")
        return self._scratch[:need].view(steps, nlanes, self.N)

    def run(self, plan, read_row, write_row):
        lanes = plan.lanes
        if not lanes:
            return
        N, ctx, lib = self.N, self.ctx, _native.lib()
        steps = max(len(l.ops) for l in lanes)
        if steps > self.max_regs:
            raise ValueError("scratch undersized for plan")        # codegen.py:359
        regs = self._regs(steps, len(lanes))
        self._keep = []
        # operand rows: which slots are read, which are stored
        rd, wr = [], []
        for lane in lanes:
            for op in lane.ops:
                rd.extend(i for k, i in op.srcs if k == SLOT)
                if op.store_slot is not None:
                    wr.append(op.store_slot)
        rd, wr = list(dict.fromkeys(rd)), list(dict.fromkeys(wr))
        host_rows = None
        ptr = {}
        if rd:
            first = read_row(plan.operand_table[rd[0]])
            host_rows = isinstance(first, np.ndarray)
        else:
            host_rows = not isinstance(write_row(plan.operand_table[wr[0]]), torch.Tensor) if wr else False
        if host_rows:
            slots = list(dict.fromkeys(rd + wr))
            stage = torch.empty((len(slots), N), dtype=torch.int32, device="cuda")
            if rd:
                from .serial import _upload_rows
                # copy each row as it is returned: the Executor hands out compressed operands
                # expanded into a small ring of reused buffers (runtime.py read_pooled)
                up = _upload_rows(np.stack([np.array(read_row(plan.operand_table[i]), dtype=np.uint64, copy=True)
                                            for i in rd]))
                idx = {s: j for j, s in enumerate(slots)}
                stage[[idx[i] for i in rd]] = up
            for j, s in enumerate(slots):
                ptr[s] = stage[j].data_ptr()
            self._keep.append(stage)
        else:
            for i in rd:
                t = read_row(plan.operand_table[i])
                assert t.is_cuda and t.dtype == torch.int32 and t.is_contiguous()
                ptr[i] = t.data_ptr()
            for i in wr:
                t = write_row(plan.operand_table[i])
                assert t.is_cuda and t.dtype == torch.int32 and t.is_contiguous()
                ptr[i] = t.data_ptr()

        stream = stream_handle()
        for s in range(steps):
            recs, srcp, ntt_lanes, stores_after = [], [], [], []
            for L, lane in enumerate(lanes):
                if s >= len(lane.ops):
                    continue
                op = lane.ops[s]
                assert op.dst_reg == s, "plan registers must follow codegen.py:160-172"
                pidx = ctx.pidx(lane.base_id)
                srcs = [regs[i, L].data_ptr() if k == REG else ptr[i] for k, i in op.srcs]
                dst = regs[s, L].data_ptr()
                store = ptr[op.store_slot] if op.store_slot is not None else 0
                rec = dict(opcode=_COPY, pidx=pidx, scalar=0, galois=0, nsrc=len(srcs), k=0, W=0,
                           pad=0, src=len(srcp), dst=dst, store=store, table=0)
                oc = op.opcode
                if oc in _NTT_OPS:
                    rec["store"] = 0                         # stored after the transform
                    ntt_lanes.append((L, pidx, oc == "INTT"))
                    if store:
                        stores_after.append(dict(rec, src=None, store=store, L=L, pidx=pidx))
                else:
                    rec["opcode"] = _OPC[oc]
                    q = int(lane.prime)
                    if oc in ("ScalarMul", "ModStep"):
                        rec["scalar"] = int(op.meta["scalar"]) % q
                    elif oc == "Automorph":
                        rec["galois"] = int(op.meta["galois"]) & ((2 * N) - 1)
                    elif oc == "BConv":
                        blob, k, m, W = ctx.bconv_table(tuple(op.meta["src_ids"]), (lane.base_id,))
                        assert k == len(srcs) and m == 1 and k <= 64
                        rec.update(k=k, W=W, table=blob.data_ptr())
                recs.append(rec)
                srcp.extend(srcs)
            self._launch(recs, srcp, stream)
            # NTT / INTT of this step's register rows, in runs of adjacent lanes
            ntt_lanes.sort()
            i = 0
            while i < len(ntt_lanes):
                j = i
                while (j + 1 < len(ntt_lanes) and ntt_lanes[j + 1][0] == ntt_lanes[j][0] + 1
                       and ntt_lanes[j + 1][2] == ntt_lanes[i][2]):
                    j += 1
                L0, inv = ntt_lanes[i][0], ntt_lanes[i][2]
                fn = lib.lf_ntt_inv if inv else lib.lf_ntt_fwd
                _native.check(fn(ctx.handle, regs[s, L0].data_ptr(), j - i + 1,
                                 _native.i32_array([x[1] for x in ntt_lanes[i: j + 1]]), stream), "lf_ntt")
                i = j + 1
            if stores_after:
                recs2, srcp2 = [], []
                for r in stores_after:
                    recs2.append(dict(opcode=_COPY, pidx=r["pidx"], scalar=0, galois=0, nsrc=1, k=0, W=0,
                                      pad=0, src=len(srcp2), dst=0, store=r["store"], table=0))
                    srcp2.append(regs[s, r["L"]].data_ptr())
                self._launch(recs2, srcp2, stream)
        if host_rows:
            if wr:
                from .serial import _download_rows
                slots = list(dict.fromkeys(rd + wr))
                idx = {s_: j for j, s_ in enumerate(slots)}
                raw = np.frombuffer(_download_rows(self._keep[0][[idx[i] for i in wr]]), dtype="<u8")
                raw = raw.reshape(len(wr), N)
                for j, i in enumerate(wr):
                    np.copyto(write_row(plan.operand_table[i]), raw[j])

    def _launch(self, recs, srcp, stream):
        if not recs:
            return
        n = len(recs)
        arr = np.array([tuple(r[k] for k in _REC.names) for r in recs], dtype=_REC)
        ptrs = np.asarray(srcp, dtype="<u8")
        # one device buffer: the records, then the source-pointer table they index into
        dev = torch.empty(arr.nbytes + ptrs.nbytes, dtype=torch.uint8, device="cuda")
        arr["src"] = dev.data_ptr() + arr.nbytes + 8 * arr["src"]
        host = np.concatenate([arr.view(np.uint8), ptrs.view(np.uint8)])
        dev.copy_(torch.from_numpy(host))
        self._keep.append(dev)
        _native.check(_native.lib().lf_plan_step(self.ctx.handle, ctypes.c_void_p(dev.data_ptr()), n, stream),
                      "lf_plan_step")
