"""CPU restatement of the reference KernelRunner — TEST INFRASTRUCTURE ONLY.

Follows /root/reference/pkg/src/limbforge/codegen.py:346-443 (KernelRunner.run / _run_lane /
_run_ntt / _run_bconv) with the oracle's own NTT, automorphism and exact base conversion
(oracle/lf_oracle.py).  Registers hold canonical residues here (every op reduces), which
gives the same stored rows as the reference's lazily reduced uint64 registers: the lazy
planner (codegen.py:212-272) only skips reductions whose omission cannot change a value mod q,
and every store is canonical.

Plans are duck-typed: the reference's KernelPlan objects and the JSON fixtures loaded by
`plan_from_json` both work.  Parity status: PINNED against the reference's own KernelRunner
output digests (tests/golden/kernel_plans_*.json, made by tests/golden/make_kernel_plans.py).
Only tests/ may import this module.
"""

from __future__ import annotations

from types import SimpleNamespace

import numpy as np

from . import lf_oracle as O

REG, SLOT = "r", "s"          # codegen.py:41-42


def plan_from_json(d):
    """A KernelPlan-shaped namespace from the fixture JSON (same field names as codegen.py:58-87)."""
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
    """codegen.py:346-361: run(plan, read_row, write_row) over caller-managed uint64 rows."""

    def __init__(self, P: O.Params):
        self.P = P
        self.N = P.N

    def run(self, plan, read_row, write_row):
        for lane in plan.lanes:
            self._run_lane(plan, lane, read_row, write_row)

    def _run_lane(self, plan, lane, read_row, write_row):        # codegen.py:363-410
        q = int(lane.prime)
        qv = np.uint64(q)
        regs = {}
        for op in lane.ops:
            srcs = [regs[i] if kind == REG else np.asarray(read_row(plan.operand_table[i]), dtype=np.uint64)
                    for kind, i in op.srcs]
            oc = op.opcode
            if oc == "Add":
                d = (srcs[0] % qv + srcs[1] % qv) % qv
            elif oc == "Sub":
                d = (srcs[0] % qv + (qv - srcs[1] % qv)) % qv
            elif oc == "Mul":
                d = (srcs[0] % qv) * (srcs[1] % qv) % qv
            elif oc == "MulAcc":
                d = (srcs[0] % qv + (srcs[1] % qv) * (srcs[2] % qv) % qv) % qv
            elif oc == "Neg":
                d = (qv - srcs[0] % qv) % qv
            elif oc == "ScalarMul":
                d = (srcs[0] % qv) * np.uint64(int(op.meta["scalar"]) % q) % qv
            elif oc == "ModStep":
                d = (srcs[0] % qv + (qv - srcs[1] % qv)) % qv * np.uint64(int(op.meta["scalar"]) % q) % qv
            elif oc == "Automorph":                                 # codegen.py:399-401
                d = srcs[0][O.automorphism_perm(self.N, int(op.meta["galois"]))]
            elif oc == "NTT":
                d = O.ntt_fwd(srcs[0] % qv, q)
            elif oc == "INTT":
                d = O.ntt_inv(srcs[0] % qv, q)
            elif oc == "BConv":                                     # codegen.py:438-443
                src_primes = tuple(int(self.P.prime(b)) for b in op.meta["src_ids"])
                d = O.bconv_row(np.stack(srcs), src_primes, q)
            else:
                raise ValueError(f"unhandled kernel op {oc}")
            regs[op.dst_reg] = np.asarray(d, dtype=np.uint64)
            if op.store_slot is not None:
                np.copyto(write_row(plan.operand_table[op.store_slot]), regs[op.dst_reg])
