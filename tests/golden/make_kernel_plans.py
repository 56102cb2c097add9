"""Golden fixtures for the KernelRunner boundary (reference codegen.py:346-443).

Run HERE, where the reference is importable (it is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_kernel_plans.py

For each workload the reference compiler lowers a real program to limb IR, fuses it and plans
the kernels (pipeline.py:117-140: hoist_rotations, merge_mod_down, lower_to_limb_ir, fuse_dag,
plan_kernels).  The plans are serialised to JSON (every field the runner reads), the input rows
are drawn from a seeded numpy Generator in `dag.inputs` order, and the reference KernelRunner
executes the whole schedule; the sha256 of every row any plan writes is recorded.  The tests
regenerate the inputs from the seed (a digest of them is stored to catch RNG drift) and compare
the rows produced by the oracle restatement (CPU) and by the B200 runner (GPU) against these
digests.
"""

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def _ser_meta(meta):
    out = {}
    for k in ("scalar", "galois", "src_ids"):
        if k in meta:
            v = meta[k]
            out[k] = [int(x) for x in v] if isinstance(v, (list, tuple)) else int(v)
    return out


def serialise_plan(plan):
    return {
        "kernel_id": int(plan.kernel_id), "opclass": plan.opclass,
        "operand_table": [int(x) for x in plan.operand_table],
        "writes": [int(x) for x in plan.writes],
        "lanes": [{
            "base_id": int(lane.base_id), "prime": int(lane.prime),
            "ops": [{"opcode": op.opcode, "dst_reg": int(op.dst_reg),
                     "srcs": [[kind, int(i)] for kind, i in op.srcs],
                     "meta": _ser_meta(op.meta),
                     "store_slot": None if op.store_slot is None else int(op.store_slot),
                     "reduce_after": bool(op.reduce_after)} for op in lane.ops]}
            for lane in plan.lanes],
    }


def input_rows(params, dag, seed):
    """(lvid -> uint64 row) in dag.inputs order; shared with the tests (same draw order)."""
    from limbforge.poly import prime_for_id
    rng = np.random.default_rng(seed)
    rows = {}
    for _, lvid in dag.inputs.items():
        q = prime_for_id(params, dag.values[lvid].base_id)
        rows[lvid] = rng.integers(0, q, params.N, dtype=np.uint64)
    return rows


def digest(row) -> str:
    return hashlib.sha256(np.ascontiguousarray(row, dtype="<u8").tobytes()).hexdigest()[:16]


def make_dag(name, params, dag, seed):
    from limbforge.codegen import CompilerConfig, KernelRunner, plan_kernels
    from limbforge.fusion import fuse_dag
    plans = plan_kernels(fuse_dag(dag), dag, params, CompilerConfig())
    return _execute(name, params, dag, plans, seed, KernelRunner)


def synth_dag(params):
    """Every elementwise opcode on two lanes (bases 0 and 1), incl. Sub / Neg / ModStep /
    ScalarMul / Automorph, which the compiled workloads above do not all reach."""
    from limbforge.limbir import (CAT_INPUT, OP_ADD, OP_AUTOMORPH, OP_MODSTEP, OP_MUL, OP_MULACC,
                                  OP_NEG, OP_SCALARMUL, OP_SUB, LimbDag)
    dag = LimbDag(params, "synth")
    outs = {}
    for base in (0, 1):
        x = [dag.input_value(("ct", f"x{i}", "b", base), base, CAT_INPUT) for i in range(4)]

        def op(code, srcs, meta=None):
            d = dag.new_value(base)
            dag.emit(code, base, d, srcs, meta)
            return d
        s1 = op(OP_SUB, (x[0], x[1]))
        n1 = op(OP_NEG, (s1,))
        m1 = op(OP_MUL, (n1, x[2]))
        a1 = op(OP_MULACC, (m1, x[3], x[0]))
        c1 = op(OP_SCALARMUL, (a1,), {"scalar": 123456789})
        ms = op(OP_MODSTEP, (c1, x[1]), {"scalar": 987654321})
        au = op(OP_AUTOMORPH, (ms,), {"galois": 5})
        outs[base] = op(OP_ADD, (au, x[2]))
    dag.outputs["out"] = {"ids": (0, 1), "b": [outs[0], outs[1]], "a": [outs[0], outs[1]],
                          "level": 1, "scale": 1}
    return dag


def make(name, params, text, seed):
    from limbforge.codegen import CompilerConfig, KernelRunner, plan_kernels
    from limbforge.fusion import fuse_dag
    from limbforge.limbir import lower_to_limb_ir
    from limbforge.parser import parse_program
    from limbforge.polyir import hoist_rotations, lower_to_poly_ir, merge_mod_down
    from limbforge.typecheck import typecheck

    typed = typecheck(parse_program(text), params)
    ir = lower_to_poly_ir(typed)
    seg = ir.steps[0]
    hoist_rotations(seg)
    merge_mod_down(seg)
    dag = lower_to_limb_ir(seg, {n: d.category for n, d in typed.program.plaintexts.items()})
    plans = plan_kernels(fuse_dag(dag), dag, params, CompilerConfig())
    return _execute(name, params, dag, plans, seed, KernelRunner)


def _execute(name, params, dag, plans, seed, KernelRunner):
    store = input_rows(params, dag, seed)
    in_digest = hashlib.sha256(b"".join(store[l].astype("<u8").tobytes()
                                        for l in store)).hexdigest()[:16]
    runner = KernelRunner(params)

    def read(lvid):
        return store[lvid]

    def write(lvid):
        if lvid not in store:
            store[lvid] = np.empty(params.N, dtype=np.uint64)
        return store[lvid]

    written = []
    for plan in plans:
        runner.run(plan, read, write)
        written.extend(plan.operand_table[w] for w in plan.writes)
    out = {
        "name": name,
        "params": {"N": params.N, "num_levels": params.max_level, "d": params.ks.d
                   if hasattr(params, "ks") else None},
        "seed": seed,
        "inputs": [[int(lvid), int(dag.values[lvid].base_id)] for _, lvid in dag.inputs.items()],
        "inputs_digest": in_digest,
        "plans": [serialise_plan(p) for p in plans],
        "written": {str(int(l)): digest(store[l]) for l in dict.fromkeys(written)},
        "opcodes": sorted({op.opcode for p in plans for lane in p.lanes for op in lane.ops}),
    }
    return out


def make_program(name, params, text, seed):
    """Every compiled segment of every function of a program (pipeline.compile_source), each
    with its own inputs, plans and written-row digests."""
    from limbforge.codegen import KernelRunner
    from limbforge.pipeline import compile_source
    comp = compile_source(text, params)
    segs = []
    for fname in sorted(comp.functions):
        for k, st in enumerate(comp.functions[fname].steps):
            if not hasattr(st, "schedule"):
                continue                                   # CallStep
            sub = _execute(f"{name}:{fname}:{k}", params, st.dag, st.schedule.plans,
                           seed + len(segs), KernelRunner)
            segs.append(sub)
    return {"name": name, "segments": segs,
            "opcodes": sorted({o for sg in segs for o in sg["opcodes"]})}


def main():
    sys.path.insert(0, "/root/reference/pkg/src")
    from limbforge.bench import bsgs64
    from limbforge.params import gen_params

    p = gen_params(256, 4, d=3, seed=3)
    bench = bsgs64(p, dim=16)
    fx = make("bsgs16_n256", p, bench.text, seed=1234)
    fx["gen_params"] = {"N": 256, "num_levels": 4, "d": 3, "seed": 3}
    from limbforge.bench import polyeval
    fx2 = make("polyeval7_n256", p, polyeval(p, degree=7).text, seed=4321)
    fx2["gen_params"] = fx["gen_params"]
    fx3 = make_dag("synth_allops_n256", p, synth_dag(p), seed=99)
    fx3["gen_params"] = fx["gen_params"]
    from limbforge.bench import tinylayer
    p10 = gen_params(256, 10, d=3, seed=3)
    fx4 = make_program("tinylayer_n256", p10, tinylayer(p10).text, seed=555)
    fx4["gen_params"] = {"N": 256, "num_levels": 10, "d": 3, "seed": 3}
    with open(os.path.join(HERE, "kernel_plans_tinylayer.json"), "w") as f:
        json.dump(fx4, f)
    print(fx4["name"], len(fx4["segments"]), "segments,", sum(len(sg["plans"]) for sg in fx4["segments"]),
          "plans,", sum(len(sg["written"]) for sg in fx4["segments"]), "rows written; opcodes", fx4["opcodes"])
    for fname, f_ in (("kernel_plans_bsgs16.json", fx), ("kernel_plans_polyeval7.json", fx2),
                      ("kernel_plans_synth.json", fx3)):
        with open(os.path.join(HERE, fname), "w") as f:
            json.dump(f_, f)
        print(f_["name"], len(f_["plans"]), "plans,", sum(len(pl["lanes"]) for pl in f_["plans"]),
              "lanes,", len(f_["written"]), "rows written; opcodes", f_["opcodes"])


if __name__ == "__main__":
    main()
