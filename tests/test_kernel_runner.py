"""KernelRunner boundary (reference codegen.py:346-443).

The fixtures hold kernel plans the reference compiler produced for three compiled programs at
N=256 (a BSGS mat-vec — the rotate-and-sum of BASELINE config 4; a degree-7 polynomial — the
polynomial activation; and the reference's `tinylayer` — mat-vec, GELU polynomial, mat-vec, the
transformer-block shape of config 5) and a synthetic plan covering every limb opcode, plus the
digests of every row the reference KernelRunner wrote
(tests/golden/make_kernel_plans.py).  CPU: the oracle restatement reproduces them.  GPU: the
B200 runner (`paper_2512_11269_b200.kernel_runner`) reproduces them with device-resident rows
and with the reference's host-row callbacks.
"""

import hashlib
import json
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")
FIXTURES = ["kernel_plans_bsgs16.json", "kernel_plans_polyeval7.json", "kernel_plans_synth.json",
            "kernel_plans_tinylayer.json"]


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _segments(fx):
    """A fixture is one compiled segment, or a program with several (tinylayer: matvec, GELU
    polynomial, matvec across three functions)."""
    for sg in fx.get("segments", [fx]):
        yield dict(sg, gen_params=fx["gen_params"])


def _digest(row) -> str:
    return hashlib.sha256(np.ascontiguousarray(row, dtype="<u8").tobytes()).hexdigest()[:16]


def _inputs(fx, prime_of):
    rng = np.random.default_rng(fx["seed"])
    rows = {}
    for lvid, base in fx["inputs"]:
        rows[lvid] = rng.integers(0, prime_of(base), fx["gen_params"]["N"], dtype=np.uint64)
    h = hashlib.sha256(b"".join(rows[l].astype("<u8").tobytes() for l in rows)).hexdigest()[:16]
    assert h == fx["inputs_digest"], "input RNG stream differs from the fixture's"
    return rows


def _host_store(fx, rows, N):
    store = dict(rows)

    def read(lvid):
        return store[lvid]

    def write(lvid):
        if lvid not in store:
            store[lvid] = np.empty(N, dtype=np.uint64)
        return store[lvid]
    return store, read, write


def _check(fx, get_row):
    bad = [l for l, d in fx["written"].items() if _digest(get_row(int(l))) != d]
    assert not bad, f"{len(bad)} of {len(fx['written'])} written rows differ, e.g. lvid {bad[:5]}"


@pytest.mark.parametrize("name", FIXTURES)
def test_oracle_runner_matches_reference(name):
    from oracle import lf_oracle as O
    from oracle.kernel_runner import KernelRunner, plan_from_json
    fx0 = _load(name)
    P = O.gen_params(**fx0["gen_params"])
    runner = KernelRunner(P)
    for fx in _segments(fx0):
        rows = _inputs(fx, P.prime)
        store, read, write = _host_store(fx, rows, P.N)
        for pl in fx["plans"]:
            runner.run(plan_from_json(pl), read, write)
        _check(fx, lambda l: store[l])
    fx = fx0
    assert set(fx["opcodes"]) <= {"Add", "Sub", "Mul", "MulAcc", "Neg", "ScalarMul", "ModStep",
                                  "Automorph", "NTT", "INTT", "BConv"}


def test_fixtures_cover_every_limb_opcode():
    ops = set()
    for name in FIXTURES:
        ops |= set(_load(name)["opcodes"])
    # limbir.py:46-56: the 11 limb opcodes
    assert ops == {"Add", "Sub", "Mul", "MulAcc", "Neg", "ScalarMul", "ModStep", "Automorph",
                   "NTT", "INTT", "BConv"}


@pytest.mark.gpu
@pytest.mark.parametrize("name", FIXTURES)
@pytest.mark.parametrize("mode", ["device", "host"])
def test_gpu_runner_matches_reference(name, mode):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2512_11269_b200 as B
    from paper_2512_11269_b200.kernel_runner import KernelRunner, plan_from_json
    fx0 = _load(name)
    p = B.gen_params(**fx0["gen_params"])
    from paper_2512_11269_b200.poly import prime_for_id
    runner = KernelRunner(p)
    for fx in _segments(fx0):
        _gpu_segment(fx, p, runner, mode, lambda b: prime_for_id(p, b))


def _gpu_segment(fx, p, runner, mode, prime_of):
    import torch
    from paper_2512_11269_b200.kernel_runner import plan_from_json
    rows = _inputs(fx, prime_of)
    plans = [plan_from_json(pl) for pl in fx["plans"]]
    if mode == "host":                  # the reference Executor's callbacks: uint64 host rows
        store, read, write = _host_store(fx, rows, p.N)
        for pl in plans:
            runner.run(pl, read, write)
        _check(fx, lambda l: store[l])
    else:                               # device-resident rows (int32 residues in HBM)
        dev = {l: torch.from_numpy(r.astype(np.int64)).to(torch.int32).cuda() for l, r in rows.items()}

        def read(lvid):
            return dev[lvid]

        def write(lvid):
            if lvid not in dev:
                dev[lvid] = torch.empty(p.N, dtype=torch.int32, device="cuda")
            return dev[lvid]
        for pl in plans:
            runner.run(pl, read, write)
        torch.cuda.synchronize()
        _check(fx, lambda l: dev[l].cpu().numpy().view(np.uint32).astype(np.uint64))
