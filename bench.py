"""Benchmark: full-level hybrid keyswitch throughput at N=2^16 (BASELINE config 2 / SURVEY
§8(d) C2: gen_params(65536, 35, d=4, seed=0, scale=2^26) -> 36 main + 9 special primes,
4 digits, ext = 45 rows).

One step = one batch of B independent full-level keyswitches (relinearisation of B
ciphertexts, one shared relinearisation key), inputs resident in HBM.  `value` is keyswitch
ops/s over the whole job (all ranks); `e2e` is the same metric through the public operator
API (`paper_2512_11269_b200.keyswitch`) with the inputs copied from pinned host memory and
the results copied back inside the timed region.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl ours|reference]

`--impl reference` times the reference itself on the host CPU cores instead: the unmodified
`limbforge.ckks.keyswitch` (installed into baseline/_ref, which travels to the GPU box), one
worker process per core; if baseline/_ref is missing it falls back to the CPU oracle
`oracle/lf_oracle.py` (a restatement of the same function) and says so (`kind: "port"`).
"""

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np
from fractions import Fraction

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

C2 = dict(N=65536, num_levels=35, d=4, seed=0, scale=2 ** 26)
ROW_BYTES = 65536 * 4
METRIC = "keyswitch ops/s"
STAGES = ["modup_in", "modup_bconv", "ks_inner", "moddown_bconv", "moddown_out"]
TRAFFIC_JSON = "r02_ncu_traffic.json"     # tools/ncu_traffic.py over a capture of this tree


def algorithmic_rows(level=35, d=4, alpha=9):
    """keyswitch(x) = (l+1) + 2*beta*ext + 2(l+1) rows of N uint32 words."""
    l1 = level + 1
    beta = min(d, l1)
    ext = l1 + alpha
    return l1 + 2 * beta * ext + 2 * l1


def key_rows(level=35, d=4, alpha=9):
    """Evaluation-key rows one keyswitch reads: 2*beta*ext (shared by a relinearisation batch)."""
    l1 = level + 1
    return 2 * min(d, l1) * (l1 + alpha)


SHOUP_MAC_PER_CLK_SM = 18.4   # profiles/r01_ubench_imad.log: one Shoup modular MAC per lane
LINE_BFLY_PER_CLK_SM = 12.1   # profiles/r02_experiments.md: 256-point line code, data on chip


def stage_butterflies(level=35, d=4, alpha=9):
    """NTT butterflies each fused kernel runs per keyswitch (N/2 per stage, 8 stages per pass)."""
    l1 = level + 1
    beta = min(d, l1)
    ext = l1 + alpha
    conv = beta * ext - l1
    per_pass = 65536 // 2 * 8
    return {"modup_in": l1 * per_pass, "modup_bconv": (l1 + conv) * per_pass,
            "ks_inner": (conv + 2 * alpha) * per_pass, "moddown_bconv": (2 * alpha + 2 * l1) * per_pass,
            "moddown_out": 2 * l1 * per_pass}


def stage_rows(level=35, d=4, alpha=9):
    """Algorithmic rows read+written by each fused kernel ('Kernels'), per
    keyswitch, the evaluation key charged per keyswitch (SURVEY §8d's definition)."""
    l1 = level + 1
    beta = min(d, l1)
    ext = l1 + alpha
    conv_rows = beta * ext - l1          # piece rows produced by base conversion
    return {
        "modup_in": l1 + l1,                                   # x in, T0 out
        "modup_bconv": l1 + conv_rows,                         # T0 in, T1 out
        "ks_inner": conv_rows + l1 + 2 * beta * ext + 2 * l1 + 2 * alpha,   # T1, x, keys in; acc, T2 out
        "moddown_bconv": 2 * alpha + 2 * l1,                   # T2 in, T3 out
        "moddown_out": 2 * l1 + 2 * l1 + 2 * l1,               # T3, acc in; out
    }


# ----------------------------------------------------------------------------------------
class ClockSampler:
    """NVML sampling of SM clock and clock-event (throttle) reasons during the timed region."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, torch_device_index, period_s=0.001):
        import threading
        self.period = period_s
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        self._thread = None
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            self.nv = pynvml
            props = torch.cuda.get_device_properties(torch_device_index)
            try:
                bus = f"{props.pci_domain_id:08x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
                self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(torch_device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self._thread = threading.Thread(target=self._run, daemon=True)
        except Exception:
            self.nv = None

    def _sample(self):
        nv = self.nv
        self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
        try:
            self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            self.reasons |= nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                pass
            time.sleep(self.period)

    def start(self):
        if self._thread:
            self._thread.start()
        return self

    def stop(self):
        if not self._thread:
            return None
        self._stop.set()
        self._thread.join()
        if not self.samples:
            try:
                self._sample()
            except Exception:
                return None
        names = sorted(n for n, bit in self.REASONS.items() if self.reasons & bit)
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples)}


# ----------------------------------------------------------------------------------------
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_module():
    """The unmodified reference package from baseline/_ref, or None when it is not installed."""
    if not os.path.isdir(os.path.join(REF_DIR, "limbforge")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import limbforge.ckks  # noqa: F401
        import limbforge.keys  # noqa: F401
        import limbforge.params  # noqa: F401
        import limbforge.poly  # noqa: F401
        import limbforge
        return limbforge
    except Exception:
        return None


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def _reference_setup(lf, level=35):
    """C2 parameters, a relinearisation-shaped key with uniform rows (keyswitch cost is
    data-independent) and warm NTT tables, all through the reference's own types."""
    from limbforge.keys import EvalKey
    from limbforge.ntt import ntt_tables
    from limbforge.poly import Domain, RnsPolynomial, extended_ids, main_ids, prime_for_id
    P = lf.params.gen_params(**C2)
    ext = extended_ids(P, P.max_level)
    rng = np.random.default_rng(7)

    def rows(ids, r):
        return np.stack([r.integers(0, prime_for_id(P, b), P.N, dtype=np.uint64) for b in ids])
    evk = EvalKey("relin", tuple((RnsPolynomial(rows(ext, rng), Domain.EVAL, ext),
                                  RnsPolynomial(rows(ext, rng), Domain.EVAL, ext)) for _ in range(P.ks.d)))
    for b in ext:
        ntt_tables(P.N, prime_for_id(P, b))
    ids = main_ids(level)
    mk = lambda seed: RnsPolynomial(rows(ids, np.random.default_rng(seed)), Domain.EVAL, ids)
    return P, evk, mk


def cpu_reference_keyswitch_sample(n_ops=2, level=35):
    """Time the reference's own limbforge.ckks.keyswitch on one core (bounded sample)."""
    lf = reference_module()
    if lf is None:
        return None
    P, evk, mk = _reference_setup(lf, level)
    xs = [mk(1000 + i) for i in range(n_ops)]
    t0 = time.perf_counter()
    for x in xs:
        lf.ckks.keyswitch(x, evk, P)
    dt = time.perf_counter() - t0
    return n_ops / dt, dt


def cpu_oracle_keyswitch_sample(n_ops=2, level=35):
    """Time the CPU oracle (restatement of limbforge ckks.keyswitch) on a bounded sample."""
    from oracle import lf_oracle as O
    P = O.gen_params(**C2)
    ext = P.ext_ids(P.L)
    rng = np.random.default_rng(7)
    evk = O.EvalKeyO("relin", [(O.sample_uniform(P, rng, ext), O.sample_uniform(P, rng, ext))
                               for _ in range(P.d)])
    ids = P.main_ids(level)
    xs = [O.sample_uniform(P, np.random.default_rng(1000 + i), ids) for i in range(n_ops)]
    O.twiddles(P.N, P.main[0])  # table build is setup, not timed
    for q in P.main + P.special:
        O.twiddles(P.N, q)
    t0 = time.perf_counter()
    for x in xs:
        O.keyswitch(P, x, evk)
    dt = time.perf_counter() - t0
    return n_ops / dt, dt


_REF_STATE = {}


def _ref_worker_init():
    lf = reference_module()
    if lf is not None:
        P, evk, mk = _reference_setup(lf)
        _REF_STATE.update(kind="reference", run=lambda seed: lf.ckks.keyswitch(mk(seed), evk, P))
        return
    from oracle import lf_oracle as O
    P = O.gen_params(**C2)
    ext = P.ext_ids(P.L)
    rng = np.random.default_rng(7)
    evk = O.EvalKeyO("relin", [(O.sample_uniform(P, rng, ext), O.sample_uniform(P, rng, ext))
                               for _ in range(P.d)])
    for q in P.main + P.special:
        O.twiddles(P.N, q)
    _REF_STATE.update(kind="port", run=lambda seed: O.keyswitch(
        P, O.sample_uniform(P, np.random.default_rng(seed), P.main_ids(P.L)), evk))


def _ref_worker_ks(seed):
    t0 = time.perf_counter()
    _REF_STATE["run"](seed)
    return time.perf_counter() - t0


def run_reference(args, rank, world):
    """--impl reference: the reference's own limbforge.ckks.keyswitch (baseline/_ref) on all
    host cores (the oracle port if the reference is not installed).  The key and twiddle tables
    are built once in the parent and shared copy-on-write with the workers."""
    if rank != 0:
        return
    import multiprocessing as mp
    cores = min(os.cpu_count() or 1, 64)
    _ref_worker_init()
    kind = _REF_STATE["kind"]
    what = "limbforge.ckks.keyswitch (baseline/_ref)" if kind == "reference" else "oracle/lf_oracle.py"
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        for w in range(args.warmup):
            pool.map(_ref_worker_ks, range(cores))
        t0 = time.perf_counter()
        for k in range(args.steps):
            pool.map(_ref_worker_ks, [10_000 + k * cores + i for i in range(cores)])
        dt = time.perf_counter() - t0
    ops = args.steps * cores
    value = ops / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "ops/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": "C2 full-level hybrid keyswitch, N=2^16, L=35, dnum=4, alpha=9",
                   "level": 35, "batch_per_step": cores, "sample": "one keyswitch per core per step"},
        "cpu_baseline": {"value": value, "unit": "ops/s", "cores": cores, "kind": kind,
                         "cpu_model": cpu_model(),
                         "sample": f"{ops} C2 keyswitches, {cores} worker processes ({what})"},
        "e2e": {"value": value, "unit": "ops/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------------------
C3 = dict(N=65536, num_levels=47, d=4, seed=0, scale=2 ** 26)


def bootstrap_latency(reps=5):
    """C3 variant ("Same p as C2 or a builder-tuned variant"): N=2^16, 48 main +
    12 special primes, d=4, h=64.  Full-slot (n=2^15) bootstrap of a level-0 encryption of
    uniform(-1,1) slots (seed 77), captured once as a CUDA graph (bootstrap.GraphedBootstrap)
    and replayed; latency = CUDA events around the call (input copy into the captured buffers,
    replay, output copy; keys and plaintext diagonals are resident).  Precision:
    max |decrypt(out) - decrypt(in)| in bits."""
    import torch
    import paper_2512_11269_b200 as B
    from paper_2512_11269_b200 import bootstrap as BT
    t0 = time.time()
    p = B.gen_params(**C3)
    sk, pk, rlk = B.keygen(p, seed=11)
    cfg = BT.BootConfig()
    planner = BT.Bootstrapper(type("P", (), {"N": p.N, "main_primes": p.rns_basis}), cfg)
    ck, rk = BT.make_bootstrap_keys(p, sk, planner.required_rotations(), seed=99)
    v = np.random.default_rng(77).uniform(-1, 1, p.n)
    ct = B.encrypt(B.encode(v, p, level=0, scale=2 ** 26), pk, p, np.random.default_rng(5))
    bt = BT.Bootstrapper(BT.GpuBackend(p, rlk, ck, rk), cfg)
    out = bt.bootstrap(ct)                   # encodes and caches the plaintext diagonals
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    bt.bootstrap(ct)
    e1.record()
    torch.cuda.synchronize()
    eager_ms = e0.elapsed_time(e1)
    graphed = BT.GraphedBootstrap(bt, ct)                 # public API: capture once, replay
    ms = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        gout = graphed(ct)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    assert np.array_equal(gout.b.numpy(), out.b.numpy()), "graph replay differs from eager"
    din, dout = B.decrypt(ct, sk, p), B.decrypt(gout, sk, p)
    err = float(np.abs(dout - din).max())
    err_v = float(np.abs(dout - v).max())
    return {"ms": statistics.median(ms), "ms_eager": eager_ms, "reps": reps,
            "params": "gen_params(65536, 47, d=4, scale=2^26), h=64, full slots n=2^15",
            "levels": f"in 0 -> out {gout.level} (L=47)", "precision_bits": -np.log2(err),
            "max_err_vs_plain": err_v, "rotation_keys": len(rk) + 1,
            "paper_1xB200_ms": 14.5, "setup_s": time.time() - t0}


def _graph_latency(be, fn, ct, reps):
    """Eager latency of fn(ct) and its CUDA-graph replay latency (median of reps), CUDA events
    on the launch stream; the replay must equal the eager output residue for residue."""
    import torch
    from paper_2512_11269_b200 import bootstrap as BT
    out = fn(ct)                                          # encodes and caches the plaintexts
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn(ct)
    e1.record()
    torch.cuda.synchronize()
    eager_ms = e0.elapsed_time(e1)
    g = BT.GraphedCircuit(be, fn, ct)
    ms = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        gout = g(ct)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    assert np.array_equal(gout.b.numpy(), out.b.numpy()), "graph replay differs from eager"
    return out, eager_ms, statistics.median(ms)


def _workload_env(kw, rotations):
    import paper_2512_11269_b200 as B
    from paper_2512_11269_b200 import bootstrap as BT
    p = B.gen_params(**kw)
    sk, pk, rlk = B.keygen(p, seed=11)
    ck, rk = BT.make_bootstrap_keys(p, sk, rotations, seed=99)
    return p, sk, pk, BT.GpuBackend(p, rlk, ck, rk), len(rk)


class _Planner:
    def __init__(self, kw):
        import paper_2512_11269_b200 as B
        self.N = kw["N"]
        self.main_primes = B.gen_params(**kw).rns_basis


C4_SHAPE = (16, 32, 32)          # ResNet-20 stage 1 on CIFAR-10: 16 channels, 32 x 32


def resnet_block_latency(reps=3):
    """C4 (BASELINE config 4): one ResNet-20 basic block relu(conv2(relu(conv1 x)) + x) on a
    16 x 32 x 32 activation (CIFAR-10 stage 1, slots c*1024 + y*32 + x, replicated 2x in
    n = 2^15), conv3x3 as a hoisted BSGS rotate-and-sum over the C*9 = 144 diagonals
    (workloads.ResNetBlock), degree-15 Chebyshev ReLU, at the C3 parameters from level 47.
    Weights default_rng(5) uniform(-1,1)/(9C); CUDA graph replay."""
    import paper_2512_11269_b200 as B
    from paper_2512_11269_b200 import workloads as WL
    t0 = time.time()
    C = C4_SHAPE[0]
    rng = np.random.default_rng(5)
    w1 = rng.uniform(-1, 1, (C, C, 3, 3)) / (9 * C)
    w2 = rng.uniform(-1, 1, (C, C, 3, 3)) / (9 * C)
    rots = WL.ResNetBlock(_Planner(C3), w1, w2, C4_SHAPE).required_rotations()
    p, sk, pk, be, nkeys = _workload_env(C3, rots)
    blk = WL.ResNetBlock(be, w1, w2, C4_SHAPE)
    act = np.random.default_rng(7).uniform(-1, 1, C4_SHAPE) * 0.5
    S = Fraction(p.rns_basis[p.max_level]) * p.rns_basis[p.max_level - 1]
    ct = B.encrypt(B.encode(blk.pack(act), p, level=p.max_level, scale=S), pk, p, np.random.default_rng(5))
    setup = time.time() - t0
    out, eager_ms, ms = _graph_latency(be, blk.forward, ct, reps)
    got = B.decrypt(out, sk, p)[: act.size].real
    err_model = float(np.abs(got - blk.plain(blk.pack(act))[: act.size]).max())
    err_true = float(np.abs(got - blk.reference(act).reshape(-1)).max())
    return {"ms": ms, "ms_eager": eager_ms, "reps": reps,
            "workload": "ResNet-20 basic block, 16x32x32 activation, two conv3x3 (144 diagonals, "
                        "BSGS 9 baby x 17 giant, hoisted) + two degree-15 Chebyshev ReLU + shortcut",
            "params": "gen_params(65536, 47, d=4, scale=2^26), h=64", "levels": f"47 -> {out.level}",
            "rotation_keys": nkeys, "max_err_vs_slot_model": err_model, "max_err_vs_network": err_true,
            "paper_context": "full ResNet-20 (9 blocks + bootstraps) 456 ms on 1xB200 (PAPER.md:688)",
            "setup_s": setup}


C5 = dict(N=65536, num_levels=52, d=4, seed=0, scale=2 ** 26)
C5_SHAPE = (128, 64)             # BERT-Base: 128 tokens, head dimension 64


def transformer_block_latency(reps=2):
    """C5 (BASELINE config 5): one single-head transformer block over T = 128 tokens x d = 64
    features (BERT-Base sequence length and head dimension; rows packed row-major, replicated
    4x): Q/K/V/O and two FFN projections as BSGS mat-vecs of I_T (x) W (127 diagonals), scores
    for all 128 offsets as ciphertext products + rotate-and-sum, softmax as Chebyshev exp and
    1/x, GELU as the reference's least-squares fit (workloads.TransformerBlock), at
    gen_params(65536, 52, d=4) from level 52 (the block uses 50 levels).  Weights
    default_rng(5) uniform(-1,1)/d; one GPU, CUDA graph replay."""
    import paper_2512_11269_b200 as B
    from paper_2512_11269_b200 import workloads as WL
    t0 = time.time()
    T, d = C5_SHAPE
    rng = np.random.default_rng(5)
    Ws = [rng.uniform(-1, 1, (d, d)) / d for _ in range(6)]
    kw = dict(T=T, d=d, score_bound=1.0, gelu_bound=2.0)
    rots = WL.TransformerBlock(_Planner(C5), *Ws, **kw).required_rotations()
    p, sk, pk, be, nkeys = _workload_env(C5, rots)
    blk = WL.TransformerBlock(be, *Ws, **kw)
    X = np.random.default_rng(8).uniform(-1, 1, (T, d)) * 0.5
    S = Fraction(p.rns_basis[p.max_level]) * p.rns_basis[p.max_level - 1]
    ct = B.encrypt(B.encode(blk.pack(X), p, level=p.max_level, scale=S), pk, p, np.random.default_rng(6))
    setup = time.time() - t0
    out, eager_ms, ms = _graph_latency(be, blk.forward, ct, reps)
    got = B.decrypt(out, sk, p)[: T * d].real.reshape(T, d)
    err = float(np.abs(got - blk.reference(X)).max())
    del blk
    sharded = shard_mul_emulation(p, 48, be.rlk)
    key_gb = nkeys * 2 * p.ks.d * (p.max_level + 1 + p.num_special) * p.N * 4 / 1e9
    return {"ms": ms, "ms_eager": eager_ms, "reps": reps,
            "workload": "single-head transformer block, 128 tokens x 64 features: 6 BSGS projections, "
                        "128-offset attention scores, Chebyshev exp + 1/x softmax, GELU lsq fit",
            "params": "gen_params(65536, 52, d=4, scale=2^26), h=64", "levels": f"52 -> {out.level}",
            "rotation_keys": nkeys, "key_gb_per_gpu_1": key_gb,
            "key_gb_per_gpu_sharded_8": key_gb / 8,
            "max_err_vs_float_block": err,
            "sharded_products_emulated": sharded,
            "paper_context": "full BERT-Base (12 layers x 12 heads, 768 hidden) 28.3 s on 1xB200 (PAPER.md:695)",
            "setup_s": setup}


def ntt_throughput(params, dev, rows=720, reps=10):
    """Standalone batched negacyclic NTT / INTT at N=2^16 over C2 primes ("integer-pipe
    utilisation for the NTT").  720 rows (189 MB) > L2, so both passes stream from HBM.
    Integer-pipe fraction: one Shoup IMAD.HI per butterfly and IMAD.HI issues at 32/clk/SM on
    B200 (tools/ubench/imad.cu, profiles/r01_ubench_imad.log)."""
    import torch
    from paper_2512_11269_b200 import poly as P
    ids = [i % (params.max_level + 1) for i in range(rows)]
    q = torch.tensor([params.rns_basis[i] for i in ids], dtype=torch.int64, device=dev)[:, None]
    g = torch.Generator(device=dev).manual_seed(5)
    x = (torch.randint(0, 2 ** 62, (rows, params.N), device=dev, generator=g, dtype=torch.int64) % q).to(torch.int32)
    for _ in range(2):
        P.ntt_rows(params, x, ids)
        P.ntt_rows(params, x, ids, inverse=True)
    torch.cuda.synchronize()
    out = {}
    bfly = rows * (params.N // 2) * (params.N.bit_length() - 1)
    for name, inv in (("fwd", False), ("inv", True)):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            P.ntt_rows(params, x, ids, inverse=inv)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        out[name] = {"us": ms * 1e3, "butterflies_per_s": bfly / (ms * 1e-3),
                     "hbm_gbs_two_passes": 4 * rows * params.N * 4 / (ms * 1e-3) / 1e9}
    return out


def batch_sweep(params, level, rlk, dev, batches=(1, 8), steps=5):
    """Per-keyswitch time at other batch sizes of SURVEY §8d C2 (B in {1, 8, 32}): same
    synthetic inputs, L2 flushed between steps, CUDA events."""
    import torch
    from paper_2512_11269_b200 import fused
    from paper_2512_11269_b200.context import get_context
    ctx = get_context(params)
    l1 = level + 1
    q = torch.tensor(params.rns_basis[:l1], dtype=torch.int64, device=dev)[:, None]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)
    out = {}
    for B in batches:
        g = torch.Generator(device=dev).manual_seed(77 + B)
        x = (torch.randint(0, 2 ** 62, (B, l1, params.N), device=dev, generator=g, dtype=torch.int64) % q).to(torch.int32)
        o = torch.empty((B, 2, l1, params.N), dtype=torch.int32, device=dev)
        ws = ctx.ks_workspace(level, B)
        for _ in range(2):
            fused.keyswitch_batch(params, level, x, rlk, out=o, ws=ws)
        ms = 0.0
        for i in range(steps):
            flush.fill_(i)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fused.keyswitch_batch(params, level, x, rlk, out=o, ws=ws)
            b.record()
            torch.cuda.synchronize()
            ms += a.elapsed_time(b)
        rec = {"keyswitch_us": ms / steps / B * 1e3}
        if B == 1:
            # latency of one keyswitch replayed from a CUDA graph (no host launch gaps)
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                fused.keyswitch_batch(params, level, x, rlk, out=o, ws=ws)
            torch.cuda.current_stream().wait_stream(side)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                fused.keyswitch_batch(params, level, x, rlk, out=o, ws=ws)
            gms = []
            for i in range(steps):
                flush.fill_(i)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                graph.replay()
                b.record()
                torch.cuda.synchronize()
                gms.append(a.elapsed_time(b))
            rec["keyswitch_us_graph"] = statistics.median(gms) * 1e3
            del graph
        out[str(B)] = rec
        del x, o, ws
    return out


def rotation_units(params, level, dev, steps=5):
    """The other C2 units of SURVEY §8d: one hom_rotate (lf_rotate, batch 1), 32 independent
    rotations in one pipeline (lf_rotate_batch, keys cycling over steps 1..8) and a hoisted
    batch of 8 rotations of one ciphertext sharing one ModUp (lf_rotate_hoisted, full
    semantics incl. ModDown).  Keys and ciphertexts are synthetic uniform rows (cost is
    data-independent); L2 flushed between timed runs; CUDA events."""
    import torch
    from types import SimpleNamespace
    from paper_2512_11269_b200 import fused
    from paper_2512_11269_b200.ntt_host import galois_element
    l1, N = level + 1, params.N
    alpha, d = params.num_special, params.ks.d
    R = params.max_level + 1 + alpha
    primes = list(params.rns_basis) + list(params.special_basis)
    g = torch.Generator(device=dev).manual_seed(4242)

    def rows(idx, lead=()):
        q = torch.tensor([primes[i] for i in idx], dtype=torch.int64, device=dev)[:, None]
        r = torch.randint(0, 2 ** 62, (*lead, len(idx), N), device=dev, generator=g, dtype=torch.int64)
        return (r % q).to(torch.int32)
    kidx = list(range(params.max_level + 1)) + list(range(params.max_level + 1, params.max_level + 1 + alpha))
    keys = [SimpleNamespace(data=rows(kidx, (d, 2)).contiguous()) for _ in range(8)]
    gs = [galois_element(N, s) for s in range(1, 9)]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)

    def ct_of(t):
        return SimpleNamespace(b=SimpleNamespace(limbs=t[0]), a=SimpleNamespace(limbs=t[1]), level=level)

    def timed(fn):
        fn()
        fn()
        ms = 0.0
        for i in range(steps):
            flush.fill_(i)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ms += a.elapsed_time(b)
        return ms / steps
    ct1 = rows(list(range(l1)) * 2).view(2, l1, N)
    one = timed(lambda: fused.rotate(params, ct_of(ct1), gs[0], keys[0]))
    cts = rows(list(range(l1)) * 2, (32,)).view(32, 2, l1, N)
    b32 = timed(lambda: fused.rotate_batch(params, level, cts, [gs[i % 8] for i in range(32)],
                                           [keys[i % 8] for i in range(32)]))
    h8 = timed(lambda: fused.rotate_hoisted(params, ct_of(ct1), gs, keys))
    beta = min(d, l1)
    ext = l1 + alpha
    h8_bytes = (2 * l1 + 8 * (2 * beta * ext + 2 * l1)) * N * 4
    rot_bytes = (4 * l1 + 2 * beta * ext) * N * 4
    return {"hom_rotate_us": one * 1e3, "rotate_batch32_us_per_op": b32 / 32 * 1e3,
            "hoisted8_us": h8 * 1e3, "hoisted8_us_per_rotation": h8 / 8 * 1e3,
            "hoisted8_algorithmic_bytes": h8_bytes,
            "hoisted8_hbm_gbs": h8_bytes / (h8 / 1e3) / 1e9,
            "rotate_algorithmic_bytes": rot_bytes,
            "keys": "synthetic uniform rows (8 rotation keys, steps 1..8)"}


def secondary_keyswitch(dev, B=32, steps=5):
    """SURVEY §8d secondary C2: gen_params(65536, 24, d=3) (25 + 9 primes, ext 34), full-level
    keyswitch at batch B; synthetic inputs and key rows (cost is data-independent)."""
    import torch
    from types import SimpleNamespace
    import paper_2512_11269_b200 as Bk
    from paper_2512_11269_b200 import fused
    from paper_2512_11269_b200.context import get_context
    p = Bk.gen_params(65536, 24, d=3, seed=0, scale=2 ** 26)
    level, N = p.max_level, p.N
    l1, alpha, d = level + 1, p.num_special, p.ks.d
    primes = list(p.rns_basis) + list(p.special_basis)
    g = torch.Generator(device=dev).manual_seed(99)

    def rows(idx, lead=()):
        q = torch.tensor([primes[i] for i in idx], dtype=torch.int64, device=dev)[:, None]
        r = torch.randint(0, 2 ** 62, (*lead, len(idx), N), device=dev, generator=g, dtype=torch.int64)
        return (r % q).to(torch.int32)
    key = SimpleNamespace(data=rows(list(range(l1 + alpha)), (d, 2)).contiguous())
    x = rows(list(range(l1)), (B,))
    out = torch.empty((B, 2, l1, N), dtype=torch.int32, device=dev)
    ws = get_context(p).ks_workspace(level, B)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)
    for _ in range(2):
        fused.keyswitch_batch(p, level, x, key, out=out, ws=ws)
    ms = 0.0
    for i in range(steps):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fused.keyswitch_batch(p, level, x, key, out=out, ws=ws)
        b.record()
        torch.cuda.synchronize()
        ms += a.elapsed_time(b)
    us = ms / steps / B * 1e3
    rows_alg = l1 + 2 * min(d, l1) * (l1 + alpha) + 2 * l1
    return {"config": "gen_params(65536, 24, d=3): 25 main + 9 special, ext 34", "batch": B,
            "keyswitch_us": us, "ops_per_s": 1e6 / us, "algorithmic_bytes": rows_alg * N * 4,
            "hbm_gbs": rows_alg * N * 4 / (us * 1e-6) / 1e9}


def shard_mul_emulation(params, level, rlk, batch=64, ks=(1, 2, 4, 8), reps=2):
    """The C5 block's dominant operation on the limb-sharded path: a batch of `batch`
    relinearised products (half the 128 score offsets) at the block's parameters, each rank's share
    of the fused pipeline run rank by rank on one GPU (k = 1: the unsharded pipeline through
    the same engine).  Per-rank device time, max over ranks; NVLink gathers not timed."""
    import torch
    from paper_2512_11269_b200.shard import ShardEngine
    l1, N = level + 1, params.N
    q = torch.tensor(params.rns_basis[:l1], dtype=torch.int64, device="cuda")[:, None]
    g = torch.Generator(device="cuda").manual_seed(11)
    c1 = (torch.randint(0, 2 ** 62, (batch, 2, l1, N), device="cuda", generator=g, dtype=torch.int64) % q).to(torch.int32)
    c2 = (torch.randint(0, 2 ** 62, (batch, 2, l1, N), device="cuda", generator=g, dtype=torch.int64) % q).to(torch.int32)
    out = {}
    for k in ks:
        eng = [ShardEngine(params, k, r) for r in range(k)]
        calls = [e.hom_mul_call(level, e.shard_rows(c1, level), e.shard_rows(c2, level), e.shard_key(rlk))[0]
                 for e in eng]
        per = [0.0] * k
        for it in range(reps + 1):
            for r, (e, c) in enumerate(zip(eng, calls)):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for ph in range(3):
                    e.phase(ph, c, level, batch)
                b.record()
                torch.cuda.synchronize()
                if it:
                    per[r] += a.elapsed_time(b) / reps
        out[str(k)] = {"per_rank_us_per_product": max(per) / batch * 1e3,
                       "key_rows_per_gpu": eng[0].info(params.max_level)["n_key_rows"]}
        del eng, calls
    out["note"] = (f"relinearised products (hom_mul, batches of {batch}: the sharded pipeline's limit) at level "
                   f"{level}, the C5 score products; ranks emulated one by one on one B200, all-gathers not timed")
    return out


def shard_emulation(params, level, rlk, dev, batch=32, ks=(2, 4, 8), reps=3):
    """SURVEY §8e on ONE GPU: the limb-sharded pipeline of k ranks run rank by rank (each rank's
    rows and key rows, the gathers as device copies): per-rank device time of its three phases
    (CUDA events, max over ranks) per keyswitch, next to the single-device pipeline.  The NVLink
    all-gathers are NOT measured here (one GPU); their bytes are reported."""
    import torch
    from paper_2512_11269_b200.shard import ShardEngine
    l1, N = level + 1, params.N
    q = torch.tensor(params.rns_basis[:l1], dtype=torch.int64, device=dev)[:, None]
    g = torch.Generator(device=dev).manual_seed(9)
    xs = (torch.randint(0, 2 ** 62, (batch, l1, N), device=dev, generator=g, dtype=torch.int64) % q).to(torch.int32)
    out = {}
    for k in ks:
        eng = [ShardEngine(params, k, r) for r in range(k)]
        calls = [e.keyswitch_call(level, e.shard_rows(xs, level), e.shard_key(rlk))[0] for e in eng]
        per = [0.0] * k
        for it in range(reps + 1):
            for r, (e, c) in enumerate(zip(eng, calls)):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for ph in range(3):
                    e.phase(ph, c, level, batch)
                b.record()
                torch.cuda.synchronize()
                if it:
                    per[r] += a.elapsed_time(b) / reps
        lay = eng[0].gather_layout(level, batch)
        out[str(k)] = {"per_rank_compute_us_per_keyswitch": max(per) / batch * 1e3,
                       "ranks_us": [x / batch * 1e3 for x in per],
                       "allgather_bytes_per_rank_per_keyswitch": (lay[1] + lay[4]) / batch,
                       "key_rows_per_gpu": eng[0].info(params.max_level)["n_key_rows"]}
        del eng, calls
    out["note"] = "per-rank kernel time of the limb-sharded pipeline, ranks emulated one by one on one B200; gathers not timed"
    return out


def ntt_summary(ntt, clocks):
    mhz = (clocks or {}).get("sm_mhz") or 1965
    peak = 32 * 148 * mhz * 1e6                  # IMAD.HI per second (one per butterfly)
    for v in ntt.values():
        v["imad_hi_frac"] = v["butterflies_per_s"] / peak
    ntt["config"] = "720 rows x 2^16, C2 primes, lf_ntt_fwd / lf_ntt_inv (column + row pass)"
    ntt["int_peak"] = f"32 IMAD.HI/clk/SM x 148 SMs x {mhz} MHz (measured rate, profiles/r01_ubench_imad.log)"
    return ntt


def run_sharded(args, rank, world):
    """N > 1: every C2 keyswitch of the step is LIMB-SHARDED over all ranks
    (main row i and special row j on rank i % k / j % k, multidev.py:55-56); each rank runs
    the fused pipeline on its rows with its rows of the key (1/k of the key resident) and the
    two all-gathers go through the library's own NCCL communicator on the launch stream
    (lf_shard_keyswitch).  The total work per step is fixed (B keyswitches), so `scaling` is
    "strong"; independent per-GPU replicas (weak scaling) are reported beside it."""
    import torch
    import torch.distributed as dist
    import paper_2512_11269_b200 as B
    from paper_2512_11269_b200 import fused
    from paper_2512_11269_b200.context import get_context
    from paper_2512_11269_b200.shard import NcclComm, ShardEngine
    dev = torch.device("cuda", torch.cuda.current_device())
    params = B.gen_params(**C2)
    level, N, Bsz = args.level, params.N, args.batch
    l1 = level + 1
    sk, pk, rlk = B.keygen(params, seed=11)           # same seed on every rank: the same key
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)
    q = torch.tensor(params.rns_basis[:l1], dtype=torch.int64, device=dev)[:, None]
    g = torch.Generator(device=dev).manual_seed(1234)                   # same inputs on every rank
    xs = [((torch.randint(0, 2 ** 62, (Bsz, l1, N), device=dev, generator=g, dtype=torch.int64) % q)
           .to(torch.int32)) for _ in range(3)]

    def timed(fn, steps):
        for i in range(args.warmup):
            fn(i)
        torch.cuda.synchronize()
        dist.barrier()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for i in range(steps):
            flush.fill_(i)
            evs[i][0].record(stream)
            fn(i)
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        t = torch.tensor([sum(a.elapsed_time(b) for a, b in evs)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # replicas (weak scaling): every rank keyswitches its own batch with the full key
    ws = get_context(params).ks_workspace(level, Bsz)
    out_full = torch.empty((Bsz, 2, l1, N), dtype=torch.int32, device=dev)
    ms_rep = timed(lambda i: fused.keyswitch_batch(params, level, xs[i % 3], rlk, out=out_full, ws=ws), args.steps)
    del ws, out_full

    # limb-sharded (strong scaling)
    comm_kind = "library NCCL communicator (lf_comm_create, ncclAllGather on the launch stream)"
    try:
        comm = NcclComm(world, rank) if dist.get_backend() == "nccl" else "torch"
        if comm == "torch":
            comm_kind = f"torch.distributed all_gather ({dist.get_backend()})"
    except Exception as e:                                               # noqa: BLE001
        comm, comm_kind = "torch", f"torch.distributed all_gather (library NCCL unavailable: {e})"
    eng = ShardEngine(params, world, rank, comm)
    key_loc = eng.shard_key(rlk)
    key_bytes_full = rlk.data.numel() * 4
    del rlk
    torch.cuda.empty_cache()
    xs_loc = [eng.shard_rows(x, level) for x in xs]
    nm = xs_loc[0].shape[1]
    out = torch.empty((Bsz, 2, nm, N), dtype=torch.int32, device=dev)
    calls = [eng.keyswitch_call(level, x, key_loc, out=out)[0] for x in xs_loc]
    clk = ClockSampler(torch.cuda.current_device()).start()
    ms = timed(lambda i: eng.run(calls[i % 3], level, Bsz), args.steps)
    clocks = clk.stop()
    value = Bsz * args.steps / (ms / 1e3)

    # batch-1 latency of one sharded keyswitch
    one = eng.keyswitch_call(level, xs_loc[0][:1].contiguous(), key_loc)[0]
    ms1 = timed(lambda i: eng.run(one, level, 1), 10) / 10

    # e2e: each rank's rows from pinned host memory, sharded keyswitch, results back
    h_in = torch.empty((Bsz, nm, N), dtype=torch.int32, pin_memory=True)
    h_in.copy_(xs_loc[0].cpu())
    h_out = torch.empty((Bsz, 2, nm, N), dtype=torch.int32, pin_memory=True)
    d_in = torch.empty_like(xs_loc[0])
    ecall = eng.keyswitch_call(level, d_in, key_loc, out=out)[0]

    def e2e(i):
        d_in.copy_(h_in, non_blocking=True)
        eng.run(ecall, level, Bsz)
        h_out.copy_(out, non_blocking=True)
    ms_e2e = timed(e2e, args.steps)
    if rank == 0:
        lay = eng.gather_layout(level, Bsz)
        line = {
            "metric": METRIC, "value": value, "unit": "ops/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u32", "data": "synthetic",
            "config": {"workload": "C2 full-level hybrid keyswitch, N=2^16, L=35, dnum=4, alpha=9",
                       "level": level, "batch_per_step": Bsz, "parallelism": f"limb-sharded{world}",
                       "l2": "256 MB flush between timed steps; inputs cycled over 3 batches"},
            "keyswitch_us": ms / args.steps / Bsz * 1e3,
            "limb_sharded": {"latency_batch1_us": ms1 * 1e3, "comm": comm_kind,
                             "allgather_bytes_per_rank_per_step": lay[1] + lay[4],
                             "key_bytes_per_gpu": key_loc.numel() * 4, "key_bytes_full": key_bytes_full,
                             "main_rows_rank0": nm},
            "replicas": {"value": world * Bsz * args.steps / (ms_rep / 1e3), "unit": "ops/s", "scaling": "weak",
                         "note": "every GPU keyswitches its own batch with the full key"},
            "gpu_launches": 5 * args.steps,
            "e2e": {"value": Bsz * args.steps / (ms_e2e / 1e3), "unit": "ops/s",
                    "h2d_bytes_per_step": Bsz * nm * N * 4 * world, "d2h_bytes_per_step": Bsz * 2 * nm * N * 4 * world,
                    "api": "ShardEngine.keyswitch per rank: local rows H2D, sharded pipeline, local results D2H"},
            "clocks": clocks, "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)


def run_ours(args, rank, world):
    import torch
    import torch.distributed as dist
    import paper_2512_11269_b200 as B
    from paper_2512_11269_b200 import fused
    from paper_2512_11269_b200.context import get_context

    dev = torch.device("cuda", torch.cuda.current_device())
    params = B.gen_params(**C2)
    level = args.level
    l1 = level + 1
    N = params.N
    sk, pk, rlk = B.keygen(params, seed=11)
    ctx = get_context(params)
    Bsz = args.batch

    # synthetic full-level inputs: NSETS distinct batches, cycled (each batch > L2 with keys/outputs)
    nsets = 3
    q = torch.tensor(params.rns_basis[:l1], dtype=torch.int64, device=dev)[:, None]
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    xs = []
    for s in range(nsets):
        r = torch.randint(0, 2 ** 62, (Bsz, l1, N), device=dev, generator=g, dtype=torch.int64)
        xs.append((r % q).to(torch.int32))
    out = torch.empty((Bsz, 2, l1, N), dtype=torch.int32, device=dev)
    ws = ctx.ks_workspace(level, Bsz)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)   # > 126 MB L2
    stream = torch.cuda.current_stream()

    def step(i):
        fused.keyswitch_batch(params, level, xs[i % nsets], rlk, out=out, ws=ws)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(torch.cuda.current_device()).start()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    for i in range(args.steps):
        flush.fill_(i)                                  # L2 flush between timed steps (untimed)
        evs[i][0].record(stream)
        step(i)
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = sum(a.elapsed_time(b) for a, b in evs)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    total_ops = Bsz * args.steps * world
    value = total_ops / (ms / 1e3)

    # per-kernel durations (CUDA events on the launch stream), averaged over 3 profiled runs
    stage = np.zeros(5)
    for i in range(3):
        flush.fill_(i)
        stage += np.array(fused.keyswitch_batch_profiled(params, level, xs[i % nsets], rlk, out, ws))
    stage /= 3
    rows = stage_rows(level)
    krows = key_rows(level)

    def batch_rows(n):          # the shared relinearisation key is read once per batch
        return rows[n] * Bsz - (krows * (Bsz - 1) if n == "ks_inner" else 0)
    stage_info = {n: {"ms": float(t), "share": float(t / stage.sum()),
                      "gbs": batch_rows(n) * ROW_BYTES / (t / 1e3) / 1e9,
                      "gbs_key_per_op": rows[n] * ROW_BYTES * Bsz / (t / 1e3) / 1e9}
                  for n, t in zip(STAGES, stage)}
    top = max(STAGES, key=lambda n: stage_info[n]["ms"])
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    ks_bytes = algorithmic_rows(level) * ROW_BYTES
    achieved_top = stage_info[top]["gbs"]
    traffic = None            # ncu dram bytes of the same kernel, per launch (profiles/, committed)
    pipes = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", TRAFFIC_JSON)))
        if top in tr and tr[top].get("batch", 8) == Bsz and level == 35:
            traffic = tr[top]["bytes_per_launch"]
            pipes = {k: tr[top].get(k) for k in ("fmaheavy_pipe_pct", "issue_active_pct", "l1tex_pct",
                                                 "dram_pct", "kernel", "tree")}
    except Exception:
        pass

    # the binding resource: NTT butterflies per second against the measured integer ceilings
    mhz = (clocks or {}).get("sm_mhz") or 1965.0
    bf = stage_butterflies(level)
    int_peak = SHOUP_MAC_PER_CLK_SM * 148 * mhz * 1e6 / 1e12
    line_peak = LINE_BFLY_PER_CLK_SM * 148 * mhz * 1e6 / 1e12
    per_stage = {}
    for name, ms_ in zip(STAGES, stage):
        tb = bf[name] * Bsz / (ms_ / 1e3) / 1e12 if ms_ > 0 else 0.0
        per_stage[name] = {"t_butterflies_per_s": tb, "frac": tb / int_peak}
    ks_bf = sum(bf.values()) / (ms / 1e3 / (Bsz * args.steps)) / 1e12
    int_roof = {"bound": "int", "unit": "T butterflies/s", "peak": int_peak,
                "peak_source": "measured Shoup modular MAC rate x 148 SMs x SM clock (profiles/r01_ubench_imad.log)",
                "line_code_peak": line_peak, "kernel": top,
                "achieved": per_stage[top]["t_butterflies_per_s"], "frac": per_stage[top]["frac"],
                "keyswitch": {"butterflies": sum(bf.values()), "achieved": ks_bf, "frac": ks_bf / int_peak,
                              "frac_of_line_code": ks_bf / line_peak},
                "stages": per_stage,
                "note": "NTT butterflies only (BConv MACs run on the tensor cores); every kernel's FMA-heavy pipe is ~50 % busy (profiles/r02_ncu_traffic.json)"}

    # e2e: public API, pinned host inputs -> device -> keyswitch -> host, every step
    host_in = torch.empty((Bsz, l1, N), dtype=torch.int32, pin_memory=True)
    host_in.copy_(xs[0].cpu())
    host_out = torch.empty((Bsz, 2, l1, N), dtype=torch.int32, pin_memory=True)
    dev_in = torch.empty((Bsz, l1, N), dtype=torch.int32, device=dev)
    ids = tuple(range(l1))

    s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()

    def e2e_step():
        """Per ciphertext: H2D copy (copy stream) -> public keyswitch API (compute stream) ->
        D2H copy (second copy stream), pipelined across the batch so PCIe traffic in both
        directions overlaps the kernels of neighbouring ciphertexts."""
        start = torch.cuda.Event()
        start.record(stream)
        s_h2d.wait_event(start)
        last = None
        keep = []            # results stay referenced until the step's D2H copies are enqueued and joined
        for b in range(Bsz):
            ev_in = torch.cuda.Event()
            with torch.cuda.stream(s_h2d):
                dev_in[b].copy_(host_in[b], non_blocking=True)
                ev_in.record(s_h2d)
            stream.wait_event(ev_in)
            kb, ka = B.keyswitch(B.RnsPolynomial(dev_in[b], B.Domain.EVAL, ids), rlk, params)
            ev_out = torch.cuda.Event()
            ev_out.record(stream)
            s_d2h.wait_event(ev_out)
            keep.append((kb, ka))
            with torch.cuda.stream(s_d2h):
                host_out[b, 0].copy_(kb.limbs, non_blocking=True)
                host_out[b, 1].copy_(ka.limbs, non_blocking=True)
                last = torch.cuda.Event()
                last.record(s_d2h)
        stream.wait_event(last)
        last.synchronize()
        keep.clear()

    for _ in range(max(1, args.warmup)):
        e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    wall_ms = (time.perf_counter() - w0) * 1e3
    e2e_ms = max(e0.elapsed_time(e1), wall_ms)
    e_t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e_t, op=dist.ReduceOp.MAX)
    e2e_value = total_ops / (float(e_t.item()) / 1e3)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        r = cpu_reference_keyswitch_sample(2, level)
        if r is not None:
            v, dt = r
            cpu = {"value": v, "unit": "ops/s", "cores": 1, "kind": "reference", "cpu_model": cpu_model(),
                   "sample": f"2 C2 full-level keyswitches, limbforge.ckks.keyswitch (baseline/_ref) on 1 core ({dt:.1f} s)"}
        else:
            v, dt = cpu_oracle_keyswitch_sample(2, level)
            cpu = {"value": v, "unit": "ops/s", "cores": 1, "kind": "port", "cpu_model": cpu_model(),
                   "sample": f"2 C2 full-level keyswitches, oracle/lf_oracle.py on 1 core ({dt:.1f} s)"}

    ntt = ntt_throughput(params, dev)
    sweep = batch_sweep(params, level, rlk, dev) if rank == 0 else None
    rot = rotation_units(params, level, dev) if rank == 0 else None
    sec = secondary_keyswitch(dev) if rank == 0 else None

    sharded = shard_emulation(params, level, rlk, dev) if rank == 0 and world == 1 else None

    boot = None
    if rank == 0 and world == 1 and not args.no_bootstrap:
        del xs, out, ws, flush
        torch.cuda.empty_cache()
        boot = bootstrap_latency()

    layers = None
    if rank == 0 and world == 1 and not args.no_workloads:
        import gc
        gc.collect()
        torch.cuda.empty_cache()
        layers = {"resnet_block": resnet_block_latency()}
        gc.collect()
        torch.cuda.empty_cache()
        layers["transformer_block"] = transformer_block_latency()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "ops/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u32", "data": "synthetic",
            "config": {"workload": "C2 full-level hybrid keyswitch, N=2^16, L=35, dnum=4, alpha=9",
                       "level": level, "batch_per_step": Bsz, "parallelism": f"replicas{world}",
                       "l2": "256 MB flush between timed steps; inputs cycled over 3 batches"},
            "keyswitch_us": ms / args.steps / Bsz * 1e3,
            "keyswitch_hbm": {"algorithmic_bytes": ks_bytes, "achieved_gbs": ks_bytes * value / world / 1e9,
                              "peak_gbs": hbm_peak, "frac": ks_bytes * value / world / 1e9 / hbm_peak,
                              "key": "charged per keyswitch (SURVEY 8d: 468 rows at C2)"},
            "keyswitch_hbm_batch": {
                "algorithmic_bytes_per_batch": (algorithmic_rows(level) * Bsz - key_rows(level) * (Bsz - 1)) * ROW_BYTES,
                "achieved_gbs": (algorithmic_rows(level) * Bsz - key_rows(level) * (Bsz - 1)) * ROW_BYTES
                                / (ms / args.steps / 1e3) / 1e9,
                "peak_gbs": hbm_peak,
                "frac": (algorithmic_rows(level) * Bsz - key_rows(level) * (Bsz - 1)) * ROW_BYTES
                        / (ms / args.steps / 1e3) / 1e9 / hbm_peak,
                "key": "the shared relinearisation key read once per batch"},
            "int_roofline": int_roof,
            "roofline": {"kernel": top, "bound": "hbm", "achieved": achieved_top, "peak": hbm_peak,
                         "unit": "GB/s", "frac": achieved_top / hbm_peak, "traffic": traffic,
                         "algorithmic_bytes_per_launch": batch_rows(top) * ROW_BYTES,
                         "ncu_pipes": pipes,
                         "peak_source": peak_src,
                         "binding_resource": "FMA-heavy integer pipe (NTT Shoup products), not HBM: see ncu_pipes",
                         "note": f"algorithmic bytes / CUDA-event time of the launch; traffic = ncu dram read+write of the same launch (profiles/{TRAFFIC_JSON})"},
            "stages": stage_info,
            "gpu_launches": 5 * args.steps,
            "e2e": {"value": e2e_value, "unit": "ops/s",
                    "h2d_bytes_per_step": Bsz * l1 * N * 4, "d2h_bytes_per_step": Bsz * 2 * l1 * N * 4,
                    "api": "paper_2512_11269_b200.keyswitch per ciphertext; H2D / compute / D2H on three streams, pipelined over the batch"},
            "clocks": clocks,
            "cpu_baseline": cpu,
            "bootstrap": boot,
            "ntt": ntt_summary(ntt, clocks),
            "batch_sweep": sweep,
            "rotation": rot,
            "secondary_c2": sec,
            "limb_sharded_emulated": sharded,
            "layers": layers,
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--level", type=int, default=35)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline sample")
    ap.add_argument("--no-bootstrap", action="store_true", help="skip the C3 bootstrap latency")
    ap.add_argument("--no-workloads", action="store_true", help="skip the C4/C5 layer latencies")
    ap.add_argument("--replicas", action="store_true", help="N > 1: independent replicas instead of limb sharding")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("LF_DIST_BACKEND", "nccl")     # gloo: several ranks on one GPU (tests)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    if world > 1 and not args.replicas:
        run_sharded(args, rank, world)
    else:
        run_ours(args, rank, world)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
