"""Drop-in re-binding of the reference evaluator onto the B200 operator API.

The reference's direct evaluator `limbforge.evaluate.run_circuit` (evaluate.py:57-113) binds
the operator names at import time (evaluate.py:12-21), so swapping the backend means
replacing those module globals.  `install(evaluate_module)` does exactly that and returns a
handle whose `restore()` puts the originals back:

    import limbforge.evaluate as ev
    from paper_2512_11269_b200 import dropin
    with dropin.install(ev):
        ct = ev.run_circuit(typed, inputs, plaintexts, keys)   # now runs on the B200 kernels

The wrappers accept reference objects (CkksParams, Ciphertext, Plaintext, EvalKey with
uint64 numpy rows) and return this package's device-resident objects, which every wrapped
operator also accepts, so a circuit stays on the GPU between operations.  Reference
evaluation keys are uploaded once and cached per key object.

The compiled pipeline (pipeline.py / runtime.py Executor) instead executes kernel plans through
`KernelRunner`; `install_runner(limbforge.runtime)` swaps that class for the B200 runner:

    import limbforge.runtime as rt
    with dropin.install_runner(rt):
        result = rt.Executor(compiled, ...).run(...)        # every kernel plan on the GPU
"""

import weakref
from fractions import Fraction

from . import ckks as C
from . import encoding as E
from .keys import EvalKey
from .params import CkksParams, KeySwitchConfig

OPERATORS = ("hom_add", "hom_sub", "hom_mul", "hom_rotate", "add_plain", "mul_plain",
             "rescale", "encode")

_PARAMS = {}
_KEYS = {}


def as_params(p) -> CkksParams:
    """This package's CkksParams for a reference (or own) parameter object."""
    if isinstance(p, CkksParams):
        return p
    got = _PARAMS.get(id(p))
    if got is None or got[0] is not p:
        own = CkksParams(N=p.N, rns_basis=tuple(int(q) for q in p.rns_basis),
                         special_basis=tuple(int(q) for q in p.special_basis),
                         scale=Fraction(p.scale), hamming_weight=p.hamming_weight,
                         ks=KeySwitchConfig(d=p.ks.d), seed=p.seed, sigma=p.sigma)
        got = (p, own)
        _PARAMS[id(p)] = got
    return got[1]


def as_key(k):
    """Device EvalKey for a reference EvalKey (uploaded once per key object)."""
    if k is None or isinstance(k, EvalKey):
        return k
    got = _KEYS.get(id(k))
    if got is None or got[0]() is not k:
        got = (weakref.ref(k), EvalKey.from_reference(k))
        _KEYS[id(k)] = got
        weakref.finalize(k, _KEYS.pop, id(k), None)     # device copy freed with the reference key
    return got[1]


def clear_cache():
    """Drop every cached device key and parameter conversion (HBM is released once the
    evaluator holds no other reference to the device keys)."""
    _KEYS.clear()
    _PARAMS.clear()


def hom_add(ct1, ct2, params):
    return C.hom_add(ct1, ct2, as_params(params))


def hom_sub(ct1, ct2, params):
    return C.hom_sub(ct1, ct2, as_params(params))


def hom_mul(ct1, ct2, relin_key, params):
    return C.hom_mul(ct1, ct2, as_key(relin_key), as_params(params))


def hom_rotate(ct, steps, rot_key, params):
    return C.hom_rotate(ct, steps, as_key(rot_key), as_params(params))


def add_plain(ct, pt, params):
    return C.add_plain(ct, pt, as_params(params))


def mul_plain(ct, pt, params):
    return C.mul_plain(ct, pt, as_params(params))


def rescale(ct, params):
    return C.rescale(ct, as_params(params))


def encode(values, params, level=None, scale=None):
    return E.encode(values, as_params(params), level=level, scale=scale)


class Installed:
    def __init__(self, module, saved):
        self.module, self.saved = module, saved

    def restore(self):
        for name, fn in self.saved.items():
            setattr(self.module, name, fn)
        self.saved = {}
        clear_cache()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.restore()
        return False


class KernelRunner:
    """Stand-in for `limbforge.codegen.KernelRunner` (codegen.py:346-361) constructed with a
    reference CkksParams, as `Executor` (runtime.py:188) and the multi-device runner
    (multidev.py:801) do; runs every plan on the B200 (kernel_runner.KernelRunner)."""

    def __init__(self, params, max_regs: int = 512):
        from .kernel_runner import KernelRunner as _Gpu
        self.params = params
        self._gpu = _Gpu(as_params(params), max_regs)

    def run(self, plan, read_row, write_row):
        self._gpu.run(plan, read_row, write_row)


def install_runner(module) -> Installed:
    """Replace the `KernelRunner` global of `module` (`limbforge.runtime` or
    `limbforge.multidev`, which bind it at import: runtime.py:21, multidev.py:29), so the
    compiled pipeline's kernels run on the B200."""
    saved = {}
    if hasattr(module, "KernelRunner"):
        saved["KernelRunner"] = module.KernelRunner
        module.KernelRunner = KernelRunner
    return Installed(module, saved)


def install(module) -> Installed:
    """Replace the operator globals of `module` (normally `limbforge.evaluate`) with the
    B200 wrappers above.  Names the module does not bind are left alone."""
    saved = {}
    for name in OPERATORS:
        if hasattr(module, name):
            saved[name] = getattr(module, name)
            setattr(module, name, globals()[name])
    return Installed(module, saved)
