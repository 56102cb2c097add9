"""Host logic of the drop-in re-binding (paper_2512_11269_b200/dropin.py): the reference
evaluator's operator globals (evaluate.py:12-21) are swapped and restored; reference
parameter objects convert field for field."""

import types
from fractions import Fraction

from paper_2512_11269_b200 import dropin
from paper_2512_11269_b200.params import gen_params


def _fake_evaluate_module():
    m = types.ModuleType("fake_evaluate")
    for name in dropin.OPERATORS:
        setattr(m, name, f"orig-{name}")
    m.run_circuit = "orig-run_circuit"
    return m


def test_install_and_restore():
    m = _fake_evaluate_module()
    with dropin.install(m) as h:
        for name in dropin.OPERATORS:
            assert getattr(m, name) is getattr(dropin, name)
        assert m.run_circuit == "orig-run_circuit"
        assert set(h.saved) == set(dropin.OPERATORS)
    for name in dropin.OPERATORS:
        assert getattr(m, name) == f"orig-{name}"


def test_install_skips_unbound_names():
    m = types.ModuleType("partial")
    m.hom_add = "x"
    h = dropin.install(m)
    assert m.hom_add is dropin.hom_add and not hasattr(m, "encode")
    h.restore()
    assert m.hom_add == "x"


def test_reference_params_convert():
    own = gen_params(4096, 6, d=3, seed=0)
    ref_like = types.SimpleNamespace(
        N=own.N, rns_basis=list(own.rns_basis), special_basis=list(own.special_basis),
        scale=Fraction(own.scale), hamming_weight=own.hamming_weight,
        ks=types.SimpleNamespace(d=3), seed=0, sigma=own.sigma)
    conv = dropin.as_params(ref_like)
    assert conv == own
    assert dropin.as_params(ref_like) is conv          # cached per object
    assert dropin.as_params(own) is own


def test_install_runner_swaps_kernel_runner():
    m = types.ModuleType("fake_runtime")
    m.KernelRunner = "orig"
    with dropin.install_runner(m):
        assert m.KernelRunner is dropin.KernelRunner
    assert m.KernelRunner == "orig"


def test_key_cache_is_weak_and_cleared_on_restore(monkeypatch):
    """Device copies of reference keys are evicted when the reference key dies and on
    restore() (no HBM leak across long-running evaluators)."""
    import gc

    class RefKey:                        # stands in for a reference EvalKey (weak-referenceable)
        pass

    monkeypatch.setattr(dropin.EvalKey, "from_reference", staticmethod(lambda k: ("device", id(k))))
    k = RefKey()
    dev = dropin.as_key(k)
    assert dropin.as_key(k) is dev and id(k) in dropin._KEYS
    kid = id(k)
    del k
    gc.collect()
    assert kid not in dropin._KEYS
    k2 = RefKey()
    dropin.as_key(k2)
    m = _fake_evaluate_module()
    dropin.install(m).restore()
    assert not dropin._KEYS
