"""The reference's OWN evaluators running on the B200 through the drop-in boundary.

The unmodified reference package (`limbforge`, installed into baseline/_ref, which travels to
the GPU box) is imported and
  * its direct evaluator `limbforge.evaluate.run_circuit` (evaluate.py:57-113) runs the
    reference's benchmark programs (bench.py: bsgs64, polyeval, tinylayer, tinylayer4) with its
    operator globals re-bound by `dropin.install` (evaluate.py:12-21): every hom_mul / rotate /
    rescale / add / plain op is a B200 kernel;
  * its compiled pipeline `limbforge.runtime.Executor` (runtime.py:188) runs the same programs
    with `dropin.install_runner(limbforge.runtime)`: every kernel plan on the B200 runner.
Both are compared residue for residue with the same reference code running on the CPU, and the
decrypted slots with the benchmark's own oracle and tolerance."""

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")


@pytest.fixture(scope="module")
def lf():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.isdir(os.path.join(REF, "limbforge")):
        pytest.skip("reference not installed in baseline/_ref (see DESIGN.md §8)")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import limbforge
    import limbforge.bench
    import limbforge.evaluate
    import limbforge.runtime
    return limbforge


def _same(got, want):
    gb = got.b.numpy() if hasattr(got.b, "numpy") else got.b.limbs
    ga = got.a.numpy() if hasattr(got.a, "numpy") else got.a.limbs
    return np.array_equal(np.asarray(gb, dtype=np.uint64), want.b.limbs) and \
        np.array_equal(np.asarray(ga, dtype=np.uint64), want.a.limbs)


@pytest.mark.parametrize("name", ["bsgs64", "polyeval", "tinylayer"])
def test_run_circuit_on_b200(lf, name):
    from limbforge.parser import parse_program
    from limbforge.typecheck import typecheck
    import paper_2512_11269_b200 as B
    from paper_2512_11269_b200 import dropin
    bench = lf.bench.SUITE[name]()
    sk, pk, keys = bench.make_keys()
    inputs = bench.encrypt_inputs(pk)
    typed = typecheck(parse_program(bench.text), bench.params)
    want = lf.evaluate.run_circuit(typed, inputs, bench.plaintexts, keys)       # reference, CPU
    with dropin.install(lf.evaluate):
        assert lf.evaluate.hom_mul is dropin.hom_mul
        got = lf.evaluate.run_circuit(typed, inputs, bench.plaintexts, keys)    # reference, B200 ops
    assert lf.evaluate.hom_mul is not dropin.hom_mul                            # restored
    assert isinstance(got, B.Ciphertext)                                        # device-resident result
    assert got.level == want.level and got.scale == want.scale
    assert _same(got, want)
    # identical residues, so the decryption is the reference's: within the benchmark's tolerance
    err = np.abs(lf.ckks.decrypt(want, sk, bench.params) - bench.oracle).max()
    assert err < bench.tolerance


@pytest.mark.parametrize("name", ["bsgs64", "polyeval", "tinylayer", "tinylayer4"])
def test_executor_on_b200_runner(lf, name):
    from paper_2512_11269_b200 import dropin
    bench = lf.bench.SUITE[name]()
    want = lf.bench.run_benchmark(bench)                        # compiled pipeline, reference runner
    with dropin.install_runner(lf.runtime):
        assert lf.runtime.KernelRunner is dropin.KernelRunner
        got = lf.bench.run_benchmark(bench)                     # same pipeline, B200 runner
    assert lf.runtime.KernelRunner is not dropin.KernelRunner
    assert np.array_equal(got["output"].b.limbs, want["output"].b.limbs)
    assert np.array_equal(got["output"].a.limbs, want["output"].a.limbs)
    assert got["pass"] and got["error"] == want["error"]
