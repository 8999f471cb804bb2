"""CPU-side checks of the product library: the C ABI loads and exports every
symbol include/dfm_b200.h declares, the host runtime (RNG, random_init,
synthetic generator) is bit-exact with the oracle, and the host API's shape
and error behaviour mirrors the reference (types.hpp, engine.cpp:173-180).
No compute kernel is launched here."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def dfm():
    import __graft_entry__ as g
    from paper_2605_19388_b200 import build as b

    b.build()
    import paper_2605_19388_b200 as m

    m._capi.load()
    return m


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "dfm_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(dfm_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol(dfm):
    lib = dfm._capi.load()
    syms = _header_symbols()
    assert len(syms) > 30
    for s in syms:
        assert hasattr(lib, s), s
    # and the ctypes table covers all of them
    assert set(syms) == set(dfm._capi.exported_symbols())


def test_shared_object_is_sm100a(dfm):
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", dfm._capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_random_init_bit_exact_with_oracle(dfm, oracle):
    for sizes, (F, T, N, K, seed) in [([2, 2], (7, 9, 3, 4, 1)), ([4, 4, 4], (5, 11, 5, 16, 42)),
                                      ([12], (3, 6, 2, 3, 9)), ([2, 3, 1], (4, 5, 2, 2, 0))]:
        got = dfm.random_init(F, T, dfm.BlockLayout(sizes), N, K, seed)
        ref = oracle.random_init(F, T, sizes, N, K, seed)
        assert np.array_equal(got.nmf.T, ref["T"])
        assert np.array_equal(got.nmf.V, ref["V"])
        assert np.array_equal(got.lambda0, ref["lam"])
        for a, b in zip(got.w0, ref["w"]):
            assert np.array_equal(a, b)


def test_generators_bit_exact_with_oracle(dfm, oracle):
    assert np.array_equal(dfm.random_observations(3, 5, 4, 9), oracle.random_observations(3, 5, 4, 9))
    for kind in (0, 1):
        a = dfm.generate_mixture(kind, 9, 13, 4, 3, 4, 5)
        b = oracle.generate_mixture(kind, 9, 13, 4, 3, 4, 5)
        assert np.array_equal(a, b)
    assert dfm._capi.load().dfm_derive_seed(1, b"gen-W", 3) == oracle.derive_seed(1, "gen-W", 3)


def test_block_layout_mirrors_reference(dfm):
    # test_dist.cpp:37-54
    L = dfm.BlockLayout([4, 4, 4])
    assert L.global_index(0, 0) == 0
    assert L.global_index(2 - 1, 3 - 1) + 1 == 7
    with pytest.raises(IndexError):
        L.global_index(3, 0)
    with pytest.raises(IndexError):
        L.global_index(0, 4)
    small = dfm.BlockLayout([2, 3])
    seen = sorted(small.global_index(l, mu) for l in range(2) for mu in range(small.sizes[l]))
    assert seen == list(range(5))
    with pytest.raises(ValueError):
        dfm.BlockLayout([2, 0])


def test_host_shape_errors_are_typed(dfm):
    x = np.zeros((3, 4, 4), complex)
    init = dfm.random_init(3, 4, dfm.BlockLayout([2, 2]), 2, 2, 0)
    with pytest.raises(dfm.ShapeMismatchError):
        dfm.fit_distributed(x, dfm.BlockLayout([2, 3]), init, 1)
    with pytest.raises(dfm.ShapeMismatchError):
        dfm.fit_distributed(np.zeros((3, 5, 4), complex), dfm.BlockLayout([2, 2]), init, 1)
    with pytest.raises(ValueError):
        dfm.fit_distributed(x, dfm.BlockLayout([2, 2]), init, -1)
    with pytest.raises(dfm.ShapeMismatchError):
        dfm.decorrelate(np.zeros((3, 4), complex), np.zeros((3, 4, 4), complex))
    assert issubclass(dfm.ShapeMismatchError, ValueError)
    assert issubclass(dfm.SingularDemixerError, RuntimeError)


def test_slice_init_and_extract_block(dfm):
    layout = dfm.BlockLayout([2, 3])
    init = dfm.random_init(4, 5, layout, 2, 2, 3)
    sub = dfm.slice_init(init, 1)
    assert sub.layout.sizes == [3]
    assert np.array_equal(sub.lambda0, init.lambda0[:, :, 2:5])
    assert np.array_equal(sub.w0[0], init.w0[1])
    x = np.arange(4 * 5 * 5).reshape(4, 5, 5).astype(complex)
    assert np.array_equal(dfm.extract_block(x, layout, 1), x[:, :, 2:])


def test_op_counts_follow_the_reference_formulas():
    # test_bench.cpp:34-52: W-stage ops per iteration and bin are M^4 + J M^3
    from paper_2605_19388_b200.fastmnmf import op_counts

    full = op_counts(4, 16, [6], 2, 6, 2, 2)
    assert full["w_update"] == 4.0 * 2 * (6 ** 4 + 16.0 * 6 ** 3)
    dist = op_counts(4, 16, [2, 2, 2], 2, 6, 2, 2)
    assert dist["w_update"] == 4.0 * 2 * 3 * (2 ** 4 + 16.0 * 2 ** 3)
    # mm: two weight builds (2FTNM each), T and V updates (2FKT per source each), Lambda (2NMT per bin)
    F, T, N, M, K = 3, 5, 2, 4, 6
    assert op_counts(F, T, [4], N, M, K, 1)["mm_update"] == 4 * F * T * N * M + 4 * N * F * K * T + 2 * F * N * M * T
