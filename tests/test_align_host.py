"""The product's host-side permutation alignment (csrc/dfm_align.cpp, through
the C ABI; no GPU involved) against the oracle's restatement of
init.cpp:14-54 / :190-250: identical permutations and bitwise-equal masks."""
import numpy as np

import init_oracle as io


def _masks(F, T, N, seed):
    rng = np.random.default_rng(seed)
    m = rng.random((F, T, N)) ** 3
    return m / m.sum(axis=2, keepdims=True)


def test_frequency_alignment_matches_oracle():
    import paper_2605_19388_b200.init as di

    for seed, (F, T, N) in enumerate([(30, 40, 2), (25, 64, 3), (12, 20, 5), (3, 5, 4), (5, 16, 8), (4, 9, 7)]):
        m = _masks(F, T, N, seed)
        # plant per-bin permutations on a smooth base so alignment has work
        for i in range(F):
            m[i] = m[i][:, np.random.default_rng(100 + i).permutation(N)]
        a = di.align_frequency_permutations(m, di.MaskOptions())
        b = io.align_frequency_permutations(m)
        assert np.array_equal(a, b)


def test_subarray_alignment_matches_oracle():
    import paper_2605_19388_b200.init as di

    base = _masks(6, 32, 3, 7)
    rng = np.random.default_rng(9)
    others = [np.maximum(0, base[:, :, p] + 0.05 * rng.standard_normal(base.shape))
              for p in ([2, 0, 1], [1, 2, 0], [0, 1, 2])]
    got = di.align_subarray_permutations([base] + others)
    ref = io.align_subarray_permutations([base] + others)
    assert got == ref.tolist()
    assert got[1] == [1, 2, 0] and got[3] == [0, 1, 2]


def test_subarray_alignment_eight_sources_matches_oracle():
    """Config 3's source count: the depth-first permutation search against the
    oracle's exhaustive next_permutation loop."""
    import paper_2605_19388_b200.init as di

    base = _masks(5, 24, 8, 11)
    rng = np.random.default_rng(12)
    perms = [rng.permutation(8) for _ in range(3)]
    others = [np.maximum(0, base[:, :, p] + 0.05 * rng.standard_normal(base.shape)) for p in perms]
    got = di.align_subarray_permutations([base] + others)
    ref = io.align_subarray_permutations([base] + others)
    assert got == ref.tolist()
