"""The probe-slice split of a multi-device engine (ssj_chunk_split, multi_device.cpp): host
logic, no GPU. Every slice goes whole to exactly one part, parts are contiguous and in C
order, the last part also takes the slots past the last slice, and the parts' work
(4|r| + k (13 + 4|r|) per slice) is balanced to within one slice."""
import numpy as np
import pytest

from paper_1812_09141_b200.verify import chunk_split


def random_chunk(rng, sizes, n_slices, max_k, trailing):
    n = sizes.size
    probes = np.sort(rng.integers(1, n, size=n_slices))
    ks = rng.integers(0, max_k + 1, size=n_slices)
    ends = np.cumsum(ks)
    CO = np.stack([probes, ends], 1).reshape(-1).astype(np.uint32)
    nC = int(ends[-1]) + trailing if n_slices else trailing
    return CO, nC, probes, ks


def work(sizes, probes, ks):
    r = sizes[probes].astype(np.float64)
    return 4 * r + ks * (13 + 4 * r)


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("parts", [1, 2, 3, 8])
def test_split_covers_and_balances(seed, parts):
    rng = np.random.default_rng(seed)
    sizes = rng.integers(1, 3000, size=5000).astype(np.uint32)
    CO, nC, probes, ks = random_chunk(rng, sizes, int(rng.integers(1, 400)), 2000,
                                      int(rng.integers(0, 50)))
    rg = chunk_split(sizes, parts, CO, nC).astype(np.int64)
    p = probes.size
    assert rg[0, 0] == 0 and rg[-1, 1] == p and rg[0, 2] == 0 and rg[-1, 3] == nC
    ends = np.concatenate([[0], CO[1::2].astype(np.int64)])
    for g in range(parts):
        a, b, lo, hi = rg[g]
        assert a <= b and lo <= hi
        assert lo == ends[a] and (hi == ends[b] or g == parts - 1)
        if g:
            assert a == rg[g - 1, 1] and lo == rg[g - 1, 3]  # contiguous, C order
    w = work(sizes, probes, ks)
    pw = [w[a:b].sum() for a, b in rg[:, :2]]
    assert max(pw) <= w.sum() / parts + w.max() + 1e-6


def test_split_edge_cases():
    sizes = np.array([3, 3, 4, 5], np.uint32)
    # more parts than slices: empty parts, trailing slots to the last one
    rg = chunk_split(sizes, 4, np.array([2, 3], np.uint32), 5)
    assert rg[:, 1].max() == 1 and rg[-1, 3] == 5 and rg[:, 3].tolist()[-1] == 5
    # empty chunk
    rg = chunk_split(sizes, 3, np.zeros(0, np.uint32), 0)
    assert rg.sum() == 0
    # zero-width slices and a probe index beyond n (weighted 0; verification reports it)
    rg = chunk_split(sizes, 2, np.array([1, 0, 9, 0, 3, 4], np.uint32), 4)
    assert rg[-1, 3] == 4 and rg[0, 0] == 0
    # malformed C_O (decreasing / beyond C) -> std::invalid_argument
    with pytest.raises(ValueError):
        chunk_split(sizes, 2, np.array([1, 3, 2, 2], np.uint32), 4)
    with pytest.raises(ValueError):
        chunk_split(sizes, 2, np.array([1, 5], np.uint32), 4)
    with pytest.raises(ValueError):
        chunk_split(sizes, 0, np.array([1, 1], np.uint32), 1)
