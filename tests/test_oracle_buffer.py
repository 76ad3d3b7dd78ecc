"""Pins for oracle.buffer (NEXT-1): the sampler's generator against splitmix64's reference
output, uniformity, and the gather as plain indexing."""
import numpy as np

from oracle import buffer


def test_splitmix64_reference_vector():
    # Reference outputs of splitmix64 seeded with 0 (the sequence of states 0x9E37..*k):
    # first outputs of the canonical C implementation (Vigna, xoshiro seeding helper).
    state = 0
    outs = []
    for _ in range(3):
        outs.append(buffer.splitmix64(state))
        state = (state + 0x9E3779B97F4A7C15) & buffer.M64
    assert outs == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_sampler_uniform_and_deterministic():
    cap, B = 97, 20000
    a = buffer.sample_indices(cap, B, seed=5, step=3)
    b = buffer.sample_indices(cap, B, seed=5, step=3)
    c = buffer.sample_indices(cap, B, seed=5, step=4)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    assert a.min() >= 0 and a.max() < cap
    counts = np.bincount(a, minlength=cap)
    chi2 = ((counts - B / cap) ** 2 / (B / cap)).sum()
    assert chi2 < 200  # 96 dof: mean 96, sd ~14


def test_gather_is_indexing():
    rng = np.random.default_rng(0)
    cap, T, D = 10, 3, 4
    buf = dict(x=rng.standard_normal((cap, T, D)), h0=rng.standard_normal((cap, 5)),
               act=rng.integers(0, 9, (cap, T, 2)), adv=rng.standard_normal((cap, T)))
    idx = [3, 3, 0, 9]
    g = buffer.gather(buf, idx)
    assert g["x"].shape == (T, 4, D) and g["h0"].shape == (4, 5)
    for j, i in enumerate(idx):
        assert np.array_equal(g["x"][:, j], buf["x"][i])
        assert np.array_equal(g["act"][:, j], buf["act"][i])
        assert np.array_equal(g["adv"][:, j], buf["adv"][i])
        assert np.array_equal(g["h0"][j], buf["h0"][i])
