"""Checks of the seeded input generator (synth/), which both sides consume."""
import numpy as np

import synth


def test_counter_generator_known_values_and_determinism():
    # SplitMix64 output function on key + idx*GAMMA; determinism and position keying
    a = synth.counter_u64(1, 0, np.arange(10, dtype=np.uint64))
    b = synth.counter_u64(1, 0, np.arange(5, 10, dtype=np.uint64))
    assert np.array_equal(a[5:], b)
    assert len(set(a.tolist())) == 10
    assert not np.array_equal(a, synth.counter_u64(2, 0, np.arange(10, dtype=np.uint64)))
    assert not np.array_equal(a, synth.counter_u64(1, 1, np.arange(10, dtype=np.uint64)))
    # scalar path agrees with the vector path
    key = synth.stream_key(1, 0)
    z = (key + 3 * synth.GAMMA) & ((1 << 64) - 1)
    assert synth._mix64_scalar(z) == int(a[3])


def test_normal_moments():
    x = synth.normals(1, 0, 400000)
    assert abs(x.mean()) < 0.01 and abs(x.std() - 1) < 0.01
    assert abs(np.mean(x ** 3)) < 0.02 and abs(np.mean(x ** 4) - 3) < 0.05
    u = synth.counter_uniform(3, 1, np.arange(100000, dtype=np.uint64))
    assert u.min() > 0 and u.max() < 1 and abs(u.mean() - 0.5) < 0.005


def test_data_at_matches_full_data():
    n, m = (5, 4, 6), (9, 8, 11)
    A, _ = synth.mode_matrices(n, m)
    y = synth.data(A, n, m, seed=4)
    ks = np.array([[0, 0, 0], [8, 7, 10], [4, 3, 5], [1, 6, 2]])
    got = synth.data_at(A, n, m, ks, seed=4)
    assert np.allclose(got, [y[tuple(k)] for k in ks], rtol=1e-14, atol=1e-15)


def test_config_shapes():
    c = synth.CONFIGS[3]
    assert c.N == 31457280 and c.Mdata == 503316480
    assert synth.CONFIGS[4].N == 536870912
    A, L = synth.mode_matrices(synth.CONFIGS[1])
    assert A[0].shape == (64, 48) and L[0].shape == (46, 48)
    assert abs(A[0].std() - 1 / 8) < 0.01
