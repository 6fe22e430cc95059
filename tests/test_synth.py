"""Properties of the seeded input generator (synth/).  CPU only."""
import numpy as np

import synth


def test_splitmix_known_values():
    # splitmix64 reference outputs for state 0 (first three draws of the public
    # splitmix64 sequence seeded with 0): x_k = h(k * gamma) in our notation.
    G = synth.GAMMA
    assert synth._h_scalar(0) == 0xE220A8397B1DCDAF
    assert synth._h_scalar(G) == 0x6E789E6AA1B965F4
    assert synth._h_scalar((2 * G) & synth.M64) == 0x06C45D188009454F
    v = synth._h_vec(np.array([0, G, (2 * G) & synth.M64], dtype=np.uint64))
    assert [int(x) for x in v] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_change_fraction_and_always_different():
    for wb in (2, 4):
        b = synth.base(200000, wb, 5, 1)
        for f in (0.0, 0.01, 0.3, 1.0):
            s = synth.step(b, 5, 1, 1, f)
            ch = s != b
            assert np.array_equal(ch, synth.change_mask(b.size, wb, 5, 1, 1, f))
            if f == 0.0:
                assert not ch.any()
            elif f == 1.0:
                assert ch.all()
            else:
                assert abs(ch.mean() - f) < 5 * np.sqrt(f * (1 - f) / b.size)


def test_s2_runs_structure():
    b = synth.base(40960, 4, 9, 2)
    s = synth.step(b, 9, 2, 1, 0.5, structure=synth.S2_RUNS)
    ch = (s != b).reshape(10, 4096)
    assert all(row.all() or not row.any() for row in ch)


def test_window_equals_full():
    full = synth.state([10000], [4], 3, 2, 0.2)[0]
    part = synth.state([1000], [4], 3, 2, 0.2, start=5000)[0]
    assert np.array_equal(full[5000:6000], part)
