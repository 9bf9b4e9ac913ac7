"""The shared seeded input generators (vp_inputs) -- host side."""
import numpy as np

import vp_inputs as I


def test_ramp_is_spec_s71():
    """pixel(i, y, x, c) = (seed*2654435761 + i*97 + y*31 + x*7 + c) mod 256."""
    f = I.frames_u8("ramp", 7, [0, 3, 11], 5, 9)
    for a, i in enumerate([0, 3, 11]):
        for y in range(5):
            for x in range(9):
                for c in range(3):
                    assert f[a, y, x, c] == (7 * 2654435761 + i * 97 + y * 31 + x * 7 + c) % 256


def test_noise_is_deterministic_and_uniformish():
    a = I.frames_u8("noise", 3, [5, 6], 64, 64)
    b = I.frames_u8("noise", 3, [5, 6], 64, 64)
    assert np.array_equal(a, b)
    assert not np.array_equal(a, I.frames_u8("noise", 4, [5, 6], 64, 64))
    h = np.bincount(a.ravel(), minlength=256)
    assert h.min() > 0 and abs(a.mean() - 127.5) < 2.0


def test_configs_shapes():
    for name, n in [("cfg1", 1), ("cfg2", 1), ("cfg3", 1), ("cfg4", 24), ("cfg5", 512)]:
        params, clips = I.config(name)
        assert len(clips) == n and params["patch_size"] == 16
