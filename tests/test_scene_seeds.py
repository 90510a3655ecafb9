"""The seeded input generators (scenes/, no method arithmetic): the config-2 noise seeds used for the
fp32 margin checks give different initial states and leave the pinned layers alone."""
import numpy as np

from scenes import generators as G


def test_config2_noise_seeds_differ_and_keep_pins():
    a = G.config2_twisted_bar(nx=4, nz=8)
    for k in (1, 2, 3):
        b = G.config2_twisted_bar(nx=4, nz=8, noise_seed=k)
        assert np.abs(a.x0 - b.x0).max() > 1e-3 * a.h
        assert np.array_equal(a.pinned, b.pinned) and np.array_equal(a.targets, b.targets)
