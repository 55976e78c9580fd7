"""CPU tier: the seeded synthetic workloads have the shapes / distributions of
BASELINE.json's configs, and every kernel is normalised (unit mass checked
through the oracle)."""
import math

import numpy as np
import pytest

import oracle_lib as OL
from paper_2507_21686_b200 import scenes


@pytest.mark.parametrize("k", [scenes.wendland_c2(), scenes.wendland_c4(), scenes.wendland_c6(),
                               scenes.generic_deg12(np.random.default_rng(scenes.SEED_BASE + 4))])
def test_kernel_normalisation(k):
    m = sum(c / (i + 2) for i, c in enumerate(k.coefficients))
    assert abs(k.normalization * 2 * math.pi * m - 1.0) < 1e-12


def test_wendland_c4_is_reference_wendland4():
    assert scenes.wendland_c4().coefficients == OL.W4
    assert scenes.wendland_c4().normalization == OL.C4


def test_cubic_spline_composition_unit_mass():
    """(1-q)^3 at h plus -1/2 (1-q')^3 at h/2 integrates to 1 over an enclosing triangle."""
    O = OL.oracle()
    tri = [-9.0, -7.0, 9.0, -7.0, 0.0, 11.0]
    total = 0.0
    for k in scenes.cubic_spline_pieces():
        st, out = OL.oracle_integrate(O, (0.1, 0.2), 1.0 * k.support_scale, tri, [1, 1, 1], k.coefficients,
                                      k.normalization)
        assert st == 0
        total += out[0]
    assert abs(total - 1.0) < 1e-14


def test_cfg1_shape():
    s = scenes.cfg1()
    assert s.particles.shape == (4096, 2) and s.triangles.shape == (1, 6) and s.h == 0.25
    assert s.particles[:, 0].min() >= -0.3 and s.particles[:, 0].max() <= 1.3


def test_cfg2_shape_and_slivers():
    s = scenes.cfg2(T=4096)
    assert s.triangles.shape == (4096, 6) and s.particles.shape == (4096 * 64, 2)
    t = s.triangles.reshape(-1, 3, 2)
    e = np.stack([np.linalg.norm(t[:, i] - t[:, (i + 1) % 3], axis=1) for i in range(3)], axis=1)
    area = 0.5 * np.abs(np.cross(t[:, 1] - t[:, 0], t[:, 2] - t[:, 0]))
    aspect = e.max(axis=1) ** 2 / (2 * area)  # longest edge / height to it
    frac = np.mean(aspect >= 99.0)
    assert abs(frac - 0.2) < 0.02
    assert np.array_equal(s.pairs[1], np.repeat(np.arange(4096), 64))


def test_cfg3_shape():
    s = scenes.cfg3(target_particles=100_000)
    assert s.triangles.shape == (8192, 6) and s.h == 0.01
    assert 80_000 < s.particles.shape[0] < 120_000
