"""CPU tests of the GPC problem setup (pure host logic of gpc.py)."""

import math

import numpy as np
import pytest


def test_dirichlet_transform_known_values():
    from paper_2503_02259_b200 import gpc

    x = np.zeros((4, 2))
    p = gpc.setup(x, [0, 1, 2, 1], alpha_eps=0.01)
    assert p.num_classes == 3
    hi, lo = math.log(1.0 / 1.01 + 1.0), math.log(1.0 / 0.01 + 1.0)
    np.testing.assert_allclose(p.noise[:, 1], [lo, hi, lo])
    raw = np.array([math.log(0.01) - lo / 2, math.log(1.01) - hi / 2, math.log(0.01) - lo / 2])
    np.testing.assert_allclose(p.targets[:, 1] + p.means, raw)
    np.testing.assert_allclose(p.targets.mean(axis=1), 0.0, atol=1e-15)


def test_setup_validation():
    from paper_2503_02259_b200 import gpc

    x = np.zeros((3, 1))
    with pytest.raises(ValueError):
        gpc.setup(x, [0, 1])
    with pytest.raises(ValueError):
        gpc.setup(x, [0, 0, 0])
    with pytest.raises(ValueError):
        gpc.setup(x, [0, 1, 5], num_classes=3)
    with pytest.raises(ValueError):
        gpc.setup(x, [0.5, 1, 0])
    assert gpc.setup(x, [0.0, 1.0, 1.0]).num_classes == 2


def test_probe_layout_and_labels():
    from paper_2503_02259_b200 import gpc

    z = gpc.generate_probes(10, 3, 4, (7, 1))
    assert z.shape == (12, 10)
    np.testing.assert_array_equal(z, gpc.generate_probes(10, 3, 4, (7, 1)))
    x = np.random.default_rng(0).standard_normal((3000, 8))
    lab = gpc.sample_latent_labels(x, 3, l=1.0, seed=0)
    counts = np.bincount(lab, minlength=3)
    assert counts.min() > 300  # every class present in a balanced-ish proportion
