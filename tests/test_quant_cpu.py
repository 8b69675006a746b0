"""Host-side pieces of the quantizer module (reference quantizer.py:31-72,
160-187): the sensitivity estimate and the containers, restating the
reference's tests (test_quantizer.py:280-310)."""

import numpy as np
import pytest


def test_sensitivity_estimate_mean_of_squares():
    from paper_2402_10517_b200 import estimate_sensitivity_diag

    est = estimate_sensitivity_diag([np.array([[2.0]]), np.array([[4.0]])])
    assert est.values.tolist() == [[10.0]] and not est.fallback
    rng = np.random.default_rng(17)
    samples = [rng.normal(size=(3, 5)) for _ in range(7)]
    est = estimate_sensitivity_diag(samples)
    assert np.allclose(est.values, np.mean([g * g for g in samples], axis=0), rtol=1e-12)


def test_sensitivity_estimate_fallbacks_and_rejections():
    from paper_2402_10517_b200 import estimate_sensitivity_diag
    from paper_2402_10517_b200.errors import ParameterError, ShapeError

    est = estimate_sensitivity_diag([np.zeros((2, 3))])
    assert est.fallback and np.array_equal(est.values, np.ones((2, 3)))
    est = estimate_sensitivity_diag([], shape=(2, 2))
    assert est.fallback and np.array_equal(est.values, np.ones((2, 2)))
    with pytest.raises(ParameterError):
        estimate_sensitivity_diag([])
    with pytest.raises(ShapeError):
        estimate_sensitivity_diag([np.ones((2, 2)), np.ones((2, 3))])


def test_containers_validate_like_the_reference():
    from paper_2402_10517_b200 import ChannelQuantization, SensitivityMap
    from paper_2402_10517_b200.errors import ParameterError, ShapeError

    with pytest.raises(ShapeError):
        SensitivityMap(np.ones(3))
    with pytest.raises(ParameterError):
        SensitivityMap(-np.ones((2, 2)))
    assert SensitivityMap.uniform((2, 3), fallback=True).fallback
    cq = ChannelQuantization(2, np.array([0, 3, 1]), np.array([0.0, 1.0, 2.0, 3.0]))
    assert cq.dequantized().tolist() == [0.0, 3.0, 1.0]
    with pytest.raises(ParameterError):
        ChannelQuantization(1, np.zeros(2, dtype=np.int64), np.zeros(2))
    with pytest.raises(ShapeError):
        ChannelQuantization(2, np.zeros(2, dtype=np.int64), np.zeros(3))
    with pytest.raises(ParameterError):
        ChannelQuantization(2, np.array([4]), np.zeros(4))
