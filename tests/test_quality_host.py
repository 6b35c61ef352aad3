"""The quality harness's host arithmetic (CPU): same assertions as
T/test_quality.py:13-80 (the control hashes `constant` / `first8bytes` and
RandomOracle are reference-only calibration controls, out of scope)."""
import numpy as np
import pytest

from paper_1612_06257_b200 import quality
from paper_1612_06257_b200.quality import BiasMatrix, HashUnderTest


def test_noise_floor_formula():
    assert quality.noise_floor(10_000) == pytest.approx(0.005)
    assert quality.noise_floor(100) == pytest.approx(0.05)


def test_bias_matrix_arithmetic():
    counts = np.full((32, 64), 5, dtype=np.int64)
    counts[0, 0] = 9
    mat = BiasMatrix(size=4, iterations=10, counts=counts)
    assert mat.flip_rate()[1, 1] == pytest.approx(0.5)
    assert mat.bias()[1, 1] == pytest.approx(0.0)
    assert mat.max_bias() == pytest.approx(0.4)


def test_median_bias_is_median_of_sample_maxima():
    def mat(max_count):
        counts = np.full((32, 64), 50, dtype=np.int64)
        counts[0, 0] = max_count
        return BiasMatrix(size=4, iterations=100, counts=counts)

    summary = quality.median_bias([mat(60), mat(80), mat(70)])
    assert summary.median_max_bias == pytest.approx(0.2)
    assert summary.sample_maxima == pytest.approx((0.1, 0.3, 0.2))
    assert summary.sample_count == 3


def test_median_bias_rejects_bad_sample_sets():
    mat4 = BiasMatrix(4, 10, np.zeros((32, 64), dtype=np.int64))
    with pytest.raises(ValueError):
        quality.median_bias([])
    with pytest.raises(ValueError):
        quality.median_bias([mat4, mat4])
    with pytest.raises(ValueError):
        quality.median_bias([mat4, mat4, BiasMatrix(5, 10, np.zeros((40, 64), dtype=np.int64))])


def test_avalanche_size_and_iteration_validation():
    h = HashUnderTest.from_name("siphash13")
    for size, iters in ((3, 10), (33, 10), (4, 0), (32, 2 ** 85)):
        with pytest.raises(ValueError):
            quality.avalanche_bias(h, size=size, iterations=iters)
    with pytest.raises(ValueError):
        HashUnderTest.from_name("md5")


def test_zero_input_and_finalization_validation():
    with pytest.raises(ValueError):
        quality.zero_input_distinctness(HashUnderTest.from_name("highway64"), max_size=0)
    with pytest.raises(ValueError):
        quality.finalization_bias_experiment(0)
