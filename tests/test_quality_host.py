"""The quality harness's host arithmetic (CPU): same assertions as
T/test_quality.py, including the calibration controls `constant`,
`first8bytes` and RandomOracle, which have no device kernel and run through
the harness's host loop exactly as in the reference (S/quality.py:119-131)."""
import numpy as np
import pytest

from paper_1612_06257_b200 import quality
from paper_1612_06257_b200.quality import BiasMatrix, HashUnderTest
from paper_1612_06257_b200.registry import RandomOracle, get_algorithm


def _hut(name):
    return HashUnderTest.from_algorithm(get_algorithm(name))


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


# T/test_quality.py:18-28 -- the control hashes.
def test_constant_hash_has_maximal_bias():
    mat = quality.avalanche_bias(_hut("constant"), size=4, iterations=50)
    assert mat.counts.shape == (32, 64)
    assert np.all(mat.counts == 0)
    assert mat.max_bias() == pytest.approx(0.5)


def test_first8bytes_is_diagonal():
    mat = quality.avalanche_bias(_hut("first8bytes"), size=8, iterations=20)
    rates = mat.flip_rate()
    assert np.all(rates[np.arange(64), np.arange(64)] == 1.0)
    off = rates.copy()
    off[np.arange(64), np.arange(64)] = 0.0
    assert np.all(off == 0.0)
    assert mat.max_bias() == pytest.approx(0.5)


def test_control_avalanche_validation():
    h = _hut("constant")
    for size, iters in ((3, 10), (33, 10), (4, 0), (32, 2 ** 85)):
        with pytest.raises(ValueError):
            quality.avalanche_bias(h, size=size, iterations=iters)


def test_run_avalanche_fails_weak_hash():
    report = quality.run_avalanche(_hut("first8bytes"), sizes=[8], iterations=100, samples=3)
    assert not report.passed
    assert report.verdicts[0].median_max_bias == pytest.approx(0.5)


def test_random_oracle_bias_is_pure_noise():
    h = HashUnderTest("oracle", 16, RandomOracle(seed=11))
    iterations = 2000
    mat = quality.avalanche_bias(h, size=4, iterations=iterations, seed=11)
    assert mat.max_bias() < 5.5 * quality.noise_floor(iterations)


def test_zero_input_controls():
    const = quality.zero_input_distinctness(_hut("constant"), max_size=64)
    assert not const.distinct
    assert len(const.collisions) == 64
    assert const.imbalance() == pytest.approx(0.5)
    assert not quality.zero_input_distinctness(_hut("first8bytes"), max_size=64).distinct
    with pytest.raises(ValueError):
        quality.zero_input_distinctness(_hut("constant"), max_size=0)


def test_hash_under_test_fields_match_reference():
    h = _hut("highway64")
    assert (h.name, h.key_size, h.kernel) == ("highway64", 32, (0, 4, 0))
    assert _hut("siptree13").kernel == (2, 1, 3)
    assert _hut("constant").kernel is None
    with pytest.raises(ValueError):
        _hut("highway256")  # no 64-bit digest
