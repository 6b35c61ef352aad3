"""GPU quality harness (§8f row 2) against the reference's own outputs.

Flip tallies must equal the reference's _kernels.avalanche_counts exactly
(integer counts); reports built from them must equal the reference's
run_avalanche / zero_input_distinctness / finalization_bias_experiment
outputs for the same seeds (tests/golden/, made by gen_golden.py)."""
import numpy as np
import pytest

from conftest import GOLDEN
from paper_1612_06257_b200 import quality, synth

pytestmark = pytest.mark.gpu


def test_counts_equal_reference_kernel():
    z = np.load(GOLDEN + "/avalanche_counts.npz")
    for tag in sorted({k.rsplit("_", 1)[0] for k in z.files}):
        parts = tag.split("_")
        alg, p1, p2 = int(parts[0][1:]), int(parts[1]), int(parts[2])
        got = quality.avalanche_counts(alg, z[tag + "_key"], z[tag + "_msgs"], p1, p2)
        assert np.array_equal(got, z[tag + "_counts"]), tag


@pytest.mark.parametrize("alg,p1,p2", [(0, 4, 0), (0, 1, 0), (1, 2, 4), (1, 1, 3), (2, 2, 4)])
def test_counts_vs_oracle_all_sizes(oracle, alg, p1, p2):
    rng = np.random.default_rng(alg * 10 + p1)
    key = rng.integers(0, 2**64, 4, dtype=np.uint64)
    if alg:
        key[2:] = 0
    for size in (1, 2, 3, 7, 8, 15, 16, 24, 31, 32):
        msgs = rng.integers(0, 256, (333, size), dtype=np.uint8)
        got = quality.avalanche_counts(alg, key, msgs, p1, p2)
        assert np.array_equal(got, oracle.avalanche_counts(alg, key, msgs, p1, p2)), size


def test_counter_messages_match_explicit(oracle):
    key = synth.key256()
    n = 5000
    msgs = np.arange(n, dtype=np.uint32).view(np.uint8).reshape(-1, 4)[:, :3].copy()
    got = quality.avalanche_counts(0, key, (n, 3), 3, 0)
    assert np.array_equal(got, oracle.avalanche_counts(0, key, msgs, 3, 0))


def test_reports_equal_reference(golden):
    q = golden["quality"]
    for name in ("highway64", "siphash24", "siphash13", "siptree24", "siptree13"):
        h = quality.HashUnderTest.from_name(name)
        rep = quality.run_avalanche(h, (4, 9, 32), iterations=300, samples=3, seed=5)
        got = [[v.size, v.median_max_bias, v.passed, v.noise_floor] for v in rep.verdicts]
        assert got == q[name], name
        z = quality.zero_input_distinctness(h, 300, seed=3)
        assert [list(c) for c in z.collisions] == q[name + "_zero"]["collisions"]
        assert [int(x) for x in z.bit_population] == q[name + "_zero"]["population"]
    for r in (1, 2, 3, 4):
        fb = quality.finalization_bias_experiment(r, inputs=2**13, seed=9)
        assert [fb.max_bias, fb.mean_bias, fb.inputs] == q[f"final_r{r}"], r


def test_noise_aware_acceptance_at_full_scale():
    """T/test_acceptance.py:166-184 at its stated scale (5 x 20,000), on the GPU."""
    for name in ("highway64", "siphash24", "siphash13", "siptree24"):
        rep = quality.run_avalanche(quality.HashUnderTest.from_name(name), (4, 16, 32),
                                    iterations=20_000, samples=5, threshold=0.02)
        assert rep.passed, (name, [v.median_max_bias for v in rep.verdicts])


def test_exhaustive_finalization_experiment_runs():
    r3 = quality.finalization_bias_experiment(3, exhaustive=True, seed=9)
    r4 = quality.finalization_bias_experiment(4, exhaustive=True, seed=9)
    assert r3.inputs == r4.inputs == 2**24
    assert 0 < r4.max_bias < r3.max_bias


def test_finalization_variant(oracle):
    """S/registry.py:200-204: hash64 at a chosen finalization depth."""
    from paper_1612_06257_b200.registry import finalization_variant

    key = bytes(range(32))
    lanes = np.frombuffer(key, np.uint64)
    for r in (0, 1, 3, 4, 6):
        f = finalization_variant(r)
        for msg in (b"", b"abc", bytes(range(33))):
            assert f(key, msg) == oracle.highway(lanes, msg, r)[0]


# T/test_quality.py, the device-side tests one by one.
def test_avalanche_seed_reproducibility():
    h = quality.HashUnderTest.from_name("siphash13")
    a = quality.avalanche_bias(h, size=4, iterations=200, seed=7)
    b = quality.avalanche_bias(h, size=4, iterations=200, seed=7)
    c = quality.avalanche_bias(h, size=4, iterations=200, seed=8)
    assert np.array_equal(a.counts, b.counts)
    assert not np.array_equal(a.counts, c.counts)


def test_run_avalanche_passes_real_hash_above_noise():
    report = quality.run_avalanche(quality.HashUnderTest.from_name("siphash24"), sizes=[4],
                                   iterations=50_000, samples=3)
    assert report.passed
    assert report.verdicts[0].noise_floor == pytest.approx(0.5 / 50_000 ** 0.5)


def test_zero_input_distinctness_real_hash():
    good = quality.zero_input_distinctness(quality.HashUnderTest.from_name("highway64"),
                                           max_size=256)
    assert good.distinct and good.imbalance() < 0.25


def test_finalization_experiment_shapes():
    res = quality.finalization_bias_experiment(4, inputs=500, seed=1)
    assert (res.rounds, res.inputs, res.exhaustive) == (4, 500, False)
    assert 0.0 <= res.max_bias <= 0.5 and 0.0 <= res.mean_bias <= res.max_bias
