"""Registry drop-in (CPU): S/registry.py's names, fields and errors, the
package-level exports of S/__init__.py:40-60, the controls' digests, and the
_kernels shim's argument checks.  Digests of real hashes need the GPU
(tests/test_gpu_registry.py)."""
import pytest

import paper_1612_06257_b200 as pkg
from paper_1612_06257_b200 import _kernels, registry


def test_package_exports_registry():
    assert pkg.ALGORITHMS is registry.ALGORITHMS
    assert pkg.get_algorithm is registry.get_algorithm
    assert {"ALGORITHMS", "get_algorithm"} <= set(pkg.__all__)


def test_names_sizes_and_controls():
    want = {"highway64": (32, 8), "highway256": (32, 32), "siphash24": (16, 8),
            "siphash13": (16, 8), "siptree24": (16, 8), "siptree13": (16, 8),
            "first8bytes": (16, 8), "constant": (16, 8)}
    for name, (ks, ds) in want.items():
        a = registry.get_algorithm(name)
        assert (a.name, a.key_size, a.digest_size) == (name, ks, ds)
    controls = {n for n, a in registry.ALGORITHMS.items() if a.control}
    assert controls == {"first8bytes", "constant"}
    assert not controls & set(registry.VECTOR_ALGORITHMS)
    assert registry.get_algorithm("highway128").digest_size == 16  # the derived addition


def test_fields_match_reference():
    a = registry.get_algorithm("highway64")
    assert callable(a.hash64) and a.kernel == (0, 4, 0)
    assert registry.get_algorithm("highway256").hash64 is None
    assert registry.get_algorithm("highway256").kernel is None
    assert registry.get_algorithm("siphash13").kernel == (1, 1, 3)
    assert registry.get_algorithm("siptree24").kernel == (2, 2, 4)
    assert registry.get_algorithm("constant").kernel is None


def test_unknown_algorithm():
    with pytest.raises(ValueError, match="unknown algorithm"):
        registry.get_algorithm("md5")


def test_control_digests():
    f8 = registry.get_algorithm("first8bytes")
    assert f8.hash64(bytes(16), b"abc") == int.from_bytes(b"abc", "little")
    assert f8.digest_hex(bytes(16), b"0123456789") == b"01234567".hex()
    h = f8.make_hasher(bytes(16))
    h.append(b"ab").append(b"cdefghijk")
    assert h.finish() == int.from_bytes(b"abcdefgh", "little")
    c = registry.get_algorithm("constant")
    assert c.hash64(bytes(16), b"x") == 0 and c.digest(bytes(16), b"x") == bytes(8)
    assert c.make_hasher(bytes(16)).append(b"x").finish() == 0
    assert c.digest_batch(bytes(16), [b"", b"a"]).shape == (2, 8)


def test_random_oracle_is_not_deterministic():
    o = registry.RandomOracle(seed=1)
    assert o(b"k", b"m") != o(b"k", b"m")
    assert registry.RandomOracle(seed=1)(b"", b"") == registry.RandomOracle(seed=1)(b"", b"")


def test_kernels_shim_rejects_bad_algo():
    with pytest.raises(ValueError):
        _kernels.hash_batch(3, [0, 0, 0, 0], None, 4, 0)
    with pytest.raises(ValueError):
        _kernels._lanes([1], 2)


def test_finalization_variant_validation():
    with pytest.raises(ValueError):
        registry.finalization_variant(-1)
