"""Vector file, CLI and per-size bench through the GPU engine (§8f rows 3-4),
against the reference's own vector file and CLI output (tests/golden/)."""
import io

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1612_06257_b200 import cli, gpubench, synth, vectors
from paper_1612_06257_b200.catalog import get_algorithm

pytestmark = pytest.mark.gpu


def _golden_lines():
    with open(GOLDEN + "/vectors_reference.txt") as f:
        return f.read().splitlines()


def test_generate_equals_reference_file():
    buf = io.StringIO()
    vectors.write(vectors.generate(), buf)
    assert buf.getvalue().splitlines() == _golden_lines()


def test_verify_reference_file_and_detect_corruption():
    with open(GOLDEN + "/vectors_reference.txt") as f:
        recs = vectors.read(f)
    assert len(recs) == 408 and vectors.verify(recs) == []
    bad = recs[:3] + [vectors.VectorRecord(recs[3].algo, recs[3].key_hex, recs[3].message_hex,
                                           "00" * (len(recs[3].digest_hex) // 2))]
    assert vectors.verify(bad) == [bad[3]]


def test_highway128_is_prefix_of_256():
    key = bytes(range(32))
    msgs = [vectors.ramp(n) for n in range(70)]
    d128 = get_algorithm("highway128").digest_batch(key, msgs)
    d256 = get_algorithm("highway256").digest_batch(key, msgs)
    assert np.array_equal(d128, d256[:, :16])


def test_cli_hash_matches_reference_cli(golden, tmp_path, capsys):
    path = tmp_path / "stream.bin"
    synth.counter_bytes(88, 200 * 1024 + 17).tofile(path)
    for name, rec in golden["cli_hash_200KiB_seed88"].items():
        argv = ["hash", "--algo", name, str(path)] + (["--key", rec["key"]] if rec["key"] else [])
        assert cli.main(argv) == 0
        out = capsys.readouterr().out.split()
        assert out == [rec["line"], str(path)], name


def test_cli_vectors_and_verify(tmp_path, capsys):
    out = tmp_path / "v.txt"
    assert cli.main(["vectors", "--out", str(out)]) == 0
    assert out.read_text().splitlines() == _golden_lines()
    assert cli.main(["verify", str(out)]) == 0
    lines = out.read_text().splitlines()
    a, k, m, d = lines[10].split(",")
    lines[10] = ",".join([a, k, m, ("0" if d[0] != "0" else "1") + d[1:]])
    out.write_text("\n".join(lines) + "\n")
    capsys.readouterr()
    assert cli.main(["verify", str(out)]) == 1
    assert "407/408" in capsys.readouterr().out


def test_cli_avalanche_and_bench(capsys):
    assert cli.main(["avalanche", "--algo", "highway64", "--sizes", "4,8", "--iters", "400",
                     "--samples", "3"]) in (0, 1)
    lines = [l for l in capsys.readouterr().out.splitlines() if l and not l.startswith("#")]
    assert [l.split(",")[1] for l in lines] == ["4", "8"]
    assert cli.main(["bench", "--algo", "siphash13,highway64", "--sizes", "8,1024",
                     "--reps", "3", "--batch-mib", "64"]) == 0
    rows = [l for l in capsys.readouterr().out.splitlines() if l.count(",") == 5]
    assert len(rows) == 4


def test_gpubench_presets():
    assert gpubench.PRESETS["table1"] == (8, 31, 32, 63, 64, 1024)
    rows = gpubench.sweep("highway64", [1, 33], batch_bytes=1 << 20, steps=2)
    assert [r.size for r in rows] == [1, 33] and all(r.msgs_per_s > 0 for r in rows)
