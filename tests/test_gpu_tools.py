"""Vector file, CLI and per-size bench through the GPU engine (§8f rows 3-4),
against the reference's own vector file and CLI output (tests/golden/)."""
import io

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1612_06257_b200 import cli, gpubench, synth, vectors
from paper_1612_06257_b200.registry import get_algorithm

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


# T/test_vectors_cli.py, one test per test (first8bytes is a reference-only
# control hash, out of scope: DESIGN.md §0).
def run_cli(capsys, *argv):
    code = cli.main(list(argv))
    cap = capsys.readouterr()
    return code, cap.out, cap.err


def test_generate_covers_all_algorithms_and_lengths():
    from paper_1612_06257_b200.registry import VECTOR_ALGORITHMS

    records = vectors.generate()
    assert len(records) == len(VECTOR_ALGORITHMS) * len(vectors.DEFAULT_LENGTHS)
    lengths = {len(r.message_hex) // 2 for r in records if r.algo == "highway64"}
    assert {0, 31, 32, 33, 64, 256, 1023, 1024} <= lengths
    assert {r.algo for r in records} == set(VECTOR_ALGORITHMS)


def test_vector_round_trip_and_verify():
    records = vectors.generate(lengths=[0, 5, 32, 33])
    buf = io.StringIO()
    vectors.write(records, buf)
    buf.seek(0)
    parsed = vectors.read(buf)
    assert parsed == records and vectors.verify(parsed) == []


def test_read_skips_comments_and_blank_lines():
    line = vectors.generate(algos=["siphash24"], lengths=[1])[0].to_line()
    assert len(vectors.read(io.StringIO(f"# header\n\n{line}\n"))) == 1


def test_cli_vectors_stdout_format(capsys):
    from paper_1612_06257_b200.registry import VECTOR_ALGORITHMS

    code, out, _ = run_cli(capsys, "vectors")
    lines = out.strip().splitlines()
    assert code == 0 and len(lines) == len(VECTOR_ALGORITHMS) * len(vectors.DEFAULT_LENGTHS)
    first = lines[0].split(",")
    assert len(first) == 4 and first[0] == "highway64"


def test_cli_hash_published_sip_vector(tmp_path, capsys):
    empty = tmp_path / "empty"
    empty.write_bytes(b"")
    code, out, _ = run_cli(capsys, "hash", "--algo", "siphash24", "--key",
                           "000102030405060708090a0b0c0d0e0f", str(empty))
    assert code == 0 and out.split()[0] == "310e0edd47db6f72"


def test_cli_hash_stdin_matches_file(tmp_path, capsys, monkeypatch):
    import sys

    data = bytes(range(200))
    path = tmp_path / "data"
    path.write_bytes(data)
    code, out_file, _ = run_cli(capsys, "hash", str(path))
    monkeypatch.setattr(sys, "stdin", type("S", (), {"buffer": io.BytesIO(data)})())
    code2, out_stdin, _ = run_cli(capsys, "hash")
    assert code == code2 == 0
    assert out_file.split()[0] == out_stdin.split()[0] and out_stdin.split()[1] == "-"


def test_cli_hash_width_256(tmp_path, capsys):
    path = tmp_path / "data"
    path.write_bytes(b"abc")
    code, out, _ = run_cli(capsys, "hash", "--algo", "highway", "--width", "256", str(path))
    assert code == 0 and len(out.split()[0]) == 64


def test_cli_hash_unreadable_input_exits_1(tmp_path, capsys):
    code, _, err = run_cli(capsys, "hash", str(tmp_path / "missing"))
    assert code == 1 and "cannot read" in err


def test_cli_avalanche_real_hash_passes(capsys):
    code, out, _ = run_cli(capsys, "avalanche", "--algo", "siphash24", "--sizes", "4",
                           "--iters", "100000", "--samples", "3")
    rows = [l for l in out.splitlines() if not l.startswith("#")]
    assert code == 0 and len(rows) == 1
    algo, size, bias, threshold, state = rows[0].split(",")
    assert (algo, size, state) == ("siphash24", "4", "pass") and float(bias) < float(threshold)


def test_cli_bench_rows(capsys):
    code, out, _ = run_cli(capsys, "bench", "--algo", "siphash13", "--sizes", "8,64", "--reps",
                           "9", "--runs", "1", "--batch-mib", "64")
    machine_rows = [l for l in out.splitlines() if l.startswith("siphash13,")]
    assert code == 0 and len(machine_rows) == 2 and machine_rows[0].split(",")[1] == "8"


def test_module_entry_point_smoke(tmp_path):
    """T/test_vectors_cli.py:205-214, with `python -m` standing in for the
    installed console script."""
    import os
    import subprocess
    import sys

    path = tmp_path / "data"
    path.write_bytes(b"hello")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    proc = subprocess.run([sys.executable, "-m", "paper_1612_06257_b200", "hash", str(path)],
                          capture_output=True, text=True, cwd=root)
    assert proc.returncode == 0
    digest = proc.stdout.split()[0]
    assert len(digest) == 16
    int(digest, 16)
