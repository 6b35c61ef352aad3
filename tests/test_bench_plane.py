"""bench.py's multi-GPU control plane on CPU (gloo, world size 2): the
self-spawn of N ranks when --gpus N runs without torchrun, message-index
shards (weak and strong), max-over-ranks time, whole-job value and the
per-rank checksum gather -- the same code the NCCL run uses."""
import json
import os

import numpy as np
import pytest

import bench


def _entry(args):
    """Stand-in for run_ours: the control plane only, on gloo."""
    plane = bench.Plane("gloo")
    ws, rank = plane.ws, plane.rank
    start, stop = bench.headline_shard(ws, rank, args.scaling, args.msgs)
    # rank-dependent fake timings: rank 1 is the slow one
    total_ms = 10.0 * (rank + 1)
    s = bench.summarise(plane, [total_ms], total_ms, (stop - start) * bench.MSG_BYTES, 1,
                        args.scaling, args.msgs * bench.MSG_BYTES)
    folds = plane.gather_u64(0xF000000000000000 + rank)
    plane.barrier()
    if rank == 0:
        with open(os.environ["PLANE_OUT"] + f".{args.scaling}", "w") as f:
            json.dump({"ws": ws, "value": s["value"], "t_max": s["t_max_ms"],
                       "bytes": s["bytes_per_step"], "folds": folds,
                       "shards": [bench.headline_shard(ws, r, args.scaling, args.msgs)
                                  for r in range(ws)]}, f)
    plane.close()
    return 0


@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_self_spawned_two_rank_plane(tmp_path, monkeypatch, scaling):
    monkeypatch.delenv("RANK", raising=False)
    out = str(tmp_path / "plane")
    monkeypatch.setenv("PLANE_OUT", out)
    argv = ["--gpus", "2", "--msgs", "1000", "--scaling", scaling]
    bench.spawn(bench.parse(argv), argv, entry=_entry)
    r = json.load(open(out + f".{scaling}"))
    assert r["ws"] == 2 and r["t_max"] == 20.0
    assert r["folds"] == [0xF000000000000000, 0xF000000000000001]
    if scaling == "weak":  # 1000 messages per rank
        assert r["shards"] == [[0, 1000], [1000, 2000]]
        assert r["bytes"] == 2000 * bench.MSG_BYTES
    else:  # one global batch of 1000 split in two
        assert r["shards"] == [[0, 500], [500, 1000]]
        assert r["bytes"] == 1000 * bench.MSG_BYTES
    assert r["value"] == pytest.approx(r["bytes"] / 0.020 / 1e9)


def test_gpus_must_match_torchrun_world(monkeypatch):
    monkeypatch.setenv("RANK", "0")
    monkeypatch.setenv("WORLD_SIZE", "2")
    with pytest.raises(SystemExit, match="WORLD_SIZE=2"):
        bench.main(["--gpus", "4"])


def test_config_identical_across_arms():
    assert bench.config_dict(1, "weak", bench.N_MSGS)["workload"].startswith("hh64_2^24x1KiB")
    assert bench.config_dict(2, "strong", 1 << 23)["global_messages"] == bench.N_MSGS


def test_reference_arm_on_cpu(capsys):
    """--impl reference runs the CPU implementation only (no GPU): one JSON
    line with the contract's keys and the same config dict as our arm."""
    assert bench.main(["--impl", "reference", "--steps", "1", "--warmup", "3",
                       "--msgs", "4096"]) == 0
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["steps"] == 1
    assert line["config"] == bench.config_dict(1, "weak", 4096)
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"
    from oracle import oracle as orc
    from paper_1612_06257_b200 import synth

    msgs = orc.synth_fill(4096 * 1024, bench.DATA_SEED).reshape(4096, 1024)
    fold = np.bitwise_xor.reduce(orc.batch_fixed(orc.ALG_HIGHWAY, synth.key256(), msgs, 64, 4))
    assert line["checksum"] == f"{int(fold):016x}"
