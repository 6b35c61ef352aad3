"""Canonical op counts of SURVEY.md §8(d) and the integer-roof arithmetic
(paper_1612_06257_b200/introof.py), CPU only."""
import pytest

from paper_1612_06257_b200 import introof


def test_canonical_counts_match_survey_table():
    assert introof.highway_mix(1024, 64).total() == 2884
    assert introof.prf_mix().total() == 420
    assert introof.sip_mix(1024, 2, 4).total() == 6813
    assert introof.sip_mix(1024, 1, 3).total() == 3693
    assert introof.siptree_mix(1024, 2, 4).total() == 7649
    assert introof.siptree_mix(1024, 1, 3).total() == 4241
    assert introof.UPDATE.total() == 80 and introof.SIPROUND.total() == 24
    # cfg3: mean over U[8, 64] of the per-length count is SURVEY's 464
    mean = sum(introof.highway_mix(L, 64).total() for L in range(8, 65)) / 57
    assert round(mean) == 464


def _peaks(alu=1.0, imad=1.0, wide=0.5, issue=2.0):
    cls = {k: {"warp_instr_per_s": alu} for k in introof.ALU}
    cls["imad"] = {"warp_instr_per_s": imad}
    cls["wide"] = {"warp_instr_per_s": wide}
    return {"classes": cls, "issue_warp_instr_per_s": issue}


def test_roof_canonical_and_balanced():
    m = introof.UPDATE  # ALU 16+16+24 + hi 16 = 72; FMA 8 wide at half rate = 16
    p = _peaks()
    assert introof.roof_seconds(m, p, balanced=False) == pytest.approx(72.0)
    # balanced: move x highs to FMA: ALU 72 - x, FMA 16 + x -> x = 16 -> 56
    assert introof.roof_seconds(m, p, balanced=True) == pytest.approx(56.0)
    # issue-bound when the issue ceiling is low
    assert introof.roof_seconds(m, _peaks(issue=1.0), balanced=True) == pytest.approx(80.0)


def test_launch_roof_scales_with_messages():
    r = introof.launch_roof(introof.highway_mix(1024), 32 * 1000, _peaks())
    assert r["canonical_ops_per_launch"] == 2884 * 32000
    assert r["t_int_balanced_ms"] <= r["t_int_canonical_ms"]


def test_slot_bound():
    # Update: 16 IADD3 + 16 LOP3 + 24 PRMT + 8 IMAD.WIDE; SipRound: 4 + 8 + 8.
    assert introof.slots(introof.UPDATE) == 64 and introof.slots(introof.SIPROUND) == 20
    p = _peaks()
    assert introof.slot_seconds(introof.UPDATE, p) == pytest.approx(64.0)
    r = introof.launch_roof(introof.sip_mix(1024, 2, 4), 32, p)
    assert r["t_int_slot_ms"] >= r["t_int_balanced_ms"]
    assert r["alu_slots_per_msg"] == introof.slots(introof.sip_mix(1024, 2, 4))
