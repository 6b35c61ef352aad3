"""Integer-pipe roofline of each hash.

The integer roof of a launch is its canonical 32-bit op mix (SURVEY §8(d):
Update = 80 ops, SipRound = 24, ...) priced at the per-class SASS rates
measured on this B200 by tools/intpeak.cu (profiles/int_peak.json).  Each
op class runs on one pipe (ALU: IADD3, LOP3, PRMT, SHF; FMA: IMAD, IMAD.X,
IMAD.WIDE), so a mix takes at least

    t = max( sum_ALU n_k / r_k ,  sum_FMA n_k / r_k ,  sum_all n_k / r_issue )

where r_k is class k's measured warp-instruction rate alone (its pipe
saturated) and r_issue the measured dual-issue ceiling.  Two variants:

* ``canonical`` -- SURVEY's mix as written: every 64-bit add is IADD3 +
  IADD3.X on the ALU pipe.
* ``balanced`` -- the same op count, but the high half of each 64-bit add
  may run as IMAD.X on the FMA pipe (what the engine does; add64_mixed in
  csrc/lh_device.cuh), split to minimise t.  This is the tighter (lower)
  bound for any implementation with the canonical op count.

* ``slot`` -- what tools/issuemix.cu measured on this B200
  (profiles/r2_issuemix.json): a 32-bit-result IMAD / IMAD.X issues beside
  an ALU-pipe instruction at no cost (1:1 mixes run at 0.95 warp
  instructions per clock per SM sub-partition), but an instruction with a
  64-bit or high-half product (IMAD.WIDE, IMAD.HI) holds the issue port of
  the ALU pipe for one ALU slot as well as its own 4 FMA clocks: x ALU
  instructions + 1 IMAD.WIDE take 2x + 2 clocks for every x >= 1.  So a mix
  needs at least (ALU-class ops + IMAD.WIDE ops) ALU slots of 2 clocks each
  per warp, however its high halves are split -- the bound that explains why
  every SipRound instruction selection runs at 40-43 clocks per warp-round
  (20 slots) and the HighwayHash Update at 138 (64 slots = 128 clocks).

Per-message op counts:
    HighwayHash  80*(floor(L/32)+4) + 96*[L%32 != 0] + 4*(w/64)
    SipHash-c-d  (floor(L/8)+1)*(4+24c) + 24d + 9
    SipTreeHash  4*Sip(Lpad/4) + Sip(32)
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass, field
from typing import Dict, Optional

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
INT_PEAK = os.path.join(ROOT, "profiles", "int_peak.json")

ALU = ("iadd3", "lop3", "prmt", "shf")
FMA = ("imad", "wide")


@dataclass
class Mix:
    """32-bit op counts by class.  ``hi`` = high halves of 64-bit adds
    (IADD3.X on ALU or IMAD.X on FMA; priced as iadd3 or imad)."""

    n: Dict[str, float] = field(default_factory=dict)
    hi: float = 0.0

    def add(self, other: "Mix", times: float = 1.0) -> "Mix":
        for k, v in other.n.items():
            self.n[k] = self.n.get(k, 0.0) + v * times
        self.hi += other.hi * times
        return self

    def total(self) -> float:
        return sum(self.n.values()) + self.hi


def _mix(hi=0.0, **n) -> Mix:
    return Mix({k: float(v) for k, v in n.items()}, float(hi))


# S/highway.py:130-150: 8 IADD3 lows + 8 highs of the 4x(v1+=p+m0) and
# 4x(v0+=m1) adds, 8+8 of the 8 zipper adds, 16 LOP3 (8 xor64), 8
# IMAD.WIDE (mul32), 24 PRMT (zipper, 6 per 16-byte pair x 4).
UPDATE = _mix(hi=16, iadd3=16, lop3=16, wide=8, prmt=24)
REMAINDER_EXTRA = _mix(iadd3=8, shf=8)  # S/highway.py:188-197: half-adds + rotates
SIPROUND = _mix(hi=4, iadd3=4, shf=8, lop3=8)  # S/sip.py:73-86


def highway_mix(L: int, width: int = 64) -> Mix:
    m = Mix().add(UPDATE, L // 32 + 4)
    if L % 32:
        m.add(UPDATE).add(REMAINDER_EXTRA)
    lanes = width // 64
    return m.add(_mix(hi=2 * lanes, iadd3=2 * lanes))  # 4 ops per output lane


def sip_mix(L: int, c: int, d: int) -> Mix:
    words = L // 8 + 1
    return Mix().add(SIPROUND, words * c + d).add(_mix(lop3=4 * words + 9))


def siptree_mix(L: int, c: int, d: int) -> Mix:
    pad = -(-L // 32) * 32
    return Mix().add(sip_mix(pad // 4, c, d), 4).add(sip_mix(32, c, d))


def prf_mix() -> Mix:
    return highway_mix(8, 64)


def load_peaks(path: str = INT_PEAK) -> Optional[dict]:
    try:
        with open(path) as f:
            j = json.load(f)
    except (OSError, ValueError):
        return None
    return j if "classes" in j and "issue_warp_instr_per_s" in j else None


def _times(mix: Mix, peaks: dict, hi_on_alu: float):
    r = {k: v["warp_instr_per_s"] for k, v in peaks["classes"].items()}
    alu = sum(mix.n.get(k, 0.0) / r[k] for k in ALU) + hi_on_alu / r["iadd3"]
    fma = sum(mix.n.get(k, 0.0) / r[k] for k in FMA) + (mix.hi - hi_on_alu) / r["imad"]
    issue = mix.total() / peaks["issue_warp_instr_per_s"]
    return alu, fma, issue


def roof_seconds(mix: Mix, peaks: dict, balanced: bool) -> float:
    """Lower bound on warp-seconds per message (multiply by messages/32)."""
    if not balanced:
        return max(_times(mix, peaks, mix.hi))
    # t_ALU grows and t_FMA shrinks linearly in the ALU share x of the
    # high halves: the minimum of the max is at an end or the crossing.
    best = min(max(_times(mix, peaks, x)) for x in (0.0, mix.hi))
    a0, f0, _ = _times(mix, peaks, 0.0)
    a1, f1, _ = _times(mix, peaks, mix.hi)
    da, df = a1 - a0, f1 - f0
    if mix.hi and da != df:
        x = mix.hi * (f0 - a0) / (da - df)
        if 0.0 <= x <= mix.hi:
            best = min(best, max(_times(mix, peaks, x)))
    return best


def slot_seconds(mix: Mix, peaks: dict) -> float:
    """ALU-slot bound (module docstring): every ALU-class op and every
    IMAD.WIDE takes one slot of the ALU pipe's measured rate; the high
    halves of 64-bit adds ride the FMA pipe for free (IMAD.X)."""
    r = {k: v["warp_instr_per_s"] for k, v in peaks["classes"].items()}
    return sum(mix.n.get(k, 0.0) / r[k] for k in ALU) + mix.n.get("wide", 0.0) / r["lop3"]


def slots(mix: Mix) -> float:
    return sum(mix.n.get(k, 0.0) for k in ALU) + mix.n.get("wide", 0.0)


def launch_roof(mix: Mix, n_msgs: float, peaks: Optional[dict] = None) -> Optional[dict]:
    """Integer roof of a launch hashing n_msgs messages of this mix:
    canonical-op totals and the two bounds in ms."""
    peaks = peaks if peaks is not None else load_peaks()
    if not peaks:
        return None
    warps = n_msgs / 32.0
    can = roof_seconds(mix, peaks, balanced=False) * warps
    bal = roof_seconds(mix, peaks, balanced=True) * warps
    slot = max(slot_seconds(mix, peaks) * warps, bal)
    return {"canonical_ops_per_msg": round(mix.total(), 2),
            "canonical_ops_per_launch": round(mix.total() * n_msgs),
            "t_int_canonical_ms": round(can * 1e3, 4),
            "t_int_balanced_ms": round(bal * 1e3, 4),
            "alu_slots_per_msg": round(slots(mix), 2),
            "t_int_slot_ms": round(slot * 1e3, 4),
            "clock_mhz": peaks.get("sm_mhz"),
            "source": "profiles/int_peak.json (tools/intpeak.cu per-class rates) x SURVEY "
                      "§8(d) canonical mix (paper_1612_06257_b200/introof.py); slot bound: "
                      "profiles/r2_issuemix.json (tools/issuemix.cu)"}
