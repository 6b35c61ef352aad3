"""lanehash.sip's host-level helpers, mirrored in paper_1612_06257_b200.sip
(CPU; no device).  Same assertions as T/test_sip.py:140-152 and
T/test_tree.py:22-38; the device-level ones are in
tests/test_gpu_sip_module.py."""
import struct

import pytest

from paper_1612_06257_b200.sip import Key128, SipParams, deinterleave, sip_round


def test_deinterleave_word_assignment():
    words = [0xA0, 0xA1, 0xA2, 0xA3, 0xB0, 0xB1, 0xB2, 0xB3]
    lanes = deinterleave(struct.pack("<8Q", *words))
    for j in range(4):
        assert struct.unpack("<2Q", lanes[j]) == (words[j], words[4 + j])


def test_deinterleave_zero_pads_to_packet_multiple():
    lanes = deinterleave(b"\x01")
    assert [len(lane) for lane in lanes] == [8, 8, 8, 8]
    assert struct.unpack("<Q", lanes[0])[0] == 1
    assert all(lanes[j] == bytes(8) for j in range(1, 4))
    assert deinterleave(b"") == (b"", b"", b"", b"")


def test_params_validation():
    with pytest.raises(ValueError):
        SipParams(0, 4)
    with pytest.raises(ValueError):
        SipParams(2, 0)


def test_key128_round_trip():
    raw = bytes(range(16))
    assert Key128.from_bytes(raw).to_bytes() == raw
    assert Key128.from_hex(raw.hex()) == Key128.from_bytes(raw)
    with pytest.raises(ValueError):
        Key128.from_bytes(bytes(8))


def test_sip_round_validates_before_device():
    with pytest.raises(ValueError):
        sip_round((1, 2, 3))
