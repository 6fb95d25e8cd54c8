"""Weight files (CPKW0001, the reference's format) and ciphertext blobs."""

import os

import numpy as np
import pytest

from paper_2102_03494_b200.netspec import WeightFileError, WeightSet, WeightTensor
from paper_2102_03494_b200.params import make_params
from paper_2102_03494_b200.rlwe import Evaluator
from paper_2102_03494_b200.wire import ct_from_bytes, ct_to_bytes, load_weights, save_weights

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_reads_a_file_written_by_the_reference():
    ws = load_weights(os.path.join(GOLD, "weights_ref.cpkw"))
    assert ws.names() == ["layer0.weight", "layer0.bias"]
    assert ws["layer0.weight"].values.tolist() == np.arange(-12, 12).reshape(2, 3, 4).tolist()
    assert ws["layer0.weight"].scale == 0.125 and ws["layer0.bias"].values.tolist() == [7, -3]


def test_round_trip_is_byte_identical_to_the_reference_writer(tmp_path):
    ws = load_weights(os.path.join(GOLD, "weights_ref.cpkw"))
    out = tmp_path / "w.cpkw"
    save_weights(ws, out)
    assert out.read_bytes() == open(os.path.join(GOLD, "weights_ref.cpkw"), "rb").read()


def test_corruption_is_detected(tmp_path):
    raw = bytearray(open(os.path.join(GOLD, "weights_ref.cpkw"), "rb").read())
    bad = tmp_path / "bad.cpkw"
    raw[-1] ^= 0xFF
    bad.write_bytes(bytes(raw))
    with pytest.raises(WeightFileError):
        load_weights(bad)
    bad.write_bytes(b"NOTAFILE" + bytes(raw[8:]))
    with pytest.raises(WeightFileError):
        load_weights(bad)
    with pytest.raises(WeightFileError):
        save_weights(WeightSet([WeightTensor("x", np.array([1 << 40]), 8, 1.0)]), tmp_path / "big.cpkw")


def test_ciphertext_blob_round_trip(golden_lib):
    P = make_params(16, [65537], levels=3, q_bits=50)
    ev = Evaluator(P, golden_lib)
    s = np.arange(2 * 32, dtype=np.uint64).reshape(1, 2, 32) % 65537
    ct = ev.encrypt(s)
    back = ct_from_bytes(ev, ct_to_bytes(ev, ct))
    assert np.array_equal(ev.read(back), ev.read(ct)) and np.array_equal(ev.decrypt(back), s)
    other = Evaluator(make_params(16, [65537], levels=3, q_bits=45), golden_lib)
    with pytest.raises(ValueError):
        ct_from_bytes(other, ct_to_bytes(ev, ct))
