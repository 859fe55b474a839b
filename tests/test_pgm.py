"""PGM frame / mask I/O (host logic; reference pkg/src/fase/pgm.py behaviour)."""

import numpy as np
import pytest

from paper_2204_14194_b200 import FormatError, ShapeError, read_mask_pgm, read_pgm, write_pgm


def test_round_trip_and_mask(tmp_path):
    img = np.arange(35, dtype=np.uint8).reshape(5, 7) * 7
    p = tmp_path / "a.pgm"
    write_pgm(p, img)
    assert p.read_bytes()[:11] == b"P5\n7 5\n255\n"
    assert np.array_equal(read_pgm(p), img)
    assert np.array_equal(read_mask_pgm(p), img == 0)


def test_write_rounds_clamps_and_drops_imaginary(tmp_path):
    p = tmp_path / "b.pgm"
    write_pgm(p, np.array([[-3.0, 0.5, 1.5, 254.6, 300.0]]))
    assert read_pgm(p).tolist() == [[0, 0, 2, 255, 255]]  # rint: half to even
    write_pgm(p, np.array([[10.2 + 99j, 3.7 - 5j]]))
    assert read_pgm(p).tolist() == [[10, 4]]


def test_header_comments_and_errors(tmp_path):
    p = tmp_path / "c.pgm"
    p.write_bytes(b"P5\n# made by hand\n2 # width\n1\n# maxval next\n255\n" + bytes([9, 200]))
    assert read_pgm(p).tolist() == [[9, 200]]
    for blob in (b"P2\n1 1\n255\n\x00", b"P5\n2 2\n255\n\x00\x01", b"P5\n1 1\n65535\n\x00\x00",
                 b"P5\n1 1", b"P5\n1 x 255\n\x00", b"P5\n0 1\n255\n"):
        p.write_bytes(blob)
        with pytest.raises(FormatError):
            read_pgm(p)
    with pytest.raises(ShapeError):
        write_pgm(p, np.zeros(4))
    with pytest.raises(ShapeError):
        write_pgm(p, np.zeros((0, 3)))
