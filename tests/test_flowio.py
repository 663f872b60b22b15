"""Wire formats (reference flowio.py) — byte-for-byte against files written
and decoded by the reference itself (tests/golden/next_flowio.npz)."""

import numpy as np
import pytest

from paper_1603_03590_b200 import flowio
from tests.conftest import golden


def test_write_flo_bytes_match_reference(tmp_path):
    g = golden("next_flowio.npz")
    p = tmp_path / "a.flo"
    flowio.write_flo(g["flo_in"], p)
    assert p.read_bytes() == g["flo_bytes"].tobytes()
    assert flowio.flo_bytes(g["flo_in"]) == g["flo_bytes"].tobytes()


def test_read_flo_matches_reference(tmp_path):
    g = golden("next_flowio.npz")
    p = tmp_path / "a.flo"
    p.write_bytes(g["flo_bytes"].tobytes())
    got = flowio.read_flo(p)
    assert got.dtype == np.float64 and np.array_equal(got, g["flo_read"])
    assert np.array_equal(flowio.flow_valid_mask(g["flo_in"]), g["mask"])


@pytest.mark.parametrize("name,suffix", [("pgm8", "pgm"), ("pgm16", "pgm"), ("ppm", "ppm")])
def test_read_image_matches_reference(tmp_path, name, suffix):
    g = golden("next_flowio.npz")
    p = tmp_path / f"x.{suffix}"
    p.write_bytes(g[f"{name}_bytes"].tobytes())
    got = flowio.read_image(p)
    assert np.array_equal(got, g[f"{name}_img"])


def test_read_frame_u8_is_exact(tmp_path):
    g = golden("next_flowio.npz")
    p = tmp_path / "x.pgm"
    p.write_bytes(g["pgm8_bytes"].tobytes())
    raw = flowio.read_frame_u8(p)
    assert raw.dtype == np.uint8
    assert np.array_equal(raw.astype(np.float64), g["pgm8_img"])


def test_write_image_bytes_match_reference(tmp_path):
    g = golden("next_flowio.npz")
    flowio.write_image(g["wimg_in"], tmp_path / "d.pgm")
    assert (tmp_path / "d.pgm").read_bytes() == g["wimg_bytes"].tobytes()
    flowio.write_image(g["wrgb_in"], tmp_path / "e.ppm")
    assert (tmp_path / "e.ppm").read_bytes() == g["wrgb_bytes"].tobytes()


def test_format_errors(tmp_path):
    with pytest.raises(flowio.FileFormatError):
        flowio.write_image(np.zeros((2, 3, 4)), tmp_path / "bad.pgm")
    p = tmp_path / "t.flo"
    p.write_bytes(b"PIEH")
    with pytest.raises(flowio.FileFormatError):
        flowio.read_flo(p)
    p.write_bytes(b"\x00" * 12)
    with pytest.raises(flowio.FileFormatError):
        flowio.read_flo(p)
    with pytest.raises(ValueError):
        flowio.write_flo(np.full((2, 2, 2), np.nan), tmp_path / "n.flo")
    with pytest.raises(ValueError):
        flowio.write_flo(np.zeros((2, 2, 3)), tmp_path / "s.flo")
    q = tmp_path / "t.pgm"
    q.write_bytes(b"P2\n1 1\n255\n0")
    with pytest.raises(flowio.FileFormatError):
        flowio.read_image(q)
    q.write_bytes(b"P5\n4 4\n255\n" + b"\x00" * 3)
    with pytest.raises(flowio.FileFormatError):
        flowio.read_image(q)
    q.write_bytes(b"P5\n4 x\n255\n")
    with pytest.raises(flowio.FileFormatError):
        flowio.read_image(q)
    q.write_bytes(b"P5\n4 4\n70000\n" + b"\x00" * 64)
    with pytest.raises(flowio.FileFormatError):
        flowio.read_image(q)
