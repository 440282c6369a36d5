"""NDTENSOR / PGM file formats, CPU only.

The B200 library's readers and writers (csrc/ndc_io.cu) are pinned against the
reference's own imageio.hpp, compiled into oracle/_ref (ref_shim.cpp ref_io_*): the
same bytes out of every writer, the same values or the same error class out of every
reader, including all truncations and random single-byte corruptions.  The case list
restates tests/test_imageio.cpp:41-190.  Where oracle/_ref is absent (it is built
by __graft_entry__.build() and travels with the tree), the committed byte fixtures in
tests/golden/io/ (written by the reference; tests/golden/make_golden_io.py) still pin
the formats.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1711_11224_b200 import ndconv as nd

GOLD_IO = os.path.join(os.path.dirname(__file__), "golden", "io")
HAVE_REF = O.available("ref")
needs_ref = pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def ref():
    return O.Oracle("ref")


def _bytes_to_file(tmp_path, data: bytes, name="t.ndt"):
    p = tmp_path / name
    p.write_bytes(data)
    return str(p)


def _ours_parse(tmp_path, data: bytes, pgm=False):
    """(kind, array|None) from the B200 reader on ``data``."""
    path = _bytes_to_file(tmp_path, data, "x.pgm" if pgm else "x.ndt")
    try:
        return "ok", (nd.read_pgm(path) if pgm else nd.read_tensor(path))
    except nd.FormatError:
        return "FormatError", None
    except nd.Error as e:
        return type(e).__name__, None


def _ref_parse(ref, data: bytes, pgm=False):
    try:
        return "ok", (ref.parse_pgm(data) if pgm else ref.parse_tensor(data))
    except O.OracleError as e:
        return e.kind, None


def _same_outcome(tmp_path, ref, data, pgm=False):
    ko, vo = _ours_parse(tmp_path, data, pgm)
    kr, vr = _ref_parse(ref, data, pgm)
    assert ko == kr, (data[:60], ko, kr)
    if ko == "ok":
        assert vo.shape == vr.shape
        assert vo.tobytes() == vr.tobytes()


def _good_tensor():
    return np.array([[1.5, -2.25, 0.0], [1e-300, -0.0, 3.0e300]], np.float64)


# --- NDTENSOR ----------------------------------------------------------------------------
def test_tensor_round_trip_bit_exact(tmp_path):
    rng = np.random.default_rng(11)
    special = np.array([0.0, -0.0, 5e-324, -5e-324, np.finfo(np.float64).max, np.finfo(np.float64).tiny])
    for shape in [(1,), (7,), (3, 4), (2, 3, 5), (2, 1, 3, 1, 2)]:
        t = rng.standard_normal(shape) * 10.0 ** rng.integers(-200, 200, size=shape)
        t.flat[: min(t.size, special.size)] = special[: min(t.size, special.size)]
        p = str(tmp_path / "r.ndt")
        nd.write_tensor(t, p)
        back = nd.read_tensor(p)
        assert back.shape == t.shape
        assert back.tobytes() == np.ascontiguousarray(t).tobytes()


def test_tensor_header_is_human_readable(tmp_path):
    p = str(tmp_path / "h.ndt")
    nd.write_tensor(np.zeros((2, 3)), p)
    data = open(p, "rb").read()
    assert data.split(b"\n", 1)[0] == b"NDTENSOR 2 2 3"
    assert len(data) == len(b"NDTENSOR 2 2 3\n") + 6 * 8


@needs_ref
def test_tensor_writer_bytes_equal_reference(tmp_path, ref):
    rng = np.random.default_rng(12)
    for shape in [(1,), (5, 4), (3, 2, 7), (2, 2, 2, 2)]:
        t = rng.standard_normal(shape)
        p = str(tmp_path / "w.ndt")
        nd.write_tensor(t, p)
        assert open(p, "rb").read() == ref.serialize_tensor(t)


MALFORMED_TENSORS = [b"", b"BADMAGIC 1 2\n", b"NDTENSOR 0\n", b"NDTENSOR -1 4\n", b"NDTENSOR 2 3\n",
                     b"NDTENSOR 1 4 junk\n", b"NDTENSOR 1 0\n", b"NDTENSOR\n", b"NDTENSOR 1 x\n",
                     b"NDTENSOR 1 2", b"NDTENSOR 2 99999999999 99999999999\n",
                     b"NDTENSOR 3 2 2 2\n" + b"\0" * 63]


@pytest.mark.parametrize("data", MALFORMED_TENSORS)
def test_malformed_tensor_headers_raise_format_errors(tmp_path, data):
    kind, _ = _ours_parse(tmp_path, data)
    assert kind == "FormatError"
    if HAVE_REF:
        assert _ref_parse(O.Oracle("ref"), data)[0] == "FormatError"


def test_trailing_bytes_rejected(tmp_path):
    p = str(tmp_path / "g.ndt")
    nd.write_tensor(_good_tensor(), p)
    good = open(p, "rb").read()
    assert _ours_parse(tmp_path, good + b"extra")[0] == "FormatError"


def test_non_finite_payloads_refused_both_directions(tmp_path):
    for bad in (np.nan, np.inf, -np.inf):
        t = _good_tensor()
        t[1, 1] = bad
        raw = b"NDTENSOR 2 2 3\n" + t.astype("<f8").tobytes()
        assert _ours_parse(tmp_path, raw)[0] == "FormatError"
        with pytest.raises(nd.NumericError):
            nd.write_tensor(t, str(tmp_path / "n.ndt"))


@needs_ref
def test_every_truncation_fails_like_reference(tmp_path, ref):
    p = str(tmp_path / "g.ndt")
    nd.write_tensor(_good_tensor(), p)
    good = open(p, "rb").read()
    for n in range(len(good)):
        assert _ours_parse(tmp_path, good[:n])[0] == "FormatError", n
        assert _ref_parse(ref, good[:n])[0] == "FormatError", n


@needs_ref
def test_random_byte_corruption_matches_reference(tmp_path, ref):
    p = str(tmp_path / "g.ndt")
    nd.write_tensor(np.arange(1.0, 13.0).reshape(3, 4), p)
    good = open(p, "rb").read()
    rng = np.random.default_rng(13)
    for _ in range(400):
        b = bytearray(good)
        pos = int(rng.integers(0, len(b)))
        b[pos] = int(rng.integers(0, 256))
        _same_outcome(tmp_path, ref, bytes(b))


def test_missing_files_are_format_errors():
    with pytest.raises(nd.FormatError):
        nd.read_tensor("/nonexistent/x.ndt")
    with pytest.raises(nd.FormatError):
        nd.read_pgm("/nonexistent/x.pgm")
    with pytest.raises(nd.FormatError):
        nd.write_tensor(np.ones(2), "/nonexistent/dir/x.ndt")


# --- PGM ---------------------------------------------------------------------------------
def test_binary_graymap_round_trips_integer_images(tmp_path):
    img = np.arange(12, dtype=np.float64).reshape(3, 4) * 20.0
    p = str(tmp_path / "i.pgm")
    nd.write_pgm(img, p, clamp=False)
    assert np.array_equal(nd.read_pgm(p), img)


def test_ascii_graymap_with_comments(tmp_path):
    data = b"P2\n# a comment\n3 2 # trailing comment\n255\n0 10 20\n30 40 255\n"
    kind, v = _ours_parse(tmp_path, data, pgm=True)
    assert kind == "ok"
    assert np.array_equal(v, np.array([[0, 10, 20], [30, 40, 255]], np.float64))


def test_wide_graymap_reads_big_endian_samples(tmp_path):
    data = b"P5 4 1 65535\n" + bytes([0, 0, 0, 255, 1, 0, 255, 255])
    kind, v = _ours_parse(tmp_path, data, pgm=True)
    assert kind == "ok"
    assert np.array_equal(v, np.array([[0, 255, 256, 65535]], np.float64))


def test_graymap_writing_validates_and_rounds_half_even(tmp_path):
    p = str(tmp_path / "r.pgm")
    nd.write_pgm(np.array([[0.4, 1.5, 2.5, 253.5]]), p, clamp=False)
    assert np.array_equal(nd.read_pgm(p), np.array([[0, 2, 2, 254]], np.float64))
    with pytest.raises(nd.ShapeError):
        nd.write_pgm(np.array([1.0, 2.0]), p)
    for bad in ([-3.0, 0.0], [0.0, 256.0], [np.nan, 0.0]):
        with pytest.raises(nd.NumericError):
            nd.write_pgm(np.array([bad]), p, clamp=False)
    nd.write_pgm(np.array([[-3.0, 300.0]]), p, clamp=True)
    assert np.array_equal(nd.read_pgm(p), np.array([[0, 255]], np.float64))


@needs_ref
def test_graymap_writer_bytes_equal_reference(tmp_path, ref):
    rng = np.random.default_rng(14)
    for clamp in (False, True):
        img = rng.uniform(-20 if clamp else 0, 280 if clamp else 255, size=(5, 7))
        img[0, :4] = [0.5, 1.5, 2.5, 254.5]
        p = str(tmp_path / "w.pgm")
        nd.write_pgm(img, p, clamp=clamp)
        assert open(p, "rb").read() == ref.serialize_pgm(img, clamp)


MALFORMED_PGMS = [b"", b"P6 2 2 255\nXXXX", b"P5 0 2 255\n", b"P5 2 2 0\n", b"P5 2 2 70000\n",
                  b"P5 2 2 255\nAB", b"P5 two 2 255\n", b"P2 2 1 255\n1", b"P2 2 1 10\n1 11\n",
                  b"P2 1 1 255\n1 junk\n", b"P5 2 1 255\nABC", b"P5 1 1 65535\nA"]


@pytest.mark.parametrize("data", MALFORMED_PGMS)
def test_malformed_graymaps_raise_format_errors(tmp_path, data):
    assert _ours_parse(tmp_path, data, pgm=True)[0] == "FormatError"
    if HAVE_REF:
        assert _ref_parse(O.Oracle("ref"), data, pgm=True)[0] == "FormatError"


@needs_ref
def test_graymap_truncations_and_corruptions_match_reference(tmp_path, ref):
    for good in (b"P5\n3 2\n255\n" + bytes(range(10, 16)), b"P2\n2 2\n100\n1 2\n3 100\n",
                 b"P5 2 1 300\n" + bytes([1, 2, 0, 7])):
        for n in range(len(good)):
            _same_outcome(tmp_path, ref, good[:n], pgm=True)
        rng = np.random.default_rng(len(good))
        for _ in range(150):
            b = bytearray(good)
            b[int(rng.integers(0, len(b)))] = int(rng.integers(0, 256))
            _same_outcome(tmp_path, ref, bytes(b), pgm=True)


# --- committed fixtures written by the reference ------------------------------------------
def test_reference_written_fixtures_read_back(tmp_path):
    man = os.path.join(GOLD_IO, "fixtures.npz")
    if not os.path.exists(man):
        pytest.skip("tests/golden/io not generated")
    want = np.load(man)
    for name in sorted(os.listdir(GOLD_IO)):
        stem, ext = os.path.splitext(name)
        if ext not in (".ndt", ".pgm"):
            continue
        path = os.path.join(GOLD_IO, name)
        got = nd.read_pgm(path) if ext == ".pgm" else nd.read_tensor(path)
        assert got.tobytes() == want[stem].tobytes(), name
        if stem.startswith("in_"):
            continue
        out = str(tmp_path / name)
        if ext == ".pgm":
            nd.write_pgm(got, out, clamp=False)
        else:
            nd.write_tensor(got, out)
        assert open(out, "rb").read() == open(path, "rb").read(), name
