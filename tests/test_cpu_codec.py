"""Host side of frame ingest / egress against the reference
(codec.cpp via oracle/_ref): PGM / PPM / PFM files byte-for-byte, read_pnm's
header grammar and its error messages. No GPU needed: the quantised bytes come
from the reference's own write_pgm."""
import os

import numpy as np
import pytest

from paper_2203_02300_b200 import dco
from paper_2203_02300_b200.config import CodecError


@pytest.fixture(scope="module")
def ref():
    from oracle import ref as r

    if not r.available():
        import oracle

        oracle.build()
    return r


def _bytes(p):
    with open(p, "rb") as f:
        return f.read()


def test_pgm_ppm_pfm_files_equal_reference(ref, tmp_path):
    rng = np.random.default_rng(3)
    img = rng.uniform(-0.2, 1.2, (7, 11)).astype(np.float32)
    img[0, 0] = np.nan
    rgb = rng.uniform(0.0, 1.0, (5, 4, 3)).astype(np.float32)
    # reference files
    ref.write_pgm(img, str(tmp_path / "r.pgm"))
    ref.write_ppm(rgb, str(tmp_path / "r.ppm"))
    fmap = rng.uniform(0.5, 3.0, (6, 9)).astype(np.float32)
    fmap[2, 3] = np.nan
    ref.write_pfm(fmap, str(tmp_path / "r.pfm"))
    # ours: the same bytes through dco_write_pnm, the map through dco_write_pfm
    gbytes = dco.read_pnm(str(tmp_path / "r.pgm"))
    cbytes = dco.read_pnm(str(tmp_path / "r.ppm"), color=True)
    assert gbytes.shape == (7, 11) and cbytes.shape == (5, 4, 3)
    lib = dco._lib()
    dco._codec(lib.dco_write_pnm, str(tmp_path / "o.pgm").encode(), gbytes.ctypes.data, 11, 7, 1)
    dco._codec(lib.dco_write_pnm, str(tmp_path / "o.ppm").encode(), cbytes.ctypes.data, 4, 5, 3)
    dco.write_pfm(str(tmp_path / "o.pfm"), fmap)
    for ext in ("pgm", "ppm", "pfm"):
        assert _bytes(tmp_path / ("o." + ext)) == _bytes(tmp_path / ("r." + ext)), ext
    # and the floats the reference reads back are bytes / 255
    assert np.array_equal(ref.read_pnm(str(tmp_path / "o.pgm")), gbytes.astype(np.float32) / np.float32(255.0))


HEADERS = [
    (b"P5\n# a comment\n3 2\n# another\n255\n", 6, None),
    (b"P5 3\t2 255 ", 6, None),
    (b"P6\n3 2\n255\n", 18, "bad magic"),
    (b"P5\n3 2\n65535\n", 6, "unsupported bit depth (maxval must be 255)"),
    (b"P5\n0 2\n255\n", 0, "degenerate dimensions"),
    (b"P5\n3 x\n255\n", 6, "malformed header"),
    (b"P5\n3 2\n255\n", 5, "truncated payload"),
    (b"P5\n3 2\n255", 0, "malformed header"),
    (b"P5\n9999999999 2\n255\n", 0, "header value out of range"),
]


@pytest.mark.parametrize("head,payload,err", HEADERS)
def test_read_pnm_grammar_and_errors(ref, tmp_path, head, payload, err):
    p = str(tmp_path / "x.pgm")
    with open(p, "wb") as f:
        f.write(head + bytes(range(payload)))
    if err is None:
        got = dco.read_pnm(p)
        assert np.array_equal(got.astype(np.float32) / np.float32(255.0), ref.read_pnm(p))
        return
    with pytest.raises(CodecError) as mine:
        dco.read_pnm(p)
    with pytest.raises(CodecError) as theirs:
        ref.read_pnm(p)
    assert err in str(mine.value)
    assert str(mine.value) == str(theirs.value)  # same text, same byte offset


def test_missing_files(ref, tmp_path):
    p = str(tmp_path / "none.pgm")
    with pytest.raises(CodecError) as mine:
        dco.read_pnm(p)
    assert str(mine.value) == p + ": cannot open file"
    with pytest.raises(CodecError):
        dco.write_pfm(os.path.join(str(tmp_path), "no", "dir.pfm"), np.zeros((2, 2), np.float32))
