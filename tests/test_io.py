"""Matrix file formats (ring.hpp:386-449): the product's host reader / writer
against the reference's own read_text / write_text / read_binary /
write_binary (oracle/_ref), byte for byte, including the io_error cases.
CPU only; the device round trip is in test_gpu_parity.py."""
import os

import numpy as np
import pytest


@pytest.fixture
def ref(O):
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    return O


@pytest.mark.parametrize("binary", [False, True], ids=["text", "binary"])
@pytest.mark.parametrize("shape,p", [((1, 1), 65521), ((3, 5), 65521), ((17, 9), 101),
                                     ((64, 33), 65521)])
def test_writer_bytes_match_reference(W, ref, tmp_path, binary, shape, p):
    a = ref.fill_random(shape[0], shape[1], 5, p)
    mine, theirs = str(tmp_path / "mine"), str(tmp_path / "ref")
    W.write_matrix_host(mine, a, p, binary)
    ref.ref_write_matrix(theirs, a, p, binary)
    assert open(mine, "rb").read() == open(theirs, "rb").read()


@pytest.mark.parametrize("binary", [False, True], ids=["text", "binary"])
def test_reader_matches_reference(W, ref, tmp_path, binary):
    a = ref.fill_random(31, 47, 9)
    f = str(tmp_path / "m")
    ref.ref_write_matrix(f, a, 65521, binary)
    got, p = W.read_matrix_host(f, binary)
    want, pw = ref.ref_read_matrix(f, binary)
    assert p == pw == 65521 and (got == want).all() and (got == a).all()
    assert W.matrix_file_info(f, binary) == (31, 47, 65521)


def test_text_reader_whitespace(W, ref, tmp_path):
    f = str(tmp_path / "ws.txt")
    open(f, "w").write("  2\t3 7\n\n1 2\n3\n4 5 6  trailing ignored\n")
    got, p = W.read_matrix_host(f)
    want, _ = ref.ref_read_matrix(f)
    assert p == 7 and got.tolist() == want.tolist() == [[1, 2, 3], [4, 5, 6]]


@pytest.mark.parametrize("content,binary", [
    ("x 2 7\n", False),                 # bad header
    ("2 2 7\n1 2 3\n", False),          # truncated
    ("2 2 7\n1 2 3 9\n", False),        # non-canonical entry
    (b"\x01\x00", True),                # truncated header
])
def test_io_errors_match_reference(W, ref, tmp_path, content, binary):
    f = str(tmp_path / "bad")
    open(f, "wb" if isinstance(content, bytes) else "w").write(content)
    with pytest.raises(ref.RefError) as re_:
        ref.ref_read_matrix(f, binary)
    with pytest.raises(W.io_error) as mine:
        W.read_matrix_host(f, binary)
    assert re_.value.code == mine.value.code == 7


def test_binary_non_canonical_and_truncated(W, ref, tmp_path):
    import struct
    f = str(tmp_path / "b")
    open(f, "wb").write(struct.pack("<5Q", 1, 2, 7, 3, 7))  # second entry == p
    with pytest.raises(W.io_error):
        W.read_matrix_host(f, True)
    with pytest.raises(ref.RefError):
        ref.ref_read_matrix(f, True)
    open(f, "wb").write(struct.pack("<4Q", 1, 2, 7, 3))  # one entry short
    with pytest.raises(W.io_error):
        W.read_matrix_host(f, True)


def test_missing_file(W, tmp_path):
    with pytest.raises(W.io_error):
        W.matrix_file_info(str(tmp_path / "nope"))
