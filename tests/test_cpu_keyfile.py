"""Host-side checks of the streaming key-file reader (keyfile.py): the ARNK
header is validated against the file size before any device work, with the
errors of deserialize_keys (reference fss.py:633-658). No GPU needed."""

import pytest

from paper_2006_04593_b200 import fss, keyfile


def _header(kind=1, n=32, count=3, version=1, lam=127, magic=b"ARNK"):
    return magic + bytes([version, kind, n]) + lam.to_bytes(2, "little") + count.to_bytes(4, "little")


@pytest.mark.parametrize("blob,msg", [
    (b"ARN", "truncated header"),
    (_header(magic=b"XRNK") + bytes(2 * 3 * 824), "bad magic"),
    (_header(version=2) + bytes(2 * 3 * 824), "unsupported version"),
    (_header(lam=128) + bytes(2 * 3 * 824), "unsupported lambda"),
    (_header(kind=2) + bytes(8), "only equality / comparison"),
    (_header() + bytes(2 * 3 * 824 - 1), "payload size mismatch"),
    (_header(kind=0, count=2) + bytes(2 * 2 * 568 + 5), "payload size mismatch"),
])
def test_header_errors(tmp_path, blob, msg):
    p = tmp_path / "k.arnk"
    p.write_bytes(blob)
    with pytest.raises(fss.KeyFormatError, match=msg):
        keyfile.load_keys(p)


def test_header_ok(tmp_path):
    p = tmp_path / "k.arnk"
    p.write_bytes(_header(kind=0, n=16, count=5) + bytes(2 * 5 * fss.eq_elem_bytes(16)))
    with open(p, "rb") as fh:
        assert keyfile.read_header(fh, p.stat().st_size) == (0, 16, 5, 5 * fss.eq_elem_bytes(16))
