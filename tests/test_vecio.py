"""§8(f3): .fvecs / .bvecs / .ivecs ingestion straight to device memory, with
io.cpp:37-85 semantics (record = i32 dim + elements; one dimension; clean end)."""
import numpy as np
import pytest

import paper_2406_10938_b200 as D
from paper_2406_10938_b200._lib import FormatError


def _write(path, rows, dtype):
    with open(path, "wb") as f:
        for r in rows:
            np.array([len(r)], np.int32).tofile(f)
            np.asarray(r, dtype).tofile(f)


def test_shape_and_errors(tmp_path):
    g = np.random.default_rng(3)
    x = g.normal(size=(7, 5)).astype(np.float32)
    p = str(tmp_path / "a.fvecs")
    _write(p, x, np.float32)
    assert D.vectors_shape(p) == (7, 5, "f32")
    b = str(tmp_path / "a.bvecs")
    _write(b, g.integers(0, 256, (4, 9)), np.uint8)
    assert D.vectors_shape(b) == (4, 9, "u8")
    with pytest.raises(ValueError):
        D.vectors_shape(str(tmp_path / "a.txt"))
    with pytest.raises(FormatError):
        D.vectors_shape(str(tmp_path / "missing.fvecs"))
    bad = str(tmp_path / "bad.fvecs")
    _write(bad, [x[0], x[1][:4]], np.float32)  # inconsistent dimension
    with pytest.raises(FormatError, match="disagree"):
        D.vectors_shape(bad)
    with open(p, "ab") as f:
        f.write(b"\x05\x00")  # truncated dimension field
    with pytest.raises(FormatError, match="truncated"):
        D.vectors_shape(p)
    t = str(tmp_path / "t.ivecs")
    _write(t, [[1, 2, 3]], np.int32)
    with open(t, "ab") as f:
        np.array([3], np.int32).tofile(f)
        np.array([1], np.int32).tofile(f)  # truncated record body
    with pytest.raises(FormatError, match="truncated record body"):
        D.vectors_shape(t)
    z = str(tmp_path / "z.fvecs")
    with open(z, "wb") as f:
        np.array([0], np.int32).tofile(f)
    with pytest.raises(FormatError, match="non-positive"):
        D.vectors_shape(z)


@pytest.mark.gpu
@pytest.mark.parametrize("ext,dtype", [("fvecs", np.float32), ("bvecs", np.uint8), ("ivecs", np.int32)])
def test_read_to_device(tmp_path, ext, dtype):
    g = np.random.default_rng(7)
    n, d = 300_001, 24  # several pinned chunks for the 1-byte kind
    if dtype == np.float32:
        x = g.normal(size=(n, d)).astype(np.float32)
    elif dtype == np.uint8:
        x = g.integers(0, 256, (n, d)).astype(np.uint8)
    else:
        x = g.integers(-2**31, 2**31 - 1, (n, d), dtype=np.int64).astype(np.int32)
    p = str(tmp_path / f"x.{ext}")
    with open(p, "wb") as f:
        hdr = np.full((n, 1), d, np.int32).view(np.uint8)
        body = np.ascontiguousarray(x).view(np.uint8).reshape(n, -1)
        np.concatenate([hdr, body], axis=1).tofile(f)
    t = D.read_vectors_device(p)
    assert tuple(t.shape) == (n, d)
    want = x.astype(np.float32)
    assert np.array_equal(t.cpu().numpy().view(np.uint32), want.view(np.uint32))
