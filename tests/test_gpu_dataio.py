"""F2 DNB containers through the Python mirror (dataio.hpp:18-150): payload
streamed file <-> HBM by dndc_file_*; the reference's round-trip, header-law,
slicing and malformed-file cases (test_dataio.cpp:26-160)."""
import numpy as np
import pytest
import torch

import paper_2007_13552_b200.api as dnd

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_round_trip_every_split(comm, tmp_path, dtype):
    data = (np.sin(np.arange(60) * 1.7 + 0.3) * 10).astype(dtype)
    shape = (5, 4, 3)
    for ss in (None, 0, 1, 2):
        for ls in (None, 0, 1, 2):
            path = str(tmp_path / f"a_{ss}_{ls}.dnb")
            dnd.dnb_save(dnd.from_global(data, shape, ss, comm), path)
            b = dnd.dnb_load(path, ls, comm)
            assert b.shape == shape and b.split == ls
            assert np.array_equal(dnd.gather(b).ravel(), data)


def test_header_law_and_foreign_file(comm, tmp_path):
    x = np.random.default_rng(2).random((1000, 18), dtype=np.float32)
    path = tmp_path / "susy_like.dnb"
    with open(path, "wb") as f:  # written without the library
        f.write(b"DNB1" + bytes([1, 2]) + np.array(x.shape, "<u8").tobytes() + x.tobytes())
    a = dnd.dnb_load(str(path), 0, comm)
    assert a.tile.dtype == torch.float32 and np.array_equal(dnd.gather(a), x)
    out = str(tmp_path / "copy.dnb")
    dnd.dnb_save(a, out)
    assert open(out, "rb").read() == open(path, "rb").read()
    assert (tmp_path / "copy.dnb").stat().st_size == 6 + 8 * 2 + 4 * x.size


def test_malformed_containers(comm, tmp_path):
    good = tmp_path / "good.dnb"
    dnd.dnb_save(dnd.from_global(np.arange(4.0), (4,), None, comm), str(good))
    raw = good.read_bytes()
    cases = {"magic": b"X" + raw[1:], "dtype_code": raw[:4] + bytes([9]) + raw[5:]}
    for needle, blob in cases.items():
        p = tmp_path / f"{needle}.dnb"
        p.write_bytes(blob)
        with pytest.raises(dnd.DataError, match=needle):
            dnd.dnb_read_header(str(p))
    short = tmp_path / "short.dnb"
    short.write_bytes(raw[:-8])
    with pytest.raises(dnd.DataError, match="truncated"):
        dnd.dnb_load(str(short), None, comm)
    with pytest.raises(dnd.DataError):
        dnd.dnb_read_header(str(tmp_path / "missing.dnb"))
