"""the FLEGVEC1 / csv vector formats (vector_io.hpp)
staged straight to and from device memory (fl_load_vector / fl_save_vector:
pinned double-buffered chunks overlapping the file I/O with the copies).
Round trips are bit-exact (test_vector_io.cpp:59-72), files are byte-identical
to the host writer's, and the reference's error messages are kept."""
import struct

import numpy as np
import pytest

import paper_1505_00354_b200 as fl

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [0, 1, 7, (1 << 20) + 3, 3 * (1 << 20)])
def test_binary_round_trip_device(tmp_path, n):
    import torch
    v = np.random.default_rng(n).standard_normal(n) * np.exp(np.random.default_rng(1).uniform(-30, 30, n))
    d = torch.from_numpy(v).cuda()
    p = tmp_path / "v.bin"
    fl.save_vector(p, d, fl.VECTOR_RAW_BINARY)
    raw = p.read_bytes()
    assert raw[:8] == b"FLEGVEC1" and struct.unpack("<Q", raw[8:16])[0] == n
    assert raw[16:] == v.astype("<f8").tobytes()  # the host writer's layout (vector_io.hpp:56-63)
    back = fl.load_vector(p, fl.VECTOR_RAW_BINARY, device="cuda")
    assert back.is_cuda and np.array_equal(back.cpu().numpy(), v)
    assert np.array_equal(fl.load_vector(p, fl.VECTOR_RAW_BINARY), v)


def test_csv_round_trip_device(tmp_path):
    import torch
    v = np.array([0.0, -0.0, 1.0, -2.5, 1e-310, 1.7976931348623157e308, np.pi, 1.0 / 3.0])
    p = tmp_path / "v.csv"
    fl.save_vector(p, torch.from_numpy(v).cuda(), fl.VECTOR_CSV)
    lines = p.read_text().splitlines()
    assert len(lines) == len(v) and all(float(s) == x for s, x in zip(lines, v))
    back = fl.load_vector(p, fl.VECTOR_CSV, device="cuda").cpu().numpy()
    assert np.array_equal(back, v) and np.signbit(back[1])


def test_dlt_from_file_through_device(tmp_path):
    """The caller either side of the path: coefficients file -> device ->
    dlt -> file, equal to the in-memory transform."""
    n = 4096
    cfg = fl.TransformConfig(n)
    c = fl.random_decaying(n, 1.0, 9)
    p = tmp_path / "c.bin"
    fl.save_vector(p, c)
    f = fl.dlt(fl.load_vector(p, device="cuda"), cfg)
    q = tmp_path / "f.bin"
    fl.save_vector(q, f)
    assert np.array_equal(fl.load_vector(q), fl.dlt(c, cfg))


def test_errors(tmp_path):
    with pytest.raises(fl.RuntimeErrorFL, match="cannot open for reading"):
        fl.load_vector(tmp_path / "missing.bin")
    p = tmp_path / "bad.bin"
    p.write_bytes(b"NOTAVEC!" + struct.pack("<Q", 1) + b"\0" * 8)
    with pytest.raises(fl.RuntimeErrorFL, match="bad magic"):
        fl.load_vector(p)
    p.write_bytes(b"FLEGVEC1" + struct.pack("<Q", 4) + b"\0" * 24)
    with pytest.raises(fl.RuntimeErrorFL, match="truncated payload"):
        fl.load_vector(p, device="cuda")
    p.write_bytes(b"FLEGVEC1\x01")
    with pytest.raises(fl.RuntimeErrorFL, match="truncated header"):
        fl.load_vector(p)
    q = tmp_path / "bad.csv"
    q.write_text("1.0\n2.0x\n")
    with pytest.raises(fl.RuntimeErrorFL, match=r"bad.csv:2: not a number"):
        fl.load_vector(q, fl.VECTOR_CSV, device="cuda")
