"""The `fastleg` command-line tool (include/fastleg/cli.hpp, built by
tests/cpp/build.sh into tests/_bin/): restates the reference's
proj/tests/test_cli.cpp. Usage (2), I/O (3) and domain (4) exit codes and
--help need no GPU; the transform cases are marked gpu.
"""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "_bin", "fastleg")


@pytest.fixture(scope="module")
def cli():
    if not os.path.exists(BIN):
        subprocess.run(["bash", os.path.join(ROOT, "tests", "cpp", "build.sh")], check=True,
                       capture_output=True)
    return BIN


def run(cli, *args):
    return subprocess.run([cli, *map(str, args)], capture_output=True, text=True, timeout=600)


def read_csv(path):
    with open(path) as f:
        return [float(line) for line in f if line.strip()]


# ---------------------------------------------------------------- no GPU needed

def test_usage_errors_exit_2(cli, tmp_path):  # test_cli.cpp "exit codes", usage part
    assert run(cli, "frobnicate").returncode == 2
    assert run(cli).returncode == 2
    assert run(cli, "dlt", "--in", "x.csv").returncode == 2            # --out missing
    assert run(cli, "nodes").returncode == 2                           # --n missing
    assert run(cli, "dlt", "--in", "a", "--out", "b", "--grid", "weird").returncode == 2
    assert run(cli, "dlt", "--in", "a", "--out", "b", "--format", "xml").returncode == 2
    assert run(cli, "nodes", "--n", "abc").returncode == 2
    assert run(cli, "dlt", "--in", "a", "--out", "b", "--bogus", "1").returncode == 2
    assert run(cli, "bench", "--min", "16", "--max", "64").returncode == 2


def test_help_exit_0(cli):
    r = run(cli, "--help")
    assert r.returncode == 0 and "dlt" in r.stdout and "compare" in r.stdout
    r = run(cli, "compare", "--help")
    assert r.returncode == 0 and "--trials" in r.stdout


def test_io_error_exit_3(cli, tmp_path):
    missing = tmp_path / "missing.csv"
    assert run(cli, "dlt", "--in", missing, "--out", tmp_path / "o.csv").returncode == 3
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"NOTMAGIC")
    assert run(cli, "leg2cheb", "--in", bad, "--out", tmp_path / "o.bin", "--format", "bin").returncode == 3


def test_empty_vector_exit_4(cli, tmp_path):  # "an empty vector has no transform"
    empty = tmp_path / "empty.csv"
    empty.write_text("")
    assert run(cli, "dlt", "--in", empty, "--out", tmp_path / "o2.csv").returncode == 4


# ---------------------------------------------------------------- on the GPU

@pytest.mark.gpu
def test_dlt_of_constant_basis_vector(cli, tmp_path):
    src, out = tmp_path / "e0.csv", tmp_path / "f.csv"
    src.write_text("1\n0\n0\n0\n0\n0\n0\n0\n")
    assert run(cli, "dlt", "--in", src, "--out", out).returncode == 0
    f = read_csv(out)
    assert len(f) == 8 and max(abs(v - 1.0) for v in f) <= 1e-14


@pytest.mark.gpu
def test_nodes_of_two_point_rule(cli, tmp_path):
    out = tmp_path / "nodes2.csv"
    assert run(cli, "nodes", "--n", 2, "--out", out).returncode == 0
    rows = [[float(x) for x in line.split(",")] for line in out.read_text().splitlines()]
    r3 = 0.57735026918962576451
    assert len(rows) == 2
    assert abs(rows[0][1] - r3) <= 4e-16 and abs(rows[1][1] + r3) <= 4e-16
    assert abs(rows[0][2] - 1.0) <= 4e-16 and abs(rows[1][2] - 1.0) <= 4e-16
    assert abs(rows[0][0] - np.arccos(r3)) <= 4e-16
    # stdout target
    r = run(cli, "nodes", "--n", 3)
    assert r.returncode == 0 and len(r.stdout.splitlines()) == 3


@pytest.mark.gpu
def test_file_round_trip_dlt_idlt(cli, tmp_path):
    import paper_1505_00354_b200 as fl
    c = fl.random_decaying(64, 1.0, 12)
    src, mid, back = tmp_path / "c.csv", tmp_path / "fvals.csv", tmp_path / "cback.csv"
    src.write_text("".join(f"{float(v)!r}\n" for v in c))
    assert run(cli, "dlt", "--in", src, "--out", mid).returncode == 0
    assert run(cli, "idlt", "--in", mid, "--out", back).returncode == 0
    rec = np.array(read_csv(back))
    assert rec.shape == (64,) and np.max(np.abs(rec - c)) <= 1e-10 * np.max(np.abs(c))
    # the CSV written is the shortest round-trip decimal: the dlt agrees with the API bitwise
    assert np.array_equal(np.array(read_csv(mid)), fl.dlt(np.array(read_csv(src)), fl.TransformConfig(64)))


@pytest.mark.gpu
def test_binary_format_round_trip(cli, tmp_path):
    import paper_1505_00354_b200 as fl
    src, out = tmp_path / "c.bin", tmp_path / "cheb.bin"
    c = fl.random_decaying(32, 0.5, 8)
    src.write_bytes(b"FLEGVEC1" + (32).to_bytes(8, "little") + c.astype("<f8").tobytes())
    assert run(cli, "leg2cheb", "--in", src, "--out", out, "--format", "bin").returncode == 0
    raw = out.read_bytes()
    assert raw[:8] == b"FLEGVEC1" and int.from_bytes(raw[8:16], "little") == 32
    cheb = np.frombuffer(raw[16:], dtype="<f8")
    assert np.array_equal(cheb, fl.leg2cheb_apply(fl.legendre_coefficients(c)).values)


@pytest.mark.gpu
def test_ndct_and_grid_selection_flags(cli, tmp_path):
    import paper_1505_00354_b200 as fl
    src, o1, o2 = tmp_path / "chebc.csv", tmp_path / "v1.csv", tmp_path / "v2.csv"
    src.write_text("".join(f"{float(v)!r}\n" for v in fl.random_decaying(24, 1.0, 9)))
    assert run(cli, "ndct", "--in", src, "--out", o1, "--grid", "cheb1").returncode == 0
    assert run(cli, "ndct", "--in", src, "--out", o2, "--grid", "chebstar", "--tol", "1e-7").returncode == 0
    v1, v2 = np.array(read_csv(o1)), np.array(read_csv(o2))
    assert v1.shape == (24,) and np.max(np.abs(v1 - v2)) <= 1e-6


@pytest.mark.gpu
def test_compare_small_errors_and_deterministic(cli, tmp_path):
    args = ["compare", "--n", 1024, "--decay", 1, "--trials", 5, "--seed", 0]
    o1, o2 = tmp_path / "cmp1.csv", tmp_path / "cmp2.csv"
    assert run(cli, *args, "--out", o1).returncode == 0
    assert run(cli, *args, "--out", o2).returncode == 0
    assert o1.read_text() == o2.read_text()
    rows = o1.read_text().splitlines()
    assert len(rows) == 5
    for line in rows:
        n, err = line.split(",")
        assert n == "1024" and float(err) <= 1e-11


@pytest.mark.gpu
def test_bench_one_row_per_size(cli, tmp_path):
    out = tmp_path / "bench.csv"
    assert run(cli, "bench", "--min", 16, "--max", 64, "--points", 3, "--out", out).returncode == 0
    rows = out.read_text().splitlines()
    assert len(rows) == 3 and rows[0].startswith("16,") and rows[2].startswith("64,")
    assert all(float(x) > 0 for x in rows[1].split(",")[1:])


@pytest.mark.gpu
def test_reference_main_unmodified(cli):
    """The reference's proj/tools/fastleg.cpp (a main calling fastleg::cli::run),
    compiled unmodified against include/fastleg/cli.hpp, behaves identically."""
    ref = os.path.join(ROOT, "tests", "_bin", "fastleg_ref_main")
    if not os.path.exists(ref):
        pytest.skip("built only where the reference checkout is present")
    a, b = run(cli, "nodes", "--n", 17), run(ref, "nodes", "--n", 17)
    assert a.returncode == b.returncode == 0 and a.stdout == b.stdout
    assert run(ref, "frobnicate").returncode == 2
