"""PGM I/O and the CLI on the CUDA path (reference test_pgmio.py / test_cli.py
behaviours).  Header parsing, P2 and the tables subcommand run on the CPU;
P5 decode/encode, filter and compute-t need the GPU."""

import csv
import io
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import REPO
from oracle import shiftbf_oracle as O
from paper_1203_5128_b200 import cli
from paper_1203_5128_b200.errors import PgmParseError
from paper_1203_5128_b200.pgmio import inspect_pgm, load_pgm, load_pgm_device, save_pgm


def _write(path, data: bytes):
    with open(path, "wb") as fh:
        fh.write(data)
    return str(path)


def test_header_and_p2_on_host(tmp_path):
    p = _write(tmp_path / "a.pgm", b"P2\n# comment\n3 2\n10\n0 1 2\n3 4 10\n")
    h = inspect_pgm(p)
    assert (h.magic, h.width, h.height, h.maxval) == ("P2", 3, 2, 10)
    np.testing.assert_array_equal(load_pgm(p), [[0, 1, 2], [3, 4, 10]])


@pytest.mark.parametrize("data,offset", [
    (b"P7\n1 1\n255\n\x00", 0),                 # bad magic at byte 0
    (b"P5\n0 1\n255\n\x00", 3),                 # width must be positive
    (b"P5\n1 1\n70000\n\x00", 7),               # maxval above 65535
    (b"P2\n2 1\n10\n3 x\n", 12),                # non-integer sample
    (b"P2\n2 1\n10\n3 11\n", 12),               # sample above maxval
])
def test_parse_errors_carry_offsets(tmp_path, data, offset):
    p = _write(tmp_path / "bad.pgm", data)
    with pytest.raises(PgmParseError) as ei:
        load_pgm(p)
    assert ei.value.offset == offset


def test_tables_subcommand(capsys):
    assert cli.main(["tables", "--which", "n0"]) == 0
    rows = list(csv.reader(io.StringIO(capsys.readouterr().out)))
    assert dict((int(a), int(b)) for a, b in rows[1:]) == {5: 1053, 10: 263, 20: 66, 30: 29,
                                                           40: 16, 60: 7, 80: 4, 100: 3}


def test_exit_codes_without_gpu(tmp_path, capsys):
    assert cli.main(["compute-t", "--input", str(tmp_path / "missing.pgm"), "--radius", "3"]) == 3
    with pytest.raises(SystemExit) as ei:
        cli.main(["filter", "--input", "x", "--output", "y", "--sigma-s", "0", "--sigma-r", "1"])
    assert ei.value.code == 2


@pytest.mark.gpu
@pytest.mark.parametrize("maxval", [255, 65535])
def test_p5_round_trip_on_device(tmp_path, maxval):
    rng = np.random.default_rng(1)
    img = rng.integers(0, maxval + 1, (37, 53)).astype(np.float64)
    p = str(tmp_path / "x.pgm")
    save_pgm(img, p, maxval=maxval)
    np.testing.assert_array_equal(load_pgm(p), img)
    assert load_pgm_device(p).dtype.is_floating_point


@pytest.mark.gpu
def test_quantisation_matches_reference_rule(tmp_path):
    vals = np.array([[-3.0, 0.49, 0.5, 1.5, 2.5, 254.5, 255.2, 300.0]])
    p = str(tmp_path / "q.pgm")
    save_pgm(vals, p, maxval=255)
    expect = np.floor(np.clip(vals, 0, 255) + 0.5)
    np.testing.assert_array_equal(load_pgm(p), expect)


@pytest.mark.gpu
def test_cli_filter_matches_oracle(tmp_path):
    rng = np.random.default_rng(2)
    img = np.round(rng.uniform(0, 255, (48, 40)))
    src = str(tmp_path / "in.pgm")
    save_pgm(img, src)
    out, raw, log = str(tmp_path / "out.pgm"), str(tmp_path / "o.f8"), str(tmp_path / "log.csv")
    rc = cli.main(["filter", "--input", src, "--output", out, "--sigma-s", "3", "--sigma-r", "30",
                   "--epsilon", "0.01", "--float-out", raw, "--csv", log])
    assert rc == 0
    got = np.fromfile(raw, dtype="<f8").reshape(img.shape)
    ref = O.shiftable_bf(img, 3.0, 30.0, 0.01)
    assert np.abs(got - ref["image"]).max() <= 1e-2
    np.testing.assert_array_equal(load_pgm(out), np.floor(np.clip(got, 0, 255) + 0.5))
    rec = cli.BenchRecord.from_csv_row(list(csv.reader(open(log)))[1])
    assert (rec.T, rec.N, rec.M) == (ref["T"], ref["N"], ref["M"])


@pytest.mark.gpu
def test_cli_compute_t_and_unsupported(tmp_path, capsys):
    rng = np.random.default_rng(3)
    img = np.round(rng.uniform(0, 255, (30, 30)))
    src = str(tmp_path / "in.pgm")
    save_pgm(img, src)
    assert cli.main(["compute-t", "--input", src, "--radius", "4"]) == 0
    assert f"T={O.compute_T(img, 4):g}" in capsys.readouterr().out
    assert cli.main(["filter", "--input", src, "--output", src + ".o", "--sigma-s", "2",
                     "--sigma-r", "30", "--kernel", "poly"]) == 4


@pytest.mark.gpu
def test_cli_direct_method_and_bench_with_direct(tmp_path, capsys):
    rng = np.random.default_rng(4)
    img = np.round(rng.uniform(0, 255, (40, 44)))
    src, raw = str(tmp_path / "in.pgm"), str(tmp_path / "d.f8")
    save_pgm(img, src)
    assert cli.main(["filter", "--input", src, "--output", src + ".o", "--sigma-s", "2",
                     "--sigma-r", "30", "--method", "direct", "--float-out", raw]) == 0
    got = np.fromfile(raw, dtype="<f8").reshape(img.shape)
    R = O.support_radius("iterated", 2.0, 3)
    ref = O.direct_bf(img, ("fir", 2.0, R), 30.0)
    assert np.abs(got - ref).max() <= 1e-2
    assert "method=direct" in capsys.readouterr().out
    log = str(tmp_path / "b.csv")
    assert cli.main(["bench", "--input", src, "--sigma-s", "2", "--sigma-r", "20,40",
                     "--repeats", "1", "--with-direct", "--csv", log]) == 0
    rows = list(csv.reader(open(log)))[1:]
    assert len(rows) == 2 and all(float(r[9]) < 5.0 for r in rows)


@pytest.mark.gpu
def test_standalone_c_caller_of_the_abi(tmp_path):
    """tests/c_abi/sbf_example.c links libsbf.so directly (no Python in the
    call path) and must reproduce the oracle."""
    import os
    import subprocess
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "sbf_example")
    lib_dir = os.path.join(repo, "paper_1203_5128_b200")
    subprocess.run(["gcc", "-O2", "-o", exe, os.path.join(repo, "tests", "c_abi", "sbf_example.c"),
                    "-I", os.path.join(repo, "include"), "-L", lib_dir, "-lsbf",
                    "-L/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{lib_dir}",
                    "-Wl,-rpath,/usr/local/cuda/lib64", "-lm"], check=True)
    for kind in ("u8", "hdr"):
        rng = np.random.default_rng(9)
        img = rng.uniform(0, 65535 if kind == "hdr" else 255, (70, 90))
        src, dst = str(tmp_path / "in.f8"), str(tmp_path / "out.f8")
        img.astype("<f8").tofile(src)
        sr = 2000.0 if kind == "hdr" else 25.0
        res = subprocess.run([exe, src, dst, "70", "90", "3.0", str(sr), "0.01"], check=True,
                             capture_output=True, text=True)
        ref = O.shiftable_bf(img, 3.0, sr, 0.01)
        assert f"N={ref['N']} M={ref['M']}" in res.stdout
        got = np.fromfile(dst, dtype="<f8").reshape(img.shape)
        assert np.abs(got - ref["image"]).max() <= 1e-2
