"""Archive / CSV / CLI compatibility with the reference (sysio.py, cli.py;
SURVEY 8(f) rank 4).  The fixture tests/golden/cli/ is a reference CLI
session (gen -> reduce -> tf, pspec), made by tests/golden/make_golden.py.
CPU tests: formats, checksums, exit codes; GPU tests: the same commands on
the GPU solvers reproduce the reference's CSVs."""

import json
import os
import shutil

import numpy as np
import pytest

from conftest import GOLDEN

import paper_1708_06290_b200 as ss
from paper_1708_06290_b200 import cli, sysio

ARCH = os.path.join(GOLDEN, "cli", "archive")


def read_csv(path):
    rows = [ln.split(",") for ln in open(path).read().splitlines() if not ln.startswith("#")]
    return rows[0], rows[1:]


def test_reference_archive_loads_and_checksums():
    chf, man = sysio.load_archive(ARCH)
    assert (chf.n, chf.m, chf.p) == (40, 3, 2)
    assert sysio.band_checksum(chf.Ahat, chf.m) == man["band_checksum"]
    assert sysio.content_hash(chf.Ahat, chf.Bhat, chf.Chat) == man["content_sha256"]


def test_archive_round_trip_is_bit_exact(tmp_path):
    chf, man = sysio.load_archive(ARCH)
    out = sysio.write_archive(tmp_path / "a", chf, reduction_stats=man["reduction"],
                              config=man["config"])
    chf2, man2 = sysio.load_archive(out)
    for X, Y in ((chf.Ahat, chf2.Ahat), (chf.Bhat, chf2.Bhat), (chf.Chat, chf2.Chat)):
        assert np.array_equal(X, Y)
    assert man2["band_checksum"] == man["band_checksum"]
    assert man2["content_sha256"] == man["content_sha256"]


def test_corrupt_and_missing_archives(tmp_path):
    bad = tmp_path / "bad"
    shutil.copytree(ARCH, bad)
    A = sysio.read_matrix(bad / "ahat.mtx")
    A[0, 0] += 1.0
    sysio.write_matrix(bad / "ahat.mtx", A)
    with pytest.raises(sysio.MatrixParseError):
        sysio.load_archive(bad)
    assert cli.main(["tf", str(bad), "--out", str(tmp_path / "x.csv"), "--w-min", "1",
                     "--w-max", "2", "--count", "2"]) == cli.EXIT_PARSE
    assert cli.main(["tf", str(tmp_path / "nowhere"), "--out", str(tmp_path / "x.csv"),
                     "--w-min", "1", "--w-max", "2", "--count", "2"]) == cli.EXIT_PARSE
    man = json.loads((bad / "manifest.json").read_text())
    man["n"] = 41
    shutil.copy(os.path.join(ARCH, "ahat.mtx"), bad / "ahat.mtx")
    (bad / "manifest.json").write_text(json.dumps(man))
    with pytest.raises(ss.DimensionMismatchError):
        sysio.load_archive(bad)


def test_tf_without_shift_source_is_a_parse_error(tmp_path):
    assert cli.main(["tf", ARCH, "--out", str(tmp_path / "x.csv")]) == cli.EXIT_PARSE


def test_shift_file_formats(tmp_path):
    f = tmp_path / "s.txt"
    f.write_text("# comment\n1.5\n2 -3\n4,5  # trailing\n\n")
    assert np.array_equal(sysio.read_shift_file(f), np.array([1.5, 2 - 3j, 4 + 5j]))
    f.write_text("1 2 3\n")
    with pytest.raises(sysio.MatrixParseError):
        sysio.read_shift_file(f)


def test_gen_matches_reference_generator(tmp_path):
    assert cli.main(["gen", "--n", "40", "--m", "3", "--p", "2", "--seed", "5",
                     "--out", str(tmp_path)]) == 0
    A = sysio.read_matrix(tmp_path / "A.mtx")
    sysb = ss.random_stable_system(40, 3, 2, seed=5, circular=False)
    assert np.array_equal(A, sysb.A)


def test_csv_layouts(tmp_path):
    G = np.arange(12, dtype=float).reshape(2, 6) * (1 + 1j)
    sysio.write_tf_csv(tmp_path / "t.csv", G, np.array([1j, 2j]), {1: 0}, p=2, m=3)
    head, rows = read_csv(tmp_path / "t.csv")
    ref_head, _ = read_csv(os.path.join(GOLDEN, "cli", "tf.csv"))
    assert head == ref_head
    assert rows[0][2] == "ok" and rows[1][2] == "singular" and rows[1][3] == "nan"
    assert float(rows[0][5]) == G[1, 0].real  # column-major p x m block


@pytest.mark.gpu
def test_tf_and_pspec_commands_match_reference(tmp_path):
    out = tmp_path / "tf.csv"
    assert cli.main(["tf", ARCH, "--out", str(out), "--w-min", "0.1", "--w-max", "100",
                     "--count", "9", "--nb", "8"]) == 0
    h1, r1 = read_csv(out)
    h0, r0 = read_csv(os.path.join(GOLDEN, "cli", "tf.csv"))
    assert h1 == h0 and len(r1) == len(r0)
    for a, b in zip(r1, r0):
        assert a[:3] == b[:3]
        x, y = np.array(a[3:], float), np.array(b[3:], float)
        assert np.linalg.norm(x - y) <= 1e-10 * np.linalg.norm(y)
    out = tmp_path / "ps.csv"
    assert cli.main(["pspec", ARCH, "--out", str(out), "--re-min", "-3", "--re-max", "1",
                     "--re-count", "4", "--im-min", "-2", "--im-max", "2", "--im-count", "3",
                     "--nb", "8"]) == 0
    h1, r1 = read_csv(out)
    h0, r0 = read_csv(os.path.join(GOLDEN, "cli", "pspec.csv"))
    assert h1 == h0
    for a, b in zip(r1, r0):
        assert a[0] == b[0] and a[1] == b[1] and a[3] == b[3]
        assert abs(float(a[2]) - float(b[2])) <= 1e-10 * abs(float(b[2]))


@pytest.mark.gpu
def test_reduce_irka_bench_commands(tmp_path):
    assert cli.main(["gen", "--n", "40", "--m", "3", "--p", "2", "--seed", "5",
                     "--out", str(tmp_path / "sys")]) == 0
    files = [str(tmp_path / "sys" / f) for f in ("A.mtx", "B.mtx", "C.mtx")]
    assert cli.main(["reduce", *files, "--out", str(tmp_path / "arch"), "--block-size", "8"]) == 0
    chf, man = sysio.load_archive(tmp_path / "arch")
    ref, _ = sysio.load_archive(ARCH)
    assert np.abs(chf.Ahat - ref.Ahat).max() <= 1e-11 * np.abs(ref.Ahat).max()
    assert cli.main(["irka", str(tmp_path / "arch"), "-r", "4", "--out", str(tmp_path / "ir"),
                     "--maxiter", "3", "--fixed-iters", "--nb", "8"]) == 0
    head, rows = read_csv(tmp_path / "ir" / "history.csv")
    assert head == ["iter", "shift_index", "re", "im", "shift_change"] and len(rows) == 12
    assert cli.main(["bench", str(tmp_path / "arch"), "--out", str(tmp_path / "b.csv")]) == 0
    head, rows = read_csv(tmp_path / "b.csv")
    assert [r[0] for r in rows] == list(ss.counters.ALL_PHASES)
    assert cli.main(["irka", str(tmp_path / "arch"), "-r", "40",
                     "--out", str(tmp_path / "ir2")]) == cli.EXIT_DIMENSION
