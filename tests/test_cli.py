"""CLI driver — argument handling, file formats and exit codes
mirror proj/tools/eigenid.cpp; the GPU runs are marked gpu."""
import os

import numpy as np
import pytest

from paper_2002_04989_b200 import cli, errors


def test_splitmix_matches_reference_bench(oracle):
    for x in (0, 1, 4096, 2**63 + 5):
        assert cli.splitmix64(x) == oracle.splitmix64(x)


def test_csv_and_matrix_market_loaders(tmp_path):
    p = tmp_path / "a.csv"
    p.write_text("2,1\n1,2\n")
    assert np.array_equal(cli.load_dense_csv(str(p)), [[2, 1], [1, 2]])
    p.write_text("1,2,3\n4,5,6\n")
    with pytest.raises(errors.DimensionMismatch):
        cli.load_dense_csv(str(p))
    p.write_text("1,x\n2,3\n")
    with pytest.raises(errors.Error):
        cli.load_dense_csv(str(p))
    m = tmp_path / "a.mtx"
    m.write_text("%%MatrixMarket matrix coordinate real symmetric\n2 2 3\n1 1 2\n2 1 1\n2 2 2\n")
    assert np.array_equal(cli.load_matrix_market(str(m)), [[2, 1], [1, 2]])
    m.write_text("%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 2 1\n")
    with pytest.raises(errors.Error):
        cli.load_matrix_market(str(m))


def test_usage_errors_exit_2(tmp_path):
    assert cli.main(["full"]) == 2                       # no source
    assert cli.main(["nonsense"]) == 2
    assert cli.main(["bench", "--sizes", "1"]) == 2      # sizes must be >= 2
    assert cli.main(["bench", "--task", "bogus"]) == 2


def test_seeded_generator_is_the_references(oracle):
    from paper_2002_04989_b200 import random_symmetric
    for seed, n, d in ((1, 7, "gaussian"), (5, 9, "uniform")):
        a = random_symmetric(seed, n, d)
        b = oracle.random_symmetric(seed, n, uniform=(d == "uniform"))
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.gpu
def test_cli_full_vector_component_bench(tmp_path, oracle, capsys):
    out = tmp_path / "m.csv"
    assert cli.main(["full", "--random", "12", "--seed", "3", "--out", str(out)]) == 0
    got = np.loadtxt(out, delimiter=",")
    want = oracle.all_magnitudes(oracle.random_symmetric(3, 12))
    assert np.max(np.abs(got - want)) <= 1e-12
    vec = tmp_path / "v.csv"
    assert cli.main(["vector", "-i", "4", "--random", "12", "--seed", "3",
                     "--out", str(vec)]) == 0
    assert open(vec).readline().strip() == "j,magnitude"
    capsys.readouterr()
    # --signs (eigenid.cpp:129-134): the signed eigenvector, %.12g per line
    assert cli.main(["vector", "-i", "4", "--random", "12", "--seed", "3", "--signs"]) == 0
    sv = np.array([float(x) for x in capsys.readouterr().out.split()])
    a = oracle.random_symmetric(3, 12)
    mags = oracle.all_magnitudes(a).reshape(12, 12)[:, 4]
    want = oracle.recover_signs(a, 4, mags, oracle.eigenvalues(a)[4])
    assert sv.shape == (12,) and np.max(np.abs(sv - want)) <= 1e-9
    csv = tmp_path / "h.csv"
    csv.write_text("2,1\n1,2\n")
    assert cli.main(["component", "-i", "0", "-j", "1", "--csv", str(csv)]) == 0
    assert capsys.readouterr().out.strip() == "0.5"
    deg = tmp_path / "d.csv"
    deg.write_text("1,0\n0,1\n")
    assert cli.main(["full", "--csv", str(deg)]) == 1    # DegenerateEigenvalue
    rec = tmp_path / "r.csv"
    plot = tmp_path / "p.csv"
    assert cli.main(["bench", "--sizes", "8", "70", "--reps", "2", "--task",
                     "all-vectors", "--out", str(rec), "--plot-out", str(plot)]) == 0
    lines = open(rec).read().splitlines()
    assert lines[0] == "n,variant,task,run,seconds,checksum" and len(lines) == 5
    assert all(abs(float(l.split(",")[5]) - int(l.split(",")[0])) < 1e-8 for l in lines[1:])
    assert open(plot).readline().strip() == "n,variant,mean_seconds,stddev_seconds"
