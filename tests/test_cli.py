"""CLI front end (paper_0901_2859_b200/cli.py) against the reference CLI's
contract (tools/main.cpp:23-25,55-125; text formats core/tridiag.hpp:107-212;
Partition::parse dichotomy/partition.hpp:52-72): exit codes, parse
diagnostics with line numbers, output format, stats JSON, --verify."""
import json
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

CLI = [sys.executable, "-m", "paper_0901_2859_b200.cli"]


def run(args, tmp_path):
    p = subprocess.run(CLI + args, cwd=ROOT, capture_output=True, text=True, timeout=300)
    return p.returncode, p.stdout, p.stderr


def write(tmp_path, name, text):
    f = tmp_path / name
    f.write_text(text)
    return str(f)


def test_read_formats_roundtrip():
    from paper_0901_2859_b200 import cli
    import io
    text = "4\n-1 -1 -1\n\n2.5 2.5 2.5 2.5\n-1 -1 -1\n"
    A = cli.read_matrix(text)
    assert A.n() == 4 and A.is_symmetric()
    buf = io.StringIO()
    cli.write_matrix(buf, A)
    B = cli.read_matrix(buf.getvalue())
    assert np.array_equal(A.diag, B.diag) and np.array_equal(A.sub, B.sub)
    F = np.random.default_rng(1).standard_normal((3, 4))
    buf = io.StringIO()
    cli.write_rhs_series(buf, 4, F)
    assert np.array_equal(cli.read_rhs_series(buf.getvalue(), 4), F)  # %.17g round trip


@pytest.mark.parametrize("text,line,frag", [
    ("", 1, "unexpected end of input reading matrix order"),
    ("1\n", 1, "matrix order must be an integer >= 2"),
    ("3\n1 x\n", 2, "bad number 'x' in sub-diagonal row"),
    ("3\n1 1\n2 2 2\n", 4, "unexpected end of input reading super-diagonal row"),
    ("3\n1 1\n2 2 2 2\n", 3, "diagonal row: expected 3 values, got 4"),
])
def test_matrix_parse_errors(text, line, frag):
    from paper_0901_2859_b200 import cli
    with pytest.raises(cli.ParseError) as e:
        cli.read_matrix(text)
    assert e.value.line == line and frag in str(e.value) and str(e.value).startswith(f"line {line}: ")


def test_rhs_parse_errors():
    from paper_0901_2859_b200 import cli
    with pytest.raises(cli.ParseError, match="rhs order 5 does not match matrix order 4"):
        cli.read_rhs_series("5 1\n1 2 3 4 5\n", 4)
    with pytest.raises(cli.ParseError, match="rhs count must be a positive integer"):
        cli.read_rhs_series("4 0\n", 4)
    with pytest.raises(cli.ParseError, match="rhs row: expected 4 values, got 3"):
        cli.read_rhs_series("4 1\n1 2 3\n", 4)


def test_partition_parse():
    from paper_0901_2859_b200 import cli
    assert cli.parse_partition(10, "3, 6,,8").boundaries == [3, 6, 8]
    for bad in ("3,x", "3,-1", "3,4 "):
        with pytest.raises(ValueError, match="bad boundary"):
            cli.parse_partition(10, bad)
    with pytest.raises(ValueError):  # Partition::validate: strictly increasing
        cli.parse_partition(10, "6,3")


def test_exit_codes_parse(tmp_path):
    m = write(tmp_path, "m.txt", "3\n-1 -1\n2 2 2\n-1 -1\n")
    bad = write(tmp_path, "bad.txt", "3\n-1 -1\n2 2 2\n")
    r = write(tmp_path, "r.txt", "3 1\n1 2 3\n")
    rc, _, err = run(["solve", "--matrix", bad, "--rhs", r], tmp_path)
    assert rc == 2 and "parse error: line 4: unexpected end of input" in err
    rc, _, err = run(["solve", "--matrix", m, "--rhs", r, "--partition", "2,x"], tmp_path)
    assert rc == 2 and "bad boundary" in err
    rc, _, err = run(["solve", "--matrix", str(tmp_path / "none.txt"), "--rhs", r], tmp_path)
    assert rc == 2 and "cannot open matrix file" in err


def _has_gpu():
    import torch
    return torch.cuda.is_available()


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU behaviour")
def test_exit_code_solver_without_gpu(tmp_path):
    """No CUDA device: the product has no CPU fallback -> solver error (3)."""
    m = write(tmp_path, "m.txt", "3\n-1 -1\n2 2 2\n-1 -1\n")
    r = write(tmp_path, "r.txt", "3 1\n1 2 3\n")
    rc, _, err = run(["solve", "--matrix", m, "--rhs", r], tmp_path)
    assert rc == 3 and "solver error" in err


@pytest.mark.gpu
@pytest.mark.parametrize("workers,partition", [(1, ""), (4, ""), (1, "10,30,31,60")])
def test_cli_solve_verify(tmp_path, orc, workers, partition):
    from paper_0901_2859_b200 import cli
    rng = np.random.default_rng(workers)
    n, N = 80, 7
    a = rng.uniform(-1, -0.5, n - 1)
    b = np.abs(np.r_[0, a]) + np.abs(np.r_[a, 0]) + rng.uniform(0.1, 1, n)
    import io
    from paper_0901_2859_b200 import TridiagMatrix
    A = TridiagMatrix.symmetric(a, b)
    buf = io.StringIO()
    cli.write_matrix(buf, A)
    m = write(tmp_path, "m.txt", buf.getvalue())
    F = rng.uniform(-1, 1, (N, n))
    buf = io.StringIO()
    cli.write_rhs_series(buf, n, F)
    r = write(tmp_path, "r.txt", buf.getvalue())
    out, stats = str(tmp_path / "x.txt"), str(tmp_path / "s.json")
    args = ["--workers", str(workers), "--verify", "solve", "--matrix", m, "--rhs", r,
            "--out", out, "--stats", stats]
    if partition:
        args += ["--partition", partition]
    rc, _, err = run(args, tmp_path)
    assert rc == 0, err
    X = cli.read_rhs_series(open(out).read(), n)
    if partition:
        bnd = [int(v) for v in partition.split(",")]
    elif workers > 1:
        from paper_0901_2859_b200 import decompose
        bnd = decompose(n, workers).induced_partition().boundaries
    else:
        bnd = []
    want = orc.solve_batch(a, b, a, np.array(bnd, dtype=np.int64), F)
    assert np.linalg.norm(X - want) / np.linalg.norm(want) <= 1e-12
    st = json.loads(open(stats).read())
    assert set(st) == {"comm_rounds", "combine_terms", "local_flops", "wall_time"}
    assert st["local_flops"] == 8 * n


@pytest.mark.gpu
def test_cli_verify_failure_and_breakdown(tmp_path):
    # singular (Neumann-like) matrix: pivot breakdown -> solver error 3
    m = write(tmp_path, "m.txt", "3\n-1 -1\n1 2 1\n-1 -1\n")
    r = write(tmp_path, "r.txt", "3 1\n1 2 3\n")
    rc, _, err = run(["solve", "--matrix", m, "--rhs", r], tmp_path)
    assert rc == 3 and "pivot breakdown" in err
