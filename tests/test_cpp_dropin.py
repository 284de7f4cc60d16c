"""The C++ drop-in header (include/parsweep_b200.hpp): reference-shaped user
types solved through parsweep::gpu::solve_batch / compute_preliminary /
solve_with_preliminary_into, and the reference exception mapping."""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, load_golden, rel_l2

EXE = os.path.join(ROOT, "paper_0901_2859_b200", "_lib", "drop_in")


def test_header_compiles_standalone(tmp_path):
    src = tmp_path / "t.cpp"
    src.write_text('#include "parsweep_b200.hpp"\nint main() { return 0; }\n')
    subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Werror",
                    f"-I{os.path.join(ROOT, 'include')}", str(src)], check=True)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c0_n1024_P4", "rand_n200_p7", "p0_n50"])
def test_cpp_drop_in_solve_batch(tmp_path, name):
    g = load_golden(name)
    n, p, N = g["diag"].size, g["bnd"].size, g["F"].shape[0]
    case = tmp_path / "case.bin"
    with open(case, "wb") as f:
        np.array([n, p, N], np.int64).tofile(f)
        for a in (g["sub"], g["diag"], g["super"]):
            np.ascontiguousarray(a, np.float64).tofile(f)
        np.ascontiguousarray(g["bnd"], np.int64).tofile(f)
        np.ascontiguousarray(g["F"], np.float64).tofile(f)
    out = tmp_path / "out.bin"
    r = subprocess.run([EXE, str(case), str(out)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    X = np.fromfile(out, np.float64).reshape(N, n)
    assert rel_l2(X, g["X"]) <= 1e-12
