"""CLI harness: same modes, flags and CSV schema as the
reference CLI (tools/cli_main.cpp)."""
import io

import pytest

from paper_2205_04194_b200 import cli


def run(argv):
    buf = io.StringIO()
    import sys
    old = sys.stdout
    sys.stdout = buf
    try:
        rc = cli.main(argv)
    finally:
        sys.stdout = old
    return rc, buf.getvalue().splitlines()


def test_errtrend_schema_and_bound(imq):
    rc, lines = run(["--mode", "errtrend"])
    assert rc == 0
    assert lines[0].startswith("# config: mode=errtrend n=0 t=1 m=10 levels=auto seed=42")
    assert lines[1] == "rho_x,M,case,E,bound"
    rows = [l.split(",") for l in lines[2:]]
    assert len(rows) == 3 * 2 * 100
    for rho, M, case, E, bound in rows:
        assert case in ("a", "b") and int(M) in (5, 10, 20)
        assert float(E) <= float(bound) * (1 + 1e-9) + 1e-15  # Theorem 1


@pytest.mark.gpu
def test_gpu_modes(imq):
    rc, lines = run(["--mode", "verify", "--n", "400", "--m", "8"])
    assert rc == 0 and lines[-1] == "# verify: 0 of 8 checks failed"
    rc, lines = run(["--mode", "bench", "--n", "3000", "--m", "6", "--levels", "1"])
    assert rc == 0 and lines[1] == "N,M,L,time_fast_s,time_dense_s,rel_err_inf"
    n, m, L, tf, td, err = lines[2].split(",")
    assert (n, m, L) == ("3000", "6", "1") and float(err) < 1e-4
    rc, lines = run(["--mode", "solve", "--n", "400", "--t", "0.03", "--m", "12"])
    assert rc == 0
    assert any(l.startswith("# solve: L=") and "converged=1" in l for l in lines)
    assert "index,coefficient" in lines and len(lines) > 400
