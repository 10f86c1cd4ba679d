"""Result tables in the reference's schema (reference
bench.py:366-419 and its tests/test_bench.py:151-183): exact CSV header, no
CR, markdown round trip, empty rows rejected — CPU; one GPU experiment row
set against the oracle's FGMRES iteration counts."""

from __future__ import annotations

import math

import numpy as np
import pytest

from paper_2512_23804_b200.tables import COLUMNS, ResultRow, emit_table

ROWS = [
    ResultRow("steady", 4, 9, 2, 1, 3, 0.1, 0.01, 1e-8, "cheb5", 1, 7, True, 0.0123456789, 3.2e-9),
    ResultRow("steady", 4, 9, 2, 1, 3, 0.1, 0.01, 1e-8, "direct", 3, 5, False, 1.5, math.nan),
]


def test_emit_empty_rows_rejected():
    with pytest.raises(ValueError):
        emit_table([])
    with pytest.raises(ValueError, match="format"):
        emit_table(ROWS, format="latex")


def test_csv_header_and_cells_exact():
    table = emit_table(ROWS, format="csv")
    lines = table.splitlines()
    assert lines[0] == ("problem,n,N_h,m_xi,p,N_xi,sigma,beta,tol,mass_solver,n_tau,"
                        "iters,converged,seconds,final_rel_res")
    assert "\r" not in table and table.endswith("\n")
    assert lines[1] == "steady,4,9,2,1,3,0.1,0.01,1e-08,cheb5,1,7,true,0.012346,3.200000e-09"
    assert lines[2].split(",")[-3:] == ["false", "1.500000", "nan"]


def test_markdown_roundtrip():
    table = emit_table(ROWS, format="markdown")
    lines = table.strip().splitlines()
    header = [c.strip() for c in lines[0].strip("|").split("|")]
    assert tuple(header) == COLUMNS
    assert lines[1] == "|" + "|".join([" --- "] * len(COLUMNS)) + "|"
    for row, line in zip(ROWS, lines[2:]):
        rec = dict(zip(header, [c.strip() for c in line.strip("|").split("|")]))
        assert int(rec["n"]) == row.n and int(rec["iters"]) == row.iterations
        assert rec["mass_solver"] == row.mass_solver and int(rec["n_tau"]) == row.n_tau
        assert float(rec["sigma"]) == row.sigma and float(rec["beta"]) == row.beta
        assert (rec["converged"] == "true") == row.converged


@pytest.mark.gpu
def test_experiment_rows_match_oracle_iterations():
    import oracle
    from paper_2512_23804_b200.problems import build_problem, steady_system
    from paper_2512_23804_b200.tables import experiment_rows

    from test_gpu_configs import _oracle_kkt

    b = build_problem(2, n=16)
    rows = experiment_rows(b, mass_solvers=("cheb5",), n_taus=[b.n_terms])
    assert len(rows) == 1 and rows[0].converged and rows[0].final_rel_res <= 1e-8
    sys_ = steady_system(b)
    o_op, _, o_bd, rhs = _oracle_kkt(sys_, b)
    _, its, conv, _ = oracle.fgmres(o_op, o_bd, rhs, 1e-8)
    assert conv and abs(rows[0].iterations - its) <= 1
    assert emit_table(rows).splitlines()[1].startswith("steady,16,225,6,3,84,0.3,0.01,1e-08,cheb5,7,")
