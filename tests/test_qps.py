"""CPU: QPS ingest against the reference's own parser
(qps.hpp, compiled in place into oracle/_ref) — identical canonical problems,
identical error messages — plus write/parse round trips."""
import numpy as np
import pytest

import oracle
import paper_2311_07710_b200 as rb
from instances import random_qp

pytestmark = pytest.mark.skipif(not oracle.have_ref(), reason="reference build absent")

# SPEC.md:116 fixture: min x^2 - 2x s.t. x <= 0.5 (default bound x >= 0)
ONE_D = """NAME          ONED
ROWS
 N  OBJ
 L  C1
COLUMNS
    X  OBJ  -2.0  C1  1.0
RHS
    RHS  C1  0.5
QUADOBJ
    X  X  2.0
ENDATA
"""

RICH = """* comment line
NAME          RICH
OBJSENSE
    MIN
ROWS
 N  COST
 L  LIM1
 G  LIM2
 E  MYEQN
 E  REQ
 L  RL
COLUMNS
    X1  COST  1.0   LIM1  1.0
    X1  LIM2  1.0
    X2  COST  2.0   LIM1  1.0
    X2  MYEQN  -1.0  REQ  2.5
    X3  COST  -1.0  MYEQN  1.0
    X3  RL  3.0
    X4  COST  0.5   REQ  1.0
    X4  LIM2  -2.0  RL  -1.0
RHS
    RHS  COST  -3.5
    RHS  LIM1  4.0   LIM2  1.0
    RHS  MYEQN  7.0  REQ  1.5
    RHS  RL  2.0
RANGES
    RNG  LIM1  2.5   LIM2  1.5
    RNG  MYEQN  -2.0  REQ  3.0
BOUNDS
 UP BND  X1  4.0
 MI BND  X2
 UP BND  X3  -1.0
 FX BND  X4  0.25
QUADOBJ
    X1  X1  2.0
    X1  X2  0.5
    X2  X2  3.0
    X3  X3  1.0
ENDATA
"""


def same_qp(a: rb.QuadraticProgram, b: rb.QuadraticProgram):
    for ma, mb in ((a.q, b.q), (a.a_ineq, b.a_ineq), (a.a_eq, b.a_eq)):
        assert (ma.n_rows, ma.n_cols) == (mb.n_rows, mb.n_cols)
        assert np.array_equal(ma.row_ptr, mb.row_ptr) and np.array_equal(ma.col_idx, mb.col_idx)
        assert np.array_equal(ma.values, mb.values)
    assert np.array_equal(a.c, b.c) and np.array_equal(a.b_ineq, b.b_ineq) and np.array_equal(a.b_eq, b.b_eq)
    assert a.obj_offset == b.obj_offset


@pytest.mark.parametrize("text", [ONE_D, RICH])
def test_parse_matches_reference(text):
    same_qp(rb.parse_qps(text), oracle.ref().parse_qps(text))


def test_one_d_fixture_shape():
    p = rb.parse_qps(ONE_D)
    # the default bound x >= 0 adds a second inequality row -x <= -0.0
    assert p.num_vars() == 1 and p.num_ineq() == 2 and p.num_eq() == 0
    assert list(p.b_ineq) == [0.5, -0.0] and np.signbit(p.b_ineq[1])
    assert p.q.to_dense()[0, 0] == 2.0 and p.c[0] == -2.0


def test_rich_semantics():
    p = rb.parse_qps(RICH)
    assert p.obj_offset == 3.5  # offset = -RHS on the objective row
    # MYEQN with range -2 -> [5, 7]: two <= rows; REQ range 3 -> [1.5, 4.5]; no pure E rows
    assert p.num_eq() == 0
    Q = p.q.to_dense()
    assert np.array_equal(Q, Q.T) and Q[0, 1] == 0.5


def test_round_trip_write_parse():
    for p in (random_qp(3, n=30, mi=12, me=4), rb.generate(rb.Gen.LASSO, 0.002, 1)):
        p.obj_offset = 1.25
        text = rb.write_qps(p)
        assert text == _ref_write(p)
        back = rb.parse_qps(text)
        # canonical form written with FR bounds: parse+canonicalize reproduces it
        same_qp(back, p)


def _ref_write(p):
    """The reference's own write_qps on the same problem."""
    return oracle.ref().write_qps(p)


@pytest.mark.parametrize("text,needle", [
    ("NAME X\nROWS\n N OBJ\nCOLUMNS\n X OBJ 1.0 C9 2.0\nRHS\nENDATA\n", "undeclared row 'C9'"),
    ("NAME X\nROWS\n N OBJ\nCOLUMNS\n X OBJ 1.0\n", "missing ENDATA"),
    ("NAME X\nROWS\n N OBJ\n L C1\nCOLUMNS\n X C1 abc\nENDATA\n", "expected a numeric value, got 'abc'"),
    ("NAME X\nNAME Y\nENDATA\n", "duplicate NAME section"),
    ("NAME X\nROWS\n N OBJ\nCOLUMNS\n M1 'MARKER' 'INTORG'\nENDATA\n", "integer markers are not supported"),
    ("NAME X\nROWS\n N OBJ\nCOLUMNS\n X OBJ 1.0\nBOUNDS\n BV B X\nENDATA\n", "unsupported bound type 'BV'"),
    ("NAME X\nOBJSENSE\n MAX\nENDATA\n", "only minimization"),
    ("NAME X\nROWS\n L C1\nCOLUMNS\n X C1 1.0\nENDATA\n", "no objective (N) row declared"),
    ("NAME X\nFOO\nENDATA\n", "unknown section 'FOO'"),
])
def test_parse_errors_match_reference(text, needle):
    with pytest.raises(rb.QpsParseError) as mine:
        rb.parse_qps(text)
    with pytest.raises(Exception) as ref:
        oracle.ref().parse_qps(text)
    assert needle in str(mine.value)
    assert str(mine.value) == str(ref.value)


def test_canonicalize_errors():
    bad = ONE_D.replace("RHS\n", "BOUNDS\n LO BND X 2.0\n UP BND X 1.0\nRHS\n").replace(
        "RHS\n    RHS  C1  0.5\n", "")
    with pytest.raises(rb.InvalidArgument, match="infeasible bounds on variable X"):
        rb.parse_qps(bad)
    asym = ONE_D.replace("QUADOBJ\n    X  X  2.0\n", "QMATRIX\n    X  X  2.0\n    X  Y  1.0\n").replace(
        "    X  OBJ  -2.0  C1  1.0\n", "    X  OBJ  -2.0  C1  1.0\n    Y  OBJ  1.0\n")
    with pytest.raises(rb.InvalidArgument, match="Q is not symmetric"):
        rb.parse_qps(asym)


def test_read_file(tmp_path):
    f = tmp_path / "oned.qps"
    f.write_text(ONE_D)
    same_qp(rb.read_qps(str(f)), rb.parse_qps(ONE_D))
    with pytest.raises(rb.QpsParseError, match="cannot open"):
        rb.read_qps(str(tmp_path / "missing.qps"))


def same_map(a: rb.CanonicalMap, b: rb.CanonicalMap):
    assert a.ineq_labels == b.ineq_labels and a.eq_labels == b.eq_labels


def test_parse_names_and_map_match_reference():
    """CanonicalMap labels (problem.hpp:95-104) and names survive the ABI."""
    for text in (ONE_D, RICH):
        a, ma = rb.parse_qps_with_map(text)
        b, mb = oracle.ref().parse_qps_with_map(text)
        same_qp(a, b)
        same_map(ma, mb)
        assert a.name == b.name and a.var_names == b.var_names
    p, mp = rb.parse_qps_with_map(RICH)
    assert p.name == "RICH" and p.var_names == ["X1", "X2", "X3", "X4"]
    assert mp.ineq_labels[:2] == ["row:LIM1:ub", "row:LIM1:lb"] and "bound:X4:ub" in mp.ineq_labels


def random_raw(seed, n=12, m=9, names=True):
    g = np.random.default_rng(seed)
    A = g.standard_normal((m, n)) * (g.random((m, n)) < 0.4)
    P = g.standard_normal((n, n)) * (g.random((n, n)) < 0.3)
    Q = P @ P.T
    def csr(M):
        r, c = np.nonzero(M)
        return rb.SparseMatrix.from_coo(M.shape[0], M.shape[1], r, c, M[r, c])
    lower = np.where(g.random(n) < 0.3, -np.inf, g.uniform(-2, 0, n))
    upper = np.where(g.random(n) < 0.3, np.inf, g.uniform(0, 2, n))
    rng = np.where(g.random(m) < 0.5, np.nan, g.uniform(-3, 3, m))
    return rb.RawProblem(q=csr(Q), c=g.standard_normal(n), a=csr(A), row_types=g.integers(0, 3, m),
                         rhs=g.standard_normal(m), lower=lower, upper=upper, range=rng,
                         obj_offset=float(g.standard_normal()), name=f"raw{seed}" if names else "",
                         row_names=[f"R{i}" for i in range(m)] if names else [],
                         var_names=[f"V{j}" for j in range(n)] if names else [])


@pytest.mark.parametrize("seed", range(6))
def test_canonicalize_matches_reference(seed):
    """rapdhg_canonicalize (RawProblem -> CanonicalProblem, problem.hpp:72-198)
    equals the reference's canonicalize: arrays, labels, names."""
    raw = random_raw(seed, names=seed % 2 == 0)
    a, ma = rb.canonicalize(raw)
    b, mb = oracle.ref().canonicalize(raw)
    same_qp(a, b)
    same_map(ma, mb)
    assert a.name == b.name and a.var_names == b.var_names
    assert a.num_rows() > 0 and len(ma.ineq_labels) == a.num_ineq() and len(ma.eq_labels) == a.num_eq()
    # write_qps with names = the reference writer's text
    assert rb.write_qps(a) == oracle.ref().write_qps(a)


def test_canonicalize_errors_match_reference():
    raw = random_raw(1)
    cases = []
    r = random_raw(1); r.c = r.c.copy(); r.c[3] = np.nan; cases.append((r, "NaN in objective vector"))
    r = random_raw(1); r.rhs = r.rhs.copy(); r.rhs[0] = np.nan; cases.append((r, "NaN in right-hand side"))
    r = random_raw(1); r.lower = r.lower.copy(); r.lower[2] = np.nan; cases.append((r, "NaN variable bound"))
    r = random_raw(1); r.lower = r.lower.copy(); r.upper = r.upper.copy(); r.lower[4], r.upper[4] = 1.0, 0.5
    cases.append((r, "infeasible bounds on variable V4"))
    r = random_raw(1, names=False); r.lower = r.lower.copy(); r.upper = r.upper.copy(); r.lower[4], r.upper[4] = 1.0, 0.5
    cases.append((r, "infeasible bounds on variable 4"))
    r = random_raw(1)
    qd = r.q.to_dense(); qd[0, 1] += 1.0
    rr, cc = np.nonzero(qd)
    r.q = rb.SparseMatrix.from_coo(qd.shape[0], qd.shape[1], rr, cc, qd[rr, cc])
    cases.append((r, "Q is not symmetric"))
    for r, msg in cases:
        with pytest.raises(rb.InvalidArgument) as mine:
            rb.canonicalize(r)
        with pytest.raises(Exception) as ref:
            oracle.ref().canonicalize(r)
        assert str(mine.value) == str(ref.value) == msg
    assert raw.num_vars() == 12


@pytest.mark.parametrize("seed", range(4))
def test_canonicalize_box_keeps_bounds_out_of_the_rows(seed):
    """keep_bounds (SolverConfig.box_projection, B200 extension): the same
    canonical problem minus the singleton bound rows canonicalize appends
    (problem.hpp:178-185), with the raw bounds carried in lower / upper."""
    raw = random_raw(seed)
    rows, mr = rb.canonicalize(raw)
    box, mb = rb.canonicalize(raw, keep_bounds=True)
    nb = int(np.isfinite(raw.lower).sum() + np.isfinite(raw.upper).sum())
    k = rows.num_ineq() - nb
    assert box.num_ineq() == k and box.num_eq() == rows.num_eq()
    assert mb.ineq_labels == mr.ineq_labels[:k] and mb.eq_labels == mr.eq_labels
    assert np.array_equal(box.a_ineq.row_ptr, rows.a_ineq.row_ptr[:k + 1])
    e = rows.a_ineq.row_ptr[k]
    assert np.array_equal(box.a_ineq.col_idx, rows.a_ineq.col_idx[:e])
    assert np.array_equal(box.a_ineq.values, rows.a_ineq.values[:e])
    assert np.array_equal(box.b_ineq, rows.b_ineq[:k])
    assert np.array_equal(box.lower, raw.lower) and np.array_equal(box.upper, raw.upper)
    assert rows.lower is None and rows.upper is None
    for ma, mb_ in ((box.q, rows.q), (box.a_eq, rows.a_eq)):
        assert np.array_equal(ma.values, mb_.values) and np.array_equal(ma.col_idx, mb_.col_idx)
    assert np.array_equal(box.c, rows.c) and box.obj_offset == rows.obj_offset


def test_bounds_from_rows_inverts_canonicalize():
    """bounds_from_rows(canonicalize(raw)) == canonicalize(raw, keep_bounds)
    when the raw rows have no singletons (they would become bounds too)."""
    g = np.random.default_rng(3)
    for seed in range(4):
        raw = random_raw(seed, n=10, m=6)
        dense = g.standard_normal((6, 10))
        r, c = np.nonzero(dense)
        raw.a = rb.SparseMatrix.from_coo(6, 10, r, c, dense[r, c])
        raw.lower[0], raw.upper[0] = -np.inf, 2.0  # one one-sided bound at least
        box, mb = rb.canonicalize(raw, keep_bounds=True)
        back = rb.bounds_from_rows(rb.canonicalize(raw)[0])
        assert back.num_ineq() == box.num_ineq()
        for ma, mb_ in ((back.a_ineq, box.a_ineq), (back.a_eq, box.a_eq)):
            assert np.array_equal(ma.row_ptr, mb_.row_ptr) and np.array_equal(ma.col_idx, mb_.col_idx)
            assert np.array_equal(ma.values, mb_.values)
        assert np.array_equal(back.b_ineq, box.b_ineq)
        assert np.array_equal(back.lower, box.lower) and np.array_equal(back.upper, box.upper)
    # a zero singleton stays a row; the tightest of two bounds wins
    a = rb.SparseMatrix.from_csr(3, 2, [0, 1, 2, 3], [0, 0, 1], [2.0, 1.0, 0.0])
    p = rb.QuadraticProgram(rb.SparseMatrix.identity(2), np.zeros(2), a, np.array([4.0, 1.5, 1.0]),
                            rb.SparseMatrix.zero(0, 2), np.zeros(0))
    q = rb.bounds_from_rows(p)
    assert q.num_ineq() == 1 and q.upper[0] == 1.5 and q.upper[1] == np.inf and q.lower is None
