"""Counter-based generators (csrc/crng.h): C2 Lasso, C3 portfolio, C4 SVM and
C5 (host.cpp + gen_device.cu; C4 also restated in numpy by oracle/synth.py
for the reference arm).
CPU: the host reference yields valid, deterministic instances with a
symmetric, diagonally dominant Q; the numpy SVM restatement equals the
library's arrays. GPU: the device generators' arrays are bit-identical to the
host reference."""
import numpy as np
import pytest

import paper_2311_07710_b200 as rb
from oracle import synth


def arrays(p):
    return [p.q.row_ptr, p.q.col_idx, p.q.values, p.a_ineq.row_ptr, p.a_ineq.col_idx, p.a_ineq.values, p.c,
            p.b_ineq, p.a_eq.row_ptr]


@pytest.mark.parametrize("kind", [rb.Gen.LARGE, rb.Gen.LARGE_LOCAL])
def test_host_large_valid_and_deterministic(kind, monkeypatch):
    monkeypatch.setenv("RAPDHG_GEN_DEVICE", "0")
    p = rb.generate(kind, 0.002, 5)
    n, m = p.num_vars(), p.num_rows()
    assert n == 20000 and m == 10000 and p.num_eq() == 0
    for mat in (p.q, p.a_ineq):
        rp, ci = mat.row_ptr, mat.col_idx
        assert rp[0] == 0 and rp[-1] == len(ci) and np.all(np.diff(rp) >= 0)
        for r in range(0, mat.n_rows, 997):  # strictly increasing columns within rows
            assert np.all(np.diff(ci[rp[r]:rp[r + 1]]) > 0)
    rows = np.repeat(np.arange(n), np.diff(p.q.row_ptr))
    dense_key = rows.astype(np.int64) * n + p.q.col_idx
    mirror = p.q.col_idx.astype(np.int64) * n + rows
    order = np.argsort(mirror)
    assert np.array_equal(np.sort(dense_key), mirror[order])          # pattern symmetric
    assert np.array_equal(p.q.values[np.argsort(dense_key)], p.q.values[order])  # values symmetric
    diag = p.q.values[rows == p.q.col_idx]
    off = np.bincount(rows[rows != p.q.col_idx], weights=np.abs(p.q.values[rows != p.q.col_idx]), minlength=n)
    assert len(diag) == n and np.all(diag >= off)                     # diagonally dominant
    q = rb.generate(kind, 0.002, 5)
    assert all(np.array_equal(a, b) for a, b in zip(arrays(p), arrays(q)))
    r = rb.generate(kind, 0.002, 6)
    assert not np.array_equal(p.c, r.c)


def test_host_large_local_pattern(monkeypatch):
    monkeypatch.setenv("RAPDHG_GEN_DEVICE", "0")
    n = 20000
    u = rb.generate(rb.Gen.LARGE, 0.002, 5)
    l = rb.generate(rb.Gen.LARGE_LOCAL, 0.002, 5)

    def home_fraction(p):
        a = p.a_ineq
        rows = np.repeat(np.arange(a.n_rows), np.diff(a.row_ptr))
        return np.mean(8 * rows // a.n_rows == 8 * a.col_idx.astype(np.int64) // n)

    assert home_fraction(l) > 0.9 and home_fraction(u) < 0.2


@pytest.mark.gpu
@pytest.mark.parametrize("kind", [rb.Gen.LARGE, rb.Gen.LARGE_LOCAL])
@pytest.mark.parametrize("scale", [0.0005, 0.01])
def test_device_generator_bit_identical(kind, scale, monkeypatch):
    monkeypatch.setenv("RAPDHG_GEN_DEVICE", "1")
    d = rb.generate(kind, scale, 5)
    monkeypatch.setenv("RAPDHG_GEN_DEVICE", "0")
    h = rb.generate(kind, scale, 5)
    for a, b in zip(arrays(d), arrays(h)):
        assert a.shape == b.shape and np.array_equal(a, b)


def svm_arrays(d):
    return [*d["q"], *d["a_ineq"], d["c"], d["b_ineq"], d["a_eq"][0]]


@pytest.mark.parametrize("scale,seed", [(0.001, 4), (0.004, 4), (0.004, 9)])
def test_svm_numpy_restatement_bit_identical(scale, seed, monkeypatch):
    monkeypatch.setenv("RAPDHG_GEN_DEVICE", "0")
    p = rb.generate(rb.Gen.SVM, scale, seed)
    d = synth.svm(scale, seed)
    for a, b in zip(arrays(p), svm_arrays(d)):
        assert a.shape == b.shape and np.array_equal(a, b)
    ns = int(round(1e6 * scale))
    nf = int(round(1e4 * scale))
    a = p.a_ineq
    assert a.n_rows == 2 * ns and p.num_vars() == nf + ns
    lens = np.diff(a.row_ptr)
    assert np.all(lens[ns:] == 1) and np.all(lens[:ns] <= 51) and lens[:ns].mean() > 0.6 * min(50, nf)
    for r in range(0, 2 * ns, 97):  # canonical rows, the t entry last
        seg = a.col_idx[a.row_ptr[r]:a.row_ptr[r + 1]]
        assert np.all(np.diff(seg) > 0) and seg[-1] == nf + r % ns


@pytest.mark.gpu
def test_device_svm_generator_bit_identical(monkeypatch):
    monkeypatch.setenv("RAPDHG_GEN_DEVICE", "1")
    d = rb.generate(rb.Gen.SVM, 0.03, 4)
    monkeypatch.setenv("RAPDHG_GEN_DEVICE", "0")
    h = rb.generate(rb.Gen.SVM, 0.03, 4)
    for a, b in zip(arrays(d), arrays(h)):
        assert a.shape == b.shape and np.array_equal(a, b)


@pytest.mark.parametrize("kind,scale", [(rb.Gen.LASSO, 0.002), (rb.Gen.PORTFOLIO, 0.002)])
def test_host_c2_c3_valid_and_deterministic(kind, scale, monkeypatch):
    """Counter-based C2 Lasso / C3 portfolio: canonical CSRs, the SURVEY
    structure, deterministic in the seed."""
    monkeypatch.setenv("RAPDHG_GEN_DEVICE", "0")
    p = rb.generate(kind, scale, 3)
    for mat in (p.q, p.a_ineq, p.a_eq):
        rp, ci = mat.row_ptr, mat.col_idx
        assert rp[0] == 0 and rp[-1] == len(ci) and np.all(np.diff(rp) >= 0)
        for r in range(mat.n_rows):
            assert np.all(np.diff(ci[rp[r]:rp[r + 1]]) > 0)
    if kind == rb.Gen.LASSO:
        nf, ns = 200, 20
        assert p.num_vars() == 2 * nf + ns and p.num_ineq() == 2 * nf and p.num_eq() == ns
        assert np.all(p.c[nf + ns:] == p.c[-1]) and p.c[-1] > 0  # lambda on t
    else:
        na, k = 2000, 2
        assert p.num_vars() == na + k and p.num_ineq() == na and p.num_eq() == k + 1
        assert np.all(p.a_eq.values[p.a_eq.row_ptr[k]:] == 1.0) and p.b_eq[k] == 1.0  # budget row
    q = rb.generate(kind, scale, 3)
    assert all(np.array_equal(a, b) for a, b in zip(arrays(p), arrays(q)))
    assert np.array_equal(p.a_eq.values, q.a_eq.values)
    assert not np.array_equal(p.a_eq.values, rb.generate(kind, scale, 4).a_eq.values)


@pytest.mark.gpu
@pytest.mark.parametrize("kind,scale", [(rb.Gen.LASSO, 0.01), (rb.Gen.LASSO, 0.3), (rb.Gen.PORTFOLIO, 0.01),
                                        (rb.Gen.PORTFOLIO, 0.2)])
def test_device_c2_c3_generators_bit_identical(kind, scale, monkeypatch):
    monkeypatch.setenv("RAPDHG_GEN_DEVICE", "1")
    d = rb.generate(kind, scale, 2)
    monkeypatch.setenv("RAPDHG_GEN_DEVICE", "0")
    h = rb.generate(kind, scale, 2)
    for a, b in zip(arrays(d) + [d.a_eq.col_idx, d.a_eq.values, d.b_eq],
                    arrays(h) + [h.a_eq.col_idx, h.a_eq.values, h.b_eq]):
        assert a.shape == b.shape and np.array_equal(a, b)
