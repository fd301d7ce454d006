"""Pin the CPU oracle against the reference's golden vectors (no GPU).

Golden vectors come from the unmodified reference (tests/golden/make_golden.py)
plus the reference test suite's own known answers (pkg/tests/test_operators.py,
SPEC.md examples), restated here as literals.
"""

import numpy as np
import pytest

import oracle as O
from conftest import graph_from_golden

SMALL_GRAPHS = ["path5", "path10", "star4", "complete5", "ring6", "ring9", "grid4x5",
                "isolated3", "twocomp", "rand700"] + [f"rand{i}" for i in range(12)]


def _pair(z, name, key):
    return z[f"{name}/pair/{key}_ptr"], z[f"{name}/pair/{key}_idx"]


@pytest.mark.parametrize("name", SMALL_GRAPHS)
def test_structure_and_values_bit_exact(golden_small, name):
    z, meta = golden_small
    n, ptr, idx, w = graph_from_golden(z, name)
    l = O.laplacian(n, ptr, idx, w)
    assert np.array_equal(l.indptr, z[f"{name}/pair/L_ptr"])
    assert np.array_equal(l.indices, z[f"{name}/pair/L_idx"])
    assert np.array_equal(l.data, z[f"{name}/pair/L_val"])
    t_ptr, t_idx = O.two_hop(n, ptr, idx)
    assert np.array_equal(t_ptr, z[f"{name}/pair/T_ptr"])
    assert np.array_equal(t_idx, z[f"{name}/pair/T_idx"])
    for lit, key in ((False, "Q"), (True, "QL")):
        q = O.q_matrix(n, t_ptr, t_idx, literal_diagonal=lit)
        assert np.array_equal(q.indptr, z[f"{name}/pair/{key}_ptr"])
        assert np.array_equal(q.indices, z[f"{name}/pair/{key}_idx"])
        assert np.array_equal(q.data, z[f"{name}/pair/{key}_val"])
    rec = meta[f"{name}/pair"]
    q = O.q_matrix(n, t_ptr, t_idx)
    eps = O.identity_shift(q)
    if n <= 512:
        assert eps == rec["eps"]          # dense branch: same LAPACK call
    else:
        assert abs(eps - rec["eps"]) <= 1e-12 * abs(rec["eps"])
    mu = O.repulsion_weight(l, q, rec["eps"])
    assert mu == rec["mu"]
    a = O.assemble(l, q, rec["mu"], rec["eps"])
    assert np.array_equal(a.indptr, z[f"{name}/pair/A_ptr"])
    assert np.array_equal(a.indices, z[f"{name}/pair/A_idx"])
    assert np.array_equal(a.data, z[f"{name}/pair/A_val"])
    if "b_error" in rec:
        with pytest.raises(O.OracleDisconnected):
            O.degree_balancing(a)
    else:
        b, gdeg = O.degree_balancing(a)
        assert np.array_equal(b, z[f"{name}/pair/b"])
        assert gdeg == rec["generalized_degree"]
        assert O.pair_diagnostics(a, q, mu, rec["eps"]) == rec["diagnostics"]


def test_reference_test_suite_known_answers():
    """Literals from pkg/tests/test_operators.py (F10's two wrong pins excluded)."""
    from paper_2112_07862_b200 import synthetic as S
    n, ptr, idx, w = S.named("path", 5)
    t_ptr, t_idx = O.two_hop(n, ptr, idx)                       # test_operators.py:28-31
    assert [list(t_idx[t_ptr[i]:t_ptr[i + 1]]) for i in range(5)] == [[2], [3], [0, 4], [1], [2]]
    q = O.q_matrix(n, t_ptr, t_idx)                             # :59-66
    d = q.dense()
    assert np.allclose(np.diag(d), [1.5, 2.0, 3.0, 2.0, 1.5])
    assert d[0, 2] == pytest.approx(-1.5) and d[1, 3] == pytest.approx(-2.0)
    assert np.max(np.abs(q.row_sums())) < 1e-12
    assert O.identity_shift(q) == pytest.approx(1.5, rel=1e-12)  # :105-107
    l = O.laplacian(n, ptr, idx, w)
    assert O.repulsion_weight(l, q, 1.5) == pytest.approx(0.25, rel=1e-12)  # :123-132
    a = O.assemble(l, q, 0.25, 1.5)                             # :164-171
    left = a.diagonal() - O.gershgorin_radii(a)
    assert np.all(left >= 0.0) and abs(left[2]) <= 1e-12
    n, ptr, idx, w = S.named("star", 4)                         # :37-42, 72-77
    t_ptr, t_idx = O.two_hop(n, ptr, idx)
    assert [list(t_idx[t_ptr[i]:t_ptr[i + 1]]) for i in range(4)] == [[], [2, 3], [1, 3], [1, 2]]
    assert np.allclose(np.diag(O.q_matrix(n, t_ptr, t_idx).dense()), [0, 2, 2, 2])
    n, ptr, idx, w = S.named("complete", 5)                     # :33-35, 68-70
    assert O.two_hop(n, ptr, idx)[1].size == 0
    omega = 0.7                                                  # :109-114
    q2 = O.CSR(2, [0, 2, 4], [0, 1, 0, 1], [omega, -omega, -omega, omega])
    assert O.identity_shift(q2) == pytest.approx(2 * omega, rel=1e-12)
    with pytest.raises(O.OracleInputError):                      # :116-119
        O.identity_shift(O.CSR(2, [0, 1, 1], [1], [1.0]))
    with pytest.raises(O.OracleInputError):                      # :144-148
        O.repulsion_weight(l, q, -1.0)
    n, ptr, idx, w = S.named("ring", 6)                          # :179-182
    pair = O.operator_pair(n, ptr, idx, w)
    assert np.allclose(pair["b"], 1.0, atol=1e-12)
    rad = np.array([1.0, 2.0, 1.0])                              # :198-207 radii (1,2,1)
    b, _ = O.balance_radii(rad)
    assert abs(np.sum(np.log(b))) < 1e-12
    assert np.allclose(rad / b, (rad / b)[0], rtol=1e-12)


@pytest.mark.parametrize("case", ["path5/embed1", "path5/embed2", "ring6/embed2", "ring9/embed3",
                                  "grid4x5/embed3", "path10/embed2", "star4/embed1"]
                         + [f"rand{i}/embed{2 + i % 3}" for i in range(12)])
def test_embed_matches_reference(golden_small, case):
    z, meta = golden_small
    name, tag = case.split("/")
    k = int(tag[len("embed"):])
    n, ptr, idx, w = graph_from_golden(z, name)
    ref = meta[case]
    emb = O.embed(n, ptr, idx, w, k, tol=1e-8, max_iter=500, seed=42, require_convergence=False)
    d = emb["diagnostics"]
    assert d["iterations"] == ref["diagnostics"]["iterations"]
    assert d["converged"] == ref["diagnostics"]["converged"]
    ev = z[f"{case}/eigenvalues"]
    assert np.allclose(emb["eigenvalues"], ev, rtol=1e-12, atol=1e-14)
    assert np.allclose(emb["P"], z[f"{case}/P"], rtol=1e-8, atol=1e-10)
    assert d["epsilon"] == ref["diagnostics"]["epsilon"]


def test_twocomp_embed_raises(golden_small):
    z, meta = golden_small
    n, ptr, idx, w = graph_from_golden(z, "twocomp")
    with pytest.raises(O.OracleDisconnected) as e:
        O.embed(n, ptr, idx, w, 1)
    assert e.value.n_components == meta["twocomp/embed1"]["n_components"]


@pytest.mark.parametrize("case", ["path10/le2", "ring9/le2", "rand3/le3"])
def test_laplacian_eigenmaps(golden_small, case):
    z, meta = golden_small
    name, tag = case.split("/")
    k = int(tag[2:])
    n, ptr, idx, w = graph_from_golden(z, name)
    emb = O.laplacian_eigenmaps(n, ptr, idx, w, k, seed=7, require_convergence=False)
    assert emb["result"]["iterations"] == meta[case]["diagnostics"]["iterations"]
    assert np.allclose(emb["eigenvalues"], z[f"{case}/eigenvalues"], rtol=1e-10, atol=1e-13)


def test_spec_lobpcg_examples(golden_small):
    z, _ = golden_small
    a = O.CSR(3, [0, 1, 2, 3], [0, 1, 2], [1.0, 2.0, 3.0])
    r = O.lobpcg(a, np.ones(3), 1)
    assert r["eigenvalues"][0] == pytest.approx(1.0, rel=1e-12)
    assert np.allclose(r["eigenvalues"], z["spec_diag123/eigenvalues"], rtol=1e-14)
    ident = O.CSR(3, [0, 1, 2, 3], [0, 1, 2], [1.0, 1.0, 1.0])
    r = O.lobpcg(ident, np.array([1.0, 2.0, 4.0]), 1)
    assert r["eigenvalues"][0] == pytest.approx(0.25, rel=1e-12)
    assert np.allclose(np.abs(r["eigenvectors"][:, 0]), [0, 0, 0.5], atol=1e-8)


def test_deflated_q_solve_trajectory(golden_small):
    """smallest_above_null's LOBPCG branch (untested by the reference suite, F12)."""
    z, meta = golden_small
    n, ptr, idx, w = graph_from_golden(z, "rand700")
    t_ptr, t_idx = O.two_hop(n, ptr, idx)
    q = O.q_matrix(n, t_ptr, t_idx)
    r = O.lobpcg(q, np.ones(n), 8, tol=1e-6, max_iter=60, seed=42,
                 deflate=np.full(n, 1 / np.sqrt(n)))
    assert r["iterations"] == meta["rand700/q_defl"]["iterations"]
    assert np.allclose(r["eigenvalues"], z["rand700/q_defl/eigenvalues"], rtol=1e-12)
    assert np.allclose(r["ritz_sum_history"], z["rand700/q_defl/history"], rtol=1e-12)


def test_c1_pair_and_solve(golden_c1):
    z, meta = golden_c1
    n = meta["graph"]["n"]
    ptr, idx, w = z["graph_ptr"], z["graph_idx"], z["graph_w"]
    pair = O.operator_pair(n, ptr, idx, w)
    assert np.array_equal(pair["A"].indices, z["A_idx"])
    assert np.array_equal(pair["Q"].data, z["Q_val"])
    assert abs(pair["eps"] - meta["pair"]["eps"]) <= 1e-12 * meta["pair"]["eps"]
    r = O.lobpcg(pair["A"], pair["b"], 3, tol=1e-8, max_iter=200, seed=42)
    assert np.allclose(r["eigenvalues"], z["eigenvalues"], rtol=1e-12)
