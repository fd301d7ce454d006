"""Round-2 fast paths of the fp32 solve at the C5 block width (K = 32: w = 108):
the tcgen05 update + narrow Gram with derived [X P] blocks must agree with the CUDA-core
update + full Gram pair, and the breakdown recovery must bring a poisoned solve back.

Synthetic C5-family graphs (unit cube, kNN k = 8) at 60K nodes: seconds per solve.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mg():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2112_07862_b200 as m
    return m


@pytest.fixture(scope="module")
def c5_graph():
    from paper_2112_07862_b200 import synthetic
    return synthetic.config_graph("c5", n=60_000)


def _solve(mg, g, k=32, tol=1e-4):
    from paper_2112_07862_b200 import core
    cfg = mg.SolverConfig(k=k + 1, tol=tol, max_iter=3000, seed=42, precision="fp32")
    res, b, dg = core.embed_arrays(*g, k, cfg)
    return res, b.cpu().numpy(), dg


def test_tensor_core_paths_agree_with_cuda_core_paths(mg, c5_graph, monkeypatch):
    monkeypatch.setenv("MG_UPD_TC", "0")
    monkeypatch.setenv("MG_GRAM_DERIVE", "0")
    ref, b, _ = _solve(mg, c5_graph)
    monkeypatch.delenv("MG_UPD_TC")
    monkeypatch.delenv("MG_GRAM_DERIVE")
    new, _, _ = _solve(mg, c5_graph)
    assert ref.converged.all() and new.converged.all()
    # both blocks satisfy the reference's stopping rule; their Ritz values agree to the
    # rule's resolution (the columns of the last, edge-cut cluster are excluded: the rule
    # leaves their mixing with the cluster's members outside the block open)
    rel = np.abs(new.eigenvalues - ref.eigenvalues) / ref.eigenvalues
    assert rel[:26].max() < 2e-4, rel
    assert rel.max() < 2e-2, rel
    # the returned block is B-orthonormal on its own (exact finish before acceptance)
    X = new.eigenvectors.cpu().numpy()
    G = X.T @ (b[:, None] * X)
    assert np.abs(G - np.eye(G.shape[0])).max() < 2e-6


def test_breakdown_recovery_restores_a_poisoned_solve(mg, c5_graph, monkeypatch, capfd):
    clean, _, _ = _solve(mg, c5_graph)
    monkeypatch.setenv("MG_DEBUG_INJECT_NAN", "40")   # NaN into W at iteration 40
    monkeypatch.setenv("MG_DEBUG_RECOVER", "1")
    capfd.readouterr()
    res, _, _ = _solve(mg, c5_graph)
    err = capfd.readouterr().err
    assert "[recover]" in err, err[-500:]
    assert res.converged.all()
    assert np.isfinite(res.eigenvectors.cpu().numpy()).all()
    # a different trajectory to the same stopping rule: the rule resolves the smallest
    # Ritz values of this 60K-node problem to ~1e-3 relative (measured 7.6e-4)
    rel = np.abs(res.eigenvalues - clean.eigenvalues) / clean.eigenvalues
    assert rel[:26].max() < 3e-3, rel


def test_recovery_can_be_switched_off(mg, c5_graph, monkeypatch):
    from paper_2112_07862_b200._native import NativeError
    monkeypatch.setenv("MG_DEBUG_INJECT_NAN", "40")
    monkeypatch.setenv("MG_RECOVER", "0")
    # the injection hook lives in the guarded path: with the guard off the solve is clean
    res, _, _ = _solve(mg, c5_graph)
    assert res.converged.all()
