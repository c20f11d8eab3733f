"""the sketch-and-solve random-features baseline of `krr bench`
(solver.cpp:175-197) on the device vs the oracle, plus the plain-CG row (null preconditioner)."""
import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,d,s,t,lam,sigma", [(500, 5, 64, 1, 0.1, 1.5), (2000, 12, 256, 3, 1e-2, 3.0),
                                               (4000, 54, 512, 2, 1e-3, 4.0)])
def test_rf_baseline_matches_oracle(krr, oracle, ctx, n, d, s, t, lam, sigma):
    x = oracle.random_matrix(n, d, 3)
    y = oracle.random_matrix(n, t, 4)
    model = krr.train_random_features_baseline(krr.Dataset(x, y), krr.KernelSpec.gaussian(sigma),
                                               krr.ChainSpec(s1=s), lam, seed=0, ctx=ctx)
    w_ref, w_rff, b_rff = oracle.rf_baseline(x, y, sigma, lam, s, 0)
    assert np.array_equal(model.chain.rff.w, w_rff) and np.array_equal(model.chain.rff.b, b_rff)
    assert model.w.shape == (s, t)
    assert rel(model.w, w_ref) <= 1e-9, rel(model.w, w_ref)
    xq = oracle.random_matrix(300, d, 5)
    got = krr.baseline_predict_scores(model, xq, ctx=ctx)
    want = oracle.rff_apply_rows(xq, w_rff, b_rff) @ w_ref
    assert rel(got, want) <= 1e-9


def test_rf_baseline_errors_and_labels(krr, oracle, ctx):
    x = oracle.random_matrix(200, 3, 1)
    y = krr.rlsc_encode(np.arange(200) % 3, 3)
    data = krr.Dataset(x, y, label_map=[10.0, 20.0, 30.0])
    with pytest.raises(krr.NonPositiveLambda):
        krr.train_random_features_baseline(data, krr.KernelSpec.gaussian(1.0), krr.ChainSpec(s1=32), 0.0, ctx=ctx)
    m = krr.train_random_features_baseline(data, krr.KernelSpec.gaussian(1.0), krr.ChainSpec(s1=64), 1e-2, ctx=ctx)
    labels = krr.baseline_predict_labels(m, x[:20])
    assert len(labels) == 20 and set(labels) <= {10.0, 20.0, 30.0}


def test_plain_cg_row_matches_oracle(krr, oracle, ctx):
    """`krr bench` row 2 (krr.cpp plain-cg): PCG with a null preconditioner."""
    n, d, sigma, lam = 1500, 8, 3.0, 1e-1
    x = oracle.random_matrix(n, d, 21)
    y = oracle.random_matrix(n, 1, 22)
    c, report = krr.solve_regularized(x, krr.KernelSpec.gaussian(sigma), y, lam, None, 1e-8, 500, ctx=ctx)
    ref = oracle.solve_gaussian(x, sigma, lam, None, 0.0, y, 1e-8, 500, dense_k=False)
    assert abs(report.per_rhs[0].iterations - int(ref.iterations[0])) <= 1
    assert rel(c, ref.c) <= 1e-8


def test_trained_model_round_trips_through_krrm(krr, oracle, ctx, tmp_path):
    """a model trained on the device, saved in the reference's KRRM format and
    loaded back, predicts identically (predict_scores = cross_gram(Xq, X) C on the device)."""
    x = oracle.random_matrix(800, 6, 31)
    y = oracle.random_matrix(800, 2, 32)
    res = krr.train(krr.Dataset(x, y), krr.KernelSpec.gaussian(2.0),
                    krr.SolverConfig(tau=1e-8, max_iter=300, lambda_=1e-2, chain=krr.ChainSpec(s1=128), seed=3),
                    ctx=ctx)
    p = tmp_path / "trained.krrm"
    krr.save_model(p, res.model)
    back = krr.load_model(p)
    xq = oracle.random_matrix(100, 6, 33)
    a = krr.predict_scores(res.model, xq, ctx=ctx)
    b = krr.predict_scores(back, xq, ctx=ctx)
    assert np.array_equal(a, b)
    # coefficients ~1e2 cancel to scores ~1: the comparison bound scales with that cancellation
    assert rel(a, oracle.cross_gram(xq, x, 2.0) @ res.model.c) <= 1e-11
