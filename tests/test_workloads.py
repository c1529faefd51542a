"""Input generators: determinism, slice-independence, GE statistics."""
import numpy as np

import workloads as W


def test_determinism():
    a = W.ge(5000, seed=3); b = W.ge(5000, seed=3); c = W.ge(5000, seed=4)
    np.testing.assert_array_equal(a.log_lik, b.log_lik)
    assert not np.array_equal(a.states, c.states)
    d1 = W.dense(16, 500, seed=2); d2 = W.dense(16, 500, seed=2)
    np.testing.assert_array_equal(d1.log_lik, d2.log_lik)
    np.testing.assert_array_equal(d1.log_A, d2.log_A)


def test_counter_based_uniform():
    u = W.uniform(9, 0, 1000)
    assert ((u >= 0) & (u < 1)).all()
    np.testing.assert_array_equal(W.uniform(9, 500, 500), u[500:])
    assert abs(u.mean() - 0.5) < 0.05


def test_ge_statistics():
    """Empirical transition / emission frequencies match Eq. 22 within 4 standard errors (T=1e6)."""
    Pi, O, pr = W.ge_model()
    T = 1_000_000
    states, obs = W.simulate_discrete(pr, Pi, O, T, seed=11)
    counts = np.zeros((4, 4))
    np.add.at(counts, (states[:-1], states[1:]), 1)
    n = counts.sum(1, keepdims=True)
    freq = counts / n
    se = np.sqrt(Pi * (1 - Pi) / n) + 1e-12
    assert (np.abs(freq - Pi) < 4 * se + 1e-9).all()
    ec = np.zeros((4, 2)); np.add.at(ec, (states, obs), 1)
    ef = ec / ec.sum(1, keepdims=True)
    ese = np.sqrt(O * (1 - O) / ec.sum(1, keepdims=True))
    assert (np.abs(ef - O) < 4 * ese + 1e-9).all()


def test_dense_model_rows_are_distributions():
    lp, la = W.dense_model(64, 5)
    rows = np.exp(la.astype(np.float64)).sum(1)
    np.testing.assert_allclose(rows, 1.0, atol=1e-5)
    assert la.min() >= -80.0
    np.testing.assert_allclose(np.exp(lp.astype(np.float64)).sum(), 1.0, atol=1e-6)


def test_planted_path_margin():
    wl = W.planted(4, 100, seed=1)
    assert wl.log_lik.shape == (100, 4)
    assert (wl.log_lik[np.arange(100), wl.states] == 0).all()
