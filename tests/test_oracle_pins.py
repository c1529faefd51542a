"""Pins for the fp64 oracle (oracle/) against things other than itself (no GPU needed).

Each test ties the oracle to: brute-force enumeration of Eqs. 1-3, fixtures printed in
SPEC.md or derived independently in SURVEY.md Appendix A, closed forms, or invariants fixed by the
paper (Z_k constancy Eq. 10; Theorem 4; filtering = forward pass
PAPER.md:177).  A dropped term, wrong sign/index or transposed operand in hmm_oracle.c fails at least
one of them (random non-symmetric models vs brute force catch transposition; unnormalised potentials
catch dropped prior/emission terms; D=1 / A=I closed forms catch offset and -inf handling).
"""
import json
import os

import numpy as np
import pytest

import oracle
from oracle import brute
import workloads as W


def _load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


def _rng_model(rng, D, T, normalized=True):
    if normalized:
        A = rng.dirichlet(np.ones(D), size=D)
        pi = rng.dirichlet(np.ones(D))
        lik = rng.uniform(0.05, 1.0, size=(T, D))
        return (np.log(pi).astype(np.float32), np.log(A).astype(np.float32), np.log(lik).astype(np.float32))
    return (rng.normal(size=D).astype(np.float32), rng.normal(size=(D, D)).astype(np.float32),
            rng.normal(size=(T, D)).astype(np.float32))


# ---------------------------------------------------------------- GE model (Eq. 22)
def test_ge_model_matches_eq22(golden_dir):
    g = _load(golden_dir, "ge_model.json")
    Pi, O, pr = W.ge_model(**g["params"])
    np.testing.assert_allclose(Pi, g["Pi"], atol=1e-15)
    np.testing.assert_allclose(O, g["O"], atol=1e-15)
    np.testing.assert_allclose(pr, g["prior"], atol=0)
    np.testing.assert_allclose(Pi.sum(1), 1.0, atol=1e-15)
    np.testing.assert_allclose(O.sum(1), 1.0, atol=1e-15)
    np.testing.assert_allclose(O[:, 0] * 0.25, g["psi1_y0"], atol=1e-16)  # psi_1 = p(y|x) p(x), Eq. 5a


def test_ge_identity_when_no_switching():
    Pi, _, _ = W.ge_model(0.0, 0.0, 0.0, 0.01, 0.1)
    np.testing.assert_array_equal(Pi, np.eye(4))


# ---------------------------------------------------------------- fixtures
def _ge_T5(golden_dir):
    g = _load(golden_dir, "ge_T5.json")
    gm = _load(golden_dir, "ge_model.json")
    O = np.array(gm["O"])
    ll = np.log(O[:, g["obs"]].T).astype(np.float32)
    return g, np.log(np.array(gm["prior"])).astype(np.float32), np.log(np.array(gm["Pi"])).astype(np.float32), ll


def _spec_D2(golden_dir):
    g = _load(golden_dir, "spec_D2_T4.json")
    B = np.array(g["B"])
    ll = np.log(B[:, g["obs"]].T).astype(np.float32)
    return g, np.log(np.array(g["prior"])).astype(np.float32), np.log(np.array(g["A"])).astype(np.float32), ll


@pytest.mark.parametrize("which", ["ge_T5", "spec_D2"])
def test_oracle_matches_fixture(golden_dir, which):
    g, lp, la, ll = (_ge_T5 if which == "ge_T5" else _spec_D2)(golden_dir)
    # fp32 rounding of the fixture's log-inputs moves values by <= ~1e-7 relative; fixtures are printed to 1e-10.
    tol = 2e-7
    s = oracle.smooth(lp, la, ll)
    assert s["info"] == 0
    assert abs(s["log_z"] - g["log_z"]) < tol * 10
    np.testing.assert_allclose(s["smoothed"], g["smoothed"], atol=tol)
    np.testing.assert_allclose(s["filtered"], g["filtered"], atol=tol)
    v = oracle.viterbi(lp, la, ll)
    assert v["path"].tolist() == g["map_path"]
    assert abs(v["log_prob"] - g["map_log_prob"]) < tol * 10


@pytest.mark.parametrize("which", ["ge_T5", "spec_D2"])
def test_brute_force_matches_fixture(golden_dir, which):
    g, lp, la, ll = (_ge_T5 if which == "ge_T5" else _spec_D2)(golden_dir)
    b = brute.smooth(lp, la, ll)
    np.testing.assert_allclose(b["smoothed"], g["smoothed"], atol=2e-7)
    np.testing.assert_allclose(b["filtered"], g["filtered"], atol=2e-7)
    m = brute.viterbi(lp, la, ll)
    assert m["path"].tolist() == g["map_path"]
    assert abs(m["gap"] - g["map_gap"]) < 1e-4


def test_spec_pairwise_and_joint_weight(golden_dir):
    g, lp, la, ll = _spec_D2(golden_dir)
    # psi_2(x_1,x_2) = p(y_2|x_2) p(x_2|x_1) (Eq. 5b) — the potential the oracle's forward step uses.
    pw = np.exp(la.astype(np.float64)) * np.exp(ll[1].astype(np.float64))[None, :]
    np.testing.assert_allclose(pw, g["pairwise0_y1"], atol=1e-7)
    w = oracle.joint_weight(lp, la, ll[:2], np.array([0, 1], np.int32))
    assert abs(w - g["joint_weight_obs01_states01"]) < 1e-6


# ---------------------------------------------------------------- brute force (Eqs. 1-3)
@pytest.mark.parametrize("normalized", [True, False])
def test_oracle_vs_brute_force_random(normalized):
    """SPEC.md:451-452 acceptance: random models D in {2,3,4}, T in {2..8} vs enumeration."""
    rng = np.random.default_rng(20260 + normalized)
    n_strict = 0
    for k in range(50):
        D = int(rng.integers(2, 5)); T = int(rng.integers(2, 9))
        if D ** T > 70000:
            T = 6
        lp, la, ll = _rng_model(rng, D, T, normalized)
        s = oracle.smooth(lp, la, ll); b = brute.smooth(lp, la, ll)
        assert s["info"] == 0
        assert abs(s["log_z"] - b["log_z"]) < 1e-10 * max(1.0, abs(b["log_z"]))
        assert abs(s["log_z_bwd"] - b["log_z"]) < 1e-10 * max(1.0, abs(b["log_z"]))
        np.testing.assert_allclose(s["smoothed"], b["smoothed"], atol=1e-10)
        np.testing.assert_allclose(s["filtered"], b["filtered"], atol=1e-10)
        v = oracle.viterbi(lp, la, ll); m = brute.viterbi(lp, la, ll)
        assert abs(v["log_prob"] - m["log_prob"]) < 1e-9
        assert abs(oracle.joint_weight(lp, la, ll, v["path"]) - m["log_prob"]) < 1e-9
        if m["gap"] > 1e-6:
            n_strict += 1
            assert v["path"].tolist() == m["path"].tolist()
        score, gap = oracle.max_marginals(lp, la, ll)
        np.testing.assert_allclose(score, brute.max_marginals(lp, la, ll), atol=1e-9)
    assert n_strict > 40


def test_oracle_viterbi_ties_smallest_index():
    """Exact ties: uniform everything -> every path ties; smallest-index rule gives all zeros."""
    D, T = 3, 5
    lp = np.full(D, -np.log(D), np.float32); la = np.full((D, D), -np.log(D), np.float32)
    ll = np.zeros((T, D), np.float32)
    v = oracle.viterbi(lp, la, ll)
    assert v["path"].tolist() == [0] * T
    assert v["path"].tolist() == brute.viterbi(lp, la, ll)["path"].tolist()


# ---------------------------------------------------------------- closed forms (any T)
def test_closed_form_D1():
    T = 1000
    rng = np.random.default_rng(1)
    lp = np.array([-0.3], np.float32); la = np.array([[-0.7]], np.float32)
    ll = rng.normal(size=(T, 1)).astype(np.float32)
    s = oracle.smooth(lp, la, ll)
    expect = float(lp[0]) + float(ll.astype(np.float64).sum()) + (T - 1) * float(la[0, 0])
    assert abs(s["log_z"] - expect) < 1e-9 * abs(expect)
    np.testing.assert_array_equal(s["smoothed"], 1.0)
    v = oracle.viterbi(lp, la, ll)
    assert (v["path"] == 0).all() and abs(v["log_prob"] - expect) < 1e-9 * abs(expect)


def test_closed_form_identity_transition():
    """A = I (off-diagonal -inf): states never move (SURVEY.md §8(c) closed form ii)."""
    D, T = 4, 2000
    rng = np.random.default_rng(2)
    lp = np.log(rng.dirichlet(np.ones(D))).astype(np.float32)
    la = np.full((D, D), -np.inf, np.float32); np.fill_diagonal(la, 0.0)
    ll = (0.05 * rng.normal(size=(T, D))).astype(np.float32)
    per_state = lp.astype(np.float64) + ll.astype(np.float64).sum(0)
    lz = np.logaddexp.reduce(per_state)
    s = oracle.smooth(lp, la, ll)
    assert abs(s["log_z"] - lz) < 1e-10 * max(1, abs(lz))
    post = np.exp(per_state - lz)
    np.testing.assert_allclose(s["smoothed"], np.broadcast_to(post, (T, D)), atol=1e-10)
    cum = lp.astype(np.float64)[None, :] + np.cumsum(ll.astype(np.float64), 0)
    filt = np.exp(cum - np.logaddexp.reduce(cum, axis=1)[:, None])
    np.testing.assert_allclose(s["filtered"], filt, atol=1e-10)
    v = oracle.viterbi(lp, la, ll)
    assert (v["path"] == int(np.argmax(per_state))).all()
    assert abs(v["log_prob"] - per_state.max()) < 1e-9


def test_closed_form_identical_rows():
    """A(i,.) = q for all i: states i.i.d.; marginals factorise (closed form iii)."""
    D, T = 5, 3000
    rng = np.random.default_rng(3)
    q = rng.dirichlet(np.ones(D)); pi = rng.dirichlet(np.ones(D))
    lp = np.log(pi).astype(np.float32); lq = np.log(q).astype(np.float32)
    la = np.tile(lq, (D, 1))
    ll = np.log(rng.uniform(0.01, 1, size=(T, D))).astype(np.float32)
    w = np.exp(lq.astype(np.float64))[None, :] * np.exp(ll.astype(np.float64))
    w[0] = np.exp(lp.astype(np.float64)) * np.exp(ll[0].astype(np.float64))
    marg = w / w.sum(1, keepdims=True)
    s = oracle.smooth(lp, la, ll)
    np.testing.assert_allclose(s["smoothed"], marg, atol=1e-12)
    np.testing.assert_allclose(s["filtered"], marg, atol=1e-12)
    assert abs(s["log_z"] - np.log(w.sum(1)).sum()) < 1e-10 * abs(s["log_z"])
    v = oracle.viterbi(lp, la, ll)
    sc = lq.astype(np.float64)[None, :] + ll.astype(np.float64)
    sc[0] = lp.astype(np.float64) + ll[0]
    assert v["path"].tolist() == np.argmax(sc, 1).tolist()


def test_closed_form_uninformative_evidence():
    """log_lik == 0, stochastic A, sum(pi)=1: log Z = 0, marginals = pi A^t (closed form iv)."""
    D, T = 4, 200
    rng = np.random.default_rng(4)
    A = rng.dirichlet(np.ones(D), size=D); pi = rng.dirichlet(np.ones(D))
    lp = np.log(pi).astype(np.float32); la = np.log(A).astype(np.float32)
    A32 = np.exp(la.astype(np.float64)); pi32 = np.exp(lp.astype(np.float64))
    ll = np.zeros((T, D), np.float32)
    s = oracle.smooth(lp, la, ll)
    # fp32 rounding makes rows sum to 1 +- 1e-7; compare with the same rounded model
    m = pi32.copy(); exp_marg = []
    zsum = np.log(pi32.sum())
    for t in range(T):
        if t > 0:
            m = m @ A32
        exp_marg.append(m / m.sum())
    np.testing.assert_allclose(s["filtered"], np.array(exp_marg), atol=1e-12)
    np.testing.assert_allclose(s["smoothed"], np.array(exp_marg), atol=1e-6)
    assert abs(s["log_z"]) < 1e-5 and abs(zsum) < 1e-6


def test_closed_form_planted_path_large_T():
    """Planted path z with margin -> Viterbi returns z exactly, gaps >= margin (closed form v)."""
    wl = W.planted(6, 100_000, seed=5, margin=4.0)
    v = oracle.viterbi(wl.log_pi, wl.log_A, wl.log_lik)
    assert v["info"] == 0
    assert np.array_equal(v["path"], wl.states)
    _, gap = oracle.max_marginals(wl.log_pi, wl.log_A, wl.log_lik)
    assert gap.min() >= 4.0 - 1e-6


# ---------------------------------------------------------------- invariants at scale
def test_invariants_ge_1e5():
    wl = W.ge(100_000, seed=1)
    s = oracle.smooth(wl.log_pi, wl.log_A, wl.log_lik)
    assert s["info"] == 0
    assert abs(s["log_z"] - s["log_z_bwd"]) < 1e-9 * abs(s["log_z"])       # Z_k constancy (k=1 vs k=T)
    np.testing.assert_allclose(s["smoothed"].sum(1), 1.0, atol=1e-12)
    np.testing.assert_allclose(s["filtered"].sum(1), 1.0, atol=1e-12)
    np.testing.assert_allclose(s["smoothed"][-1], s["filtered"][-1], atol=1e-12)
    assert -0.4 < s["log_z"] / wl.T < -0.2                                   # SURVEY App. A.1 entropy-rate scale
    v = oracle.viterbi(wl.log_pi, wl.log_A, wl.log_lik)
    assert v["log_prob"] <= s["log_z"]
    assert abs(oracle.joint_weight(wl.log_pi, wl.log_A, wl.log_lik, v["path"]) - v["log_prob"]) < 1e-7
    score, gap = oracle.max_marginals(wl.log_pi, wl.log_A, wl.log_lik)
    # Theorem 4 / Eq. 21: max_x (log psi~f_k + log psi~b_k) is the MAP log-prob at every k.
    np.testing.assert_allclose(score.max(1), v["log_prob"], atol=1e-6)
    # Raw GE has exact ties: the tie count is small but non-zero.
    assert 0 < int((gap < 1e-9).sum()) < 0.02 * wl.T


def test_time_reversal_symmetry():
    """Symmetric doubly-stochastic A + uniform prior: reversing the evidence reverses the marginals."""
    D, T = 4, 500
    rng = np.random.default_rng(6)
    P = sum(w * np.eye(D)[rng.permutation(D)] for w in rng.dirichlet(np.ones(3)))
    A = 0.5 * (P + P.T)
    lp = np.full(D, -np.log(D), np.float32)
    la = np.log(A).astype(np.float32)
    la = np.minimum(la, la.T)  # exact symmetry after rounding
    ll = np.log(rng.uniform(0.01, 1, size=(T, D))).astype(np.float32)
    a = oracle.smooth(lp, la, ll); b = oracle.smooth(lp, la, ll[::-1].copy())
    np.testing.assert_allclose(a["smoothed"], b["smoothed"][::-1], atol=1e-11)
    assert abs(a["log_z"] - b["log_z"]) < 1e-10 * abs(a["log_z"])


# ---------------------------------------------------------------- impossible evidence (info)
def test_info_impossible_evidence():
    D, T = 3, 20
    rng = np.random.default_rng(7)
    lp, la, ll = _rng_model(rng, D, T)
    ll[5, :] = -np.inf
    assert oracle.smooth(lp, la, ll)["info"] == 6
    assert oracle.viterbi(lp, la, ll)["info"] == 6
    # zero transitions: stuck in state 0 (A = I), evidence says state 1 at t=3
    lp2 = np.array([0.0, -np.inf], np.float32)
    la2 = np.array([[0.0, -np.inf], [-np.inf, 0.0]], np.float32)
    ll2 = np.zeros((6, 2), np.float32); ll2[3, 0] = -np.inf
    assert oracle.smooth(lp2, la2, ll2)["info"] == 4
    assert oracle.viterbi(lp2, la2, ll2)["info"] == 4
    ll3 = ll2.copy(); ll3[2, 1] = np.nan
    assert oracle.smooth(lp2, la2, ll3)["info"] == -1


def test_batched_oracle_matches_single():
    wl = W.dense_batch(6, 8, 300)
    sb = oracle.smooth_batched(wl.log_pi, wl.log_A, wl.log_lik, nthreads=3)
    vb = oracle.viterbi_batched(wl.log_pi, wl.log_A, wl.log_lik, nthreads=3)
    for b in range(6):
        s = oracle.smooth(wl.log_pi, wl.log_A, wl.log_lik[b])
        np.testing.assert_array_equal(sb["smoothed"][b], s["smoothed"])
        assert sb["log_z"][b] == s["log_z"]
        v = oracle.viterbi(wl.log_pi, wl.log_A, wl.log_lik[b])
        np.testing.assert_array_equal(vb["path"][b], v["path"])


# ---------------------------------------------------------------- sampled smoother (full-size checks)
@pytest.mark.parametrize("D,T", [(4, 5000), (3, 777), (1, 50), (8, 2000)])
def test_smooth_sampled_matches_full_oracle(D, T):
    """oracle.smooth_sampled is Algorithm 1 with O(samples) memory: at every sampled step it must give
    the same numbers as the full oracle (same recursions, same operation order -> bitwise equal)."""
    wl = W.ge(T, seed=3) if D == 4 else W.dense(D, T, seed=D)
    full = oracle.smooth(wl.log_pi, wl.log_A, wl.log_lik)
    ts = np.unique(np.r_[0, T - 1, np.random.default_rng(D).integers(0, T, 40)])
    s = oracle.smooth_sampled(wl.log_pi, wl.log_A, wl.log_lik, ts)
    assert s["info"] == 0 and s["log_z"] == full["log_z"]
    assert np.array_equal(s["filtered"], full["filtered"][ts])
    assert np.array_equal(s["smoothed"], full["smoothed"][ts])


def test_smooth_sampled_info():
    wl = W.ge(3000, seed=4)
    wl.log_lik[1234, :] = -np.inf
    assert oracle.smooth_sampled(wl.log_pi, wl.log_A, wl.log_lik, [5, 10])["info"] == 1235


# ---------------------------------------------------------------- Baum-Welch E-step statistics (f2)
@pytest.mark.parametrize("seed", range(12))
def test_smooth_stats_brute_force(seed):
    """xi_sum / gamma_sum from the forward-backward potentials equal the enumeration of all D^T paths."""
    rng = np.random.default_rng(100 + seed)
    D, T = int(rng.integers(2, 5)), int(rng.integers(2, 7))
    if seed % 2:
        wl = W.random_potentials(D, T, seed=seed)
    else:
        wl = W.dense(D, T, seed=seed)
    o = oracle.smooth_stats(wl.log_pi, wl.log_A, wl.log_lik)
    b = brute.pair_stats(wl.log_pi, wl.log_A, wl.log_lik)
    assert o["info"] == 0
    np.testing.assert_allclose(o["xi_sum"], b["xi_sum"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(o["gamma_sum"], b["gamma_sum"], rtol=1e-10, atol=1e-12)


def test_smooth_stats_invariants():
    wl = W.ge(20_000, seed=3)
    o = oracle.smooth_stats(wl.log_pi, wl.log_A, wl.log_lik)
    sm = oracle.smooth(wl.log_pi, wl.log_A, wl.log_lik)["smoothed"]
    T = 20_000
    assert abs(o["xi_sum"].sum() - (T - 1)) < 1e-8 * T
    # marginalising xi over x_t gives the occupancies of x_{t-1} (t = 0..T-2), and vice versa
    np.testing.assert_allclose(o["xi_sum"].sum(1), sm[:-1].sum(0), rtol=1e-9)
    np.testing.assert_allclose(o["xi_sum"].sum(0), sm[1:].sum(0), rtol=1e-9)
    np.testing.assert_allclose(o["gamma_sum"], sm.sum(0), rtol=1e-12)


# ---------------------------------------------------------------- symbol inputs (f1)
@pytest.mark.parametrize("which", ["ge_T5", "spec_D2"])
def test_symbol_oracle_matches_fixture(golden_dir, which):
    """Discrete observations through the emission matrix: the printed fixture values."""
    if which == "ge_T5":
        g = _load(golden_dir, "ge_T5.json"); gm = _load(golden_dir, "ge_model.json")
        lp, la, B = np.log(gm["prior"]), np.log(gm["Pi"]), np.array(gm["O"])
    else:
        g = _load(golden_dir, "spec_D2_T4.json")
        lp, la, B = np.log(g["prior"]), np.log(g["A"]), np.array(g["B"])
    y = np.array(g["obs"], np.uint8)
    o = oracle.smooth_symbols(lp, la, np.log(B), y)
    assert abs(o["log_z"] - g["log_z"]) < 1e-7
    np.testing.assert_allclose(o["smoothed"], g["smoothed"], atol=1e-7)
    v = oracle.viterbi_symbols(lp, la, np.log(B), y)
    if "map_path" in g:
        assert list(v["path"]) == g["map_path"]


def test_symbol_workload_matches_loglik_workload():
    """ge_symbols is the same chain as ge: gathering log O at y reproduces ge's log_lik exactly."""
    ws = W.ge_symbols(10_000, 3)
    wl = W.ge(10_000, 3)
    np.testing.assert_array_equal(oracle.symbols_loglik(ws.log_B, ws.y), wl.log_lik)
    d = W.discrete(5, 7, 1000, 2)
    assert d.y.max() < 7 and np.allclose(np.exp(d.log_B.astype(np.float64)).sum(1), 1.0, atol=1e-6)


def test_golden_fixtures_regenerate_from_enumeration():
    """tests/golden/ge_T5.json and spec_D2_T4.json are what tools/make_golden.py computes with
    oracle/brute.py alone (Eqs. 1-3 by enumeration): no stored value is hand-copied."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "make_golden", os.path.join(os.path.dirname(os.path.dirname(__file__)), "tools", "make_golden.py"))
    mg = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mg)
    assert mg.check(mg.compute()) == []


@pytest.mark.parametrize("D,T,seed", [(4, 100_000, 1), (3, 9_000, 2), (1, 5000, 3), (8, 4097, 4), (2, 1, 5)])
def test_max_marginal_gap_o_t_memory_is_bitwise_the_full_routine(D, T, seed):
    """oracle.max_marginal_gap (checkpointed, O(T) memory, used at T = 1e8) returns exactly the gap of
    oracle.max_marginals (pinned to enumeration below) rounded to float32, block boundaries included."""
    wl = W.ge(T, seed, jitter=0.1) if D == 4 else W.random_potentials(D, T, seed)
    _, gap = oracle.max_marginals(wl.log_pi, wl.log_A, wl.log_lik)
    g32 = oracle.max_marginal_gap(wl.log_pi, wl.log_A, wl.log_lik)
    assert np.array_equal(g32, gap.astype(np.float32))


def test_joint_weight_diff_matches_difference_of_weights():
    """Eq. 6 term-wise difference == difference of the full joint weights (small T, no cancellation issue)."""
    rng = np.random.default_rng(7)
    for k in range(20):
        D, T = int(rng.integers(2, 6)), int(rng.integers(1, 300))
        wl = W.random_potentials(D, T, 100 + k)
        a = rng.integers(0, D, T).astype(np.int32)
        b = a.copy()
        flip = rng.random(T) < 0.2
        b[flip] = rng.integers(0, D, int(flip.sum()))
        d = oracle.joint_weight_diff(wl.log_pi, wl.log_A, wl.log_lik, a, b)
        ref = oracle.joint_weight(wl.log_pi, wl.log_A, wl.log_lik, a) - oracle.joint_weight(wl.log_pi, wl.log_A,
                                                                                             wl.log_lik, b)
        assert abs(d - ref) <= 1e-9 * max(1.0, abs(ref))
        assert oracle.joint_weight_diff(wl.log_pi, wl.log_A, wl.log_lik, a, a) == 0.0


# ---------------------------------------------------------------- paper-faithful variants
from oracle import variants  # noqa: E402


@pytest.mark.parametrize("seed", range(40))
def test_alg5_and_path_elements_vs_brute_force(seed):
    """Algorithm 5 (Eq. 21 assembly) and the Def. 4 reduction both give the enumerated MAP on inputs
    whose best sequence is unique by a margin (Theorem 4 / Corollary 1)."""
    rng = np.random.default_rng(7000 + seed)
    D = int(rng.integers(2, 5)); T = int(rng.integers(2, 8))
    lp, la, ll = _rng_model(rng, D, T, normalized=bool(seed % 2))
    bv = brute.viterbi(lp, la, ll)
    x, w = bv["path"], bv["log_prob"]
    if bv["gap"] < 1e-6:
        pytest.skip("tied instance")
    a5 = variants.viterbi_maxproduct(lp, la, ll)
    np.testing.assert_array_equal(a5["path"], x)
    assert abs(a5["log_prob"] - w) <= 1e-9 * max(1, abs(w))
    assert abs(a5["path_weight"] - w) <= 1e-9 * max(1, abs(w)) and a5["coherent"]
    pe = variants.viterbi_path_elements(lp, la, ll)
    np.testing.assert_array_equal(pe["path"], x)
    assert abs(pe["log_prob"] - w) <= 1e-9 * max(1, abs(w))


def test_alg5_incoherent_under_ties_closed_form():
    """Two MAP paths (0,1,0,1,..) and (1,0,1,0,..) tie; Eq. 21 takes the smallest index at every (tied)
    step and assembles (0,0,...,0), whose weight is log(pi_0) + (T-1) log(eps) + sum ll: SPEC's
    diagnostic must flag it, and the Def. 4 reduction must still return a MAP path."""
    eps, T = 0.1, 6
    lp = np.log(np.array([0.5, 0.5])).astype(np.float32)
    la = np.log(np.array([[eps, 1 - eps], [1 - eps, eps]])).astype(np.float32)
    ll = np.zeros((T, 2), np.float32)
    a5 = variants.viterbi_maxproduct(lp, la, ll)
    np.testing.assert_array_equal(a5["path"], np.zeros(T, np.int32))
    map_w = float(np.float64(lp[0]) + (T - 1) * np.float64(la[0, 1]))
    bad_w = float(np.float64(lp[0]) + (T - 1) * np.float64(la[0, 0]))
    assert abs(a5["log_prob"] - map_w) <= 1e-12
    assert abs(a5["path_weight"] - bad_w) <= 1e-12
    assert not a5["coherent"] and a5["n_tied"] == T
    pe = variants.viterbi_path_elements(lp, la, ll)
    assert abs(pe["log_prob"] - map_w) <= 1e-12
    assert abs(oracle.joint_weight(lp, la, ll, pe["path"]) - map_w) <= 1e-12


def test_path_elements_vs_alg4_on_ge():
    """Near-tie-free GE sequence (jittered, SURVEY §8(d) recipe): the Def. 4 reduction, Algorithm 5 and
    the Algorithm 4 oracle agree on the path exactly and on the weight to 1e-9."""
    wl = W.ge(256, seed=3, jitter=0.1)
    v = oracle.viterbi(wl.log_pi, wl.log_A, wl.log_lik)
    _, gap = oracle.max_marginals(wl.log_pi, wl.log_A, wl.log_lik)
    assert gap.min() >= 1e-3
    pe = variants.viterbi_path_elements(wl.log_pi, wl.log_A, wl.log_lik)
    a5 = variants.viterbi_maxproduct(wl.log_pi, wl.log_A, wl.log_lik)
    np.testing.assert_array_equal(pe["path"], v["path"])
    np.testing.assert_array_equal(a5["path"], v["path"])
    assert abs(pe["log_prob"] - v["log_prob"]) <= 1e-9 * abs(v["log_prob"])
    assert abs(a5["log_prob"] - v["log_prob"]) <= 1e-9 * abs(v["log_prob"])


def test_alg5_raw_ge_flags_ties():
    """Raw GE observations have exact max-marginal ties: the diagnostic counts them and
    any incoherent assembly is flagged (path weight below the MAP)."""
    wl = W.ge(10_000, seed=0)
    a5 = variants.viterbi_maxproduct(wl.log_pi, wl.log_A, wl.log_lik)
    v = oracle.viterbi(wl.log_pi, wl.log_A, wl.log_lik)
    assert a5["n_tied"] > 0
    assert abs(a5["log_prob"] - v["log_prob"]) <= 1e-9 * abs(v["log_prob"])
    assert a5["coherent"] == (a5["path_weight"] >= v["log_prob"] - 1e-9 * abs(v["log_prob"]))
    assert a5["path_weight"] <= v["log_prob"] + 1e-9 * abs(v["log_prob"])


def test_path_elements_cap():
    wl = W.ge(variants.PATH_ELEMENT_MAX_T + 1, seed=0)
    with pytest.raises(ValueError):
        variants.viterbi_path_elements(wl.log_pi, wl.log_A, wl.log_lik)
