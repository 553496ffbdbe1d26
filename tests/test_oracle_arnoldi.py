"""Pins of the oracle's Arnoldi reduced-order net model (O12; SURVEY.md
§8(f) row 1) against closed forms, dense
linear algebra (numpy / scipy, independent of the oracle's tree recursion),
a transient simulation and degenerate cases."""
import numpy as np
import pytest
from scipy.linalg import eigh, lu_factor, lu_solve
from scipy.optimize import brentq

import oracle
import synth


def random_tree(rng, n):
    parent = np.array([-1] + [int(rng.integers(0, i)) for i in range(1, n)], np.int32)
    res = np.concatenate([[0.0], rng.uniform(0.05, 2.0, n - 1)]).astype(np.float32)
    cap = np.concatenate([[rng.uniform(0, 1)], rng.uniform(0.1, 3.0, n - 1)])
    return parent, res, cap


def dense(parent, res, cap):
    """G (conductance Laplacian of the non-root nodes), C, b: C v' + G v = b u."""
    n = parent.size
    G = np.zeros((n - 1, n - 1))
    b = np.zeros(n - 1)
    for i in range(1, n):
        g = 1.0 / float(res[i])
        G[i - 1, i - 1] += g
        p = parent[i]
        if p == 0:
            b[i - 1] += g
        else:
            G[p - 1, p - 1] += g
            G[i - 1, p - 1] -= g
            G[p - 1, i - 1] -= g
    return G, np.diag(cap[1:]), b


def exact_moments(parent, res, cap, K):
    G, C, b = dense(parent, res, cap)
    A = np.linalg.solve(G, C)
    x = np.linalg.solve(G, b)                # = 1
    out = []
    for _ in range(K):
        out.append(x.copy())
        x = A @ x
    return out, C


def test_single_pole_closed_form():
    # one RC segment (R = 2, C = 3): lam = RC; step input: delay RC ln 2, 20-80 slew RC ln 4
    qq, lam, r = oracle.arnoldi_reduce([-1, 0], [0, 2.0], [0.0, 3.0], 4)
    assert qq == 1 and abs(lam[0] - 6.0) < 1e-12 and abs(r[1, 0] - 1.0) < 1e-12
    d, s = oracle.arnoldi_delay(lam, r[1, :qq], 0.0)
    assert abs(d - 6.0 * np.log(2)) < 2e-6 and abs(s - 6.0 * np.log(4)) < 2e-6


@pytest.mark.parametrize("slew", [3.0, 40.0])
def test_single_pole_ramp_vs_independent_root(slew):
    # ramp of 20-80 slew s (duration D = s / 0.6) through one pole: the closed
    # form response solved by scipy's brentq, not by the oracle's bisection
    R, C = 1.5, 4.0
    lam = R * C
    D = slew / 0.6

    def y(t):
        r = lambda x: x - lam * (1 - np.exp(-x / lam)) if x > 0 else 0.0
        return (r(t) - (r(t - D) if t > D else 0.0)) / D

    hi = D + 60 * lam
    t50, t20, t80 = (brentq(lambda t: y(t) - th, 0, hi, xtol=1e-12) for th in (0.5, 0.2, 0.8))
    qq, lm, rr = oracle.arnoldi_reduce([-1, 0], [0, R], [0.0, C], 4)
    d, s = oracle.arnoldi_delay(lm, rr[1, :qq], slew)
    assert abs(d - (t50 - D / 2)) < 2e-6 and abs(s - (t80 - t20)) < 2e-6


@pytest.mark.parametrize("seed", range(10))
def test_moment_matching(seed):
    # per node the first q moments A^k 1 (k < q) are matched exactly; the
    # C-weighted quadratic form 1^T C A^k 1 for k <= 2q - 1 (Lanczos)
    rng = np.random.default_rng(seed)
    n = int(rng.integers(6, 25))
    q = int(rng.integers(2, 5))
    parent, res, cap = random_tree(rng, n)
    qq, lam, resid = oracle.arnoldi_reduce(parent, res, cap, q)
    assert qq == q
    mu, C = exact_moments(parent, res, cap, 2 * q)
    for k in range(q):
        model = resid[1:, :qq] @ (lam ** k)
        np.testing.assert_allclose(model, mu[k], rtol=1e-9, atol=0)
    one = np.ones(n - 1)
    for k in range(2 * q):
        model = np.diag(C) @ (resid[1:, :qq] @ (lam ** k))
        exact = one @ C @ mu[k]
        assert abs(model - exact) <= 1e-9 * abs(exact)


def test_first_moment_is_elmore():
    # m_1 = A 1 = the Elmore delay of O3 at every sink (cross-check against the pinned O3)
    rng = np.random.default_rng(7)
    parent, res, cap = random_tree(rng, 15)
    mu, _ = exact_moments(parent, res, cap, 2)
    qq, lam, resid = oracle.arnoldi_reduce(parent, res, cap, 4)
    # brute-force Elmore: sum over nodes k of C_k * R(path(root, k) ∩ path(root, i))
    def path(i):
        s = set()
        while i > 0:
            s.add(i)
            i = parent[i]
        return s
    for i in range(1, 15):
        el = sum(cap[k] * sum(float(res[a]) for a in path(i) & path(k)) for k in range(1, 15))
        assert abs(resid[i, :qq] @ lam - el) < 1e-9 * el
        assert abs(mu[1][i - 1] - el) < 1e-9 * el


@pytest.mark.parametrize("seed", range(4))
def test_full_order_spectrum_and_transient(seed):
    # q >= n - 1: the reduced time constants are the exact spectrum (generalized
    # eigenproblem G phi = mu C phi, lam = 1 / mu) and the ramp delay matches a
    # transient (trapezoidal) simulation within 0.5 %
    rng = np.random.default_rng(20 + seed)
    n = int(rng.integers(4, 8))
    parent, res, cap = random_tree(rng, n)
    qq, lam, resid = oracle.arnoldi_reduce(parent, res, cap, 8)
    assert qq == n - 1
    G, C, b = dense(parent, res, cap)
    mu = eigh(G, C, eigvals_only=True)
    np.testing.assert_allclose(np.sort(lam), np.sort(1.0 / mu), rtol=1e-9)
    slew = 5.0
    D = slew / 0.6
    # trapezoidal (second-order) transient of C v' + G v = b u(t): a step of
    # 1 % of the fastest time constant
    h = 1e-2 * min(1.0 / mu.max(), D)
    T = D + 12.0 / mu.min()
    lu = lu_factor(C / h + G / 2)
    Mr = C / h - G / 2
    v = np.zeros(n - 1)
    t, u_prev = 0.0, 0.0
    i_out = n - 1
    trace_t, trace_v = [0.0], [0.0]
    while t < T:
        t += h
        u = min(t / D, 1.0)
        v = lu_solve(lu, Mr @ v + b * (u + u_prev) / 2)
        u_prev = u
        trace_t.append(t)
        trace_v.append(v[i_out - 1])
    tt, vv = np.array(trace_t), np.array(trace_v)
    k = int(np.argmax(vv >= 0.5))
    t50 = tt[k - 1] + (0.5 - vv[k - 1]) * (tt[k] - tt[k - 1]) / (vv[k] - vv[k - 1])
    d, _ = oracle.arnoldi_delay(lam, resid[i_out, :qq], slew)
    assert abs(d - (t50 - D / 2)) <= 5e-3 * (t50 - D / 2) + 1e-6


def test_zero_resistance_and_bounds():
    # zero-R net: no dynamics: delay 0, the slew passes through
    qq, lam, resid = oracle.arnoldi_reduce([-1, 0, 1], [0, 0, 0], [0.0, 1.0, 2.0], 4)
    d, s = oracle.arnoldi_delay(lam, resid[2, :qq], 12.0)
    assert abs(d) < 2e-6 and abs(s - 12.0) < 2e-6
    # 0 <= delay <= (sum R)(sum C) on trees
    rng = np.random.default_rng(3)
    for _ in range(10):
        parent, res, cap = random_tree(rng, 12)
        qq, lam, resid = oracle.arnoldi_reduce(parent, res, cap, 4)
        bound = float(res.astype(np.float64).sum()) * float(cap.sum())
        for i in range(1, 12):
            d, s = oracle.arnoldi_delay(lam, resid[i, :qq], float(rng.uniform(0, 30)))
            assert -1e-6 <= d <= bound and s > 0


def test_update_arnoldi_integration():
    # a PI driving one RC segment to a PO: the sink's arrival is the PI
    # arrival plus the single-pole ramp delay (brentq above), its slew the
    # ramp's 20-80 width; on a design whose wires have no resistance the
    # Arnoldi update equals the Elmore update
    d = synth.generate(400, 10, seed=9, period=300.0)
    zr = synth.RcTree(d.rc[0].rc_ptr, d.rc[0].parent, d.rc[0].node_pin, np.zeros_like(d.rc[0].res),
                      d.rc[0].cap)
    import copy
    d0 = copy.copy(d)
    d0.rc = [zr]
    a = oracle.update(d0, net_model="arnoldi")
    e = oracle.update(d0)
    fin = np.isfinite(e["at"])
    assert np.array_equal(fin, np.isfinite(a["at"]))
    np.testing.assert_allclose(a["at"][fin], e["at"][fin], rtol=0, atol=1e-5)
    np.testing.assert_allclose(a["slew"][fin], e["slew"][fin], rtol=0, atol=1e-5)
    # the Arnoldi model changes the answer on resistive wires (not a no-op)
    a1 = oracle.update(d, net_model="arnoldi")
    e1 = oracle.update(d)
    assert np.nanmax(np.abs(np.where(fin, a1["at"] - e1["at"], 0))) > 1e-3


def test_update_single_net_by_hand():
    R, Cw, Cpin = 2.0, 1.0, 0.5
    lam = R * (Cw + Cpin)
    pin_at, pin_slew = 10.0, 12.0
    D = pin_slew / 0.6

    def y(t):
        r = lambda x: x - lam * (1 - np.exp(-x / lam)) if x > 0 else 0.0
        return (r(t) - (r(t - D) if t > D else 0.0)) / D

    t50 = brentq(lambda t: y(t) - 0.5, 0, D + 60 * lam, xtol=1e-12)
    t20 = brentq(lambda t: y(t) - 0.2, 0, D + 60 * lam, xtol=1e-12)
    t80 = brentq(lambda t: y(t) - 0.8, 0, D + 60 * lam, xtol=1e-12)
    lib = synth.Library.from_tables([synth.design.constant_table(1.0)] * 4)
    cons = synth.Constraints(100.0, 5.0, np.array([0], np.uint32), np.full((1, 4), pin_at, np.float32),
                             np.full((1, 4), pin_slew, np.float32), np.array([1], np.uint32),
                             np.zeros((1, 2), np.float32), np.zeros((1, 2), np.float32), np.zeros(1, np.float32))
    rc = synth.RcTree(np.array([0, 2], np.uint32), np.array([-1, 0], np.int32), np.array([0, 1], np.uint32),
                      np.array([0.0, R], np.float32), np.array([0.0, Cw], np.float32))
    dsg = synth.Design(num_pins=2, pin_cap=np.array([0.0, Cpin], np.float32), pin_role=np.array([1, 2], np.uint8),
                       net_ptr=np.array([0, 2], np.uint32), net_pins=np.array([0, 1], np.uint32),
                       arc_from=np.zeros(0, np.uint32), arc_to=np.zeros(0, np.uint32),
                       arc_sense=np.zeros(0, np.uint8), arc_tab=np.zeros(0, np.uint32),
                       chk_d=np.zeros(0, np.uint32), chk_ck=np.zeros(0, np.uint32), chk_tab=np.zeros(0, np.uint32),
                       libs=[lib], rc=[rc], cons=cons, name="arn1")
    out = oracle.update(dsg, net_model="arnoldi")
    np.testing.assert_allclose(out["at"][1], pin_at + (t50 - D / 2), atol=2e-6)
    np.testing.assert_allclose(out["slew"][1], t80 - t20, atol=2e-6)
    # backward through the net arc with the same delay: RAT_late(PI) = T - out_max - d,
    # RAT_early(PI) = -out_min - d
    np.testing.assert_allclose(out["rat"][0][2:], 100.0 - (t50 - D / 2), atol=2e-6)
    np.testing.assert_allclose(out["rat"][0][:2], -(t50 - D / 2), atol=2e-6)
