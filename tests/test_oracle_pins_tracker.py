"""Pins of the f1 tracker oracle (Kalman update Eqs. 11-13, association, spawn/prune; no GPU).

P20  Eqs. 11-13: hand-computed gains, zero innovation, the information form
     P'^-1 = P^-1 + H^T R^-1 H and the Joseph form (independent algebra, numpy), singular S.
P21  greedy gated association: SPEC examples and, on random instances of at most
     4 x 4, the unique stable matching found by brute-force enumeration of all matchings.
P22  tracker tick: spawn, prune, coincident detections, capacity; with Q = 0 the
     filtered state equals the batch weighted least-squares (MAP) estimate of the initial state
     propagated forward (normal equations solved by numpy), and trace(H P H^T) decreases.
"""
import itertools
import math

import numpy as np
import pytest

H = np.array([[1.0, 0, 0, 0], [0, 1.0, 0, 0]])


def _A(dt):
    A = np.eye(4)
    A[0, 2] = A[1, 3] = dt
    return A


def _spd(rng, n, scale=1.0):
    M = rng.normal(size=(n, n))
    return scale * (M @ M.T + n * np.eye(n) * 0.1)


# --------------------------------------------------------------------- P20
def test_p20_hand_gain(orc):
    # P = I, R = I: S = 2 I, K = [0.5 I; 0], x' = x + (z - Hx) / 2, P' = diag(1/2, 1/2, 1, 1)
    st, x, P = orc.kalman_update([1.0, -2.0, 3.0, 4.0], np.eye(4), [3.0, 0.0], np.eye(2))
    assert st == 0
    assert x.tolist() == [2.0, -1.0, 3.0, 4.0]
    assert P.tolist() == np.diag([0.5, 0.5, 1.0, 1.0]).tolist()
    # 1D-like slice with correlation: P = [[2, 0, 1, 0], [0, 1, 0, 0], [1, 0, 1, 0], [0, 0, 0, 1]], R = I
    # S = diag(3, 2); K = P H^T S^-1 = [[2/3, 0], [0, 1/2], [1/3, 0], [0, 0]]
    P0 = np.array([[2.0, 0, 1, 0], [0, 1, 0, 0], [1, 0, 1, 0], [0, 0, 0, 1]])
    st, x, P = orc.kalman_update([0.0, 0.0, 0.0, 0.0], P0, [3.0, 2.0], np.eye(2))
    assert np.allclose(x, [2.0, 1.0, 1.0, 0.0], atol=1e-15)
    # P' = (I - K H) P: P'_00 = 2 - 4/3, P'_02 = 1 - 2/3, P'_22 = 1 - 1/3, P'_11 = 1/2
    assert np.allclose(P, [[2 / 3, 0, 1 / 3, 0], [0, 0.5, 0, 0], [1 / 3, 0, 2 / 3, 0], [0, 0, 0, 1]], atol=1e-15)


def test_p20_zero_innovation_shrinks(orc):
    rng = np.random.default_rng(2)
    for _ in range(50):
        P0 = _spd(rng, 4)
        x0 = rng.normal(size=4)
        R = _spd(rng, 2, 0.1)
        st, x, P = orc.kalman_update(x0, P0, H @ x0, R)
        assert st == 0 and np.allclose(x, x0, atol=1e-12)
        assert np.trace(P) < np.trace(P0)
        assert np.array_equal(P, P.T)


def test_p20_information_and_joseph_forms(orc):
    rng = np.random.default_rng(3)
    for _ in range(200):
        P0 = _spd(rng, 4, rng.uniform(0.01, 3))
        R = _spd(rng, 2, rng.uniform(0.001, 1))
        x0 = rng.normal(size=4)
        z = rng.normal(size=2)
        st, x, P = orc.kalman_update(x0, P0, z, R)
        assert st == 0
        Pinfo = np.linalg.inv(np.linalg.inv(P0) + H.T @ np.linalg.inv(R) @ H)
        xinfo = Pinfo @ (np.linalg.solve(P0, x0) + H.T @ np.linalg.solve(R, z))
        K = np.linalg.solve((H @ P0 @ H.T + R).T, (P0 @ H.T).T).T
        IKH = np.eye(4) - K @ H
        Pjos = IKH @ P0 @ IKH.T + K @ R @ K.T
        sc = max(1.0, np.abs(Pinfo).max())
        assert np.abs(P - Pinfo).max() < 1e-9 * sc
        assert np.abs(P - Pjos).max() < 1e-9 * sc
        assert np.abs(x - xinfo).max() < 1e-9 * max(1.0, np.abs(xinfo).max())


def test_p20_singular_innovation(orc):
    P0 = np.diag([0.0, 0.0, 1.0, 1.0])
    st, x, P = orc.kalman_update([1, 2, 3, 4], P0, [0, 0], np.zeros((2, 2)))
    assert st == -1 and x.tolist() == [1, 2, 3, 4] and np.array_equal(P, P0)


# --------------------------------------------------------------------- P21
def test_p21_spec_examples(orc):
    mt, du = orc.associate([[1.0, 1.0]], [[1.05, 1.0]], 0.5)
    assert mt.tolist() == [0] and du.tolist() == [True]
    mt, du = orc.associate([[1.0, 1.0]], [[1.6, 1.0]], 0.5)
    assert mt.tolist() == [-1] and du.tolist() == [False]
    # crossed: tracks at (0,0), (1,0); detections at (0.9,0), (0.2,0) -> closest pair (1,0)-(0.9,0) first
    mt, _ = orc.associate([[0, 0], [1, 0]], [[0.9, 0], [0.2, 0]], 1.0)
    assert mt.tolist() == [1, 0]
    # ties: equal distances -> lower track, then lower detection
    mt, _ = orc.associate([[0, 0], [2, 0]], [[1, 0]], 1.5)
    assert mt.tolist() == [0, -1]
    mt, _ = orc.associate([[1, 0]], [[0, 0], [2, 0]], 1.5)
    assert mt.tolist() == [0]
    assert orc.associate(np.zeros((0, 2)), [[1, 1]], 1.0)[1].tolist() == [False]


def _stable_matchings(d, g2):
    n, m = d.shape
    out = []
    for k in range(0, min(n, m) + 1):
        for ti in itertools.permutations(range(n), k):
            for dj in itertools.permutations(range(m), k):
                if any(d[i, j] > g2 for i, j in zip(ti, dj)):
                    continue
                mt = [-1] * n
                md = [-1] * m
                for i, j in zip(ti, dj):
                    mt[i], md[j] = j, i
                cur_t = [d[i, mt[i]] if mt[i] >= 0 else math.inf for i in range(n)]
                cur_d = [d[md[j], j] if md[j] >= 0 else math.inf for j in range(m)]
                blocking = any(d[i, j] <= g2 and d[i, j] < cur_t[i] and d[i, j] < cur_d[j]
                               for i in range(n) for j in range(m) if mt[i] != j)
                if not blocking:
                    out.append(tuple(mt))
    return sorted(set(out))


def test_p21_greedy_is_the_unique_stable_matching(orc):
    rng = np.random.default_rng(4)
    for _ in range(150):
        n, m = int(rng.integers(0, 5)), int(rng.integers(0, 5))
        p = rng.uniform(0, 2, (n, 2))
        z = rng.uniform(0, 2, (m, 2))
        gate = rng.uniform(0.2, 1.5)
        d = ((z[None, :, :] - p[:, None, :]) ** 2).sum(-1) if n and m else np.zeros((n, m))
        st = _stable_matchings(d, gate * gate)
        assert len(st) == 1
        mt, du = orc.associate(p, z, gate)
        assert tuple(mt.tolist()) == st[0]
        assert sorted(j for j in mt.tolist() if j >= 0) == [j for j in range(m) if du[j]]


# --------------------------------------------------------------------- P22
def test_p22_spawn_prune_coincident(orc):
    st, tr, mis = orc.track_step(np.zeros((0, 20)), [], [[1.0, 2.0]])
    assert st == 0 and len(tr) == 1 and mis.tolist() == [0]
    assert tr[0, :4].tolist() == [1.0, 2.0, 0.0, 0.0]
    assert tr[0, 4:].reshape(4, 4).tolist() == np.diag([0.25, 0.25, 1.0, 1.0]).tolist()
    st, tr, _ = orc.track_step(np.zeros((0, 20)), [], [[1.0, 2.0], [1.0, 2.0]])
    assert len(tr) == 2                                   # no de-duplication
    t = np.zeros((2, 20))
    t[:, 4:] = np.eye(4).reshape(16)
    st, tr, mis = orc.track_step(t, [10, 9], np.zeros((0, 2)))
    assert len(tr) == 1 and mis.tolist() == [10]          # missed 11 > 10 pruned, 10 kept
    st, tr, mis = orc.track_step(t, [0, 0], [[5.0, 5.0], [6.0, 6.0], [7.0, 7.0]], max_tracks=3)
    assert st == orc.W_TRUNCATED and len(tr) == 3 and tr[2, :2].tolist() == [5.0, 5.0]


def test_p22_constant_velocity_equals_batch_map(orc):
    dt, sz = 0.1, 0.05
    rng = np.random.default_rng(5)
    A = _A(dt)
    R = sz * sz * np.eye(2)
    for trial in range(5):
        p0 = rng.uniform(0, 5, 2)
        v = rng.uniform(-0.5, 0.5, 2)
        zs = [p0 + v * dt * k + rng.normal(0, sz, 2) * (trial % 2) for k in range(25)]
        st, tr, mis = orc.track_step(np.zeros((0, 20)), [], [zs[0]], dt=dt, Q=np.zeros(16))
        m0 = np.array([zs[0][0], zs[0][1], 0.0, 0.0])
        P0 = np.diag([0.25, 0.25, 1.0, 1.0])
        prev_tr = None
        for k in range(1, 25):
            st, tr, mis = orc.track_step(tr, mis, [zs[k]], dt=dt, Q=np.zeros(16))
            assert st == 0 and mis.tolist() == [0]
            # MAP of the initial state: (P0^-1 + sum Ai^T H^T R^-1 H Ai) s0 = P0^-1 m0 + sum Ai^T H^T R^-1 z_i
            Ninf = np.linalg.inv(P0)
            rhs = Ninf @ m0
            for i in range(1, k + 1):
                Ai = np.linalg.matrix_power(A, i)
                Ninf = Ninf + Ai.T @ H.T @ np.linalg.inv(R) @ H @ Ai
                rhs = rhs + Ai.T @ H.T @ np.linalg.solve(R, zs[i])
            s0 = np.linalg.solve(Ninf, rhs)
            Ak = np.linalg.matrix_power(A, k)
            assert np.abs(tr[0, :4] - Ak @ s0).max() < 1e-9
            Pk = Ak @ np.linalg.inv(Ninf) @ Ak.T
            assert np.abs(tr[0, 4:].reshape(4, 4) - Pk).max() < 1e-10
            if prev_tr is not None:   # trace(H P H^T) strictly decreases with Q = 0
                pp = prev_tr[4:].reshape(4, 4)
                assert np.trace(H @ tr[0, 4:].reshape(4, 4) @ H.T) < np.trace(H @ (A @ pp @ A.T) @ H.T)
            prev_tr = tr[0].copy()


def test_p22_missed_tick_keeps_prediction(orc):
    t = np.zeros((1, 20))
    t[0, :4] = (1.0, 1.0, 0.5, -0.5)
    t[0, 4:] = (np.eye(4) * 0.01).reshape(16)
    Q = np.zeros(16)
    st, tr, mis = orc.track_step(t, [3], [[9.0, 9.0]], dt=0.1, Q=Q, gate=0.5)
    assert mis.tolist() == [4, 0] and len(tr) == 2
    assert np.allclose(tr[0, :4], [1.05, 0.95, 0.5, -0.5], atol=1e-15)
    assert tr[1, :2].tolist() == [9.0, 9.0]
