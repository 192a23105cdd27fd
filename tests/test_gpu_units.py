"""GPU parity of the hot-path pieces against the reference itself:
solve_qp (qp.hpp:183-357) on the reference's own test QPs, and apply_barrier
(barrier.hpp:132-205) on random teams, through the C ABI unit entry points."""
import ctypes

import numpy as np
import pytest

import paper_2505_06771_b200 as m
from paper_2505_06771_b200 import _lib

pytestmark = pytest.mark.gpu
P = ctypes.POINTER


def gpu_qp(A, b, lo, hi, u, fp64, tol):
    count, mm, n = A.shape
    uo = np.zeros((count, n))
    st = np.zeros(count, dtype=np.int32)
    it = np.zeros(count, dtype=np.int32)
    d = lambda a: np.ascontiguousarray(a, dtype=np.float64).ctypes.data_as(P(ctypes.c_double))  # noqa: E731
    rc = _lib.lib().mrsim_qp_solve_batch(0, int(fp64), count, n, mm, d(A), d(b), d(lo), d(hi), d(u), tol,
                                          uo.ctypes.data_as(P(ctypes.c_double)),
                                          st.ctypes.data_as(P(ctypes.c_int32)), it.ctypes.data_as(P(ctypes.c_int32)))
    assert rc == 0
    return uo, st, it


@pytest.mark.parametrize("fp64", [True, False])
def test_qp_matches_enumeration_oracle_1000(fp64, ref):
    # test_qp.cpp:91-107: 1000 random feasible QPs (qp_oracle.hpp:119-140), seed 2024
    n, mm, A, b, u = ref.random_qps(2024, 1000)
    objs = []
    for t in range(1000):
        nt, mt = n[t], mm[t]
        # pad to a common (m, n) with vacuous rows so one batch launch covers all problems
        objs.append(ref.qp_enumeration(A[t, :mt, :nt], b[t, :mt], u[t, :nt]))
    maxn, maxm = 8, 12
    Ap = np.zeros((1000, maxm, maxn))
    bp = np.ones((1000, maxm))          # padded rows 0.u <= 1 are vacuous
    up = np.zeros((1000, maxn))
    for t in range(1000):
        Ap[t, :mm[t], :n[t]] = A[t, :mm[t], :n[t]]
        bp[t, :mm[t]] = b[t, :mm[t]]
        up[t, :n[t]] = u[t, :n[t]]
    lo = np.full((1000, maxn), -1e30)
    hi = np.full((1000, maxn), 1e30)
    uo, st, it = gpu_qp(Ap, bp, lo, hi, up, fp64, 1e-9 if fp64 else 2e-6)
    assert (st == 0).all()
    tol = 1e-6 if fp64 else 2e-4
    for t in range(1000):
        nt = n[t]
        obj = 0.5 * np.sum((uo[t, :nt] - up[t, :nt]) ** 2)
        assert objs[t] is not None
        assert abs(obj - objs[t][1]) <= tol * max(1.0, abs(objs[t][1])), (t, obj, objs[t][1])
        # and the solution itself equals the reference solver's
        sr, ur, _, _ = ref.solve_qp(A[t, :mm[t], :nt], b[t, :mm[t]], np.full(nt, -1e30), np.full(nt, 1e30),
                                    u[t, :nt])
        assert sr == 0
        np.testing.assert_allclose(uo[t, :nt], ur, atol=1e-9 if fp64 else 2e-4)


@pytest.mark.parametrize("fp64", [True, False])
def test_qp_closed_forms(fp64):
    # test_qp.cpp:9-72
    def one(A, b, lo, hi, u):
        A = np.asarray(A, dtype=np.float64).reshape(1, -1, len(u))
        return gpu_qp(A, np.asarray(b, dtype=np.float64).reshape(1, -1), np.asarray(lo).reshape(1, -1),
                      np.asarray(hi).reshape(1, -1), np.asarray(u, dtype=np.float64).reshape(1, -1), fp64,
                      1e-9 if fp64 else 2e-6)
    inf = 1e30
    uo, st, _ = one(np.zeros((0, 2)), np.zeros(0), [-inf, -inf], [inf, inf], [0.1, -0.05])
    assert st[0] == 0 and np.allclose(uo[0], [0.1, -0.05], atol=1e-7)
    uo, st, _ = one([[1.0, 0.0]], [0.0], [-inf, -inf], [inf, inf], [0.1, 0.0])
    assert st[0] == 0 and np.allclose(uo[0], [0.0, 0.0], atol=1e-7)
    uo, st, _ = one(np.zeros((0, 3)), np.zeros(0), [-1, -1, -1], [1, 1, 1], [2.0, -3.0, 0.25])
    assert st[0] == 0 and np.allclose(uo[0], [1.0, -1.0, 0.25], atol=1e-6)
    _, st, _ = one([[1.0], [-1.0]], [0.0, -1.0], [-inf], [inf], [0.0])
    assert st[0] == 1
    _, st, _ = one([[-1.0, -1.0]], [-3.0], [-1, -1], [1, 1], [0.0, 0.0])
    assert st[0] == 1


def gpu_barrier(cfg, poses, nominal, obstacles=None, masks=None, fp64=True):
    count, N, _ = poses.shape
    nob = 0 if obstacles is None else obstacles.shape[1]
    cmds = np.zeros((count, N, 2))
    inf = np.zeros(count, dtype=np.int32)
    d = lambda a: np.ascontiguousarray(a, dtype=np.float64).ctypes.data_as(P(ctypes.c_double))  # noqa: E731
    ob = obstacles if nob else np.zeros((count, 1, 3))
    mk = np.ascontiguousarray(masks if masks is not None else np.zeros((count, max(nob, 1))), dtype=np.uint64)
    rc = _lib.lib().mrsim_apply_barrier_batch(0, int(fp64), ctypes.byref(cfg.raw), count, d(poses), d(nominal),
                                              nob, d(ob), mk.ctypes.data_as(P(ctypes.c_uint64)),
                                              cmds.ctypes.data_as(P(ctypes.c_double)),
                                              inf.ctypes.data_as(P(ctypes.c_int32)))
    return rc, cmds, inf


def random_team(rng, N, sep=0.2):
    poses = []
    while len(poses) < N:
        p = (rng.uniform(-1.3, 1.3), rng.uniform(-0.7, 0.7), rng.uniform(-np.pi, np.pi))
        if all(np.hypot(p[0] - q[0], p[1] - q[1]) >= sep for q in poses):
            poses.append(p)
    return np.array(poses)


@pytest.mark.parametrize("N", [2, 4, 6, 10])
@pytest.mark.parametrize("fp64", [True, False])
def test_apply_barrier_matches_reference(N, fp64, ref):
    # the reference's "filtered commands always respect actuation limits" setup
    # (test_barrier.cpp:106-133), compared command by command with apply_barrier
    rng = np.random.default_rng(321 + N)
    count = 300
    poses = np.stack([random_team(rng, N, sep=0.2 if N <= 6 else 0.15) for _ in range(count)])
    nominal = np.stack([np.stack([rng.uniform(-0.2, 0.2, N), rng.uniform(-3.6, 3.6, N)], axis=1)
                        for _ in range(count)])
    cfg = m.make_default_config("navigation")
    cfg.set_num_robots(N)
    rb = ref.RefBatch(ref.spec("navigation", num_robots=N))
    rc, cmds, inf = gpu_barrier(cfg, poses, nominal, fp64=fp64)
    assert rc == 0
    tv, tw = (1e-9, 1e-8) if fp64 else (1e-4, 2e-3)
    for t in range(count):
        rcmd, rinf, _ = ref.apply_barrier(rb, poses[t], nominal[t])
        assert bool(inf[t]) == rinf
        np.testing.assert_allclose(cmds[t, :, 0], rcmd[:, 0], atol=tv, err_msg=f"team {t}")
        np.testing.assert_allclose(cmds[t, :, 1], rcmd[:, 1], atol=tw, err_msg=f"team {t}")
        assert np.all(np.abs(cmds[t, :, 0]) <= 0.2 + 1e-6) and np.all(np.abs(cmds[t, :, 1]) <= 3.6 + 1e-5)


@pytest.mark.parametrize("fp64", [True, False])
def test_apply_barrier_with_masked_obstacles(fp64, ref):
    rng = np.random.default_rng(7)
    N, count, nob = 4, 200, 6
    poses = np.stack([random_team(rng, N) for _ in range(count)])
    nominal = np.stack([np.stack([rng.uniform(-0.2, 0.2, N), rng.uniform(-3.6, 3.6, N)], axis=1)
                        for _ in range(count)])
    obstacles = np.zeros((count, nob, 3))
    masks = np.zeros((count, nob), dtype=np.uint64)
    for t in range(count):
        for o in range(nob):
            # keep obstacles off the robots' projected points
            while True:
                c = (rng.uniform(-1.2, 1.2), rng.uniform(-0.7, 0.7))
                if np.min(np.hypot(poses[t, :, 0] - c[0], poses[t, :, 1] - c[1])) > 0.3:
                    break
            obstacles[t, o] = (c[0], c[1], 0.12)
            masks[t, o] = rng.integers(0, 16)
    cfg = m.make_default_config("navigation")
    cfg.set_num_robots(N)
    rb = ref.RefBatch(ref.spec("navigation", num_robots=N))
    rc, cmds, inf = gpu_barrier(cfg, poses, nominal, obstacles, masks, fp64=fp64)
    assert rc == 0
    tv, tw = (1e-9, 1e-8) if fp64 else (1e-4, 2e-3)
    for t in range(count):
        rcmd, rinf, _ = ref.apply_barrier(rb, poses[t], nominal[t], obstacles[t], masks[t])
        assert bool(inf[t]) == rinf
        np.testing.assert_allclose(cmds[t], rcmd, atol=max(tv, tw))


@pytest.mark.parametrize("fp64", [True, False])
def test_head_on_keeps_separation(fp64):
    # test_barrier.cpp:86-104
    cfg = m.make_default_config("navigation")
    cfg.set_num_robots(2)
    for d in (0.18, 0.25, 0.3, 0.4, 0.6):
        poses = np.array([[[-d / 2, 0.0, 0.0], [d / 2, 0.0, np.pi]]])
        nominal = np.array([[[0.2, 0.0], [0.2, 0.0]]])
        rc, cmds, inf = gpu_barrier(cfg, poses, nominal, fp64=fp64)
        assert rc == 0 and inf[0] == 0
        a = poses[0, 0, :2] + cmds[0, 0, 0] * np.array([1, 0]) * 0.033
        b = poses[0, 1, :2] + cmds[0, 1, 0] * np.array([-1, 0]) * 0.033
        assert np.hypot(*(a - b)) >= 0.17 - 1e-6


def test_coincident_robots_are_a_domain_error():
    cfg = m.make_default_config("navigation")
    cfg.set_num_robots(2)
    poses = np.array([[[0.1, 0.2, 0.3], [0.1, 0.2, 0.3]]])
    rc, _, _ = gpu_barrier(cfg, poses, np.zeros((1, 2, 2)))
    assert rc == m.DomainError.code
