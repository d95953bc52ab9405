"""Pins of the tabled-trajectory oracle (NEXT-2, reading R23; the paper's position LUT, and
its continual-motion model): the interpolant against analytic trajectories, the delay
against a closed form and against bisection, and the full sum against the pinned constant-velocity
and stop-and-hop definitions."""
import numpy as np
import pytest

import oracle
import synth

C = 1500.0


def _quad(r0, v, a, t):
    return r0 + v * t + 0.5 * a * t * t


@pytest.mark.parametrize("K", [3, 4, 7])
def test_interpolant_reproduces_quadratic_motion(K):
    """Central tangents inside, second-order one-sided tangents at the ends: any quadratic
    trajectory is reproduced exactly, inside the table and on the continued end cubics."""
    rng = np.random.default_rng(K)
    r0, v, a = rng.normal(size=3) * 10, rng.normal(size=3), rng.normal(size=3) * 3
    dt = 0.013
    lut = np.stack([_quad(r0, v, a, k * dt) for k in range(K)])
    for t in np.concatenate([rng.uniform(-dt, K * dt, 40), np.arange(K) * dt]):
        np.testing.assert_allclose(oracle.nav_eval(lut, dt, t), _quad(r0, v, a, t), rtol=0, atol=1e-12)


def test_interpolant_hand_values():
    """Nodes (0, 1, 4) at dt = 1 (x = t^2): x(0.5) = 0.25, x(1.5) = 2.25, x(3) = 9 (continued);
    a non-quadratic table (0, 1, 0, 1) at t = 1.5: tangents m1 = (0 - 0)/2 = 0, m2 = (1 - 1)/2 = 0,
    so x = h00 * 1 + h01 * 0 = 0.5; at t = 0.5: m0 = (-0 + 4 - 0)/2 = 2, m1 = 0 ->
    x = h10 * 2 + h01 * 1 = 0.125 * 2 + 0.5 = 0.75."""
    lut = np.array([[0.0, 0, 0], [1.0, 0, 0], [4.0, 0, 0]])
    for t, x in ((0.5, 0.25), (1.5, 2.25), (3.0, 9.0), (-1.0, 1.0)):
        assert oracle.nav_eval(lut, 1.0, t)[0] == pytest.approx(x, abs=1e-14)
    lut2 = np.array([[0.0, 0, 0], [1.0, 0, 0], [0.0, 0, 0], [1.0, 0, 0]])
    assert oracle.nav_eval(lut2, 1.0, 1.5)[0] == pytest.approx(0.5, abs=1e-14)
    assert oracle.nav_eval(lut2, 1.0, 0.5)[0] == pytest.approx(0.75, abs=1e-14)


def test_delay_closed_form_accelerating_receiver():
    """Collinear geometry: tx at 0, point at D on the x axis, receiver at r(t) = r0 + v t + a t^2/2
    between them: c tau = D + D - r(tau) -> (a/2) tau^2 + (c + v) tau - (2 D - r0) = 0."""
    D, r0, v, a = 60.0, 0.7, 2.0, 4.0
    dt = 0.02
    lut = np.stack([np.array([_quad(r0, v, a, k * dt), 0.0, 0.0]) for k in range(6)])
    tau = oracle.delay_nav([D, 0, 0], [0, 0, 0], lut, dt, C)
    exact = (-(C + v) + np.sqrt((C + v) ** 2 + 2 * a * (2 * D - r0))) / a
    assert tau == pytest.approx(exact, rel=1e-14)
    # stop-and-hop would be (2 D - r0) / c: the motion must matter at this level
    assert abs(tau - (2 * D - r0) / C) > 1e-6


def test_delay_matches_bisection_on_a_turning_lever_arm():
    """The fixed point equals the root of f(tau) = c tau - |x - tx| - |x - r(tau)| (monotone for
    element speeds below c) found by bisection with the same interpolant."""
    rng = np.random.default_rng(5)
    dt, K = 0.01, 9
    w, L = 0.3, np.array([1.2, 0.4, 0.0])
    t = np.arange(K) * dt
    lut = np.stack([np.array([np.cos(w * tk) * L[0] - np.sin(w * tk) * L[1] + 1.5 * tk,
                              np.sin(w * tk) * L[0] + np.cos(w * tk) * L[1], -0.2 * tk]) for tk in t])
    for _ in range(5):
        x = rng.normal(size=3) * 20 + np.array([0, 40, 5])
        tx = rng.normal(size=3)
        tau = oracle.delay_nav(x, tx, lut, dt, C)
        f = lambda s: C * s - np.linalg.norm(x - tx) - np.linalg.norm(x - oracle.nav_eval(lut, dt, s))
        lo, hi = 0.0, 1.0
        for _ in range(200):
            m = 0.5 * (lo + hi)
            lo, hi = (m, hi) if f(m) < 0 else (lo, m)
        assert tau == pytest.approx(0.5 * (lo + hi), abs=1e-15)


def test_linear_table_equals_constant_velocity_oracle():
    """A table of the constant-velocity trajectory rx + v t is the R16 definition."""
    s = synth.scenario(1, reduced=True)
    e = s.echoes()
    vel = np.random.default_rng(1).normal(size=(s.P, 3)) * np.array([1.5, 0.5, 0.1])
    lut, dt = synth.nav_table(s, K=5, accel=0.0, yaw_rate_deg=0.0, vel=vel)
    pts = s.pixel_centre(s.sample_pixels(60, window=5))
    got = oracle.tdbp_points_nav(e, s.tx, lut, dt, s.t0, s.fc, s.fs, s.c, pts)
    ref = oracle.tdbp_points_motion(e, s.tx, s.rx, s.t0, vel, s.fc, s.fs, s.c, pts)
    assert np.max(np.abs(got - ref)) <= 1e-9 * np.max(np.abs(ref))


def test_fixed_table_is_stop_and_hop():
    s = synth.scenario(1, reduced=True)
    e = s.echoes()
    lut = np.repeat(s.rx[:, :, None, :], 4, axis=2)
    pts = s.pixel_centre(s.sample_pixels(40, window=5))
    got, n1 = oracle.tdbp_points_nav(e, s.tx, lut, 1e-3, s.t0, s.fc, s.fs, s.c, pts, with_count=True)
    ref, n2 = oracle.tdbp_points(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, pts, with_count=True)
    # (the interpolant of a constant table equals it to rounding: h00 + h01 = 1 in exact arithmetic)
    assert np.max(np.abs(got - ref)) <= 1e-8 * np.max(np.abs(ref))
    assert np.array_equal(n1, n2)


def test_gated_nav_reduces_to_gated_motion_and_to_nav():
    """Gated + tabled (R22 + R23): with a linear table it is the pinned gated-motion sum; with an
    open gate it is the ungated tabled sum."""
    s = synth.scenario(1, reduced=True)
    e = s.echoes()
    vel = np.random.default_rng(2).normal(size=(s.P, 3)) * np.array([1.5, 0.5, 0.1])
    lut, dt = synth.nav_table(s, K=6, accel=0.0, yaw_rate_deg=0.0, vel=vel)
    pts = s.pixel_centre(s.sample_pixels(40, window=5))
    az = 2 * np.arcsin(s.sin_half_beam) * 0.5
    got, n1 = oracle.tdbp_points_gated_nav(e, s.tx, s.rx, lut, dt, s.t0, s.fc, s.fs, s.c, pts, az, bistatic=True,
                                           with_count=True)
    ref, n2 = oracle.tdbp_points_gated_motion(e, s.tx, s.rx, s.t0, vel, s.fc, s.fs, s.c, pts, az, bistatic=True,
                                              with_count=True)
    assert np.array_equal(n1, n2) and n1.min() < s.P * s.E
    assert np.max(np.abs(got - ref)) <= 1e-9 * max(np.max(np.abs(ref)), 1e-30)
    lut2, dt2 = synth.nav_table(s, K=6, seed=3)
    op = oracle.tdbp_points_gated_nav(e, s.tx, s.rx, lut2, dt2, s.t0, s.fc, s.fs, s.c, pts, np.pi)
    un = oracle.tdbp_points_nav(e, s.tx, lut2, dt2, s.t0, s.fc, s.fs, s.c, pts)
    assert np.max(np.abs(op - un)) <= 1e-12 * np.max(np.abs(un))


def test_mutations_of_the_interpolant_are_caught():
    """Sanity of the pins themselves: a table interpolated with first-order end tangents (a
    plausible slip) misses the quadratic reproduction by far more than the pin's 1e-12."""
    dt, K = 0.013, 4
    r0, v, a = np.array([1.0, 2, 3]), np.array([0.5, -1, 2]), np.array([3.0, 1, -2])
    lut = np.stack([_quad(r0, v, a, k * dt) for k in range(K)])
    t = 0.3 * dt
    m0_first_order = (lut[1] - lut[0])          # dt * one-sided first-order tangent
    m0 = 0.5 * (-3 * lut[0] + 4 * lut[1] - lut[2])
    assert np.max(np.abs(m0_first_order - m0)) > 1e-5
    np.testing.assert_allclose(oracle.nav_eval(lut, dt, t), _quad(r0, v, a, t), atol=1e-12)
