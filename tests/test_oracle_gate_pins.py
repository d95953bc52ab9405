"""Pins of the oracle's gated variants and of the whitening frequency orientation (round 2).

Each gated function is checked against a hand-built geometry whose admitted (ping, element)
set is decided on paper (angles worked out in the comments, not by calling the gate), so the
gated sum must equal the plain (already pinned) sum over exactly those channels:
  * the bistatic receive-cone gate of oracle_tdbp_points_gated ("bistatic
    ray-culling"; reading R15),
  * both gates of oracle_tdbp_points_gated_weighted (R15 + R18),
  * the gated moving-receiver and gated refracted sums (R15 + R16 / R17, reading R22: the gate
    is the straight line-of-sight cone from the sensor positions recorded at transmit),
and the whitening gain / whitened compression against a complex tone, whose spectrum is NOT
symmetric in f, so the sign of the periodogram exponent and of the FIR's imaginary part are
both fixed (Eq. 9; reading R21).
"""
import numpy as np
import pytest

import oracle

FC, FS, C = 120e3, 120e3, 1500.0
SIN_HALF = 0.3                      # azimuth half-width: |v.a| <= |v| * 0.3
AZ = 2 * np.arcsin(SIN_HALF)
X = np.array([[0.0, 10.0, 0.0]])    # the scatterer position; a = +x, b = +y (default axes)

# Sensors on the x axis at s = (sx, 0, 0): v = x - s = (-sx, 10, 0), |v.a| / |v| = |sx| / sqrt(sx^2 + 100):
#   sx = 0   -> 0       (inside)
#   sx = 2   -> 0.196   (inside)
#   sx = 3.1 -> 0.2961  (inside; the boundary 0.3 is at sx = 3.145)
#   sx = 5   -> 0.447   (outside)
TX = np.array([[0.0, 0, 0], [5.0, 0, 0]])                  # ping 0 tx inside, ping 1 tx outside
RX = np.array([[[0.0, 0, 0], [5.0, 0, 0], [3.1, 0, 0]],     # ping 0: in, out, in
               [[0.0, 0, 0], [2.0, 0, 0], [-2.0, 0, 0]]])   # ping 1: all in (but its tx is out)
# admitted channels, worked out above:
MONO = [(0, 0), (0, 1), (0, 2)]          # tx gate only: every element of ping 0
BIST = [(0, 0), (0, 2)]                  # tx and rx gates


def _echoes(seed=3, Ns=4096):
    rng = np.random.default_rng(seed)
    return ((rng.normal(size=(2, 3, Ns)) + 1j * rng.normal(size=(2, 3, Ns))) / np.sqrt(2)).astype(np.complex64)


def _subset_sum(fn, e, chans, *extra, vel=None):
    """Sum of the plain (ungated) oracle over single channels: one P = E = 1 call per channel."""
    tot = 0.0 + 0.0j
    for p, k in chans:
        args = [e[p:p + 1, k:k + 1], TX[p:p + 1], RX[p:p + 1, k:k + 1], None]
        if vel is not None:
            args.append(vel[p:p + 1])
        tot += fn(*args, *extra, X)[0]
    return tot


def test_gated_bistatic_receive_cone_admits_exactly_the_hand_set():
    e = _echoes()
    base = (FC, FS, C)
    mono, nm = oracle.tdbp_points_gated(e, TX, RX, None, *base, X, az=AZ, bistatic=False, with_count=True)
    bist, nb = oracle.tdbp_points_gated(e, TX, RX, None, *base, X, az=AZ, bistatic=True, with_count=True)
    want_m = _subset_sum(oracle.tdbp_points, e, MONO, *base)
    want_b = _subset_sum(oracle.tdbp_points, e, BIST, *base)
    assert abs(want_m - want_b) > 1e-3                          # channel (0, 1) matters
    assert abs(mono[0] - want_m) <= 1e-12 * abs(want_m)
    assert abs(bist[0] - want_b) <= 1e-12 * abs(want_b)
    assert nm[0] == len(MONO) and nb[0] == len(BIST)


def test_gated_weighted_both_gates_hand_set():
    e = _echoes(4)
    base = (FC, FS, C)
    for bist, chans in ((False, MONO), (True, BIST)):
        got = oracle.tdbp_points_gated_weighted(e, TX, RX, None, *base, X, az=AZ, bistatic=bist)[0]
        want = _subset_sum(oracle.tdbp_points_weighted, e, chans, *base)
        assert abs(got - want) <= 1e-12 * abs(want), bist
    # the weight is on: a gated-weighted term is R_tx R_rx (~100 m^2) times the unweighted one
    one = oracle.tdbp_points_gated_weighted(e[:1, :1], TX[:1], RX[:1, :1], None, *base, X, az=AZ)[0]
    plain = oracle.tdbp_points(e[:1, :1], TX[:1], RX[:1, :1], None, *base, X)[0]
    assert abs(one - 100.0 * plain) <= 1e-12 * abs(one)


def test_gated_motion_gates_on_transmit_time_positions():
    """Element (0, 2) at sx = 3.1 is inside the cone at transmit; moving at 10 m/s along +x during
    the ~13.65 ms reception it reaches sx = 3.24 (|v.a|/|v| = 0.308, outside).  Reading R22 gates on
    the recorded (transmit-time) positions, so it stays admitted."""
    e = _echoes(5)
    vel = np.array([[10.0, 0, 0], [10.0, 0, 0]])
    tau = oracle.delay_moving(X[0], TX[0], RX[0, 2], vel[0], C)
    rx_rec = RX[0, 2] + vel[0] * tau
    assert abs(rx_rec[0]) / np.hypot(rx_rec[0], 10.0) > SIN_HALF   # outside at reception
    base = (FC, FS, C)
    for bist, chans in ((False, MONO), (True, BIST)):
        got, n = oracle.tdbp_points_gated_motion(e, TX, RX, None, vel, *base, X, az=AZ, bistatic=bist,
                                                 with_count=True)
        want = _subset_sum(oracle.tdbp_points_motion, e, chans, *base, vel=vel)
        assert abs(got[0] - want) <= 1e-12 * abs(want), bist
        assert n[0] == len(chans)


def test_gated_motion_limits():
    """v = 0 is the (pinned) gated sum exactly; a wide-open gate is the (pinned) motion sum."""
    e = _echoes(6)
    base = (FC, FS, C)
    pts = np.array([[0.3, 9.0, 0.2], [0.0, 10.0, 0.0], [-1.0, 11.0, 0.5]])
    z = np.zeros((2, 3))
    vel = np.array([[1.5, 0.2, 0.0], [1.7, -0.1, 0.05]])
    g0 = oracle.tdbp_points_gated_motion(e, TX, RX, None, z, *base, pts, az=AZ, bistatic=True)
    assert np.array_equal(g0, oracle.tdbp_points_gated(e, TX, RX, None, *base, pts, az=AZ, bistatic=True))
    op = oracle.tdbp_points_gated_motion(e, TX, RX, None, vel, *base, pts, az=np.pi, bistatic=True)
    assert np.array_equal(op, oracle.tdbp_points_motion(e, TX, RX, None, vel, *base, pts))


def test_gated_refracted_hand_set_and_limits():
    """The scatterer 0.5 m below a flat interface at z = 0.5 (sensors in the water at z = 0): the
    gate is the straight line-of-sight cone (the horizontal geometry above is unchanged by the
    z offset: |v.a| / |v| = |sx| / sqrt(sx^2 + 100 + 1), same in/out classes), every admitted term
    takes the Fermat delay."""
    e = _echoes(7)
    x = np.array([[0.0, 10.0, 1.0]])
    zb, c2 = 0.5, 1700.0
    base = (FC, FS, C)
    for bist, chans in ((False, MONO), (True, BIST)):
        got, n = oracle.tdbp_points_gated_refracted(e, TX, RX, None, zb, c2, *base, x, az=AZ, bistatic=bist,
                                                    with_count=True)
        want = 0.0 + 0.0j
        for p, k in chans:
            want += oracle.tdbp_points_refracted(e[p:p + 1, k:k + 1], TX[p:p + 1], RX[p:p + 1, k:k + 1], None,
                                                 zb, c2, *base, x)[0]
        assert abs(got[0] - want) <= 1e-12 * abs(want), bist
        assert n[0] == len(chans)
    pts = np.array([[0.3, 9.0, 0.2], [0.0, 10.0, 1.0], [-1.0, 11.0, 0.9]])
    op = oracle.tdbp_points_gated_refracted(e, TX, RX, None, zb, c2, *base, pts, az=np.pi, bistatic=True)
    assert np.array_equal(op, oracle.tdbp_points_refracted(e, TX, RX, None, zb, c2, *base, pts))
    eq = oracle.tdbp_points_gated_refracted(e, TX, RX, None, zb, C, *base, pts, az=AZ, bistatic=True)
    ref = oracle.tdbp_points_gated(e, TX, RX, None, *base, pts, az=AZ, bistatic=True)
    assert np.max(np.abs(eq - ref)) <= 1e-9 * np.max(np.abs(ref))   # c2 = c: straight rays


# ---------------------------------------------------------------- whitening orientation (R21)

def _tone(k0, M=16, B=4, nch=2):
    n = np.arange(M * B)
    return np.tile(np.exp(2j * np.pi * k0 * n / M), (nch, 1)).astype(np.complex64)


def test_whitening_periodogram_of_a_complex_tone_peaks_at_its_own_bin():
    """x[n] = exp(+j 2 pi 3 n / 16): |sum_n x[n] exp(-j 2 pi k n / M)|^2 = M^2 delta[k - 3], so P = 256 at
    bin 3 (not at bin 13 = -3); with gamma = 1, mean P = 16 and G = h(1 / (16 + P)) = 1 except
    G[3] = 16 / 272 = 1/17 (hand values)."""
    M = 16
    G, P = oracle.whitening_gain(_tone(3), M, 1.0)
    assert int(np.argmax(P)) == 3
    assert abs(P[3] - 256.0) <= 1e-4 and np.max(np.abs(np.delete(P, 3))) <= 1e-4   # complex64 tone
    want = np.ones(M)
    want[3] = 1.0 / 17.0
    assert np.max(np.abs(G - want)) <= 1e-6


def test_whitened_fir_attenuates_the_tone_bin_not_its_mirror():
    """With G[3] = 1/17 (else 1) the frequency-sampling FIR has amplitude response sqrt(G) at
    f = k fs / M: away from the record edges a tone at bin 3 comes out scaled by sqrt(1/17), a tone
    at bin -3 (= 13) unchanged (the replica r = [1] makes the compression the identity).  Derivation:
    sum_i w[i] exp(-j 2 pi 3 i / M) over one period = (1/M) sum_k sqrt(G_k) sum_i exp(j 2 pi (k-3) i / M)
    = sqrt(G_3)."""
    M = 16
    G = np.ones(M)
    G[3] = 1.0 / 17.0
    r = np.array([1.0], dtype=np.complex64)
    inner = slice(M, 4 * M - M)
    for k0, gain in ((3, np.sqrt(1.0 / 17.0)), (-3, 1.0), (13, 1.0), (5, 1.0)):
        x = _tone(k0)
        y = oracle.rangecompress_whitened(x, r, G)
        assert np.max(np.abs(y[:, inner] - gain * x[:, inner])) <= 1e-6, k0
