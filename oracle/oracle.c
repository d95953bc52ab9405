/*
 * oracle/oracle.c -- plain, slow, obviously-correct fp64 CPU oracle for the
 * time-domain backprojection (TDBP) hot path of Gerg et al., "GPU Acceleration
 * for Synthetic Aperture Sonar Image Reconstruction" (arXiv 2101.05888).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2101_05888_b200/) never links, imports or calls it,
 * and this file shares no code, header, table or constant with the CUDA path.
 *
 * Citation key: P:n = /root/reference/PAPER.md line n (sections / equations as
 * labelled there); readings R1..R13 are listed in DESIGN.md ("Readings").
 *
 * What it computes:
 *
 *   I(x) = sum_{p=0}^{P-1} sum_{e=0}^{E-1}  ehat_{p,e}(u_{p,e}(x)) * exp(+j 2 pi fc tau_{p,e}(x))
 *
 *   tau_{p,e}(x) = (|x - tx_p| + |x - rx_{p,e}|) / c      -- delay argument of
 *                  Eq. (eqn:backprojection), tx stationary during
 *                  transmit; stop-and-hop per element (R5)
 *   u_{p,e}(x)   = (tau - t0_p) * fs                      -- sample n is taken
 *                  t0_p + n/fs after ping p's transmit (R4)
 *   ehat(u)      = (1-a) d[k] + a d[k+1],  k = floor(u), a = u - k,
 *                  d[n] = 0 for n outside 0..Ns-1         -- linear, zero-extended (R1, R2)
 *   exp(+j...)   -- re-modulation of basebanded echoes (R3)
 *   weight 1, no FOV gate, no normalisation (R6, R7, R10), pixel centre =
 *   origin + ix*step_x + iy*step_y + iz*step_z (R8), single sound speed (R9).
 *
 * Every quantity is fp64 (positions, tau, u, phase, std sin/cos, accumulator);
 * only the echoes are complex64, because that is what the caller provides.
 * Loop order per pixel: ping-major, then element (R11).
 *
 * Range compression (the paper presumes compressed data,
 * S:195):  y[n] = sum_{m=0}^{Nr-1} x[n+m] * conj(r[m]),  x[k] = 0 for k >= Ns,
 * the direct O(Ns*Nr) correlation in fp64.
 *
 * NEXT rows: gating (R15), moving receiver (R16; tabled trajectories R23), sediment refraction (R17),
 * and the NEXT-4 interpolation / conditioning variants -- spreading weight R_tx R_rx (R18),
 * 8-tap windowed-sinc xU upsampling (R19), passband basebanding (R20) and spectral whitening
 * (R21).
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>
#include <stdlib.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_TWO_PI 6.283185307179586476925286766559

/* d[n] with zero extension outside 0..Ns-1 (reading R2). */
static inline void sample_at(const float* ch, int32_t Ns, int64_t n, double* re, double* im) {
  if (n < 0 || n >= (int64_t)Ns) { *re = 0.0; *im = 0.0; return; }
  *re = (double)ch[2 * n];
  *im = (double)ch[2 * n + 1];
}

/* Euclidean distance |a - b| in fp64. */
static inline double dist3(const double* a, const double* b) {
  double dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
  return sqrt(dx * dx + dy * dy + dz * dz);
}

/* Pixel centre (reading R8): origin + ix*step_x + iy*step_y + iz*step_z. */
void oracle_pixel_centre(const double* origin, const double* step_x, const double* step_y,
                         const double* step_z, int64_t ix, int64_t iy, int64_t iz, double* out) {
  for (int a = 0; a < 3; ++a)
    out[a] = origin[a] + (double)ix * step_x[a] + (double)iy * step_y[a] + (double)iz * step_z[a];
}

/*
 * One term of the sum for one pixel x, ping p, element e (the whole method for
 * one (pixel, ping, element) triple).  Returns 1 if the interpolation support
 * meets the recorded window, i.e. u in (-1, Ns), else 0 (the term is then 0).
 */
static int one_term_tau(const double* x, const float* ch, int32_t Ns, double tau, double t0, double fc, double fs,
                        double* acc_re, double* acc_im) {
  double u = (tau - t0) * fs;                                /* R4 */
  double kf = floor(u);
  double a = u - kf;
  int64_t k = (int64_t)kf;
  double d0r, d0i, d1r, d1i;
  sample_at(ch, Ns, k, &d0r, &d0i);
  sample_at(ch, Ns, k + 1, &d1r, &d1i);
  double er = (1.0 - a) * d0r + a * d1r;                     /* R1 linear */
  double ei = (1.0 - a) * d0i + a * d1i;
  double ph = ORACLE_TWO_PI * fc * tau;                      /* R3 exp(+j 2 pi fc tau) */
  double cs = cos(ph), sn = sin(ph);
  *acc_re += er * cs - ei * sn;
  *acc_im += er * sn + ei * cs;
  return (u > -1.0 && u < (double)Ns) ? 1 : 0;
}

static int one_term(const double* x, const float* ch, int32_t Ns, const double* tx, const double* rx,
                    double t0, double fc, double fs, double c, double* acc_re, double* acc_im) {
  double tau = (dist3(x, tx) + dist3(x, rx)) / c;           /* Eq. 1 delay */
  return one_term_tau(x, ch, Ns, tau, t0, fc, fs, acc_re, acc_im);
}

/*
 * Two-way delay with the receiver moving during reception (NEXT-2, reading R16): the platform
 * moves with constant velocity v during the ping (first-order kinematics; the
 * paper's motion model assumes continual motion), the transmitter is stationary during
 * the instantaneous transmit, and the echo from x is received at tau, when the
 * element is at rx + v tau:
 *     tau = ( |x - tx| + |x - rx - v tau| ) / c .
 * Solved by fixed-point iteration from the stop-and-hop delay (a contraction with factor
 * <= |v|/c) until the update is below 1e-18 s.
 */
static double delay_moving(const double* x, const double* tx, const double* rx, const double* v, double c) {
  const double rt = dist3(x, tx);
  double tau = (rt + dist3(x, rx)) / c;
  for (int it = 0; it < 64; ++it) {
    double r[3] = {rx[0] + v[0] * tau, rx[1] + v[1] * tau, rx[2] + v[2] * tau};
    double nt = (rt + dist3(x, r)) / c;
    double d = fabs(nt - tau);
    tau = nt;
    if (d <= 1e-18) break;
  }
  return tau;
}

/*
 * TDBP at an explicit list of N points (fp64 NED metres).
 *   echoes : complex64 [P][E][Ns] interleaved (re, im)
 *   tx     : [P][3], rx : [P][E][3], t0 : [P] or NULL (= 0)
 *   out    : complex128 [N] interleaved; n_in : [N] or NULL, count of terms
 *            with u in (-1, Ns) (SURVEY §8(d) N_u)
 * Returns 0, or -1 on invalid sizes.
 */
int oracle_tdbp_points(const float* echoes, int32_t P, int32_t E, int32_t Ns, const double* tx,
                       const double* rx, const double* t0, double fc, double fs, double c,
                       const double* pts, int64_t N, double* out, int64_t* n_in) {
  if (P < 1 || E < 1 || Ns < 1 || N < 0 || !(c > 0) || !(fs > 0)) return -1;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < N; ++i) {
    const double* x = pts + 3 * i;
    double ar = 0.0, ai = 0.0;
    int64_t cnt = 0;
    for (int32_t p = 0; p < P; ++p) {            /* ping-major (R11) */
      double t0p = t0 ? t0[p] : 0.0;
      for (int32_t e = 0; e < E; ++e) {
        const float* ch = echoes + 2 * ((int64_t)p * E + e) * (int64_t)Ns;
        cnt += one_term(x, ch, Ns, tx + 3 * p, rx + 3 * ((int64_t)p * E + e), t0p, fc, fs, c, &ar, &ai);
      }
    }
    out[2 * i] = ar;
    out[2 * i + 1] = ai;
    if (n_in) n_in[i] = cnt;
  }
  return 0;
}

/*
 * Field-of-view gate of a sensor at position s for the scattering location x (NEXT-1 row:
 * "every pixel must query the sonar geometry and determine if it is in the sonar field of
 * view"; hard FWHM cones; reading R15 in DESIGN.md):
 *   v = x - s;  a = along-track unit axis, b = boresight unit axis of the ping (NED);
 *   azimuth   : |v.a| <= |v| sin(az/2)                (skipped when az >= pi)
 *   elevation : v.b > 0 and |v.c| <= (v.b) tan(el/2),  c = a x b   (skipped when el <= 0 or el >= pi)
 */
static int in_fov(const double* x, const double* s, const double* a, const double* b, double az, double el) {
  double v[3] = {x[0] - s[0], x[1] - s[1], x[2] - s[2]};
  double nv = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
  if (az < 3.141592653589793) {
    double va = v[0] * a[0] + v[1] * a[1] + v[2] * a[2];
    if (fabs(va) > nv * sin(0.5 * az)) return 0;
  }
  if (el > 0 && el < 3.141592653589793) {
    double c[3] = {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
    double vb = v[0] * b[0] + v[1] * b[1] + v[2] * b[2];
    double vc = v[0] * c[0] + v[1] * c[1] + v[2] * c[2];
    if (!(vb > 0) || fabs(vc) > vb * tan(0.5 * el)) return 0;
  }
  return 1;
}

/*
 * Gated TDBP at explicit points (NEXT-1): the sum of the definition restricted to the terms
 * whose pixel lies in the transmitter's field of view (and, when bistatic != 0, also in the
 * receiving element's, P:310 / P:315 "bistatic ray-culling"):
 *   I_g(x) = sum_{p,e} [x in FOV(tx_p)] [bistatic -> x in FOV(rx_{p,e})] term_{p,e}(x)
 *   axes : [P][2][3] per-ping unit along-track axis a_p and boresight b_p, or NULL for
 *          a = (1,0,0), b = (0,1,0) (side-looking to starboard)
 */
int oracle_tdbp_points_gated(const float* echoes, int32_t P, int32_t E, int32_t Ns, const double* tx,
                             const double* rx, const double* t0, double fc, double fs, double c,
                             const double* axes, double az, double el, int32_t bistatic,
                             const double* pts, int64_t N, double* out, int64_t* n_in) {
  if (P < 1 || E < 1 || Ns < 1 || N < 0 || !(c > 0) || !(fs > 0)) return -1;
  static const double def_a[3] = {1.0, 0.0, 0.0}, def_b[3] = {0.0, 1.0, 0.0};
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < N; ++i) {
    const double* x = pts + 3 * i;
    double ar = 0.0, ai = 0.0;
    int64_t cnt = 0;
    for (int32_t p = 0; p < P; ++p) {
      const double* a = axes ? axes + 6 * p : def_a;
      const double* b = axes ? axes + 6 * p + 3 : def_b;
      if (!in_fov(x, tx + 3 * p, a, b, az, el)) continue;
      double t0p = t0 ? t0[p] : 0.0;
      for (int32_t e = 0; e < E; ++e) {
        const double* r = rx + 3 * ((int64_t)p * E + e);
        if (bistatic && !in_fov(x, r, a, b, az, el)) continue;
        const float* ch = echoes + 2 * ((int64_t)p * E + e) * (int64_t)Ns;
        cnt += one_term(x, ch, Ns, tx + 3 * p, r, t0p, fc, fs, c, &ar, &ai);
      }
    }
    out[2 * i] = ar;
    out[2 * i + 1] = ai;
    if (n_in) n_in[i] = cnt;
  }
  return 0;
}

/*
 * One-way travel time from a sensor s in the water to x across a flat sediment-water
 * interface (NEXT-3, reading R17; "include a sediment-water interface refraction model in
 * determining propagation time"): interface the horizontal plane z = zb (NED,
 * z down), sound speed c1 above (water) and c2 below (sediment).  For x above the interface the
 * path is straight; for x below, Fermat's principle gives
 *     t = min_xi  sqrt(xi^2 + h1^2)/c1 + sqrt((D - xi)^2 + h2^2)/c2,
 * D = horizontal distance s -> x, h1 = zb - s_z, h2 = x_z - zb (Snell's law at the minimum);
 * solved by Newton's method on the convex objective from the straight-line crossing, to
 * |d xi| < 1e-14 (D + h1 + h2).
 */
static double travel_refracted(const double* x, const double* s, double zb, double c1, double c2) {
  const double h2 = x[2] - zb;
  if (h2 <= 0.0) return dist3(x, s) / c1;
  const double h1 = zb - s[2];
  const double dx = x[0] - s[0], dy = x[1] - s[1];
  const double D = sqrt(dx * dx + dy * dy);
  double xi = D * h1 / (h1 + h2);
  for (int it = 0; it < 100; ++it) {
    const double L1 = sqrt(xi * xi + h1 * h1), L2 = sqrt((D - xi) * (D - xi) + h2 * h2);
    const double f1 = xi / (c1 * L1) - (D - xi) / (c2 * L2);
    const double f2 = h1 * h1 / (c1 * L1 * L1 * L1) + h2 * h2 / (c2 * L2 * L2 * L2);
    double nx = xi - f1 / f2;
    if (nx < 0.0) nx = 0.5 * xi;
    if (nx > D) nx = 0.5 * (xi + D);
    const double step = fabs(nx - xi);
    xi = nx;
    if (step <= 1e-14 * (D + h1 + h2)) break;
  }
  return sqrt(xi * xi + h1 * h1) / c1 + sqrt((D - xi) * (D - xi) + h2 * h2) / c2;
}

/*
 * TDBP through a flat sediment-water interface (NEXT-3): the definition with the straight-path
 * delay replaced by tau = travel_refracted(x, tx) + travel_refracted(x, rx).  Sensors must be in
 * the water (tx_z, rx_z < zb); c is the water sound speed c1.
 */
int oracle_tdbp_points_refracted(const float* echoes, int32_t P, int32_t E, int32_t Ns, const double* tx,
                                 const double* rx, const double* t0, double zb, double c2, double fc, double fs,
                                 double c, const double* pts, int64_t N, double* out, int64_t* n_in) {
  if (P < 1 || E < 1 || Ns < 1 || N < 0 || !(c > 0) || !(fs > 0) || !(c2 > 0)) return -1;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < N; ++i) {
    const double* x = pts + 3 * i;
    double ar = 0.0, ai = 0.0;
    int64_t cnt = 0;
    for (int32_t p = 0; p < P; ++p) {
      double t0p = t0 ? t0[p] : 0.0;
      const double tt = travel_refracted(x, tx + 3 * p, zb, c, c2);
      for (int32_t e = 0; e < E; ++e) {
        const float* ch = echoes + 2 * ((int64_t)p * E + e) * (int64_t)Ns;
        const double tau = tt + travel_refracted(x, rx + 3 * ((int64_t)p * E + e), zb, c, c2);
        cnt += one_term_tau(x, ch, Ns, tau, t0p, fc, fs, &ar, &ai);
      }
    }
    out[2 * i] = ar;
    out[2 * i + 1] = ai;
    if (n_in) n_in[i] = cnt;
  }
  return 0;
}

/* One-way refracted travel time alone (for the pins). */
double oracle_travel_refracted(const double* x, const double* s, double zb, double c1, double c2) {
  return travel_refracted(x, s, zb, c1, c2);
}

/*
 * TDBP with continuous receiver motion at explicit points (NEXT-2): the definition with the
 * stop-and-hop delay replaced by delay_moving (per-ping velocity vel[P][3], NED m/s).
 */
int oracle_tdbp_points_motion(const float* echoes, int32_t P, int32_t E, int32_t Ns, const double* tx,
                              const double* rx, const double* t0, const double* vel, double fc, double fs,
                              double c, const double* pts, int64_t N, double* out, int64_t* n_in) {
  if (P < 1 || E < 1 || Ns < 1 || N < 0 || !(c > 0) || !(fs > 0) || !vel) return -1;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < N; ++i) {
    const double* x = pts + 3 * i;
    double ar = 0.0, ai = 0.0;
    int64_t cnt = 0;
    for (int32_t p = 0; p < P; ++p) {
      double t0p = t0 ? t0[p] : 0.0;
      for (int32_t e = 0; e < E; ++e) {
        const float* ch = echoes + 2 * ((int64_t)p * E + e) * (int64_t)Ns;
        double tau = delay_moving(x, tx + 3 * p, rx + 3 * ((int64_t)p * E + e), vel + 3 * p, c);
        cnt += one_term_tau(x, ch, Ns, tau, t0p, fc, fs, &ar, &ai);
      }
    }
    out[2 * i] = ar;
    out[2 * i + 1] = ai;
    if (n_in) n_in[i] = cnt;
  }
  return 0;
}

/* The moving-receiver delay alone (for the closed-form pins): tau for one (x, tx, rx, v). */
double oracle_delay_moving(const double* x, const double* tx, const double* rx, const double* v, double c) {
  return delay_moving(x, tx, rx, v, c);
}

/*
 * TDBP at grid pixels given by index triples idx[N][3] = (ix, iy, iz) of the
 * grid (origin, step_x, step_y, step_z), reading R8.
 */
int oracle_tdbp_grid_pixels(const float* echoes, int32_t P, int32_t E, int32_t Ns, const double* tx,
                            const double* rx, const double* t0, double fc, double fs, double c,
                            const double* origin, const double* step_x, const double* step_y,
                            const double* step_z, const int64_t* idx, int64_t N, double* out,
                            int64_t* n_in) {
  if (N < 0) return -1;
  int rc = 0;
  /* chunked so the point list stays small */
  const int64_t CHUNK = 4096;
  double pts[3 * 4096];
  for (int64_t s = 0; s < N && rc == 0; s += CHUNK) {
    int64_t n = (N - s) < CHUNK ? (N - s) : CHUNK;
    for (int64_t i = 0; i < n; ++i) {
      const int64_t* q = idx + 3 * (s + i);
      oracle_pixel_centre(origin, step_x, step_y, step_z, q[0], q[1], q[2], pts + 3 * i);
    }
    rc = oracle_tdbp_points(echoes, P, E, Ns, tx, rx, t0, fc, fs, c, pts, n, out + 2 * s,
                            n_in ? n_in + s : NULL);
  }
  return rc;
}

/*
 * Direct matched-filter correlation (row a1):
 *   y[n] = sum_{m=0}^{Nr-1} x[n+m] * conj(r[m]),  n = 0..Ns-1,  x[k] = 0 for k >= Ns.
 *   raw : complex64 [nch][Ns], replica : complex64 [Nr], out : complex128 [nch][Ns].
 */
int oracle_rangecompress(const float* raw, int64_t nch, int32_t Ns, const float* replica, int32_t Nr,
                         double* out) {
  if (nch < 0 || Ns < 1 || Nr < 1) return -1;
#pragma omp parallel for schedule(static)
  for (int64_t ch = 0; ch < nch; ++ch) {
    const float* x = raw + 2 * ch * (int64_t)Ns;
    double* y = out + 2 * ch * (int64_t)Ns;
    for (int32_t n = 0; n < Ns; ++n) {
      double yr = 0.0, yi = 0.0;
      for (int32_t m = 0; m < Nr && n + m < Ns; ++m) {
        double xr = x[2 * (n + m)], xi = x[2 * (n + m) + 1];
        double rr = replica[2 * m], ri = -(double)replica[2 * m + 1];  /* conj(r[m]) */
        yr += xr * rr - xi * ri;
        yi += xr * ri + xi * rr;
      }
      y[2 * n] = yr;
      y[2 * n + 1] = yi;
    }
  }
  return 0;
}

/*
 * Spreading-compensated TDBP at explicit points (NEXT-4, reading R18): every term of the
 * definition multiplied by w = |x - tx_p| |x - rx_{p,e}|, the inverse of the spherical-spreading
 * amplitude 1/(|x_TX - x| |x_RX - x|) of Eq. (eqn:backprojection) ("spreading
 * compensation (multiplying by R_tx R_rx)").
 */
int oracle_tdbp_points_weighted(const float* echoes, int32_t P, int32_t E, int32_t Ns, const double* tx,
                                const double* rx, const double* t0, double fc, double fs, double c,
                                const double* pts, int64_t N, double* out, int64_t* n_in) {
  if (P < 1 || E < 1 || Ns < 1 || N < 0 || !(c > 0) || !(fs > 0)) return -1;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < N; ++i) {
    const double* x = pts + 3 * i;
    double ar = 0.0, ai = 0.0;
    int64_t cnt = 0;
    for (int32_t p = 0; p < P; ++p) {
      double t0p = t0 ? t0[p] : 0.0;
      const double rt = dist3(x, tx + 3 * p);
      for (int32_t e = 0; e < E; ++e) {
        const float* ch = echoes + 2 * ((int64_t)p * E + e) * (int64_t)Ns;
        const double rr = dist3(x, rx + 3 * ((int64_t)p * E + e));
        double tr = 0.0, ti = 0.0;
        cnt += one_term_tau(x, ch, Ns, (rt + rr) / c, t0p, fc, fs, &tr, &ti);
        ar += rt * rr * tr;                                    /* w = R_tx R_rx (R18) */
        ai += rt * rr * ti;
      }
    }
    out[2 * i] = ar;
    out[2 * i + 1] = ai;
    if (n_in) n_in[i] = cnt;
  }
  return 0;
}

/*
 * The 8-tap windowed-sinc interpolation kernel (NEXT-4, reading R19; "band-limited
 * via 8-tap windowed-sinc"; the paper is silent on interpolation): the Lanczos window of
 * order 4,
 *     L(s) = sinc(s) sinc(s/4)  for |s| < 4,   0 otherwise,   sinc(s) = sin(pi s)/(pi s), sinc(0) = 1.
 */
static double lanczos4(double s) {
  const double PI = 3.141592653589793238462643383279;
  if (s == 0.0) return 1.0;
  if (fabs(s) >= 4.0) return 0.0;
  return (sin(PI * s) / (PI * s)) * (sin(PI * s / 4.0) / (PI * s / 4.0));
}

double oracle_lanczos4(double s) { return lanczos4(s); }

/*
 * Band-limited xU upsampling of complex channels by the 8-tap kernel (NEXT-4, R19):
 *     y[U n + r] = sum_{m=-3}^{4} x[n + m] L(r/U - m),   r = 0..U-1,  n = 0..Ns-1,
 * x zero-extended outside 0..Ns-1 (reading R2).  Output sample j = U n + r sits at the input
 * time n + r/U, so the upsampled series has rate U fs and the same t0.
 *   x : complex64 [nch][Ns], out : complex128 [nch][U Ns].
 */
int oracle_upsample(const float* x, int64_t nch, int32_t Ns, int32_t U, double* out) {
  if (nch < 0 || Ns < 1 || U < 1) return -1;
#pragma omp parallel for schedule(static)
  for (int64_t ch = 0; ch < nch; ++ch) {
    const float* xc = x + 2 * ch * (int64_t)Ns;
    double* y = out + 2 * ch * (int64_t)Ns * U;
    for (int32_t n = 0; n < Ns; ++n) {
      for (int32_t r = 0; r < U; ++r) {
        double yr = 0.0, yi = 0.0;
        for (int32_t m = -3; m <= 4; ++m) {
          double dr, di;
          sample_at(xc, Ns, (int64_t)n + m, &dr, &di);
          const double w = lanczos4((double)r / (double)U - (double)m);
          yr += w * dr;
          yi += w * di;
        }
        y[2 * ((int64_t)U * n + r)] = yr;
        y[2 * ((int64_t)U * n + r) + 1] = yi;
      }
    }
  }
  return 0;
}

/*
 * Basebanding of real passband channels (the optional input; reading
 * R20): mix down by the carrier measured from the ping's transmit instant (R3, R4), low-pass
 * with the caller's FIR taps h[0..Nh-1] (Nh odd, centred) and keep every D-th sample:
 *     z[n] = x[n] exp(-j 2 pi fc (t0_p + n / fs_in)),       z[n] = 0 outside 0..Nin-1
 *     y[m] = sum_{k=0}^{Nh-1} h[k] z[m D + (Nh-1)/2 - k],     m = 0..Nout-1
 * Output sample m is taken at t0_p + m D / fs_in: rate fs_in / D, same t0.
 *   x : float [P][E][Nin], t0 : [P] or NULL (= 0), out : complex128 [P][E][Nout].
 */
int oracle_baseband(const float* x, int32_t P, int32_t E, int32_t Nin, double fs_in, double fc,
                    const double* t0, const float* h, int32_t Nh, int32_t D, int32_t Nout, double* out) {
  if (P < 1 || E < 1 || Nin < 1 || Nh < 1 || (Nh % 2) == 0 || D < 1 || Nout < 1 || !(fs_in > 0)) return -1;
  const int64_t nch = (int64_t)P * E;
  const int32_t half = (Nh - 1) / 2;
#pragma omp parallel for schedule(static)
  for (int64_t ch = 0; ch < nch; ++ch) {
    const float* xc = x + ch * (int64_t)Nin;
    const double t0p = t0 ? t0[ch / E] : 0.0;
    double* y = out + 2 * ch * (int64_t)Nout;
    for (int32_t m = 0; m < Nout; ++m) {
      double yr = 0.0, yi = 0.0;
      for (int32_t k = 0; k < Nh; ++k) {
        const int64_t n = (int64_t)m * D + half - k;
        if (n < 0 || n >= Nin) continue;
        const double ph = -ORACLE_TWO_PI * fc * (t0p + (double)n / fs_in);
        yr += (double)h[k] * (double)xc[n] * cos(ph);
        yi += (double)h[k] * (double)xc[n] * sin(ph);
      }
      y[2 * m] = yr;
      y[2 * m + 1] = yi;
    }
  }
  return 0;
}

/*
 * Spectral whitening (NEXT-4, reading R21; Eq. (eqn:whitening)):
 *     G(f) = h( 1 / (gamma * mean_f P(f) + P(f)) ),   h = scaling so that max G = 1 (0 dB minimum
 *     attenuation, "h is a normalization function ensuring the minimum attenuation is 0 dB")
 * with the power estimate P the batch-mean periodogram on an M-point frequency grid:
 *     P[k] = (1 / (nch B)) sum_ch sum_{b<B} | sum_{n<M} x_ch[b M + n] exp(-j 2 pi k n / M) |^2,
 *     B = max(1, floor(Ns / M)) blocks per channel, x zero past Ns.
 *   raw : complex64 [nch][Ns]; G, P : fp64 [M] out.  Returns -2 if gamma*mean + P[k] <= 0 for
 *   some k (an all-zero batch has no spectrum), -1 on invalid sizes.
 */
int oracle_whitening_gain(const float* raw, int64_t nch, int32_t Ns, int32_t M, double gamma, double* G, double* P) {
  const double TWO_PI = ORACLE_TWO_PI;
  if (nch < 1 || Ns < 1 || M < 1 || !(gamma >= 0)) return -1;
  const int32_t B = Ns / M > 0 ? Ns / M : 1;
  for (int32_t k = 0; k < M; ++k) P[k] = 0.0;
  for (int64_t ch = 0; ch < nch; ++ch) {
    const float* x = raw + 2 * ch * (int64_t)Ns;
    for (int32_t b = 0; b < B; ++b) {
      for (int32_t k = 0; k < M; ++k) {
        double re = 0.0, im = 0.0;
        for (int32_t n = 0; n < M; ++n) {
          double xr, xi;
          sample_at(x, Ns, (int64_t)b * M + n, &xr, &xi);
          const double a = -TWO_PI * (double)(((int64_t)k * n) % M) / (double)M;
          re += xr * cos(a) - xi * sin(a);
          im += xr * sin(a) + xi * cos(a);
        }
        P[k] += re * re + im * im;
      }
    }
  }
  double mean = 0.0;
  for (int32_t k = 0; k < M; ++k) {
    P[k] /= (double)nch * (double)B;
    mean += P[k];
  }
  mean /= (double)M;
  double gmax = 0.0;
  for (int32_t k = 0; k < M; ++k) {
    const double den = gamma * mean + P[k];
    if (!(den > 0)) return -2;
    G[k] = 1.0 / den;
    if (G[k] > gmax) gmax = G[k];
  }
  for (int32_t k = 0; k < M; ++k) G[k] /= gmax;
  return 0;
}

/*
 * Whitened range compression (NEXT-4, R21): G of Eq. 9 is a POWER gain (it flattens P: with
 * gamma = 0, G P is constant; SPEC S:208-209 gives its values in dB as 10 log10 G), so the signal
 * is filtered with the amplitude response sqrt(G[k]) at f = k fs / M -- the M-tap
 * frequency-sampling FIR over one centred period,
 *     w[i] = (1/M) sum_k sqrt(G[k]) exp(+j 2 pi k i / M),   i = -M/2 .. M/2 - 1   (M even; M = 1: w = [sqrt G0])
 * -- followed by the matched filter of R14:
 *     x_w[n] = sum_i w[i] x[n - i]          (x zero outside 0..Ns-1, x_w not truncated)
 *     y[n]   = sum_{m<Nr} x_w[n + m] conj(r[m]),   n = 0..Ns-1.
 *   raw : complex64 [nch][Ns], replica complex64 [Nr], G fp64 [M], out complex128 [nch][Ns].
 */
int oracle_rangecompress_whitened(const float* raw, int64_t nch, int32_t Ns, const float* replica, int32_t Nr,
                                  const double* G, int32_t M, double* out) {
  const double TWO_PI = ORACLE_TWO_PI;
  if (nch < 0 || Ns < 1 || Nr < 1 || M < 1 || (M > 1 && (M % 2) != 0)) return -1;
  const int32_t i0 = -(M / 2);
  double* w = (double*)malloc(sizeof(double) * 2 * (size_t)M);
  if (!w) return -1;
  for (int32_t t = 0; t < M; ++t) {
    const int32_t i = i0 + t;
    double re = 0.0, im = 0.0;
    for (int32_t k = 0; k < M; ++k) {
      const int64_t km = (((int64_t)k * i) % M + M) % M;
      const double a = TWO_PI * (double)km / (double)M;
      re += sqrt(G[k]) * cos(a);
      im += sqrt(G[k]) * sin(a);
    }
    w[2 * t] = re / M;
    w[2 * t + 1] = im / M;
  }
#pragma omp parallel for schedule(static)
  for (int64_t ch = 0; ch < nch; ++ch) {
    const float* x = raw + 2 * ch * (int64_t)Ns;
    double* y = out + 2 * ch * (int64_t)Ns;
    for (int32_t n = 0; n < Ns; ++n) {
      double yr = 0.0, yi = 0.0;
      for (int32_t m = 0; m < Nr; ++m) {
        double xwr = 0.0, xwi = 0.0;                            /* x_w[n + m] */
        for (int32_t t = 0; t < M; ++t) {
          double xr, xi;
          sample_at(x, Ns, (int64_t)n + m - (i0 + t), &xr, &xi);
          xwr += w[2 * t] * xr - w[2 * t + 1] * xi;
          xwi += w[2 * t] * xi + w[2 * t + 1] * xr;
        }
        const double rr = replica[2 * m], ri = -(double)replica[2 * m + 1];   /* conj(r[m]) */
        yr += xwr * rr - xwi * ri;
        yi += xwr * ri + xwi * rr;
      }
      y[2 * n] = yr;
      y[2 * n + 1] = yi;
    }
  }
  free(w);
  return 0;
}

/*
 * Gated AND spreading-weighted TDBP (NEXT-1 gate R15 combined with the NEXT-4 weight R18): the
 * gated sum of oracle_tdbp_points_gated with every admitted term multiplied by R_tx R_rx.
 */
int oracle_tdbp_points_gated_weighted(const float* echoes, int32_t P, int32_t E, int32_t Ns, const double* tx,
                                      const double* rx, const double* t0, double fc, double fs, double c,
                                      const double* axes, double az, double el, int32_t bistatic,
                                      const double* pts, int64_t N, double* out) {
  if (P < 1 || E < 1 || Ns < 1 || N < 0 || !(c > 0) || !(fs > 0)) return -1;
  static const double def_a[3] = {1.0, 0.0, 0.0}, def_b[3] = {0.0, 1.0, 0.0};
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < N; ++i) {
    const double* x = pts + 3 * i;
    double ar = 0.0, ai = 0.0;
    for (int32_t p = 0; p < P; ++p) {
      const double* a = axes ? axes + 6 * p : def_a;
      const double* b = axes ? axes + 6 * p + 3 : def_b;
      if (!in_fov(x, tx + 3 * p, a, b, az, el)) continue;
      const double t0p = t0 ? t0[p] : 0.0;
      const double rt = dist3(x, tx + 3 * p);
      for (int32_t e = 0; e < E; ++e) {
        const double* r = rx + 3 * ((int64_t)p * E + e);
        if (bistatic && !in_fov(x, r, a, b, az, el)) continue;
        const float* ch = echoes + 2 * ((int64_t)p * E + e) * (int64_t)Ns;
        const double rr = dist3(x, r);
        double tr = 0.0, ti = 0.0;
        one_term_tau(x, ch, Ns, (rt + rr) / c, t0p, fc, fs, &tr, &ti);
        ar += rt * rr * tr;
        ai += rt * rr * ti;
      }
    }
    out[2 * i] = ar;
    out[2 * i + 1] = ai;
  }
  return 0;
}

/*
 * Gated TDBP with the receiver moving during reception (NEXT-1 gate R15 combined with the NEXT-2
 * delay R16; reading R22 in DESIGN.md): the FOV decision is taken on the sensor positions at the
 * transmit instant (tx_p, rx_{p,e} as recorded; the paper tests the sonar geometry per ping,
 * P:160) along the straight line of sight, and every admitted term takes the moving-receiver
 * delay of oracle_tdbp_points_motion:
 *   I(x) = sum_{p,e} [x in FOV(tx_p)] [bistatic -> x in FOV(rx_{p,e})] term(x; tau = delay_moving)
 */
int oracle_tdbp_points_gated_motion(const float* echoes, int32_t P, int32_t E, int32_t Ns, const double* tx,
                                    const double* rx, const double* t0, const double* vel, double fc, double fs,
                                    double c, const double* axes, double az, double el, int32_t bistatic,
                                    const double* pts, int64_t N, double* out, int64_t* n_in) {
  if (P < 1 || E < 1 || Ns < 1 || N < 0 || !(c > 0) || !(fs > 0) || !vel) return -1;
  static const double def_a[3] = {1.0, 0.0, 0.0}, def_b[3] = {0.0, 1.0, 0.0};
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < N; ++i) {
    const double* x = pts + 3 * i;
    double ar = 0.0, ai = 0.0;
    int64_t cnt = 0;
    for (int32_t p = 0; p < P; ++p) {
      const double* a = axes ? axes + 6 * p : def_a;
      const double* b = axes ? axes + 6 * p + 3 : def_b;
      if (!in_fov(x, tx + 3 * p, a, b, az, el)) continue;
      const double t0p = t0 ? t0[p] : 0.0;
      for (int32_t e = 0; e < E; ++e) {
        const double* r = rx + 3 * ((int64_t)p * E + e);
        if (bistatic && !in_fov(x, r, a, b, az, el)) continue;
        const float* ch = echoes + 2 * ((int64_t)p * E + e) * (int64_t)Ns;
        const double tau = delay_moving(x, tx + 3 * p, r, vel + 3 * p, c);
        cnt += one_term_tau(x, ch, Ns, tau, t0p, fc, fs, &ar, &ai);
      }
    }
    out[2 * i] = ar;
    out[2 * i + 1] = ai;
    if (n_in) n_in[i] = cnt;
  }
  return 0;
}

/*
 * Gated TDBP through a flat sediment-water interface (NEXT-1 gate R15 combined with the NEXT-3
 * delay R17; reading R22; the paper's near-field craft uses bistatic culling and the refraction
 * model together): the FOV decision is the straight line-of-sight cone test from the
 * recorded sensor positions, every admitted term takes the Fermat delay of
 * oracle_tdbp_points_refracted.
 */
int oracle_tdbp_points_gated_refracted(const float* echoes, int32_t P, int32_t E, int32_t Ns, const double* tx,
                                       const double* rx, const double* t0, double zb, double c2, double fc,
                                       double fs, double c, const double* axes, double az, double el,
                                       int32_t bistatic, const double* pts, int64_t N, double* out, int64_t* n_in) {
  if (P < 1 || E < 1 || Ns < 1 || N < 0 || !(c > 0) || !(fs > 0) || !(c2 > 0)) return -1;
  static const double def_a[3] = {1.0, 0.0, 0.0}, def_b[3] = {0.0, 1.0, 0.0};
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < N; ++i) {
    const double* x = pts + 3 * i;
    double ar = 0.0, ai = 0.0;
    int64_t cnt = 0;
    for (int32_t p = 0; p < P; ++p) {
      const double* a = axes ? axes + 6 * p : def_a;
      const double* b = axes ? axes + 6 * p + 3 : def_b;
      if (!in_fov(x, tx + 3 * p, a, b, az, el)) continue;
      const double t0p = t0 ? t0[p] : 0.0;
      const double tt = travel_refracted(x, tx + 3 * p, zb, c, c2);
      for (int32_t e = 0; e < E; ++e) {
        const double* r = rx + 3 * ((int64_t)p * E + e);
        if (bistatic && !in_fov(x, r, a, b, az, el)) continue;
        const float* ch = echoes + 2 * ((int64_t)p * E + e) * (int64_t)Ns;
        const double tau = tt + travel_refracted(x, r, zb, c, c2);
        cnt += one_term_tau(x, ch, Ns, tau, t0p, fc, fs, &ar, &ai);
      }
    }
    out[2 * i] = ar;
    out[2 * i + 1] = ai;
    if (n_in) n_in[i] = cnt;
  }
  return 0;
}

/* Number of OpenMP threads the oracle will use (for the cpu_baseline "cores"). */
int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/*
 * Receiver position during reception from a position table (NEXT-2, reading R23 in DESIGN.md;
 * the paper keeps the navigation in a position look-up table, and its motion model
 * assumes continual motion).  For one (ping, element) the table holds K >= 3 positions
 * r_k at the times t_k = k dt after the ping's transmit; between nodes the position is the cubic
 * Hermite spline through them with the tangents
 *     m_k     = (r_{k+1} - r_{k-1}) / (2 dt)                 0 < k < K-1
 *     m_0     = (-3 r_0 + 4 r_1 - r_2) / (2 dt)
 *     m_{K-1} = (3 r_{K-1} - 4 r_{K-2} + r_{K-3}) / (2 dt)
 * (all exact for quadratic motion, so a quadratic trajectory is reproduced exactly); before t_0
 * and after t_{K-1} the first / last segment's cubic is continued.  On segment k with
 * s = t/dt - k:
 *     r(t) = h00(s) r_k + h10(s) dt m_k + h01(s) r_{k+1} + h11(s) dt m_{k+1},
 *     h00 = (1 + 2s)(1 - s)^2,  h10 = s (1 - s)^2,  h01 = s^2 (3 - 2s),  h11 = s^2 (s - 1).
 */
static void nav_tangent_dt(const double* lut, int32_t K, int32_t k, double m[3]) {   /* dt * m_k */
  for (int i = 0; i < 3; ++i) {
    if (k == 0)
      m[i] = 0.5 * (-3.0 * lut[i] + 4.0 * lut[3 + i] - lut[6 + i]);
    else if (k == K - 1)
      m[i] = 0.5 * (3.0 * lut[3 * (K - 1) + i] - 4.0 * lut[3 * (K - 2) + i] + lut[3 * (K - 3) + i]);
    else
      m[i] = 0.5 * (lut[3 * (k + 1) + i] - lut[3 * (k - 1) + i]);
  }
}

static void nav_eval(const double* lut, int32_t K, double dt, double t, double r[3]) {
  double s = t / dt;
  int32_t k = (int32_t)floor(s);
  if (k < 0) k = 0;
  if (k > K - 2) k = K - 2;
  s -= (double)k;
  const double h00 = (1.0 + 2.0 * s) * (1.0 - s) * (1.0 - s);
  const double h10 = s * (1.0 - s) * (1.0 - s);
  const double h01 = s * s * (3.0 - 2.0 * s);
  const double h11 = s * s * (s - 1.0);
  double m0[3], m1[3];
  nav_tangent_dt(lut, K, k, m0);
  nav_tangent_dt(lut, K, k + 1, m1);
  for (int i = 0; i < 3; ++i)
    r[i] = h00 * lut[3 * k + i] + h10 * m0[i] + h01 * lut[3 * (k + 1) + i] + h11 * m1[i];
}

/*
 * Two-way delay with the receiver on the tabled trajectory (R23): the echo from x reaches the
 * element at tau, when it is at r(tau), the transmitter stationary at tx:
 *     tau = ( |x - tx| + |x - r(tau)| ) / c ,
 * fixed-point iteration from tau = (|x - tx| + |x - r(0)|)/c (a contraction for element speeds
 * below c) until the update is below 1e-18 s.
 */
static double delay_nav(const double* x, const double* tx, const double* lut, int32_t K, double dt, double c) {
  const double rt = dist3(x, tx);
  double r[3];
  nav_eval(lut, K, dt, 0.0, r);
  double tau = (rt + dist3(x, r)) / c;
  for (int it = 0; it < 200; ++it) {
    nav_eval(lut, K, dt, tau, r);
    const double nt = (rt + dist3(x, r)) / c;
    const double d = fabs(nt - tau);
    tau = nt;
    if (d <= 1e-18) break;
  }
  return tau;
}

/*
 * TDBP with tabled receiver trajectories at explicit points (NEXT-2, R23): the definition with
 * the delay of delay_nav.  lut: fp64 [P][E][K][3] (NED metres), node spacing dt (s).
 */
int oracle_tdbp_points_nav(const float* echoes, int32_t P, int32_t E, int32_t Ns, const double* tx,
                           const double* lut, int32_t K, double dt, const double* t0, double fc, double fs,
                           double c, const double* pts, int64_t N, double* out, int64_t* n_in) {
  if (P < 1 || E < 1 || Ns < 1 || N < 0 || K < 3 || !(dt > 0) || !(c > 0) || !(fs > 0) || !lut) return -1;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < N; ++i) {
    const double* x = pts + 3 * i;
    double ar = 0.0, ai = 0.0;
    int64_t cnt = 0;
    for (int32_t p = 0; p < P; ++p) {
      const double t0p = t0 ? t0[p] : 0.0;
      for (int32_t e = 0; e < E; ++e) {
        const int64_t ch = (int64_t)p * E + e;
        const float* d = echoes + 2 * ch * (int64_t)Ns;
        const double tau = delay_nav(x, tx + 3 * p, lut + 3 * (int64_t)K * ch, K, dt, c);
        cnt += one_term_tau(x, d, Ns, tau, t0p, fc, fs, &ar, &ai);
      }
    }
    out[2 * i] = ar;
    out[2 * i + 1] = ai;
    if (n_in) n_in[i] = cnt;
  }
  return 0;
}

/* The table interpolant and the delay alone (for the pins). */
void oracle_nav_eval(const double* lut, int32_t K, double dt, double t, double* r) { nav_eval(lut, K, dt, t, r); }
double oracle_delay_nav(const double* x, const double* tx, const double* lut, int32_t K, double dt, double c) {
  return delay_nav(x, tx, lut, K, dt, c);
}

/*
 * Gated TDBP with tabled receiver trajectories (NEXT-1 gate R15 with the NEXT-2 delay R23;
 * reading R22): the FOV decision is the straight line-of-sight cone test from the positions
 * recorded at the transmit instant (tx_p, rx_{p,e}); every admitted term takes delay_nav.
 */
int oracle_tdbp_points_gated_nav(const float* echoes, int32_t P, int32_t E, int32_t Ns, const double* tx,
                                 const double* rx, const double* lut, int32_t K, double dt, const double* t0,
                                 double fc, double fs, double c, const double* axes, double az, double el,
                                 int32_t bistatic, const double* pts, int64_t N, double* out, int64_t* n_in) {
  if (P < 1 || E < 1 || Ns < 1 || N < 0 || K < 3 || !(dt > 0) || !(c > 0) || !(fs > 0) || !lut) return -1;
  static const double def_a[3] = {1.0, 0.0, 0.0}, def_b[3] = {0.0, 1.0, 0.0};
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < N; ++i) {
    const double* x = pts + 3 * i;
    double ar = 0.0, ai = 0.0;
    int64_t cnt = 0;
    for (int32_t p = 0; p < P; ++p) {
      const double* a = axes ? axes + 6 * p : def_a;
      const double* b = axes ? axes + 6 * p + 3 : def_b;
      if (!in_fov(x, tx + 3 * p, a, b, az, el)) continue;
      const double t0p = t0 ? t0[p] : 0.0;
      for (int32_t e = 0; e < E; ++e) {
        const int64_t ch = (int64_t)p * E + e;
        if (bistatic && !in_fov(x, rx + 3 * ch, a, b, az, el)) continue;
        const float* d = echoes + 2 * ch * (int64_t)Ns;
        const double tau = delay_nav(x, tx + 3 * p, lut + 3 * (int64_t)K * ch, K, dt, c);
        cnt += one_term_tau(x, d, Ns, tau, t0p, fc, fs, &ar, &ai);
      }
    }
    out[2 * i] = ar;
    out[2 * i + 1] = ai;
    if (n_in) n_in[i] = cnt;
  }
  return 0;
}
