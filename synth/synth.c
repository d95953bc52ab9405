/*
 * synth/synth.c -- seeded synthetic echo generator (forward model only).
 *
 * Shared by tests and bench as the INPUT generator for both the CUDA path and
 * the oracle.  It holds none of the backprojection method's arithmetic: it
 * evaluates the forward model Eq. (eqn:backprojection) for a
 * sparse point-scatterer scene, in the range-compressed, basebanded form
 * (SURVEY §8(d) "Synthetic inputs"; S:278 superposition, S:310 closed-form pulse):
 *
 *   e_{p,e}[n] = sum_s  sigma_s / (R_tx R_rx) * sinc(B (t_n - tau_s)) * exp(-j 2 pi fc tau_s)
 *   t_n = t0_p + n / fs,   tau_s = (R_tx + R_rx) / c,
 *
 * with the compressed pulse truncated to |t_n - tau_s| * fs <= half_support and an
 * optional hard azimuth fan-beam gate tested from the transmitter in the body
 * frame: keep scatterer s for ping p iff |v_x| <= |v| sin(theta/2),
 * v = R_p^T (x_s - tx_p).
 *
 * Random numbers (scene, speckle, nav perturbations) are drawn in synth/__init__.py
 * with numpy's seeded PCG64 and passed in; this file is deterministic.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#define SYN_PI 3.14159265358979323846264338328

/* Forward-model one-way time from a sensor s (in water) to a scatterer x across the flat
 * interface z = zb (c1 above, c2 below), Fermat path; also returns the geometric path length. */
static double syn_travel(const double* x, const double* s, double zb, double c1, double c2, double* len) {
  double dx = x[0] - s[0], dy = x[1] - s[1], dz = x[2] - s[2];
  double h2 = x[2] - zb;
  if (h2 <= 0.0) {
    *len = sqrt(dx * dx + dy * dy + dz * dz);
    return *len / c1;
  }
  double h1 = zb - s[2], D = sqrt(dx * dx + dy * dy);
  double lo = 0.0, hi = D;   /* bisection on the derivative of the convex objective (robust) */
  for (int it = 0; it < 200 && hi - lo > 1e-15 * (D + 1.0); ++it) {
    double m = 0.5 * (lo + hi);
    double g = m / (c1 * sqrt(m * m + h1 * h1)) - (D - m) / (c2 * sqrt((D - m) * (D - m) + h2 * h2));
    if (g > 0) hi = m; else lo = m;
  }
  double xi = 0.5 * (lo + hi);
  double L1 = sqrt(xi * xi + h1 * h1), L2 = sqrt((D - xi) * (D - xi) + h2 * h2);
  *len = L1 + L2;
  return L1 / c1 + L2 / c2;
}

/*
 * echoes   : float32 [P][E][Ns][2], accumulated into (caller zeroes it)
 * tx       : [P][3]; rx : [P][E][3]; t0 : [P]
 * body_rot : [P][9] row-major body->world rotation, or NULL (identity)
 * scat     : [S][3]; sigma : [S][2] complex amplitude
 * sin_half_beam : gate parameter; <= 0 disables the gate (omni elements)
 */
int synth_echoes(float* echoes, int32_t P, int32_t E, int32_t Ns, const double* tx, const double* rx,
                 const double* t0, const double* body_rot, double fc, double B, double fs, double c,
                 int32_t half_support, const double* scat, const double* sigma, int64_t S,
                 double sin_half_beam, const double* vel, int32_t refract, double zb, double c2) {
  if (P < 1 || E < 1 || Ns < 1 || S < 0 || !(fs > 0) || !(c > 0) || !(B > 0)) return -1;
  const double step = SYN_PI * B / fs; /* sinc argument increment (radians of pi x) */
  const double cst = cos(step), snt = sin(step);
#pragma omp parallel for schedule(dynamic, 1)
  for (int32_t p = 0; p < P; ++p) {
    const double* T = tx + 3 * p;
    const double* Rm = body_rot ? body_rot + 9 * p : NULL;
    for (int64_t s = 0; s < S; ++s) {
      const double* X = scat + 3 * s;
      double vx = X[0] - T[0], vy = X[1] - T[1], vz = X[2] - T[2];
      double rtx = sqrt(vx * vx + vy * vy + vz * vz);
      if (rtx <= 0) continue;
      if (sin_half_beam > 0) {
        /* body-frame forward component: (R^T v)_x = R[0][0] vx + R[1][0] vy + R[2][0] vz */
        double bx = Rm ? (Rm[0] * vx + Rm[3] * vy + Rm[6] * vz) : vx;
        if (fabs(bx) > rtx * sin_half_beam) continue;
      }
      for (int32_t e = 0; e < E; ++e) {
        const double* Rx = rx + 3 * ((int64_t)p * E + e);
        double wx = X[0] - Rx[0], wy = X[1] - Rx[1], wz = X[2] - Rx[2];
        double rrx = sqrt(wx * wx + wy * wy + wz * wz);
        if (rrx <= 0) continue;
        double tau = (rtx + rrx) / c;
        if (refract) {   /* sediment-water interface: both legs follow Fermat paths */
          double lt, lr;
          tau = syn_travel(X, T, zb, c, c2, &lt) + syn_travel(X, Rx, zb, c, c2, &lr);
          rrx = lr;
          (void)lt;
        } else if (vel) {  /* receiver moving with the platform during reception: tau = (R_tx + |x - rx - v tau|)/c */
          const double* V = vel + 3 * p;
          for (int it = 0; it < 8; ++it) {
            double qx = wx - V[0] * tau, qy = wy - V[1] * tau, qz = wz - V[2] * tau;
            rrx = sqrt(qx * qx + qy * qy + qz * qz);
            tau = (rtx + rrx) / c;
          }
        }
        double amp_r = sigma[2 * s] / (rtx * rrx), amp_i = sigma[2 * s + 1] / (rtx * rrx);
        /* carrier exp(-j 2 pi fc tau), phase reduced in cycles first */
        double cyc = fc * tau;
        cyc -= floor(cyc);
        double cr = cos(2.0 * SYN_PI * cyc), ci = -sin(2.0 * SYN_PI * cyc);
        double ar = amp_r * cr - amp_i * ci, ai = amp_r * ci + amp_i * cr;
        double u = (tau - t0[p]) * fs; /* fractional sample of the echo peak */
        int64_t n_lo = (int64_t)ceil(u - half_support), n_hi = (int64_t)floor(u + half_support);
        if (n_lo < 0) n_lo = 0;
        if (n_hi > Ns - 1) n_hi = Ns - 1;
        if (n_lo > n_hi) continue;
        float* ch = echoes + 2 * ((int64_t)p * E + e) * (int64_t)Ns;
        /* x_n = B (t_n - tau) = (n - u) B / fs ; sin(pi x_n) by rotation */
        double x0 = ((double)n_lo - u) * B / fs;
        double sr = sin(SYN_PI * x0), cr0 = cos(SYN_PI * x0);
        for (int64_t n = n_lo; n <= n_hi; ++n) {
          double x = ((double)n - u) * B / fs;
          double sinc = (fabs(x) < 1e-12) ? 1.0 : sr / (SYN_PI * x);
          ch[2 * n] += (float)(ar * sinc);
          ch[2 * n + 1] += (float)(ai * sinc);
          double ns = sr * cst + cr0 * snt, nc = cr0 * cst - sr * snt;
          sr = ns; cr0 = nc;
        }
      }
    }
  }
  return 0;
}
