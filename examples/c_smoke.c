/*
 * c_smoke.c -- the C ABI used from plain C (no Python, no torch): image one point target.
 *
 * 16 pings along x at 10 m altitude, 2 receive elements, a point target at (1.0, 8.0, 0);
 * the echoes are the analytic compressed baseband pulse sinc(B (t - tau)) exp(-j 2 pi fc tau)
 * (the forward model of Eq. 1, with unit amplitude).  The program forms a 48 x 48 image
 * around the target through libsasbp.so and checks that the peak is the target pixel.
 *
 *   gcc -std=c11 -O2 -I include examples/c_smoke.c -L paper_2101_05888_b200 -lsasbp -lm \
 *       -Wl,-rpath,$PWD/paper_2101_05888_b200 -o c_smoke && ./c_smoke
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "sasbp.h"

#define P 16
#define E 2
#define NS 1024
#define N 48

int main(void) {
  const double PI = 3.141592653589793, c = 1500.0, fc = 120e3, B = 30e3, fs = 4 * B, t0 = 0.012;
  const double tgt[3] = {1.0, 8.0, 0.0};
  static double tx[P][3], rx[P][E][3];
  static float echoes[P][E][NS][2];
  for (int p = 0; p < P; ++p) {
    tx[p][0] = 0.6 + 0.05 * p; tx[p][1] = 0.0; tx[p][2] = -10.0;
    for (int e = 0; e < E; ++e) {
      rx[p][e][0] = tx[p][0] + 0.02 * (e - 0.5); rx[p][e][1] = 0.0; rx[p][e][2] = -10.0;
      double dt[3], dr[3];
      for (int a = 0; a < 3; ++a) { dt[a] = tgt[a] - tx[p][a]; dr[a] = tgt[a] - rx[p][e][a]; }
      const double tau = (sqrt(dt[0] * dt[0] + dt[1] * dt[1] + dt[2] * dt[2]) +
                          sqrt(dr[0] * dr[0] + dr[1] * dr[1] + dr[2] * dr[2])) / c;
      for (int n = 0; n < NS; ++n) {
        const double x = B * (t0 + n / fs - tau);
        const double s = fabs(x) < 1e-12 ? 1.0 : sin(PI * x) / (PI * x);
        echoes[p][e][n][0] = (float)(s * cos(-2 * PI * fc * tau));
        echoes[p][e][n][1] = (float)(s * sin(-2 * PI * fc * tau));
      }
    }
  }
  sas_grid g = {{tgt[0] - 0.005 * (N / 2), tgt[1] - 0.005 * (N / 2), 0.0},
                {0.005, 0, 0}, {0, 0.005, 0}, {0, 0, 1.0}, N, N, 1};
  sas_bp_t h = NULL;
  sas_status st = sas_bp_create(fc, B, fs, c, &g, &h);
  if (st != SAS_OK) { printf("create: %d %s\n", st, sas_last_error()); return st == SAS_E_UNSUPPORTED ? 77 : 1; }
  double t0s[P];
  for (int p = 0; p < P; ++p) t0s[p] = t0;
  st = sas_bp_set_pings(h, &echoes[0][0][0][0], P, E, NS, &tx[0][0], &rx[0][0][0], t0s);
  if (st != SAS_OK) { printf("set_pings: %s\n", sas_last_error()); return 1; }
  float* img = (float*)malloc(sizeof(float) * 2 * N * N);
  st = sas_bp_form(h, img);
  if (st != SAS_OK) { printf("form: %s\n", sas_last_error()); return 1; }
  int best = 0;
  double bm = -1;
  for (int i = 0; i < N * N; ++i) {
    const double m = hypot(img[2 * i], img[2 * i + 1]);
    if (m > bm) { bm = m; best = i; }
  }
  const int ix = best % N, iy = best / N;
  printf("%s: peak |I| = %.3f at (%d, %d), target pixel (%d, %d), phase %.2e rad\n", sas_version(), bm, ix, iy,
         N / 2, N / 2, atan2(img[2 * best + 1], img[2 * best]));
  sas_bp_destroy(h);
  free(img);
  return (ix == N / 2 && iy == N / 2 && bm > 0.9 * P * E) ? 0 : 2;
}
