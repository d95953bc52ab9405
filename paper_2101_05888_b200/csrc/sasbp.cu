// sasbp.cu -- host side of libsasbp.so: the C ABI declared in include/sasbp.h.
//
// Owns: argument validation, the per-grid plan (tile shape, window capacity, precision
// mode), the one-time device allocations (image + workspace, the paper's slab idea P:156),
// ping uploads and the K2/K3 launches.  No torch types cross this boundary.
#include "sasbp.h"

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <new>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "k2_launch.cuh"


namespace {

thread_local char g_err[512] = "";
thread_local int g_last_occ = 0;   // resident CTAs per SM of the last K2 launch on this thread
thread_local int g_last_split = 0; // wave-tail split factor of the last K2 launch on this thread

sas_status fail(sas_status st, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return st;
}

bool finite3(const double* v) { return std::isfinite(v[0]) && std::isfinite(v[1]) && std::isfinite(v[2]); }
double norm3(const double* v) { return std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]); }

using Variant = sasbp::K2Variant;
constexpr Variant V2D = sasbp::kV2D, V2D_DZ = sasbp::kV2D_DZ, V3D = sasbp::kV3D;

}  // namespace

struct sas_bp_s {
  int device = -1;
  double fc = 0, bandwidth = 0, fs = 0, c = 0;
  sas_grid grid{};
  // plan
  Variant variant = V2D;
  int TX = 32, TY = 32, TZ = 1;
  int tiles_x = 0, tiles_y = 0, tiles_z = 0;
  double d_max = 0;  // max |pixel - tile centre| (m)
  double hw = 0;     // half window, samples
  int W = 0;         // window slots per channel
  int mode = 0;      // receive-leg mode: sasbp::kSeries3 / kSeries4 / kExact
  bool axis = false; // diagonal grid steps (compact per-pixel geometry kernels)
  // device memory
  float2* image = nullptr;
  float2* echoes_owned = nullptr;
  size_t echoes_cap = 0;
  const float2* echoes = nullptr;
  double* geo = nullptr;  // tx [P*3] | rx [P*E*3] | t0 [P]
  size_t geo_cap = 0;
  unsigned long long* counter = nullptr;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;   // H2D of ping chunks in sas_bp_form_streamed
  // Completion of the last K2/K3 launch queued on a caller stream (sas_bp_form_device): every call
  // that rewrites the workspace (nav, owned echoes, axes, velocities) first waits for it, so a
  // setter can never overwrite data a still-running kernel reads (sasbp.h "Ordering").
  cudaEvent_t busy = nullptr;
  bool busy_pending = false;
  int P = 0, E = 0, Ns = 0;
  // TMA descriptor of the current echoes (row staging), rebuilt when the ping set changes
  sasbp::TmaDesc tmap{};
  bool use_tma = false;
  int tma_W = -1;        // window the descriptor's box was encoded for (a launch with another W re-encodes)
  int ctas_per_sm = 0;   // measured occupancy of the last form
  int tail_split = 0;    // wave-tail split of the last form
  // field-of-view gating (sas_bp_set_beam; NEXT-1)
  int gate = 0, cull = 0, az_on = 0, el_on = 0;
  double half_az = 0, sin_half_az = 0, half_el = 0, tan_half_el = 0;
  double* axes = nullptr;
  int axes_P = 0;
  // continuous receiver motion (sas_bp_set_motion; NEXT-2)
  double* vel = nullptr;
  int vel_P = 0;
  // tabled receiver trajectories (sas_bp_set_nav; NEXT-2, R23): [P*E][K][3]
  double* nav = nullptr;
  int nav_P = 0, nav_E = 0, nav_K = 0;
  double nav_dt = 0, nav_rmin = INFINITY;   // smallest node-to-grid distance (series truncation bound)
  double rmin = INFINITY;                   // smallest sensor-to-grid distance of the ping set
  // sediment-water interface (sas_bp_set_medium; NEXT-3)
  int refract = 0;
  double zb = 0, c2 = 0;
  // spreading weight R_tx R_rx (sas_bp_set_weighting; NEXT-4, R18)
  int weight = 0;
  double max_sensor_z = -INFINITY;   // of the current ping set
  bool has_pings = false;
  bool broken = false;
  size_t bytes = 0;
};

namespace {

sas_status cuda_fail(sas_bp_t h, cudaError_t e, const char* what) {
  if (h) h->broken = true;
  return fail(SAS_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define CK_H(h, call)                                          \
  do {                                                         \
    cudaError_t e_ = (call);                                   \
    if (e_ != cudaSuccess) return cuda_fail((h), e_, #call);   \
  } while (0)

size_t smem_bytes(int W) { return sasbp::k2_smem_bytes(W); }

// Host-blocking wait for the last asynchronous launch that reads the workspace.
sas_status wait_idle(sas_bp_t h) {
  if (h->busy_pending) {
    CK_H(h, cudaEventSynchronize(h->busy));
    h->busy_pending = false;
  }
  return SAS_OK;
}

// Mode combinations and per-ping array sizes, checked against the ping set about to be used
// (P, largest sensor z) BEFORE any state changes.
sas_status check_modes(sas_bp_t h, int32_t P, double max_sensor_z, int32_t E = -1) {
  if (E < 0) E = h->E;
  if (h->gate && h->axes && h->axes_P != P) return fail(SAS_E_STATE, "beam axes were given for %d pings, the ping set has %d", h->axes_P, P);
  if (h->vel && h->vel_P != P) return fail(SAS_E_STATE, "velocities were given for %d pings, the ping set has %d", h->vel_P, P);
  if (h->nav && (h->nav_P != P || h->nav_E != E))
    return fail(SAS_E_STATE, "receiver tables were given for %d x %d channels, the ping set has %d x %d", h->nav_P, h->nav_E, P, E);
  if (h->refract && (h->vel || h->nav)) return fail(SAS_E_UNSUPPORTED, "refraction and receiver motion cannot be combined");
  if (h->refract && !(max_sensor_z < h->zb)) return fail(SAS_E_INVALID, "with an interface every sensor must be in the water (z < zb)");
  if (h->weight && (h->vel || h->nav || h->refract)) return fail(SAS_E_UNSUPPORTED, "the spreading weight is defined for stop-and-hop straight rays only");
  return SAS_OK;
}

double max_z(int32_t P, int32_t E, const double* tx, const double* rx) {
  double m = -INFINITY;
  for (int32_t p = 0; p < P; ++p) m = std::fmax(m, tx[3 * (size_t)p + 2]);
  for (size_t i = 0; i < (size_t)P * E; ++i) m = std::fmax(m, rx[3 * i + 2]);
  return m;
}

// Receive-leg mode from the series truncation bound: sqrt(1+e) - 1 truncated
// after n terms leaves |rem| <= r * |c_{n+1}| e^{n+1} / (1 - e) (alternating, decreasing terms),
// c = 1/2, -1/8, 1/16, -5/128, 7/256; with |e| <= 2 d/r + (d/r)^2 the worst case is at the
// smallest element-to-grid distance r_min.  Allowed: 3e-5 wavelength of path (1.9e-4 rad).
int choose_mode(double d_max, double r_min, double lambda) {
  if (!(r_min > 0)) return sasbp::kExact;
  const double eps = 2.0 * d_max / r_min + (d_max / r_min) * (d_max / r_min);
  if (eps > 0.3) return sasbp::kExact;
  const double tol = 3e-5 * lambda;
  if (r_min * (5.0 / 128.0) * std::pow(eps, 4.0) / (1.0 - eps) <= tol) return sasbp::kSeries3;
  if (r_min * (7.0 / 256.0) * std::pow(eps, 5.0) / (1.0 - eps) <= tol) return sasbp::kSeries4;
  return sasbp::kExact;
}

// distance from point p to the axis-aligned bounding box of the grid's pixel centres
double dist_to_box(const double* p, const double lo[3], const double hi[3]) {
  double s = 0;
  for (int a = 0; a < 3; ++a) {
    double d = 0;
    if (p[a] < lo[a]) d = lo[a] - p[a];
    else if (p[a] > hi[a]) d = p[a] - hi[a];
    s += d * d;
  }
  return std::sqrt(s);
}

// Encode the TMA descriptor for the echo array [P*E][Ns] of 8-byte samples, box = one window
// row.  Returns false (cp.async fallback) when the layout does not meet TMA's rules: 16-B
// aligned base and row pitch (Ns even), box <= 256 samples.
bool encode_tma(sas_bp_t h, int W) {
  const char* no = getenv("SASBP_NO_TMA");
  if (no && no[0] == '1') return false;
  const int box = sasbp::box_samples(W);
  if ((h->Ns & 1) || box > 256 || (((uintptr_t)h->echoes) & 15)) return false;
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return false;
    encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }
  cuuint64_t dims[2] = {(cuuint64_t)h->Ns, (cuuint64_t)h->P * (cuuint64_t)h->E};
  cuuint64_t strides[1] = {(cuuint64_t)h->Ns * 8};
  cuuint32_t boxd[2] = {(cuuint32_t)box, 1};
  cuuint32_t estr[2] = {1, 1};
  sasbp::TmaDesc t{};
  CUresult r = encode(reinterpret_cast<CUtensorMap*>(&t), CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, (void*)h->echoes,
                      dims, strides, boxd, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  h->tmap = t;
  h->tma_W = W;
  return true;
}

// receive-leg mode of a launch: tabled receivers may come closer to the grid than the ping set's
// positions, so the truncation bound takes the nearest table node as well
int rx_mode(sas_bp_t h) {
  if (!h->nav) return h->mode;
  return choose_mode(h->d_max, std::fmin(h->rmin, h->nav_rmin), h->c / h->fc);
}

// bounding box of the pixel centres grown by the tile sphere radius
void grid_box(sas_bp_t h, double lo[3], double hi[3]) {
  const sas_grid& g = h->grid;
  for (int a = 0; a < 3; ++a) {
    double v0 = g.origin[a];
    double ex = (g.nx - 1) * g.step_x[a], ey = (g.ny - 1) * g.step_y[a], ez = (g.nz - 1) * g.step_z[a];
    lo[a] = v0 + std::fmin(ex, 0.0) + std::fmin(ey, 0.0) + std::fmin(ez, 0.0) - h->d_max;
    hi[a] = v0 + std::fmax(ex, 0.0) + std::fmax(ey, 0.0) + std::fmax(ez, 0.0) + h->d_max;
  }
}

cudaError_t launch_tdbp(sas_bp_t h, float2* image, unsigned long long* counter, int accumulate,
                        bool count, cudaStream_t st, int ch_lo = 0, int ch_hi = -1) {
  sasbp::TdbpParams prm{};
  prm.echoes = h->echoes;
  prm.tx = h->geo;
  prm.rx = h->geo + 3 * (size_t)h->P;
  prm.t0 = h->geo + 3 * (size_t)h->P + 3 * (size_t)h->P * h->E;
  prm.image = image;
  prm.counter = counter;
  for (int a = 0; a < 3; ++a) {
    prm.origin[a] = h->grid.origin[a];
    prm.sx[a] = h->grid.step_x[a];
    prm.sy[a] = h->grid.step_y[a];
    prm.sz[a] = h->grid.step_z[a];
  }
  prm.fc = h->fc; prm.fs = h->fs; prm.c = h->c;
  prm.k_s = h->fs / h->c; prm.k_c = h->fc / h->c; prm.k_r = h->fc / h->fs; prm.inv_e = 1.0 / h->E;
  prm.kph_f = (float)(6.283185307179586 * prm.k_r); prm.kfs_f = (float)prm.k_s;
  prm.hw = h->hw;
  prm.P = h->P; prm.E = h->E; prm.Ns = h->Ns;
  prm.nx = h->grid.nx; prm.ny = h->grid.ny; prm.nz = h->grid.nz;
  prm.tiles_x = h->tiles_x; prm.tiles_y = h->tiles_y; prm.tiles_z = h->tiles_z;
  prm.W = h->W;
  prm.accumulate = accumulate;
  prm.ch_lo = ch_lo;
  prm.ch_hi = ch_hi < 0 ? h->P * h->E : ch_hi;
  prm.gate = h->gate; prm.cull = h->cull; prm.az_on = h->az_on; prm.el_on = h->el_on;
  prm.axes = h->axes;
  prm.sin_half_az = h->sin_half_az; prm.half_az = h->half_az;
  prm.tan_half_el = h->tan_half_el; prm.half_el = h->half_el;
  prm.d_max = h->d_max;
  prm.vel = h->vel;
  prm.nav = h->nav; prm.nav_k = h->nav_K; prm.nav_dt = h->nav_dt;
  prm.refract = h->refract; prm.zb = h->zb; prm.c2 = h->c2;
  prm.mode = h->refract ? sasbp::kRefract : rx_mode(h);
  if (h->refract) {   // the window must cover the slowest medium: |grad tau| <= 2 / min(c, c2)
    prm.hw = 2.0 * h->d_max * h->fs / std::min(h->c, h->c2);
    prm.W = (int)std::ceil(2.0 * prm.hw + 4.0) + 3;
  }
  // the TMA box must match the window this launch stages (the refracted plan widens it): a
  // descriptor encoded for another W would never complete the batch's mbarrier transaction
  bool tma = h->use_tma;
  if (tma && h->tma_W != prm.W) tma = encode_tma(h, prm.W);
  const char* na = getenv("SASBP_NO_AXIS");   // A/B and test switch: force the general-geometry kernel
  const bool no_axis = na && na[0] == '1';
  sasbp::K2Launch L{tma, h->axis && !no_axis, rx_mode(h), count, st, &g_last_occ, &g_last_split};
  // A/B knob: the two-launch gated form (IN pairs mask-free, then the edge pairs); config 2 with the
  // generator's beam: 125.4-126.1 ms against 122.9 ms for one launch (profiles/ab_r02.txt), so off
  const char* g2 = getenv("SASBP_GATE_TWO");
  L.gsplit = g2 && g2[0] == '1';
  g_last_occ = 0;
  g_last_split = 0;
  const bool g = prm.gate && !count;
  if (h->weight && !count) {
    switch (h->variant) {
      case V2D: return sasbp::k2_launch_2d_w(prm, h->tmap, L);
      case V2D_DZ: return sasbp::k2_launch_2ddz_w(prm, h->tmap, L);
      default: return sasbp::k2_launch_3d_w(prm, h->tmap, L);
    }
  }
  switch (h->variant) {
    case V2D: return g ? sasbp::k2_launch_2d_gate(prm, h->tmap, L) : sasbp::k2_launch_2d(prm, h->tmap, L);
    case V2D_DZ: return g ? sasbp::k2_launch_2ddz_gate(prm, h->tmap, L) : sasbp::k2_launch_2ddz(prm, h->tmap, L);
    default: return g ? sasbp::k2_launch_3d_gate(prm, h->tmap, L) : sasbp::k2_launch_3d(prm, h->tmap, L);
  }
}

sas_status validate_geo(int32_t P, int32_t E, int32_t Ns, const double* tx, const double* rx, const double* t0) {
  if (P < 1 || E < 1 || Ns < 1) return fail(SAS_E_INVALID, "P, E, Ns must be >= 1 (got %d, %d, %d)", P, E, Ns);
  if (!tx || !rx) return fail(SAS_E_INVALID, "tx and rx must not be NULL");
  const long double tot = (long double)P * E * Ns;
  if (tot > 9.0e15L || (long double)P * E > 2.0e9L) return fail(SAS_E_INVALID, "P*E*Ns too large");
  for (int32_t p = 0; p < P; ++p) {
    if (!finite3(tx + 3 * (size_t)p)) return fail(SAS_E_INVALID, "non-finite tx[%d]", p);
    if (t0 && !std::isfinite(t0[p])) return fail(SAS_E_INVALID, "non-finite t0[%d]", p);
  }
  for (size_t i = 0; i < (size_t)P * E; ++i)
    if (!finite3(rx + 3 * i)) return fail(SAS_E_INVALID, "non-finite rx[%zu]", i);
  return SAS_OK;
}

// upload nav, decide the precision mode of the plan for this ping set
sas_status upload_geo(sas_bp_t h, int32_t P, int32_t E, int32_t Ns, const double* tx, const double* rx,
                      const double* t0, cudaStream_t st) {
  const size_t n = 3 * (size_t)P + 3 * (size_t)P * E + (size_t)P;
  if (sas_status w = wait_idle(h); w != SAS_OK) return w;
  if (n > h->geo_cap) {
    if (h->geo) { cudaFree(h->geo); h->bytes -= h->geo_cap * sizeof(double); h->geo = nullptr; h->geo_cap = 0; }
    cudaError_t e = cudaMalloc(&h->geo, n * sizeof(double));
    if (e != cudaSuccess) { h->geo = nullptr; return fail(SAS_E_NOMEM, "cudaMalloc(nav): %s", cudaGetErrorString(e)); }
    h->geo_cap = n;
    h->bytes += n * sizeof(double);
  }
  std::vector<double> host(n);
  memcpy(host.data(), tx, 3 * (size_t)P * sizeof(double));
  memcpy(host.data() + 3 * (size_t)P, rx, 3 * (size_t)P * E * sizeof(double));
  for (int32_t p = 0; p < P; ++p) host[3 * (size_t)P + 3 * (size_t)P * E + p] = t0 ? t0[p] : 0.0;
  CK_H(h, cudaMemcpyAsync(h->geo, host.data(), n * sizeof(double), cudaMemcpyHostToDevice, st));
  CK_H(h, cudaStreamSynchronize(st));  // host vector goes out of scope
  // precision mode: smallest element-to-grid distance decides Taylor vs exact rx leg
  const sas_grid& g = h->grid;
  double lo[3], hi[3];
  for (int a = 0; a < 3; ++a) {
    double v0 = g.origin[a];
    double ex = (g.nx - 1) * g.step_x[a], ey = (g.ny - 1) * g.step_y[a], ez = (g.nz - 1) * g.step_z[a];
    lo[a] = v0 + std::fmin(ex, 0.0) + std::fmin(ey, 0.0) + std::fmin(ez, 0.0) - h->d_max;
    hi[a] = v0 + std::fmax(ex, 0.0) + std::fmax(ey, 0.0) + std::fmax(ez, 0.0) + h->d_max;
  }
  double rmin = INFINITY;
  for (size_t i = 0; i < (size_t)P * E; ++i) rmin = std::fmin(rmin, dist_to_box(rx + 3 * i, lo, hi));
  for (int32_t p = 0; p < P; ++p) rmin = std::fmin(rmin, dist_to_box(tx + 3 * (size_t)p, lo, hi));   // tx leg series too
  h->max_sensor_z = max_z(P, E, tx, rx);
  // sample indices must stay far inside int32 (window starts, TMA coordinates): reject geometries
  // whose delays exceed 1e9 samples (e.g. t0 in the wrong unit)
  {
    double bc[3], hd2 = 0, far_t = 0, far_r = 0, t0max = 0;
    for (int a = 0; a < 3; ++a) { bc[a] = 0.5 * (lo[a] + hi[a]); hd2 += 0.25 * (hi[a] - lo[a]) * (hi[a] - lo[a]); }
    const double hd = std::sqrt(hd2);
    auto dist = [&](const double* q) {
      return std::sqrt((q[0] - bc[0]) * (q[0] - bc[0]) + (q[1] - bc[1]) * (q[1] - bc[1]) + (q[2] - bc[2]) * (q[2] - bc[2]));
    };
    for (int32_t p = 0; p < P; ++p) {
      far_t = std::fmax(far_t, dist(tx + 3 * (size_t)p) + hd);
      if (t0) t0max = std::fmax(t0max, std::fabs(t0[p]));
    }
    for (size_t i = 0; i < (size_t)P * E; ++i) far_r = std::fmax(far_r, dist(rx + 3 * i) + hd);
    if ((far_t + far_r) * h->fs / h->c + t0max * h->fs > 1e9)
      return fail(SAS_E_INVALID, "delays beyond 1e9 samples (check t0 units and sensor positions)");
  }
  h->mode = choose_mode(h->d_max, rmin, h->c / h->fc);
  h->rmin = rmin;
  h->P = P; h->E = E; h->Ns = Ns;
  return SAS_OK;
}

}  // namespace

extern "C" {

const char* sas_last_error(void) { return g_err; }

// internal (not in sasbp.h): lets the other translation units report through sas_last_error
__attribute__((visibility("hidden"))) void sasbp_set_error(const char* msg) {
  snprintf(g_err, sizeof(g_err), "%s", msg ? msg : "");
}

const char* sas_version(void) { return "sasbp 0.1.0 sm_100a"; }

sas_status sas_bp_create(double fc, double bandwidth, double fs, double c, const sas_grid* grid, sas_bp_t* out) {
  g_err[0] = 0;
  if (!out) return fail(SAS_E_INVALID, "out must not be NULL");
  *out = nullptr;
  if (!grid) return fail(SAS_E_INVALID, "grid must not be NULL");
  if (!(std::isfinite(fc) && fc > 0)) return fail(SAS_E_INVALID, "fc must be finite and > 0");
  if (!(std::isfinite(fs) && fs > 0)) return fail(SAS_E_INVALID, "fs must be finite and > 0");
  if (!(std::isfinite(c) && c > 0)) return fail(SAS_E_INVALID, "c must be finite and > 0");
  if (!(std::isfinite(bandwidth) && bandwidth > 0 && bandwidth <= fs))
    return fail(SAS_E_INVALID, "bandwidth must satisfy 0 < bandwidth <= fs");
  const sas_grid& g = *grid;
  if (g.nx < 1 || g.ny < 1 || g.nz < 1) return fail(SAS_E_INVALID, "grid dims must be >= 1");
  if ((long double)g.nx * g.ny * g.nz > 2147483647.0L) return fail(SAS_E_INVALID, "grid has more than 2^31 pixels");
  if (!finite3(g.origin) || !finite3(g.step_x) || !finite3(g.step_y) || !finite3(g.step_z))
    return fail(SAS_E_INVALID, "grid origin/steps must be finite");
  const double nxs = norm3(g.step_x), nys = norm3(g.step_y), nzs = norm3(g.step_z);
  if ((g.nx > 1 && !(nxs > 0)) || (g.ny > 1 && !(nys > 0)) || (g.nz > 1 && !(nzs > 0)))
    return fail(SAS_E_INVALID, "zero step on an axis with more than one pixel");
  // independence of the used step vectors
  {
    const double* v[3] = {g.step_x, g.step_y, g.step_z};
    int used[3] = {g.nx > 1, g.ny > 1, g.nz > 1};
    for (int a = 0; a < 3; ++a)
      for (int b = a + 1; b < 3; ++b)
        if (used[a] && used[b]) {
          double cx = v[a][1] * v[b][2] - v[a][2] * v[b][1], cy = v[a][2] * v[b][0] - v[a][0] * v[b][2],
                 cz = v[a][0] * v[b][1] - v[a][1] * v[b][0];
          if (!(std::sqrt(cx * cx + cy * cy + cz * cz) > 1e-12 * norm3(v[a]) * norm3(v[b])))
            return fail(SAS_E_INVALID, "grid step vectors are linearly dependent");
        }
  }
  int dev = -1;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail(SAS_E_UNSUPPORTED, "no CUDA device: %s", cudaGetErrorString(e));
  int major = 0;
  e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (e != cudaSuccess) return fail(SAS_E_UNSUPPORTED, "cudaDeviceGetAttribute: %s", cudaGetErrorString(e));
  if (major != 10) return fail(SAS_E_UNSUPPORTED, "libsasbp is built for sm_100a only (device cc major %d)", major);

  sas_bp_t h = new (std::nothrow) sas_bp_s();
  if (!h) return fail(SAS_E_NOMEM, "host allocation failed");
  h->device = dev;
  h->fc = fc; h->bandwidth = bandwidth; h->fs = fs; h->c = c;
  h->grid = g;
  const bool flat_z = (g.nz == 1) && g.step_x[2] == 0.0 && g.step_y[2] == 0.0;
  // 3D grids with each step along its own axis (off-diagonal components exactly zero) run the
  // compact-geometry instantiation (A/B on config 4: +7.9 %; on 2D planes it lost 1.8 %)
  h->axis = (g.nz > 1 || SASBP_AXIS2D) && g.step_x[1] == 0.0 && g.step_x[2] == 0.0 && g.step_y[0] == 0.0 && g.step_y[2] == 0.0 &&
            g.step_z[0] == 0.0 && g.step_z[1] == 0.0;
  if (g.nz == 1) { h->variant = flat_z ? V2D : V2D_DZ; h->TX = 8 * SASBP_KX2D; h->TY = 4 * SASBP_KY2D * SASBP_WY2D; h->TZ = 1; }
  else { h->variant = V3D; h->TX = 16; h->TY = 4 * SASBP_KY3D; h->TZ = SASBP_KZ3D * SASBP_WZ3D; }
  h->tiles_x = (g.nx + h->TX - 1) / h->TX;
  h->tiles_y = (g.ny + h->TY - 1) / h->TY;
  h->tiles_z = (g.nz + h->TZ - 1) / h->TZ;
  // max |d| over the tile: a convex function of the offsets, maximal at a corner
  {
    double best = 0;
    for (int sxn = -1; sxn <= 1; sxn += 2)
      for (int syn = -1; syn <= 1; syn += 2)
        for (int szn = -1; szn <= 1; szn += 2) {
          double ax = sxn * 0.5 * (h->TX - 1), ay = syn * 0.5 * (h->TY - 1), az = szn * 0.5 * (h->TZ - 1);
          double d[3];
          for (int a = 0; a < 3; ++a) d[a] = ax * g.step_x[a] + ay * g.step_y[a] + az * g.step_z[a];
          best = std::fmax(best, norm3(d));
        }
    h->d_max = best;
  }
  h->hw = 2.0 * h->d_max * fs / c;
  h->W = (int)std::ceil(2.0 * h->hw + 4.0) + 3;  // + 1 cell for the even (TMA-aligned) window start
  if (smem_bytes(h->W) > 200 * 1024) {
    delete h;
    return fail(SAS_E_UNSUPPORTED, "tile window of %d samples does not fit shared memory (pixel step too large for fs)", 0);
  }
  e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) { delete h; return fail(SAS_E_CUDA, "cudaStreamCreate: %s", cudaGetErrorString(e)); }
  e = cudaEventCreateWithFlags(&h->busy, cudaEventDisableTiming);
  if (e != cudaSuccess) { cudaStreamDestroy(h->stream); delete h; return fail(SAS_E_CUDA, "cudaEventCreate: %s", cudaGetErrorString(e)); }
  const size_t npx = (size_t)g.nx * g.ny * g.nz;
  e = cudaMalloc(&h->image, npx * sizeof(float2));
  if (e != cudaSuccess) { cudaEventDestroy(h->busy); cudaStreamDestroy(h->stream); delete h; return fail(SAS_E_NOMEM, "cudaMalloc(image): %s", cudaGetErrorString(e)); }
  e = cudaMalloc(&h->counter, sizeof(unsigned long long));
  if (e != cudaSuccess) { cudaFree(h->image); cudaEventDestroy(h->busy); cudaStreamDestroy(h->stream); delete h; return fail(SAS_E_NOMEM, "cudaMalloc(counter)"); }
  h->bytes = npx * sizeof(float2) + sizeof(unsigned long long);
  *out = h;
  return SAS_OK;
}

void sas_bp_destroy(sas_bp_t h) {
  if (!h) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  if (h->busy) { if (h->busy_pending) cudaEventSynchronize(h->busy); cudaEventDestroy(h->busy); }
  cudaFree(h->image);
  cudaFree(h->echoes_owned);
  cudaFree(h->geo);
  cudaFree(h->counter);
  cudaFree(h->axes);
  cudaFree(h->vel);
  cudaFree(h->nav);
  if (h->stream) cudaStreamDestroy(h->stream);
  if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
  if (prev >= 0) cudaSetDevice(prev);
  delete h;
}

sas_status sas_bp_set_pings(sas_bp_t h, const float* echoes, int32_t P, int32_t E, int32_t Ns, const double* tx,
                            const double* rx, const double* t0) {
  g_err[0] = 0;
  if (!h) return fail(SAS_E_INVALID, "handle is NULL");
  if (h->broken) return fail(SAS_E_CUDA, "handle is in a failed CUDA state; destroy it");
  if (!echoes) return fail(SAS_E_INVALID, "echoes must not be NULL");
  sas_status st = validate_geo(P, E, Ns, tx, rx, t0);
  if (st != SAS_OK) return st;
  CK_H(h, cudaSetDevice(h->device));
  if ((st = wait_idle(h)) != SAS_OK) return st;
  const size_t n = (size_t)P * E * Ns;
  if (n > h->echoes_cap) {
    if (h->echoes_owned) { cudaFree(h->echoes_owned); h->bytes -= h->echoes_cap * sizeof(float2); }
    h->echoes_owned = nullptr; h->echoes_cap = 0;
    cudaError_t e = cudaMalloc(&h->echoes_owned, n * sizeof(float2));
    if (e != cudaSuccess) { h->echoes_owned = nullptr; h->has_pings = false; return fail(SAS_E_NOMEM, "cudaMalloc(echoes, %zu B): %s", n * sizeof(float2), cudaGetErrorString(e)); }
    h->echoes_cap = n;
    h->bytes += n * sizeof(float2);
  }
  h->has_pings = false;   // the owned echoes change now; valid again once the nav is in
  CK_H(h, cudaMemcpyAsync(h->echoes_owned, echoes, n * sizeof(float2), cudaMemcpyHostToDevice, h->stream));
  st = upload_geo(h, P, E, Ns, tx, rx, t0, h->stream);  // synchronises the stream
  if (st != SAS_OK) { h->has_pings = false; return st; }
  h->echoes = h->echoes_owned;
  h->use_tma = encode_tma(h, h->W);
  h->has_pings = true;
  return SAS_OK;
}

sas_status sas_bp_set_pings_device(sas_bp_t h, const void* echoes_dev, int32_t P, int32_t E, int32_t Ns,
                                   const double* tx, const double* rx, const double* t0, void* cuda_stream) {
  g_err[0] = 0;
  if (!h) return fail(SAS_E_INVALID, "handle is NULL");
  if (h->broken) return fail(SAS_E_CUDA, "handle is in a failed CUDA state; destroy it");
  if (!echoes_dev) return fail(SAS_E_INVALID, "echoes_dev must not be NULL");
  if (((uintptr_t)echoes_dev) & 7) return fail(SAS_E_INVALID, "echoes_dev must be 8-byte aligned");
  sas_status st = validate_geo(P, E, Ns, tx, rx, t0);
  if (st != SAS_OK) return st;
  CK_H(h, cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)cuda_stream;
  st = upload_geo(h, P, E, Ns, tx, rx, t0, s);
  if (st != SAS_OK) { h->has_pings = false; return st; }
  h->echoes = (const float2*)echoes_dev;
  h->use_tma = encode_tma(h, h->W);
  h->has_pings = true;
  return SAS_OK;
}

sas_status sas_bp_form_device(sas_bp_t h, void* image_dev, void* cuda_stream, int32_t flags) {
  g_err[0] = 0;
  if (!h) return fail(SAS_E_INVALID, "handle is NULL");
  if (h->broken) return fail(SAS_E_CUDA, "handle is in a failed CUDA state; destroy it");
  if (!image_dev) return fail(SAS_E_INVALID, "image_dev must not be NULL");
  if (((uintptr_t)image_dev) & 7) return fail(SAS_E_INVALID, "image_dev must be 8-byte aligned");
  if (flags & ~SAS_FORM_ACCUMULATE) return fail(SAS_E_INVALID, "unknown flags 0x%x", flags);
  if (!h->has_pings) return fail(SAS_E_STATE, "sas_bp_form before sas_bp_set_pings");
  if (sas_status st = check_modes(h, h->P, h->max_sensor_z); st != SAS_OK) return st;
  CK_H(h, cudaSetDevice(h->device));
  CK_H(h, launch_tdbp(h, (float2*)image_dev, h->counter, (flags & SAS_FORM_ACCUMULATE) ? 1 : 0, false,
                      (cudaStream_t)cuda_stream));
  CK_H(h, cudaEventRecord(h->busy, (cudaStream_t)cuda_stream));
  h->busy_pending = true;
  h->ctas_per_sm = g_last_occ;
  h->tail_split = g_last_split;
  return SAS_OK;
}

sas_status sas_bp_form(sas_bp_t h, float* image_out) {
  g_err[0] = 0;
  if (!h) return fail(SAS_E_INVALID, "handle is NULL");
  if (h->broken) return fail(SAS_E_CUDA, "handle is in a failed CUDA state; destroy it");
  if (!image_out) return fail(SAS_E_INVALID, "image_out must not be NULL");
  if (!h->has_pings) return fail(SAS_E_STATE, "sas_bp_form before sas_bp_set_pings");
  if (sas_status st = check_modes(h, h->P, h->max_sensor_z); st != SAS_OK) return st;
  CK_H(h, cudaSetDevice(h->device));
  CK_H(h, launch_tdbp(h, h->image, h->counter, 0, false, h->stream));
  h->ctas_per_sm = g_last_occ;
  h->tail_split = g_last_split;
  const size_t npx = (size_t)h->grid.nx * h->grid.ny * h->grid.nz;
  CK_H(h, cudaMemcpyAsync(image_out, h->image, npx * sizeof(float2), cudaMemcpyDeviceToHost, h->stream));
  CK_H(h, cudaStreamSynchronize(h->stream));
  return SAS_OK;
}

sas_status sas_bp_form_streamed(sas_bp_t h, const float* echoes, int32_t P, int32_t E, int32_t Ns, const double* tx,
                                const double* rx, const double* t0, float* image_out, int32_t chunks) {
  g_err[0] = 0;
  if (!h) return fail(SAS_E_INVALID, "handle is NULL");
  if (h->broken) return fail(SAS_E_CUDA, "handle is in a failed CUDA state; destroy it");
  if (!echoes || !image_out) return fail(SAS_E_INVALID, "echoes and image_out must not be NULL");
  if (chunks < 0) return fail(SAS_E_INVALID, "chunks must be >= 0");
  sas_status st = validate_geo(P, E, Ns, tx, rx, t0);
  if (st != SAS_OK) return st;
  // every check that can fail without a CUDA error runs before the handle's state changes
  if ((st = check_modes(h, P, max_z(P, E, tx, rx), E)) != SAS_OK) return st;
  CK_H(h, cudaSetDevice(h->device));
  if ((st = wait_idle(h)) != SAS_OK) return st;
  const size_t n = (size_t)P * E * Ns;
  h->has_pings = false;   // from here on the owned echoes are being replaced
  if (n > h->echoes_cap) {
    if (h->echoes_owned) { cudaFree(h->echoes_owned); h->bytes -= h->echoes_cap * sizeof(float2); }
    h->echoes_owned = nullptr; h->echoes_cap = 0;
    cudaError_t e = cudaMalloc(&h->echoes_owned, n * sizeof(float2));
    if (e != cudaSuccess) { h->echoes_owned = nullptr; return fail(SAS_E_NOMEM, "cudaMalloc(echoes, %zu B): %s", n * sizeof(float2), cudaGetErrorString(e)); }
    h->echoes_cap = n;
    h->bytes += n * sizeof(float2);
  }
  if (!h->copy_stream) CK_H(h, cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
  st = upload_geo(h, P, E, Ns, tx, rx, t0, h->stream);  // small, synchronous
  if (st != SAS_OK) return st;
  h->echoes = h->echoes_owned;
  h->use_tma = encode_tma(h, h->W);
  const int nch = P * E;
  int nchunk = chunks > 0 ? chunks : 8;
  nchunk = std::max(1, std::min(nchunk, (nch + 63) / 64));   // >= 64 channels per chunk
  std::vector<cudaEvent_t> ev(nchunk, nullptr);
  for (auto& x : ev) CK_H(h, cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
  cudaError_t err = cudaSuccess;
  for (int c = 0; c < nchunk && err == cudaSuccess; ++c) {
    const int c0 = (int)((long long)nch * c / nchunk), c1 = (int)((long long)nch * (c + 1) / nchunk);
    err = cudaMemcpyAsync(h->echoes_owned + (size_t)c0 * Ns, echoes + 2 * (size_t)c0 * Ns,
                          (size_t)(c1 - c0) * Ns * sizeof(float2), cudaMemcpyHostToDevice, h->copy_stream);
    if (err == cudaSuccess) err = cudaEventRecord(ev[c], h->copy_stream);
    if (err == cudaSuccess) err = cudaStreamWaitEvent(h->stream, ev[c], 0);
    if (err == cudaSuccess) err = launch_tdbp(h, h->image, h->counter, c > 0 ? 1 : 0, false, h->stream, c0, c1);
  }
  const size_t npx = (size_t)h->grid.nx * h->grid.ny * h->grid.nz;
  if (err == cudaSuccess)
    err = cudaMemcpyAsync(image_out, h->image, npx * sizeof(float2), cudaMemcpyDeviceToHost, h->stream);
  if (err == cudaSuccess) err = cudaStreamSynchronize(h->stream);
  for (auto& x : ev) cudaEventDestroy(x);
  if (err != cudaSuccess) return cuda_fail(h, err, "sas_bp_form_streamed");
  h->has_pings = true;   // the whole ping set is resident now (form / form_device may reuse it)
  return SAS_OK;
}

sas_status sas_bp_count_terms(sas_bp_t h, uint64_t* dense, uint64_t* in_win) {
  g_err[0] = 0;
  if (!h) return fail(SAS_E_INVALID, "handle is NULL");
  if (h->broken) return fail(SAS_E_CUDA, "handle is in a failed CUDA state; destroy it");
  if (!h->has_pings) return fail(SAS_E_STATE, "sas_bp_count_terms before sas_bp_set_pings");
  if (sas_status st = check_modes(h, h->P, h->max_sensor_z); st != SAS_OK) return st;
  const uint64_t npx = (uint64_t)h->grid.nx * h->grid.ny * h->grid.nz;
  if (dense) *dense = npx * (uint64_t)h->P * (uint64_t)h->E;
  if (in_win) {
    CK_H(h, cudaSetDevice(h->device));
    CK_H(h, cudaMemsetAsync(h->counter, 0, sizeof(unsigned long long), h->stream));
    CK_H(h, launch_tdbp(h, h->image, h->counter, 0, true, h->stream));
    unsigned long long v = 0;
    CK_H(h, cudaMemcpyAsync(&v, h->counter, sizeof(v), cudaMemcpyDeviceToHost, h->stream));
    CK_H(h, cudaStreamSynchronize(h->stream));
    *in_win = v;
  }
  return SAS_OK;
}

size_t sas_bp_workspace_bytes(sas_bp_t h) { return h ? h->bytes : 0; }

sas_status sas_bp_set_beam(sas_bp_t h, const sas_beam* beam, const double* axes, int32_t P) {
  g_err[0] = 0;
  if (!h) return fail(SAS_E_INVALID, "handle is NULL");
  if (h->broken) return fail(SAS_E_CUDA, "handle is in a failed CUDA state; destroy it");
  if (!beam) {   // back to the dense sum
    h->gate = 0;
    return SAS_OK;
  }
  const double pi = 3.141592653589793;
  if (!std::isfinite(beam->az_fwhm) || !(beam->az_fwhm > 0) || !std::isfinite(beam->el_fwhm))
    return fail(SAS_E_INVALID, "az_fwhm must be finite and > 0, el_fwhm finite");
  if (beam->bistatic != 0 && beam->bistatic != 1) return fail(SAS_E_INVALID, "bistatic must be 0 or 1");
  if (beam->cull != 0 && beam->cull != 1) return fail(SAS_E_INVALID, "cull must be 0 or 1");
  if (axes) {
    if (P < 1) return fail(SAS_E_INVALID, "P must be >= 1 when axes are given");
    for (int32_t p = 0; p < P; ++p) {
      const double* a = axes + 6 * (size_t)p;
      const double* b = a + 3;
      if (!finite3(a) || !finite3(b)) return fail(SAS_E_INVALID, "non-finite axes of ping %d", p);
      if (std::fabs(norm3(a) - 1.0) > 1e-6 || std::fabs(norm3(b) - 1.0) > 1e-6 ||
          std::fabs(a[0] * b[0] + a[1] * b[1] + a[2] * b[2]) > 1e-6)
        return fail(SAS_E_INVALID, "axes of ping %d must be orthonormal (a along track, b boresight)", p);
    }
    CK_H(h, cudaSetDevice(h->device));
    if (sas_status w = wait_idle(h); w != SAS_OK) return w;
    if (h->axes_P != P || !h->axes) {
      if (h->axes) { cudaFree(h->axes); h->bytes -= (size_t)h->axes_P * 6 * sizeof(double); h->axes = nullptr; }
      cudaError_t e = cudaMalloc(&h->axes, (size_t)P * 6 * sizeof(double));
      if (e != cudaSuccess) { h->axes = nullptr; h->axes_P = 0; h->gate = 0; return fail(SAS_E_NOMEM, "cudaMalloc(axes)"); }
      h->bytes += (size_t)P * 6 * sizeof(double);
    }
    CK_H(h, cudaMemcpy(h->axes, axes, (size_t)P * 6 * sizeof(double), cudaMemcpyHostToDevice));
    h->axes_P = P;
  } else if (h->axes) {
    if (sas_status w = wait_idle(h); w != SAS_OK) return w;
    cudaFree(h->axes);
    h->bytes -= (size_t)h->axes_P * 6 * sizeof(double);
    h->axes = nullptr;
    h->axes_P = 0;
  }
  h->az_on = beam->az_fwhm < pi ? 1 : 0;
  h->half_az = 0.5 * beam->az_fwhm;
  h->sin_half_az = std::sin(0.5 * beam->az_fwhm);   // same libm expression as the oracle's
  h->el_on = (beam->el_fwhm > 0 && beam->el_fwhm < pi) ? 1 : 0;
  h->half_el = 0.5 * beam->el_fwhm;
  h->tan_half_el = h->el_on ? std::tan(0.5 * beam->el_fwhm) : 0.0;
  h->cull = beam->cull;
  h->gate = beam->bistatic ? 2 : 1;
  return SAS_OK;
}

sas_status sas_bp_set_motion(sas_bp_t h, const double* vel, int32_t P) {
  g_err[0] = 0;
  if (!h) return fail(SAS_E_INVALID, "handle is NULL");
  if (h->broken) return fail(SAS_E_CUDA, "handle is in a failed CUDA state; destroy it");
  if (!vel) {   // stop-and-hop
    if (sas_status w = wait_idle(h); w != SAS_OK) return w;
    if (h->vel) { cudaFree(h->vel); h->bytes -= (size_t)h->vel_P * 3 * sizeof(double); }
    h->vel = nullptr; h->vel_P = 0;
    return SAS_OK;
  }
  if (P < 1) return fail(SAS_E_INVALID, "P must be >= 1");
  for (int32_t p = 0; p < P; ++p) {
    const double* v = vel + 3 * (size_t)p;
    if (!finite3(v)) return fail(SAS_E_INVALID, "non-finite velocity of ping %d", p);
    if (norm3(v) > 0.01 * h->c) return fail(SAS_E_INVALID, "velocity of ping %d exceeds c/100", p);
  }
  CK_H(h, cudaSetDevice(h->device));
  if (sas_status w = wait_idle(h); w != SAS_OK) return w;
  if (h->vel_P != P || !h->vel) {
    if (h->vel) { cudaFree(h->vel); h->bytes -= (size_t)h->vel_P * 3 * sizeof(double); h->vel = nullptr; }
    cudaError_t e = cudaMalloc(&h->vel, (size_t)P * 3 * sizeof(double));
    if (e != cudaSuccess) { h->vel = nullptr; h->vel_P = 0; return fail(SAS_E_NOMEM, "cudaMalloc(vel)"); }
    h->bytes += (size_t)P * 3 * sizeof(double);
  }
  CK_H(h, cudaMemcpy(h->vel, vel, (size_t)P * 3 * sizeof(double), cudaMemcpyHostToDevice));
  h->vel_P = P;
  if (h->nav) {   // one motion model at a time: velocities replace a receiver table
    cudaFree(h->nav);
    h->bytes -= (size_t)h->nav_P * h->nav_E * h->nav_K * 3 * sizeof(double);
    h->nav = nullptr; h->nav_P = h->nav_E = h->nav_K = 0; h->nav_dt = 0; h->nav_rmin = INFINITY;
  }
  return SAS_OK;
}

sas_status sas_bp_set_nav(sas_bp_t h, const double* lut, int32_t P, int32_t E, int32_t K, double dt) {
  g_err[0] = 0;
  if (!h) return fail(SAS_E_INVALID, "handle is NULL");
  if (h->broken) return fail(SAS_E_CUDA, "handle is in a failed CUDA state; destroy it");
  auto drop = [&]() {
    if (h->nav) { cudaFree(h->nav); h->bytes -= (size_t)h->nav_P * h->nav_E * h->nav_K * 3 * sizeof(double); }
    h->nav = nullptr; h->nav_P = h->nav_E = h->nav_K = 0; h->nav_dt = 0; h->nav_rmin = INFINITY;
  };
  if (!lut) {   // back to the ping set's fixed receivers (or velocities, if set)
    if (sas_status w = wait_idle(h); w != SAS_OK) return w;
    drop();
    return SAS_OK;
  }
  if (P < 1 || E < 1) return fail(SAS_E_INVALID, "P and E must be >= 1");
  if (K < 3 || K > 65536) return fail(SAS_E_INVALID, "K must be in 3..65536 (K = %d)", K);
  if (!(dt > 0) || !std::isfinite(dt)) return fail(SAS_E_INVALID, "dt must be finite and > 0");
  if ((double)P * E * K > 4.0e9) return fail(SAS_E_INVALID, "P*E*K too large");
  const size_t nch = (size_t)P * E;
  double lo[3], hi[3];
  grid_box(h, lo, hi);
  double rmin = INFINITY;
  for (size_t ch = 0; ch < nch; ++ch) {
    const double* L = lut + ch * (size_t)K * 3;
    for (int32_t k = 0; k < K; ++k) {
      if (!finite3(L + 3 * k)) return fail(SAS_E_INVALID, "non-finite table node %d of channel %zu", k, ch);
      rmin = std::fmin(rmin, dist_to_box(L + 3 * k, lo, hi));
      if (k > 0) {
        const double d[3] = {L[3 * k] - L[3 * k - 3], L[3 * k + 1] - L[3 * k - 2], L[3 * k + 2] - L[3 * k - 1]};
        if (norm3(d) > 0.01 * h->c * dt) return fail(SAS_E_INVALID, "channel %zu moves faster than c/100 between nodes %d and %d", ch, k - 1, k);
      }
    }
  }
  CK_H(h, cudaSetDevice(h->device));
  if (sas_status w = wait_idle(h); w != SAS_OK) return w;
  const size_t n = nch * (size_t)K * 3;
  if (!h->nav || (size_t)h->nav_P * h->nav_E * h->nav_K * 3 != n) {
    drop();
    cudaError_t e = cudaMalloc(&h->nav, n * sizeof(double));
    if (e != cudaSuccess) { h->nav = nullptr; return fail(SAS_E_NOMEM, "cudaMalloc(nav)"); }
    h->bytes += n * sizeof(double);
  }
  CK_H(h, cudaMemcpy(h->nav, lut, n * sizeof(double), cudaMemcpyHostToDevice));
  h->nav_P = P; h->nav_E = E; h->nav_K = K; h->nav_dt = dt; h->nav_rmin = rmin;
  if (h->vel) { cudaFree(h->vel); h->bytes -= (size_t)h->vel_P * 3 * sizeof(double); h->vel = nullptr; h->vel_P = 0; }
  return SAS_OK;
}

sas_status sas_bp_set_medium(sas_bp_t h, double zb, double c2) {
  g_err[0] = 0;
  if (!h) return fail(SAS_E_INVALID, "handle is NULL");
  if (!std::isfinite(zb) || !std::isfinite(c2)) return fail(SAS_E_INVALID, "zb and c2 must be finite");
  if (c2 <= 0) { h->refract = 0; return SAS_OK; }   // isovelocity (R9)
  const double Wn = std::ceil(2.0 * (2.0 * h->d_max * h->fs / std::min(h->c, c2)) + 4.0) + 3;
  if (smem_bytes((int)Wn) > 200 * 1024) return fail(SAS_E_UNSUPPORTED, "sediment speed too low for the tile window");
  h->refract = 1; h->zb = zb; h->c2 = c2;
  return SAS_OK;
}

sas_status sas_bp_set_weighting(sas_bp_t h, int32_t spreading) {
  g_err[0] = 0;
  if (!h) return fail(SAS_E_INVALID, "handle is NULL");
  if (spreading != 0 && spreading != 1) return fail(SAS_E_INVALID, "spreading must be 0 or 1");
  h->weight = spreading;
  return SAS_OK;
}

sas_status sas_bp_get_plan(sas_bp_t h, sas_bp_plan* out) {
  g_err[0] = 0;
  if (!h || !out) return fail(SAS_E_INVALID, "NULL argument");
  out->tile[0] = h->TX; out->tile[1] = h->TY; out->tile[2] = h->TZ;
  out->window = h->W;
  out->rx_mode = h->has_pings ? (h->refract ? 3 : rx_mode(h)) : -1;
  out->tma = h->has_pings ? (h->use_tma ? 1 : 0) : -1;
  out->batch = sasbp::kNB;
  out->ctas_per_sm = h->ctas_per_sm;
  out->tail_split = h->tail_split;
  return SAS_OK;
}

}  // extern "C"
