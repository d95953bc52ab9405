// tdbp_kernel.cuh -- the time-domain backprojection kernel (K2) and the in-window term counter
// (K3) for sm_100a.
//
// Computes, for every pixel of a CTA tile and every channel (ping p, element e), the term
//   ehat_{p,e}(u) * exp(+j 2 pi fc tau),  tau = (|x - tx_p| + |x - rx_{p,e}|)/c,  u = (tau - t0_p) fs
// of the inversion of Eq. (eqn:backprojection) ("integrate the time-series
// into the appropriate complex pixels") and accumulates it in registers.
//
// Design (DESIGN.md §4 "K2"):
//  * one CTA = one pixel tile (2D: 32x32, 3D: 16x8x8), 128 threads, K = 8 pixels per thread held
//    as 4 x-adjacent PAIRS so the per-pixel fp32 geometry runs on the sm_100 paired FP32 path
//    (FFMA2 / FADD2 / FMUL2: two lanes of math per issue slot); complex accumulators live in
//    registers across ALL channels; one image store per tile;
//  * channels are processed in batches of kNB.  Per batch a fp64 prologue (row a2) computes each
//    channel's tile-centre reference geometry: leg lengths, window start k_lo, the
//    window-relative reference index and the reference phase reduced mod 2 pi -- the ~1e5-rad
//    carrier phase never passes through fp32 (range-relative delays);
//  * software pipeline: while batch b is computed, batch b+1's prologue runs and its sample
//    windows stream global -> shared with cp.async (zero-filled outside 0..Ns-1, reading R2);
//    after a barrier each window is rewritten as (intercept, slope) float4 cells:
//      cell j: slope = d[k_lo+j+1] - d[k_lo+j], intercept = mid_j - (j - Wh) * slope
//    so the linear interpolation (row a4) at window coordinate U is one LDS.128 + one FFMA2:
//      ehat = intercept_j + U * slope_j,  j = rn(U) + Wh;
//  * per term (rows a3-a5): q = 2u.d + |d|^2; dU_rx = q h(q / r^2) with h the truncated series of
//    (sqrt(1+eps) - 1)/eps (3 or 4 terms by a plan-time error bound) or the exact form for
//    near-field plans; U = dU_tx + dU_rx + u_ref; j via the 1.5*2^23 rounding trick;
//    phase = U * 2 pi fc/fs + phi0 -> MUFU sin/cos; the complex MAC is 2 FFMA2 into
//    A += Re(ehat)(cos, sin), B += Im(ehat)(cos, sin); I = (A.x - B.y, A.y + B.x).
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#ifndef SASBP_FLAT_TRANSFORM
#define SASBP_FLAT_TRANSFORM 0
#endif
#ifndef SASBP_WY2D
#define SASBP_WY2D 4   // warps per 2D CTA (tile = 32 x 8*SASBP_WY2D pixels)
#endif

namespace sasbp {

#ifndef SASBP_MINB
#define SASBP_MINB 4   // resident 4-warp CTAs per SM the register allocation targets
#endif
#ifndef SASBP_MINB_AXIS
#define SASBP_MINB_AXIS 4   // the same for axis-aligned grids (A/B on config 4: 5 CTAs/SM -0.7 %)
#endif
#ifndef SASBP_MINB_3D
#define SASBP_MINB_3D 2   // 3D volume kernels (16 voxels per thread): 2 CTAs/SM, up to 255 registers
                          // (config 4 A/B: 16x8x16 tiles at 2 CTAs/SM 1431 Gterm/s, 16x8x12 at 3 1399,
                          // 16x8x8 at 4 1367; profiles/ab_r02.txt)
#endif
#ifndef SASBP_MINB_GATE
#define SASBP_MINB_GATE SASBP_MINB   // the same for the gated (NEXT-1) kernels
#endif
#ifndef SASBP_CUNROLL2
#define SASBP_CUNROLL2 0
#endif
#ifndef SASBP_CC_LDS
#define SASBP_CC_LDS 0   // A/B knob: channel constants via explicit ld.shared (see lds_struct)
#endif
#ifndef SASBP_AXIS_PAIRS
#define SASBP_AXIS_PAIRS 0   // A/B knob: AXIS kernels keep dy / dz per row as register pairs
#endif
#ifndef SASBP_GATE_SPLIT
#define SASBP_GATE_SPLIT 0   // A/B knob: gated kernels take the per-pixel mask selects only on edge channels
#endif
#ifndef SASBP_GATE_PREF
#define SASBP_GATE_PREF 0   // A/B knob: gated series kernels load the next channel's hot constants one channel ahead
#endif
#ifndef SASBP_GATE_PRED
// gated kernels: a gated-out pixel skips its two accumulate FFMA2s under a per-pixel predicate
// (0: it reads a zero cell instead, an address select of ~3 ALU instructions per pixel)
#define SASBP_GATE_PRED 0   // A/B on config 2: 135.3 ms (1) vs 123.0 ms (0): the predicated MUFUs cost more than the selects
#endif
#ifndef SASBP_GATE_NOINLINE
#define SASBP_GATE_NOINLINE 0   // A/B knob: the fp64 per-pixel cone tests of edge tiles as out-of-line calls
#endif
#ifndef SASBP_AXIS_SEPQ
#define SASBP_AXIS_SEPQ 1   // AXIS kernels form q = |d|^2 + 2u.d per axis (x pair + y row + z plane):
                            // 6 fewer FMA-pipe cycles per warp-channel on the 3D plan (A/B +0.6 %, profiles/ab_r02.txt)
#endif
#ifndef SASBP_AXIS2D
#define SASBP_AXIS2D 0       // A/B knob: instantiate / select the AXIS kernels for 2D planes as well
#endif
#ifndef SASBP_CC_PREFETCH
// dense series kernels on axis-aligned 3D grids: load the next channel's hot constants one channel
// ahead (A/B config 4: +1.6 %; the register-tighter 2D kernel lost 1.5 % with it)
#define SASBP_CC_PREFETCH 1
#endif
#ifndef SASBP_GRIDCONST
#define SASBP_GRIDCONST 1   // K2 params as __grid_constant__ (gate_mask() takes their address without a copy)
#endif
#if SASBP_GRIDCONST
#define SASBP_PRM_QUAL const __grid_constant__
#else
#define SASBP_PRM_QUAL const
#endif
#ifndef SASBP_KPH_PARAM
#define SASBP_KPH_PARAM 1   // 2 pi fc/fs and fs/c as host-computed floats (0: derived on the device)
#endif
#ifndef SASBP_TAILSPLIT
#define SASBP_TAILSPLIT 1   // wave-tail split support in K2 (0: kernel without it, host never splits; A/B)
#endif
#ifndef SASBP_XFORM_CURSOR
#define SASBP_XFORM_CURSOR 1   // window transform with per-lane cursors (0: indexed form, A/B)
#endif
#ifndef SASBP_XFORM_CURSOR_GATE
#define SASBP_XFORM_CURSOR_GATE 0   // A/B knob: the cursor form in the gated kernels too
#endif
#ifndef SASBP_LAZY_RANGE
#define SASBP_LAZY_RANGE 0   // A/B knob: the CTA tile / channel range re-derived at each use (raised the 3D kernel 123 -> 128 registers)
#endif
#ifndef SASBP_XFORM_CURSOR_GIN
#define SASBP_XFORM_CURSOR_GIN 0   // A/B knob: the cursor form in the mask-free gated (GIN) kernels
#endif
#ifndef SASBP_DIV_MULHI
#define SASBP_DIV_MULHI 1
#endif
#ifndef SASBP_TX_SERIES
#define SASBP_TX_SERIES 1   // series plans evaluate the transmit leg with the same series (no MUFU)
#endif
#ifndef SASBP_BININDEX
// 1: the window cell index comes from the exponent-aligned window coordinate V = u - k_lo + 2^kb
//    by integer ops (SHF + LOP3 + IADD3 on the ALU pipe); the phase and the lerp use the small
//    tile-relative delay U' directly.  0: the original magic-number rounding (FADD2 + IMAD on the
//    FMA pipe).  Both compute the same sum; A/B on config 2: 1271 (1) vs 1328 (0) Gterm/s, so 0 is
//    the default (moving the index off the FMA pipe does not help: MUFU / latency bound).
#define SASBP_BININDEX 0
#endif
#ifndef SASBP_TILE_GROUP
#define SASBP_TILE_GROUP 8   // tiles per side of the square groups the launch order walks
#endif
#ifndef SASBP_NB
#define SASBP_NB 16
#endif
constexpr int kNB = SASBP_NB;   // channels per batch

// receive-leg evaluation modes
constexpr int kSeries3 = 0;     // 3-term series in eps
constexpr int kSeries4 = 1;     // 4-term series in eps
constexpr int kExact = 2;       // q / (sqrt(r^2 + q) + r)
constexpr int kRefract = 3;     // Fermat path through a flat sediment interface (NEXT-3), per-term Newton

struct TdbpParams {
  const float2* echoes;   // [P*E][Ns]
  const double* tx;       // [P][3]
  const double* rx;       // [P*E][3]
  const double* t0;       // [P]
  float2* image;          // [nz][ny][nx]
  unsigned long long* counter;  // K3: in-window term total
  double origin[3], sx[3], sy[3], sz[3];
  double fc, fs, c;
  double k_s;             // fs / c   (samples per metre of path)
  double k_c;             // fc / c   (carrier cycles per metre of path)
  double k_r;             // fc / fs  (carrier cycles per sample)
  double inv_e;           // 1 / E
  float kph_f;            // (float)(2 pi k_r): radians of carrier phase per sample (host-computed, so
                          // the kernel never re-derives it in fp64 under register pressure)
  float kfs_f;            // (float)k_s
  double hw;              // half window in samples: 2 * d_max * fs / c
  int P, E, Ns;
  int nx, ny, nz;
  int tiles_x, tiles_y, tiles_z;
  int W;                  // window cells per channel (cells j = 0..W-1 use samples k_lo+j, k_lo+j+1)
  int accumulate;
  int ch_lo, ch_hi;       // channel range [ch_lo, ch_hi) of this launch (ch = p * E + e)
  int resident;           // co-resident CTAs of the launch (SMs x CTAs/SM) for the channel rotation
  // wave-tail split: tiles [tail0, ntiles) are launched tsplit (= 2) times, each CTA summing half of
  // the channels and adding its partial image with an atomic float2 add into a zeroed image (0 + a + b
  // = 0 + b + a exactly: still deterministic); tsplit = 1 -> one CTA per tile
  int tail0, tsplit;
  // field-of-view gating (NEXT-1, reading R15); gate = 0 -> dense sum
  int gate;               // 1 = gate at tx; 2 = gate at tx and at each rx (bistatic)
  int cull;               // skip (tile, channel) pairs whose tile sphere misses a cone
  int gpart;              // two-launch gated form: 0 = every class, 1 = only (tile, channel) pairs
                          // wholly inside the cone(s), 2 = only the others (edge / unculled out)
  int az_on, el_on;
  const double* axes;     // [P][2][3] per-ping along-track axis a, boresight b; NULL = (+x, +y)
  double sin_half_az, half_az, tan_half_el, half_el;
  double d_max;           // tile sphere radius (m)
  // continuous receiver motion (NEXT-2, reading R16): per-ping velocity [P][3] or NULL
  const double* vel;
  // tabled receiver trajectories (NEXT-2, reading R23): [P*E][nav_k][3] positions nav_dt apart
  // from the transmit, or NULL (vel and nav are never both set)
  const double* nav;
  int nav_k;
  double nav_dt;
  // sediment-water interface (NEXT-3, reading R17): z = zb, sediment speed c2 (refract != 0)
  int refract;
  double zb, c2;
  int mode;               // receive-leg mode of the plan (kSeries3 / kSeries4 / kExact / kRefract)
};

// per-channel constants in shared memory (fp64 prologue output)
struct __align__(16) ChanConst {
  float ux2, uy2, uz2, kap0;    // rx leg: 2 (c_T - rx'); moving receiver scale (1 for stop-and-hop)
  float a0, a1, a2, a3;         // rx leg series in q: dU = q (a0 + a1 q + a2 q^2 + a3 q^3), see prologue
  float urr, phi0, r_r, r2_r;   // centred window coordinate offset; phase offset (rad); r_r; r_r^2
  float tx2x, tx2y, tx2z, r2_t; // tx leg: 2 (c_T - tx), r_t^2
  float r_t, kgx, kgy, kgz;     // r_t; moving receiver: U = dU (kap0 + kg.d) + urr (kg = 0 stop-and-hop)
  int ping, woff, klo, gate;    // ping index; LDS byte offset of cell Wh minus MAGIC*16; window start;
                                // gate classes: bits 0-1 tx, 2-3 rx (kGIn/kGEdge/kGOut), bit 4 = culled
};

constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23: x + kMagic rounds x to an integer in the low bits
constexpr int kMagicBits = 0x4B400000;

__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ float2 lds64(uint32_t addr) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
  return v;
}
// ChanConst read through a 32-bit shared-window address (ld.shared): a generic pointer into dynamic
// shared memory makes ptxas rematerialise its base with S2R SR_CgaCtaId inside the channel loop
// under register pressure
template <typename T>
__device__ __forceinline__ T lds_struct(uint32_t addr) {
  static_assert(sizeof(T) % 16 == 0, "16-byte multiple");
  T v;
  float4* p = reinterpret_cast<float4*>(&v);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(T) / 16); ++i) p[i] = lds128(addr + 16u * i);
  return v;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rsqrt_approx(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// Denominator sqrt(r^2 + q) + r of dR = q / (sqrt(r^2 + q) + r), safe when the pixel coincides
// with the sensor: r^2 + q (which can round to 0 or slightly below there) is floored at 1e-30, so
// sqrt = x rsqrt(x) >= 1e-15 > 0 and no 0 * inf or negative root arises (dR stays bounded by the
// window; q / den -> 0 when the tile centre is on the sensor as well)
__device__ __forceinline__ float leg_den(float r2, float r) {
  const float r2c = fmaxf(r2, 1e-30f);
  return fmaf(r2c, rsqrt_approx(r2c), r);
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src, bool valid) {
  // 8-byte global -> shared copy; src-size 0 writes zeros (zero extension, reading R2)
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }

// ---------------------------------------------------------------- refraction (NEXT-3, R17)
// One-way Fermat time through the interface, fp64 (prologue reference): same definition as the
// test-side reference, Newton from the straight-line crossing with bisection-style safeguards.
__device__ inline double refr_time64(const double x[3], const double s[3], double zb, double c1, double c2) {
  const double h2 = x[2] - zb;
  const double dx = x[0] - s[0], dy = x[1] - s[1];
  if (h2 <= 0.0) return sqrt(dx * dx + dy * dy + (x[2] - s[2]) * (x[2] - s[2])) / c1;
  const double h1 = zb - s[2];
  const double D = sqrt(dx * dx + dy * dy);
  double xi = D * h1 / (h1 + h2);
  for (int it = 0; it < 60; ++it) {
    const double L1 = sqrt(xi * xi + h1 * h1), L2 = sqrt((D - xi) * (D - xi) + h2 * h2);
    const double f1 = xi / (c1 * L1) - (D - xi) / (c2 * L2);
    const double f2 = h1 * h1 / (c1 * L1 * L1 * L1) + h2 * h2 / (c2 * L2 * L2 * L2);
    double nx = xi - f1 / f2;
    if (nx < 0.0) nx = 0.5 * xi;
    if (nx > D) nx = 0.5 * (xi + D);
    const double st = fabs(nx - xi);
    xi = nx;
    if (st <= 1e-14 * (D + h1 + h2)) break;
  }
  return sqrt(xi * xi + h1 * h1) / c1 + sqrt((D - xi) * (D - xi) + h2 * h2) / c2;
}

// Per-term fp32 version in SAMPLES (k1 = fs/c1, k2 = fs/c2), tile-relative coordinates: voxel
// offset e = d - s from the sensor, depth below the interface h2 = d_z - zbr, sensor height above
// it h1 = zbr - s_z.  Newton on the convex objective (3 steps from the straight-line crossing,
// each clamped to [0, D]); the time is stationary at the minimum, so the residual refraction-
// point error enters only at second order.
__device__ __forceinline__ float refr_time32(float ex, float ey, float ez, float h1, float h2, float k1, float k2) {
  if (h2 <= 0.f) return sqrtf(fmaf(ex, ex, fmaf(ey, ey, ez * ez))) * k1;
  const float D = sqrtf(fmaf(ex, ex, ey * ey));
  float xi = D * h1 * rcp_approx(h1 + h2);
#pragma unroll
  for (int it = 0; it < 3; ++it) {
    const float a = xi, b = D - xi;
    const float i1 = rsqrt_approx(fmaf(a, a, h1 * h1)), i2 = rsqrt_approx(fmaf(b, b, h2 * h2));
    const float f1 = a * k1 * i1 - b * k2 * i2;
    const float f2 = h1 * h1 * k1 * i1 * i1 * i1 + h2 * h2 * k2 * i2 * i2 * i2;
    xi = fminf(fmaxf(xi - f1 * rcp_approx(f2), 0.f), D);
  }
  const float a = xi, b = D - xi;
  return sqrtf(fmaf(a, a, h1 * h1)) * k1 + sqrtf(fmaf(b, b, h2 * h2)) * k2;
}

// ---------------------------------------------------------------- FOV gate (NEXT-1, R15)
constexpr int kGIn = 0, kGEdge = 1, kGOut = 2;

__device__ __forceinline__ void ping_axes(const TdbpParams& prm, int p, double a[3], double b[3]) {
  if (prm.axes) {
#pragma unroll
    for (int i = 0; i < 3; ++i) { a[i] = prm.axes[6 * p + i]; b[i] = prm.axes[6 * p + 3 + i]; }
  } else {
    a[0] = 1.0; a[1] = 0.0; a[2] = 0.0; b[0] = 0.0; b[1] = 1.0; b[2] = 0.0;
  }
}

// Classify a whole tile (sphere of radius d_max around its centre, v = centre - sensor) against
// one sensor's cone: kGIn (every point inside), kGOut (every point outside) or kGEdge.  Exact
// spherical bounds: the angle to the plane perpendicular to a ranges over alpha -/+ beta; the
// elevation condition depends only on the projection onto span(b, c), a disk of radius d_max.
__device__ inline int cone_class(const TdbpParams& prm, const double v[3], const double a[3], const double b[3]) {
  const double rho = prm.d_max, eps = 1e-9;
  const double nv = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
  if (!(nv > rho)) return kGEdge;
  int cls = kGIn;
  if (prm.az_on) {
    const double beta = asin(rho / nv);
    const double alpha = asin(fmin(1.0, fabs(v[0] * a[0] + v[1] * a[1] + v[2] * a[2]) / nv));
    if (alpha - beta > prm.half_az + eps) return kGOut;
    if (!(alpha + beta < prm.half_az - eps)) cls = kGEdge;
  }
  if (prm.el_on) {
    const double c[3] = {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
    const double vb = v[0] * b[0] + v[1] * b[1] + v[2] * b[2];
    const double vc = v[0] * c[0] + v[1] * c[1] + v[2] * c[2];
    const double rp = sqrt(vb * vb + vc * vc);
    if (!(rp > rho)) return kGEdge;
    const double be = asin(rho / rp), el = atan2(fabs(vc), vb);
    if (el - be > prm.half_el + eps) return kGOut;
    if (!(el + be < prm.half_el - eps)) cls = kGEdge;
  }
  return cls;
}

// Per-point test, evaluated in fp64 in the definition's order of operations (no contraction),
// so the decision is the plain fp64 one the test-side reference takes (R15).
__device__ inline bool in_fov_px(const TdbpParams& prm, const double x[3], const double* s, const double a[3],
                          const double b[3]) {
  const double v0 = __dsub_rn(x[0], s[0]), v1 = __dsub_rn(x[1], s[1]), v2 = __dsub_rn(x[2], s[2]);
  if (prm.az_on) {
    const double nv = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(v0, v0), __dmul_rn(v1, v1)), __dmul_rn(v2, v2)));
    const double va = __dadd_rn(__dadd_rn(__dmul_rn(v0, a[0]), __dmul_rn(v1, a[1])), __dmul_rn(v2, a[2]));
    if (fabs(va) > __dmul_rn(nv, prm.sin_half_az)) return false;
  }
  if (prm.el_on) {
    const double c0 = __dsub_rn(__dmul_rn(a[1], b[2]), __dmul_rn(a[2], b[1]));
    const double c1 = __dsub_rn(__dmul_rn(a[2], b[0]), __dmul_rn(a[0], b[2]));
    const double c2 = __dsub_rn(__dmul_rn(a[0], b[1]), __dmul_rn(a[1], b[0]));
    const double vb = __dadd_rn(__dadd_rn(__dmul_rn(v0, b[0]), __dmul_rn(v1, b[1])), __dmul_rn(v2, b[2]));
    const double vc = __dadd_rn(__dadd_rn(__dmul_rn(v0, c0), __dmul_rn(v1, c1)), __dmul_rn(v2, c2));
    if (!(vb > 0) || fabs(vc) > __dmul_rn(vb, prm.tan_half_el)) return false;
  }
  return true;
}

// Pixel centre in fp64, oracle order: ((origin + ix sx) + iy sy) + iz sz (reading R8)
__device__ __forceinline__ void pixel_centre64(const TdbpParams& prm, int ix, int iy, int iz, double x[3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
    x[i] = __dadd_rn(__dadd_rn(__dadd_rn(prm.origin[i], __dmul_rn((double)ix, prm.sx[i])),
                               __dmul_rn((double)iy, prm.sy[i])),
                     __dmul_rn((double)iz, prm.sz[i]));
}

// Receiver position r and velocity v at time t on a channel's tabled trajectory L [K][3] (R23;
// the paper's position LUT): the cubic Hermite spline through the nodes (dt apart) with
// central-difference tangents inside and second-order one-sided tangents at the two ends, the
// first / last segment's cubic continued outside the table.
__device__ __forceinline__ void nav_pv(const double* __restrict__ L, int K, double dt, double t, double r[3],
                                       double v[3]) {
  double s = t / dt;
  const int k = (int)fmin(fmax(floor(s), 0.0), (double)(K - 2));
  s -= (double)k;
  const double s2 = s * s, s3 = s2 * s;
  const double h00 = 2.0 * s3 - 3.0 * s2 + 1.0, h10 = s3 - 2.0 * s2 + s, h01 = 3.0 * s2 - 2.0 * s3, h11 = s3 - s2;
  const double g00 = 6.0 * s2 - 6.0 * s, g10 = 3.0 * s2 - 4.0 * s + 1.0, g11 = 3.0 * s2 - 2.0 * s;
  const double* a = L + 3 * k;   // node k; node k + 1 at a + 3
  for (int i = 0; i < 3; ++i) {
    const double p0 = a[i], p1 = a[3 + i];
    // dt * tangent at nodes k and k + 1
    const double m0 = k == 0 ? 0.5 * (4.0 * p1 - 3.0 * p0 - a[6 + i]) : 0.5 * (p1 - a[i - 3]);
    const double m1 = k + 1 == K - 1 ? 0.5 * (3.0 * p1 - 4.0 * p0 + a[i - 3]) : 0.5 * (a[6 + i] - p0);
    r[i] = h00 * p0 + h10 * m0 + h01 * p1 + h11 * m1;
    v[i] = (g00 * (p0 - p1) + g10 * m0 + g11 * m1) / dt;
  }
}

// fp64 prologue for one channel (row a2): reference geometry at the tile centre ct (and, for
// gated kernels, the tile's cone classes).
template <bool GATE, bool MOTION = false, bool REFRACT = false>
__device__ __forceinline__ ChanConst chan_prologue(const TdbpParams& prm, int ch, const double ct[3], int slot,
                                                   uint32_t win_base) {
  const int p = (int)(((double)ch + 0.5) * prm.inv_e);   // ch / E, exact for ch < 2^40
  const double* T = prm.tx + 3 * p;
  const double* R = prm.rx + 3 * (size_t)ch;
  const double utx = ct[0] - T[0], uty = ct[1] - T[1], utz = ct[2] - T[2];
  const double urx = ct[0] - R[0], ury = ct[1] - R[1], urz = ct[2] - R[2];
  int gate_bits = 0;
  if (GATE && prm.gate) {   // cone classes of the tile first: a culled channel needs nothing else
    double a[3], b[3];
    ping_axes(prm, p, a, b);
    const double vt[3] = {utx, uty, utz};
    const int ct_cls = cone_class(prm, vt, a, b);
    int cr_cls = kGIn;
    if (prm.gate == 2 && !(prm.cull && ct_cls == kGOut)) {
      const double vr[3] = {urx, ury, urz};
      cr_cls = cone_class(prm, vr, a, b);
    }
    if (prm.cull && (ct_cls == kGOut || cr_cls == kGOut)) {
      ChanConst k{};
      k.ping = p;
      k.gate = 16;
      return k;
    }
    const bool in_all = ct_cls == kGIn && cr_cls == kGIn;
    if ((prm.gpart == 1 && !in_all) || (prm.gpart == 2 && in_all)) {   // the other launch's share
      ChanConst k{};
      k.ping = p;
      k.gate = 16;
      return k;
    }
    // without culling an OUT class is evaluated per pixel like an edge
    gate_bits = (ct_cls == kGOut ? kGEdge : ct_cls) | ((cr_cls == kGOut ? kGEdge : cr_cls) << 2);
  }
  const double r_t = sqrt(utx * utx + uty * uty + utz * utz);
  double urx_m = urx, ury_m = ury, urz_m = urz;   // centre minus the receiver at its reception time
  double r_r = sqrt(urx * urx + ury * ury + urz * urz);
  double kap0 = 1.0, kg[3] = {0.0, 0.0, 0.0};
  if (MOTION && (prm.vel || prm.nav)) {
    // reference delay with the receiver moving at v during reception: c tau = r_t + |c_T - rx - v tau|
    // (fixed point from stop-and-hop, contraction |v|/c); the rx leg below is then taken w.r.t.
    // rx' = rx + v tau_ref, and per pixel tau - tau_ref = (dR_t + dR_r') / (c + w.v), w = unit(x - rx'),
    // i.e. U = dU / (1 + g), g = w.v / c = g0 + g1.d to first order in the pixel offset d.
    // Tabled trajectories (R23): c tau = r_t + |c_T - r(tau)| from r(0), then rx' = r(tau_ref) and
    // v = r'(tau_ref): over one tile's delay spread the trajectory is its tangent line (the neglected
    // |r''| dtau^2 / 2 is ~1e-7 m for 1 m/s^2 over 0.5 ms).
    double V[3];
    if (prm.nav) {
      const double* L = prm.nav + (size_t)ch * (size_t)prm.nav_k * 3;
      double rp[3];
      nav_pv(L, prm.nav_k, prm.nav_dt, 0.0, rp, V);
      urx_m = ct[0] - rp[0]; ury_m = ct[1] - rp[1]; urz_m = ct[2] - rp[2];
      r_r = sqrt(urx_m * urx_m + ury_m * ury_m + urz_m * urz_m);
      double tau = (r_t + r_r) / prm.c;
      for (int it = 0; it < 8; ++it) {
        nav_pv(L, prm.nav_k, prm.nav_dt, tau, rp, V);
        urx_m = ct[0] - rp[0]; ury_m = ct[1] - rp[1]; urz_m = ct[2] - rp[2];
        r_r = sqrt(urx_m * urx_m + ury_m * ury_m + urz_m * urz_m);
        tau = (r_t + r_r) / prm.c;
      }
    } else {
      V[0] = prm.vel[3 * p]; V[1] = prm.vel[3 * p + 1]; V[2] = prm.vel[3 * p + 2];
      double tau = (r_t + r_r) / prm.c;
      for (int it = 0; it < 6; ++it) {
        urx_m = urx - V[0] * tau; ury_m = ury - V[1] * tau; urz_m = urz - V[2] * tau;
        r_r = sqrt(urx_m * urx_m + ury_m * ury_m + urz_m * urz_m);
        tau = (r_t + r_r) / prm.c;
      }
    }
    if (prm.mode == kExact) {
      // near-field plans: the kernel evaluates kappa = |x - rx'| / (|x - rx'| + (u + d).v / c) exactly
      // per pixel (the first-order expansion below is only accurate for |d| << R); pass (u.v)/c, v/c
      kap0 = (urx_m * V[0] + ury_m * V[1] + urz_m * V[2]) / prm.c;
      kg[0] = V[0] / prm.c; kg[1] = V[1] / prm.c; kg[2] = V[2] / prm.c;
    } else if (r_r > 1e-9) {   // (a receiver exactly at the tile centre keeps kappa = 1: no direction defined)
      const double ux = urx_m / r_r, uy = ury_m / r_r, uz = urz_m / r_r;
      const double uv = ux * V[0] + uy * V[1] + uz * V[2];
      kap0 = 1.0 / (1.0 + uv / prm.c);
      const double s1 = -kap0 * kap0 / (prm.c * r_r);   // d kappa = -kap0^2 g1.d, g1 = (v - (u.v) u) / (c r)
      kg[0] = s1 * (V[0] - uv * ux); kg[1] = s1 * (V[1] - uv * uy); kg[2] = s1 * (V[2] - uv * uz);
    }
  }
  double S = r_t + r_r;
  double At = 0.0, Ar = 0.0;   // refraction: reference one-way times in samples
  if (REFRACT) {
    const double ctr[3] = {ct[0], ct[1], ct[2]};
    const double tt = refr_time64(ctr, T, prm.zb, prm.c, prm.c2);
    const double tr = refr_time64(ctr, R, prm.zb, prm.c, prm.c2);
    S = prm.c * (tt + tr);          // c tau_ref: Uref and the reference phase below follow
    At = tt * prm.fs; Ar = tr * prm.fs;
  }
  const double Uref = fma(S, prm.k_s, -prm.t0[p] * prm.fs);   // absolute sample index at tile centre
  const double klo_d = floor(Uref - prm.hw) - 2.0;
  // even window start: a TMA box must start 16-B aligned (2 samples); the plan's W has one
  // spare cell for this
  const int klo = ((int)fmax(fmin(klo_d, 2.0e9), -2.0e9)) & ~1;
  const int Wh = prm.W >> 1;
  // window coordinate U = u - k_lo - 0.5 - Wh, so cell j = rn(U) + Wh
  const double urr = Uref - (double)(klo + Wh) - 0.5;
#if SASBP_BININDEX
  double ph = S * prm.k_c;                                    // reference phase (cycles) at U' = 0 (tau = tau_ref)
#else
  double ph = fma(-urr, prm.k_r, S * prm.k_c);                // reference phase (cycles) at U = 0
#endif
  ph -= floor(ph);
  ChanConst k;
  k.ux2 = (float)(2.0 * urx_m); k.uy2 = (float)(2.0 * ury_m); k.uz2 = (float)(2.0 * urz_m);
  k.kap0 = (float)kap0; k.kgx = (float)kg[0]; k.kgy = (float)kg[1]; k.kgz = (float)kg[2];
  // series coefficients only need fp32 relative accuracy
  const float ir = 1.0f / (float)r_r;
  const float ir2 = ir * ir;
  // (sqrt(1+e)-1)/e = 1/2 - e/8 + e^2/16 - 5e^3/128 + ..., e = q / r^2; folded into a polynomial
  // in q so the kernel needs no e = q / r^2 multiply: a_n = c_n (fs/c) / r^(2n+1)
  const float g = (float)prm.k_s * ir;
  k.a0 = 0.5f * g; k.a1 = -0.125f * g * ir2; k.a2 = 0.0625f * g * ir2 * ir2; k.a3 = -0.0390625f * g * ir2 * ir2 * ir2;
  k.urr = (float)urr;
  k.phi0 = (float)(6.283185307179586 * ph);
  k.r_r = (float)r_r; k.r2_r = (float)(r_r * r_r);
  k.tx2x = (float)(2.0 * utx); k.tx2y = (float)(2.0 * uty); k.tx2z = (float)(2.0 * utz);
  k.r2_t = (float)(r_t * r_t); k.r_t = (float)r_t;
  if (REFRACT) {   // sensor positions relative to the tile centre and reference times (samples)
    k.ux2 = (float)(R[0] - ct[0]); k.uy2 = (float)(R[1] - ct[1]); k.uz2 = (float)(R[2] - ct[2]);
    k.tx2x = (float)(T[0] - ct[0]); k.tx2y = (float)(T[1] - ct[1]); k.tx2z = (float)(T[2] - ct[2]);
    k.a1 = (float)Ar; k.r_t = (float)At;
  }
  k.ping = p;
#if SASBP_BININDEX
  k.woff = (int)(win_base + (uint32_t)(slot * prm.W) * 16u);   // cell 0 of this channel's window
#else
  k.woff = (int)(win_base + (uint32_t)(slot * prm.W + Wh) * 16u - (uint32_t)kMagicBits * 16u);
#endif
  k.klo = klo;
  k.gate = gate_bits;
  return k;
}

// tile bookkeeping shared by K2 and K3
template <int KX, int KY, int KZ, int WY, int WZ>
struct TileMap {
  static constexpr int K = KX * KY * KZ;
  static constexpr int NP = K / 2;  // x-adjacent pixel pairs per thread
  static constexpr int TX = 8 * KX, TY = 4 * KY * WY, TZ = KZ * WZ;
  int x0, y0, z0, lx, ly, wy, wz;
  __device__ TileMap(const TdbpParams& prm, int tile = -1) {
    if (tile < 0) tile = (int)blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    lx = lane >> 2; ly = lane & 3;          // quarter-warp = 4 (y) x 2 (x) pixel patch
    wy = warp % WY; wz = warp / WY;
    // Tile order: square groups of G x G tiles (row-major inside a group, groups row-major)
    // so the CTAs resident at one time cover a compact patch of the image; their windows
    // of a channel then overlap and a channel comes from DRAM once per wave (L2 reuse).
    const int nxy = prm.tiles_x * prm.tiles_y;
    const int b = tile % nxy, bz = tile / nxy;
    constexpr int G = SASBP_TILE_GROUP;
    const int sr = b / (G * prm.tiles_x);                       // super-row of G tile rows
    const int gh = min(G, prm.tiles_y - sr * G);
    const int r = b - sr * G * prm.tiles_x;
    const int gi = r / (G * gh);                                 // group (G columns) in the super-row
    const int gw = min(G, prm.tiles_x - gi * G);
    const int rr = r - gi * G * gh;
    const int tix = gi * G + rr % gw, tiy = sr * G + rr / gw;
    x0 = tix * TX; y0 = tiy * TY; z0 = bz * TZ;
  }
  // pixel k = ((kz * KY + ky) * KX + kx); pairs are (kx even, kx odd)
  __device__ int ix(int k) const { return x0 + lx + 8 * (k % KX); }
  __device__ int iy(int k) const { return y0 + ly + 4 * ((k / KX) % KY) + 4 * KY * wy; }
  __device__ int iz(int k) const { return z0 + (k / (KX * KY)) + KZ * wz; }
  __device__ void centre(const TdbpParams& prm, double ct[3]) const {
    const double cxr = x0 + 0.5 * (TX - 1), cyr = y0 + 0.5 * (TY - 1), czr = z0 + 0.5 * (TZ - 1);
#pragma unroll
    for (int a = 0; a < 3; ++a) ct[a] = prm.origin[a] + cxr * prm.sx[a] + cyr * prm.sy[a] + czr * prm.sz[a];
  }
  __device__ void offset(const TdbpParams& prm, int k, float& dx, float& dy, float& dz) const {
    const float rxi = (float)(ix(k) - x0) - 0.5f * (TX - 1);
    const float ryi = (float)(iy(k) - y0) - 0.5f * (TY - 1);
    const float rzi = (float)(iz(k) - z0) - 0.5f * (TZ - 1);
    dx = rxi * (float)prm.sx[0] + ryi * (float)prm.sy[0] + rzi * (float)prm.sz[0];
    dy = rxi * (float)prm.sx[1] + ryi * (float)prm.sy[1] + rzi * (float)prm.sz[1];
    dz = rxi * (float)prm.sx[2] + ryi * (float)prm.sy[2] + rzi * (float)prm.sz[2];
  }
  __device__ bool valid(const TdbpParams& prm, int k) const {
    return ix(k) < prm.nx && iy(k) < prm.ny && iz(k) < prm.nz;
  }
};

// shared-memory layout of K2 (bytes):
//   cc[2][kNB] ChanConst | mbarrier (16 B) | raw[kNB] slots of RS bytes (128-B aligned, TMA
//   destinations) | win[kNB][W] float4 (intercept, slope) cells
__host__ __device__ inline int box_samples(int W) { return (W + 1 + 1) & ~1; }      // even => 16-B rows
__host__ __device__ inline size_t raw_slot_bytes(int W) { return ((size_t)box_samples(W) * 8 + 127) & ~(size_t)127; }
#ifndef SASBP_BPW
#define SASBP_BPW 2   // batches per warp in one prologue group (lanes = BPW * kNB <= 32)
#endif
constexpr int kBPW = SASBP_BPW;
static_assert(kBPW * kNB <= 32, "one prologue group runs kBPW batches of kNB channels on the 32 lanes of a warp");
constexpr int kRing = 8 * kBPW;   // ChanConst batches kept in shared memory (prologues run ahead)
// after the ring: mbarrier (8 B, +8 pad), zero cell (16 B), per-slot batch-live flags (kRing ints)
__host__ __device__ inline size_t k2_raw_off() {
  return (kRing * kNB * sizeof(ChanConst) + 32 + kRing * 4 + 127) & ~(size_t)127;
}
__host__ __device__ inline size_t k2_win_off(int W) { return k2_raw_off() + kNB * raw_slot_bytes(W); }
__host__ __device__ inline size_t k2_smem_bytes(int W) { return k2_win_off(W) + (size_t)kNB * W * sizeof(float4) + 128; }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
  return ok != 0;
}
// Wait for a batch's TMA transaction.  A transaction that never completes (a byte count that does
// not match what was issued) is a bug: trap -- the launch fails with an error -- instead of
// spinning forever (each try_wait already suspends for a hardware time slice).
#ifndef SASBP_MBAR_TRAP
#define SASBP_MBAR_TRAP 0   // debug option: trap instead of spinning on a transaction that never completes (costs 3 % on 3D plans)
#endif
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
#if SASBP_MBAR_TRAP
  // the poll loop stays in PTX (a C++ loop around try_wait cost 3 % on the 3D plan); the counter
  // only runs while the transaction is incomplete
  asm volatile(
      "{\n .reg .pred p, q;\n .reg .u32 n;\n"
      " mov.u32 n, 0;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @p bra DONE_%=;\n"
      " add.u32 n, n, 1;\n"
      " setp.lt.u32 q, n, 4194304;\n"
      " @q bra WAIT_%=;\n"
      " trap;\n"
      "DONE_%=:\n}\n" ::"r"(bar), "r"(parity) : "memory");
#else
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(bar), "r"(parity) : "memory");
#endif
}
__device__ __forceinline__ void tma_load_row(uint32_t dst, const void* tmap, int x, int y, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(dst), "l"(tmap), "r"(x), "r"(y), "r"(bar) : "memory");
}

// TMA descriptor of the echo array seen as a 2D tensor of 8-byte samples [P*E][Ns] (inner dim
// Ns); box = box_samples(W) x 1; out-of-bounds samples read as zero (reading R2).
struct __align__(64) TmaDesc { unsigned char bytes[128]; };

// Per-pixel fp64 cone masks of one thread's pixels (edge tiles only).  Out of line under
// SASBP_GATE_NOINLINE: the fp64 temporaries then never compete with the pixel loop's registers
// (the call saves what is live around it, once per edge ping / channel).
#if SASBP_GATE_NOINLINE
#define SASBP_MASK_FN __device__ __noinline__
#else
#define SASBP_MASK_FN __device__ __forceinline__
#endif
template <class TM, int NPIX>
SASBP_MASK_FN uint32_t gate_mask(const TdbpParams* prm, const TM tm, int ping, const double* sensor, uint32_t in) {
  double a[3], bb[3], x[3];
  ping_axes(*prm, ping, a, bb);
  uint32_t m = in;
#pragma unroll
  for (int k = 0; k < NPIX; ++k) {
    pixel_centre64(*prm, tm.ix(k), tm.iy(k), tm.iz(k), x);
    if (!in_fov_px(*prm, x, sensor, a, bb)) m &= ~(1u << k);
  }
  return m;
}

// HAS_DZ = false means the grid is a z-level plane (step_x, step_y have no z component).  AXIS =
// true for grids with diagonal steps (each step along its own axis): the pixel offsets are kept
// per column / row / plane instead of per pixel pair (fewer registers, same arithmetic).
// WEIGHT = true multiplies every term by the spreading weight R_tx R_rx (NEXT-4, reading R18).
// GIN = true (gated kernels, prm.gpart = 1): only (tile, channel) pairs wholly inside the cone(s)
// reach the pixel loop, so it carries no per-pixel gate masks (the dense kernel's loop).
template <int KX, int KY, int KZ, int WY, int WZ, bool HAS_DZ, int MODE, bool USE_TMA, bool GATE = false,
          bool MOTION = false, bool AXIS = false, bool WEIGHT = false, bool GIN = false>
__global__ void __launch_bounds__(32 * WY * WZ, (KZ > 1 ? SASBP_MINB_3D : GATE ? SASBP_MINB_GATE : AXIS ? SASBP_MINB_AXIS : SASBP_MINB) * 4 / (WY * WZ))
    tdbp_kernel(SASBP_PRM_QUAL TdbpParams prm,
                                                                          const __grid_constant__ TmaDesc tmap) {
  using TM = TileMap<KX, KY, KZ, WY, WZ>;
  constexpr int NP = TM::NP;
  constexpr int kWarps = WY * WZ;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // the dynamic smem base is only guaranteed 16-B aligned: align it to 128 B ourselves
  unsigned char* sbase = smem_raw + ((128 - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 127)) & 127);
  ChanConst* cc = reinterpret_cast<ChanConst*>(sbase);                       // [kRing][kNB]
  const uint32_t bar = (uint32_t)__cvta_generic_to_shared(sbase + kRing * kNB * sizeof(ChanConst));
  const uint32_t zcell = bar + 16;   // a zero float4: the cell gated-out terms read
  volatile int* blive = reinterpret_cast<int*>(sbase + kRing * kNB * sizeof(ChanConst) + 32);   // [kRing]
  const int W = prm.W;
  const uint32_t rsb = (uint32_t)raw_slot_bytes(W);
  unsigned char* rawp = sbase + k2_raw_off();
  float4* win = reinterpret_cast<float4*>(sbase + k2_win_off(W));
  const uint32_t win_base = (uint32_t)__cvta_generic_to_shared(win);
  const uint32_t raw_base = (uint32_t)__cvta_generic_to_shared(rawp);

  // tile of this CTA and its channel range (a wave-tail tile is shared by tsplit CTAs)
#if SASBP_LAZY_RANGE
  // recomputed at each (per-batch) use from blockIdx and the launch constants instead of being kept
  // in registers (A/B knob: it raised the 3D kernel from 123 to 128 registers)
  auto red_cta = [&]() -> bool { return SASBP_TAILSPLIT && prm.tsplit > 1 && (int)blockIdx.x >= prm.tail0; };
  auto ch_edge = [&](int k) -> int {   // k = 0: first channel, k = 1: one past the last
    if (!red_cta()) return k ? prm.ch_hi : prm.ch_lo;
    const int sp = ((int)blockIdx.x - prm.tail0) % prm.tsplit + k;
    return prm.ch_lo + (int)(((long long)prm.ch_hi - prm.ch_lo) * sp / prm.tsplit);
  };
  const int tile = red_cta() ? prm.tail0 + ((int)blockIdx.x - prm.tail0) / prm.tsplit : (int)blockIdx.x;
#else
  int tile = (int)blockIdx.x, ch_lo_v = prm.ch_lo, ch_hi_v = prm.ch_hi;
  bool red_v = false;
  if (SASBP_TAILSPLIT && prm.tsplit > 1 && tile >= prm.tail0) {
    const int r = tile - prm.tail0, sp = r % prm.tsplit;
    const long long n = (long long)prm.ch_hi - prm.ch_lo;
    tile = prm.tail0 + r / prm.tsplit;
    ch_lo_v = prm.ch_lo + (int)(n * sp / prm.tsplit);
    ch_hi_v = prm.ch_lo + (int)(n * (sp + 1) / prm.tsplit);
    red_v = true;
  }
  auto red_cta = [&]() -> bool { return red_v; };
  auto ch_edge = [&](int k) -> int { return k ? ch_hi_v : ch_lo_v; };
#endif
  const TM tm(prm, tile);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double ct[3];
  tm.centre(prm, ct);

  // Per-pixel geometry.  General grids keep the offsets of every pixel pair; axis-aligned grids
  // (diagonal steps, AXIS) keep dx per x-pair column, dy per ky row and dz per kz plane -- the
  // same arithmetic from ~20 fewer registers (occupancy).  Pixel k = ((kz KY + ky) KX + kx), pair
  // p = k / 2: x-pair column p % NXP, row (p / NXP) % KY, plane p / (NXP KY).
  constexpr int NXP = KX / 2;
  constexpr bool AXP = AXIS && SASBP_AXIS_PAIRS;   // dy, dz as register pairs (else broadcast scalars)
  // SEPQ: q = (dx^2 + ux dx) + (dy^2 + uy dy) + (dz^2 + uz dz) evaluated per column / row / plane and
  // added per pixel pair (the squares are kept per axis instead of |d|^2 per pair)
  constexpr bool SEPQ = AXIS && !AXP && SASBP_AXIS_SEPQ;
  float2 DX[AXIS ? NXP : NP], DY[AXP ? KY : (AXIS ? 1 : NP)], DZ[AXP ? KZ : (AXIS ? 1 : NP)], DD[SEPQ ? 1 : NP], BT[NP];
  float DYA[AXIS ? KY : 1], DZA[AXIS ? KZ : 1];
  float2 DX2[SEPQ ? NXP : 1];
  float DY2[SEPQ ? KY : 1], DZ2[SEPQ ? KZ : 1];
  float2 A[2 * NP], B[2 * NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    float dx0, dy0, dz0, dx1, dy1, dz1;
    tm.offset(prm, 2 * p, dx0, dy0, dz0);
    tm.offset(prm, 2 * p + 1, dx1, dy1, dz1);
    if (!HAS_DZ) { dz0 = 0.f; dz1 = 0.f; }
    if constexpr (AXP) {
      DX[p % NXP] = make_float2(dx0, dx1); DY[(p / NXP) % KY] = f2(dy0); DZ[p / (NXP * KY)] = f2(dz0);
    } else if constexpr (AXIS) {
      DX[p % NXP] = make_float2(dx0, dx1); DYA[(p / NXP) % KY] = dy0; DZA[p / (NXP * KY)] = dz0;
    } else {
      DX[p] = make_float2(dx0, dx1); DY[p] = make_float2(dy0, dy1); DZ[p] = make_float2(dz0, dz1);
    }
    if constexpr (SEPQ) {
      DX2[p % NXP] = make_float2(dx0 * dx0, dx1 * dx1); DY2[(p / NXP) % KY] = dy0 * dy0; DZ2[p / (NXP * KY)] = dz0 * dz0;
    } else {
      DD[p] = make_float2(dx0 * dx0 + dy0 * dy0 + dz0 * dz0, dx1 * dx1 + dy1 * dy1 + dz1 * dz1);
    }
    BT[p] = f2(0.f);
    A[2 * p] = f2(0.f); A[2 * p + 1] = f2(0.f); B[2 * p] = f2(0.f); B[2 * p + 1] = f2(0.f);
  }
  auto dxp = [&](int p) -> float2 { if constexpr (AXIS) return DX[p % NXP]; else return DX[p]; };
  auto dyp = [&](int p) -> float2 {
    if constexpr (AXP) return DY[(p / NXP) % KY]; else if constexpr (AXIS) return f2(DYA[(p / NXP) % KY]); else return DY[p];
  };
  auto dzp = [&](int p) -> float2 {
    if constexpr (AXP) return DZ[p / (NXP * KY)]; else if constexpr (AXIS) return f2(DZA[p / (NXP * KY)]); else return DZ[p];
  };
  // q = 2 u.d + |d|^2 of pixel pair p for the leg with 2u = (ux, uy, uz)
  auto qpair = [&](int p, float ux, float uy, float uz) -> float2 {
    if constexpr (SEPQ) {
      const float y = fmaf(DYA[(p / NXP) % KY], uy, DY2[(p / NXP) % KY]);
      const float z = HAS_DZ ? fmaf(DZA[p / (NXP * KY)], uz, DZ2[p / (NXP * KY)]) : 0.f;
      return __fadd2_rn(__ffma2_rn(DX[p % NXP], f2(ux), DX2[p % NXP]), f2(y + z));
    } else {
      float2 q = __ffma2_rn(f2(uy), dyp(p), DD[p]);
      q = __ffma2_rn(f2(ux), dxp(p), q);
      if (HAS_DZ) q = __ffma2_rn(f2(uz), dzp(p), q);
      return q;
    }
  };

#if SASBP_KPH_PARAM
  const float kph = prm.kph_f;
  const float kfs = prm.kfs_f;
#else
  const float kph = (float)(6.283185307179586 * prm.k_r);
  const float kfs = (float)prm.k_s;
#endif
  // spreading weight (R18): w = R_tx R_rx = (r_t k_s + dU_tx)(r_r k_s + dU_rx) / k_s^2, in samples
  const float inv_ks2 = (float)(1.0 / (prm.k_s * prm.k_s));
#if SASBP_BININDEX
  // V = U' + urr + Wh + 0.5 + 2^kb = u - k_lo + 2^kb lies in the binade [2^kb, 2^(kb+1)) for every
  // window coordinate u - k_lo in [0, W) (W <= 2^kb): the cell index floor(u - k_lo) is the top kb
  // mantissa bits, and (bits >> (19 - kb)) & ((2^kb - 1) << 4) is already its byte offset (16 B cells)
  const int vkb = 32 - __clz(max(prm.W - 1, 1));
  const float voff = (float)(prm.W >> 1) + 0.5f + (float)(1 << vkb);
  const uint32_t vsh = (uint32_t)(19 - vkb), vmask = ((1u << vkb) - 1u) << 4;
#endif
  // refraction: interface height relative to the tile centre, slownesses in samples per metre
  const float zbr = MODE == kRefract ? (float)(prm.zb - ct[2]) : 0.f;
  const float k1r = (float)(prm.fs / prm.c), k2r = MODE == kRefract ? (float)(prm.fs / prm.c2) : 0.f;
  const int nch = ch_edge(1) - ch_edge(0);
  const int nbatch = (nch + kNB - 1) / kNB;
  // Channel order: every tile visits all batches, starting at a batch offset proportional to
  // its launch rank among the resident CTAs (blockIdx / resident).  CTAs that are resident at
  // the same time then stream the same channels at the same time, so a channel's windows come
  // from DRAM once per wave and from L2 for the other tiles.  Deterministic (depends on
  // blockIdx only); the sum is order-free up to fp32 rounding (R11).
  const int rot = prm.resident > 0
      ? (int)(((long long)(blockIdx.x % prm.resident) * nbatch) / prm.resident) : 0;
  auto bat = [&](int i) { const int t = i + rot; return t >= nbatch ? t - nbatch : t; };
  const int Wh = W >> 1;
  const int nbox = box_samples(W);
#if SASBP_FLAT_TRANSFORM
  const float inv_w = 1.0f / (float)W;
#endif
  const int P2 = (W + 1) >> 1;                // cell pairs per channel
  [[maybe_unused]] const float inv_p2 = 1.0f / (float)P2;
  // i / P2 as a multiply-high (exact for i < 2^32 / P2^2): keeps the transform's index math off
  // the XU (the float trick below is an I2F + F2I pair per lane-step)
  const uint32_t mp2 = 0xFFFFFFFFu / (uint32_t)P2 + 1u;

  if (tid == 0) {
    if (USE_TMA) {
      mbar_init(bar, kWarps);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("st.shared.v4.f32 [%0], {%1, %1, %1, %1};" ::"r"(zcell), "f"(0.f) : "memory");
    for (int i = 0; i < kRing; ++i) blive[i] = 1;
  }
  __syncthreads();

  // fp64 prologues run in groups: warp w computes all kNB channels of batch g + w (one lane per
  // channel), four batches ahead of use, into a ring of kRing constant batches -- one pass of
  // the prologue code per warp per kWarps batches instead of one per batch.
  constexpr int kGroup = kWarps * kBPW;   // batches per prologue group
  auto prologue_group = [&](int g) {
    const int sub = lane / kNB, cl = lane % kNB;
    const int bb = g + warp * kBPW + sub;
    bool live = false;
    if (sub < kBPW && bb < nbatch) {
      const int nbb = min(kNB, nch - bat(bb) * kNB);
      if (cl < nbb) {
        const ChanConst k = chan_prologue<GATE, MOTION, MODE == kRefract>(prm, ch_edge(0) + bat(bb) * kNB + cl, ct, cl,
                                                                         win_base);
        cc[(bb % kRing) * kNB + cl] = k;
        live = !(k.gate & 16);
      }
    }
    if (GATE) {   // a batch with every channel culled is skipped as a whole
      const unsigned m = __ballot_sync(0xffffffffu, live);
      if (cl == 0 && sub < kBPW && bb < nbatch) blive[bb % kRing] = ((m >> (sub * kNB)) & ((1u << kNB) - 1u)) != 0u;
    }
  };
  // window loads of batch b: warp w issues the rows of channels [w*kCW, (w+1)*kCW); every warp
  // arrives once on the batch's mbarrier with the byte count of its rows.
  static_assert(kNB % kWarps == 0, "each warp issues the window rows of kNB / kWarps channels");
  constexpr int kCW = kNB / kWarps;
  auto issue = [&](int b) {
    if (GATE && !blive[b % kRing]) return;   // dead batch: no loads, no mbarrier phase
    const int nb = min(kNB, nch - bat(b) * kNB);
    const int ch0 = ch_edge(0) + bat(b) * kNB;
    const ChanConst* cb = cc + (b % kRing) * kNB;
    const int c0 = warp * kCW;
    const int mine = max(0, min(kCW, nb - c0));
    if (USE_TMA) {
      if (lane == 0) {
        int live = mine;
        if (GATE)
          for (int c = c0; c < c0 + mine; ++c) live -= (cb[c].gate >> 4) & 1;
        mbar_expect_tx(bar, (uint32_t)(live * nbox * 8));
        for (int c = c0; c < c0 + mine; ++c)
          if (!GATE || !(cb[c].gate & 16)) tma_load_row(raw_base + c * rsb, &tmap, cb[c].klo, ch0 + c, bar);
      }
    } else {
      for (int c = c0; c < c0 + mine; ++c) {
        if (GATE && (cb[c].gate & 16)) continue;
        const int klo = cb[c].klo;
        const float2* row = prm.echoes + (size_t)(ch0 + c) * prm.Ns;
        const uint32_t dst = raw_base + c * rsb;
        for (int j = lane; j < nbox; j += 32) {
          const int n = klo + j;
          const bool ok = (n >= 0) && (n < prm.Ns);
          cp_async8(dst + 8u * j, ok ? (const void*)(row + n) : (const void*)row, ok);
        }
      }
      cp_async_commit();
    }
  };

  prologue_group(0);
  __syncthreads();
  issue(0);
  int cur_ping = -1;
  static_assert(2 * NP <= 32, "per-pixel gate masks are 32-bit");
  constexpr uint32_t kAllPx = 2 * NP == 32 ? 0xFFFFFFFFu : (1u << (2 * NP)) - 1u;   // every pixel of a thread
  uint32_t mtx = kAllPx;   // transmit-cone pixel mask of the current ping (GATE)

  uint32_t phase = 0;   // mbarrier parity of the next live batch
  for (int b = 0; b < nbatch; ++b) {
    const int nb = min(kNB, nch - bat(b) * kNB);
    const bool live = !GATE || blive[b % kRing] != 0;   // warp-uniform (set >= 2 barriers ago)
    if (live) {
      if (USE_TMA) { mbar_wait(bar, phase); phase ^= 1u; }
      else cp_async_wait_all();
    }
    __syncthreads();   // raw(b) landed; every warp is done with win(b-1)
    if (live) {
    // rewrite raw windows as (intercept, slope) cells; cell j serves u in [k_lo+j, k_lo+j+1]:
    //   slope = d1 - d0,  intercept = d0 + (0.5 - (j - Wh)) * slope   (ehat = intercept + U slope)
#if SASBP_FLAT_TRANSFORM
    {  // warp w takes channels w, w+kWarps, ...; flattened over (channel, cell)
      const int nmine = (nb - warp + kWarps - 1) / kWarps;
      const int tot = nmine * W;
      for (int i = lane; i < tot; i += 32) {
        const int q = (int)(((float)i + 0.5f) * inv_w);   // i / W (exact: i < 2^20)
        const int j = i - q * W;
        const int c = warp + q * kWarps;
        const float2* rw = reinterpret_cast<const float2*>(rawp + c * rsb);
        const float2 d0 = rw[j], d1 = rw[j + 1];
        const float2 sl = __fadd2_rn(d1, make_float2(-d0.x, -d0.y));
#if SASBP_BININDEX
        const float2 ic = __ffma2_rn(sl, f2(0.5f - (float)(j - Wh) + cc[(b % kRing) * kNB + c].urr), d0);
#else
        const float2 ic = __ffma2_rn(sl, f2(0.5f - (float)(j - Wh)), d0);
#endif
        win[c * W + j] = make_float4(ic.x, ic.y, sl.x, sl.y);
      }
    }
#else
    if constexpr (SASBP_XFORM_CURSOR && !SASBP_BININDEX && (!GATE || SASBP_XFORM_CURSOR_GATE || (GIN && SASBP_XFORM_CURSOR_GIN))) {
       // warp w rewrites channels w, w+kWarps, ...: two cells per lane-step, flattened over
       // (channel, cell pair) so the lanes stay busy across channel boundaries.  Each lane keeps
       // cursors (raw source, cell destination, cell coordinate) and advances them by 32 pairs,
       // wrapping to its next channel when it runs past the P2 pairs of one: no division and no
       // re-derived smem offsets per step (the indexed form spent ~50 of 62 instructions per
       // step on index math the compiler rematerialised under register pressure).
      const int nmine = (nb - warp + kWarps - 1) / kWarps;
      const int tot = nmine * P2;
      int t = lane, q = 0;
      while (t >= P2) { t -= P2; ++q; }
      const unsigned char* rp = rawp + (warp + q * kWarps) * rsb + 16 * t;
      float4* wp = win + (warp + q * kWarps) * W + 2 * t;
      const ChanConst* gp = cc + (b % kRing) * kNB + warp + q * kWarps;
      float j0 = (float)(Wh - 2 * t) + 0.5f;
      const int rwrap = kWarps * (int)rsb - 16 * P2, wwrap = kWarps * W - 2 * P2;
      for (int i = lane; i < tot; i += 32) {
        if (!GATE || !(gp->gate & 16)) {
          const float4 d01 = *reinterpret_cast<const float4*>(rp);
          const float2 d2 = *reinterpret_cast<const float2*>(rp + 16);
          const float2 d0 = make_float2(d01.x, d01.y), d1 = make_float2(d01.z, d01.w);
          const float2 s0 = __fadd2_rn(d1, make_float2(-d0.x, -d0.y));
          const float2 s1 = __fadd2_rn(d2, make_float2(-d1.x, -d1.y));
          const float2 i0 = __ffma2_rn(s0, f2(j0), d0);
          const float2 i1 = __ffma2_rn(s1, f2(j0 - 1.0f), d1);
          wp[0] = make_float4(i0.x, i0.y, s0.x, s0.y);
          if (2 * t + 1 < W) wp[1] = make_float4(i1.x, i1.y, s1.x, s1.y);
        }
        t += 32; rp += 512; wp += 64; j0 -= 64.f;
        while (t >= P2) { t -= P2; rp += rwrap; wp += wwrap; j0 += (float)(2 * P2); gp += kWarps; }
      }
    } else {
       // indexed form (the gated kernels: the cursor form cost them 7 % in register allocation,
       // profiles/ab_r02.txt): flattened over (channel, cell pair) so the lanes stay busy
      const int nmine = (nb - warp + kWarps - 1) / kWarps;
      const int tot = nmine * P2;
      for (int i = lane; i < tot; i += 32) {
#if SASBP_DIV_MULHI
        const int q = (int)__umulhi((uint32_t)i, mp2);        // i / P2
#else
        const int q = (int)(((float)i + 0.5f) * inv_p2);   // i / P2, exact for i < 2^20
#endif
        const int t = i - q * P2;
        const int c = warp + q * kWarps;
        if (GATE && (cc[(b % kRing) * kNB + c].gate & 16)) continue;
        const float2* rw = reinterpret_cast<const float2*>(rawp + c * rsb) + 2 * t;
        const float4 d01 = *reinterpret_cast<const float4*>(rw);
        const float2 d2 = rw[2];
        const float2 d0 = make_float2(d01.x, d01.y), d1 = make_float2(d01.z, d01.w);
        const float2 s0 = __fadd2_rn(d1, make_float2(-d0.x, -d0.y));
        const float2 s1 = __fadd2_rn(d2, make_float2(-d1.x, -d1.y));
#if SASBP_BININDEX
        // the cells take the channel's fractional window offset: ehat = ic' + U' slope
        const float j0 = (float)(Wh - 2 * t) + 0.5f + cc[(b % kRing) * kNB + c].urr;
#else
        const float j0 = (float)(Wh - 2 * t) + 0.5f;
#endif
        const float2 i0 = __ffma2_rn(s0, f2(j0), d0);
        const float2 i1 = __ffma2_rn(s1, f2(j0 - 1.0f), d1);
        float4* wc = win + c * W + 2 * t;
        wc[0] = make_float4(i0.x, i0.y, s0.x, s0.y);
        if (2 * t + 1 < W) wc[1] = make_float4(i1.x, i1.y, s1.x, s1.y);
      }
    }
#endif
    __syncthreads();   // win(b) complete; raw free
    }
    if (b + 1 < nbatch) issue(b + 1);
    if ((b + 2) % kGroup == 0) prologue_group(b + 2);   // batches b+2 .. b+1+kGroup (ring slots not in use)
    if (!live) continue;
    const ChanConst* cb = cc + (b % kRing) * kNB;
#if SASBP_CC_LDS
    const uint32_t cb_s = (uint32_t)__cvta_generic_to_shared(cc) + (uint32_t)((b % kRing) * kNB) * (uint32_t)sizeof(ChanConst);
#endif

    // hot channel constants of the dense series kernels (ux2 uy2 uz2 kap0 | a0..a3 | urr phi0 | ping
    // woff), loaded one channel ahead so the loads' latency overlaps the previous channel's terms
#if SASBP_CC_PREFETCH
    constexpr bool kPref = ((AXIS && !GATE) || (GATE && SASBP_GATE_PREF)) && !MOTION && !WEIGHT &&
                           (MODE == kSeries3 || MODE == kSeries4);
#else
    constexpr bool kPref = false;
#endif
    const uint32_t cb_a = (uint32_t)__cvta_generic_to_shared(cb);
    float4 pf0, pf1, pf5;
    float2 pf2;
    auto hot = [&](int c) {
      const uint32_t a = cb_a + (uint32_t)c * (uint32_t)sizeof(ChanConst);
      pf0 = lds128(a); pf1 = lds128(a + 16u); pf2 = lds64(a + 32u);
      if (GATE) pf5 = lds128(a + 80u);   // ping woff klo gate
      else { const float2 t = lds64(a + 80u); pf5.x = t.x; pf5.y = t.y; }
    };
    if constexpr (kPref) hot(0);

#if SASBP_CUNROLL2
#pragma unroll 2
#else
#pragma unroll 1
#endif
    for (int c = 0; c < nb; ++c) {
      ChanConst kc;
      if constexpr (kPref) {
        const float4 r0 = pf0, r1 = pf1, r5 = pf5;
        const float2 r2 = pf2;
        if (c + 1 < nb) hot(c + 1);
        kc.ux2 = r0.x; kc.uy2 = r0.y; kc.uz2 = r0.z; kc.kap0 = r0.w;
        kc.a0 = r1.x; kc.a1 = r1.y; kc.a2 = r1.z; kc.a3 = r1.w;
        kc.urr = r2.x; kc.phi0 = r2.y;
        kc.ping = __float_as_int(r5.x); kc.woff = __float_as_int(r5.y);
        if (GATE) kc.gate = __float_as_int(r5.w);
      } else {
#if SASBP_CC_LDS
        kc = lds_struct<ChanConst>(cb_s + (uint32_t)c * (uint32_t)sizeof(ChanConst));
#else
        kc = cb[c];
#endif
      }
      if (GATE && (kc.gate & 16)) continue;                 // culled: tile outside a cone
      if (kc.ping != cur_ping) {
        cur_ping = kc.ping;
        if constexpr (kPref) {   // the transmit-leg constants, once per ping
          kc.tx2x = cb[c].tx2x; kc.tx2y = cb[c].tx2y; kc.tx2z = cb[c].tx2z; kc.r2_t = cb[c].r2_t; kc.r_t = cb[c].r_t;
        }
        if (GATE && !GIN) {   // transmit-cone mask of this thread's pixels for the new ping
          mtx = kAllPx;
          if ((kc.gate & 3) == kGEdge)
            mtx = gate_mask<TM, 2 * NP>(&prm, tm, cur_ping, prm.tx + 3 * cur_ping, kAllPx);
        }
        // transmit leg, exact range-relative form: dR = q / (sqrt(r^2 + q) + r), in samples
#if SASBP_TX_SERIES
        // series plans: dU_tx = q (a0 + a1 q + a2 q^2 [+ a3 q^3]), a_n = c_n (fs/c) / r_t^(2n+1)
        // (the plan's truncation bound covers the transmitter too)
        float ta0 = 0.f, ta1 = 0.f, ta2 = 0.f, ta3 = 0.f;
        if (MODE == kSeries3 || MODE == kSeries4) {
          const float ir = rcp_approx(kc.r_t), ir2 = ir * ir, g = kfs * ir;
          ta0 = 0.5f * g; ta1 = -0.125f * g * ir2; ta2 = 0.0625f * g * ir2 * ir2; ta3 = -0.0390625f * g * ir2 * ir2 * ir2;
        }
#endif
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          if (MODE == kRefract) {   // Fermat time through the interface minus the tile reference
            const float t0v = refr_time32(dxp(p).x - kc.tx2x, dyp(p).x - kc.tx2y, dzp(p).x - kc.tx2z, zbr - kc.tx2z,
                                          dzp(p).x - zbr, k1r, k2r);
            const float t1v = refr_time32(dxp(p).y - kc.tx2x, dyp(p).y - kc.tx2y, dzp(p).y - kc.tx2z, zbr - kc.tx2z,
                                          dzp(p).y - zbr, k1r, k2r);
            BT[p] = make_float2(t0v - kc.r_t, t1v - kc.r_t);
            continue;
          }
          const float2 q = qpair(p, kc.tx2x, kc.tx2y, kc.tx2z);
#if SASBP_TX_SERIES
          if (MODE == kSeries3 || MODE == kSeries4) {   // far field: the rx leg's series, no MUFU
            float2 h = MODE == kSeries4 ? __ffma2_rn(f2(ta3), q, f2(ta2)) : f2(ta2);
            h = __ffma2_rn(h, q, f2(ta1));
            h = __ffma2_rn(h, q, f2(ta0));
            BT[p] = __fmul2_rn(q, h);
            continue;
          }
#endif
          const float2 r2 = __fadd2_rn(q, f2(kc.r2_t));
          const float den0 = leg_den(r2.x, kc.r_t);
          const float den1 = leg_den(r2.y, kc.r_t);
          BT[p] = __fmul2_rn(__fmul2_rn(q, make_float2(rcp_approx(den0), rcp_approx(den1))), f2(kfs));
        }
      }
      uint32_t msk = kAllPx;
      bool masked = false;
      if (GATE && !GIN) {
        msk = mtx;
        if (((kc.gate >> 2) & 3) == kGEdge) {   // receive-cone mask (bistatic), per channel
          const int chg = ch_edge(0) + bat(b) * kNB + c;
          msk = gate_mask<TM, 2 * NP>(&prm, tm, kc.ping, prm.rx + 3 * (size_t)chg, msk);
        }
        masked = (kc.gate & 3) == kGEdge || ((kc.gate >> 2) & 3) == kGEdge;   // warp-uniform
        if (SASBP_GATE_PRED && !masked) msk = 0xFFFFFFFFu;   // IN channel: every pixel accumulates
      }
#if SASBP_BININDEX
      const float urrv = kc.urr + voff;                            // V = U' + urrv
#endif
      const float rtk = WEIGHT ? kc.r_t * kfs : 0.f;               // r_t, r_r in samples
      const float rrk = WEIGHT ? kc.r_r * kfs * inv_ks2 : 0.f;
      // the pixel loop; MSK = per-pixel gate selects (edge channels).  With SASBP_GATE_SPLIT the
      // selects are compiled into a second copy taken only by channels whose tile straddles a cone
      // edge (warp-uniform branch); otherwise every channel of a gated kernel pays them.
      auto pixels = [&](auto msk_tag) {
        constexpr bool MSK = decltype(msk_tag)::value;
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          const float2 q = qpair(p, kc.ux2, kc.uy2, kc.uz2);
          float2 U;
          float2 wgt = f2(1.f);
          float2 srr = f2(0.f);   // exact-mode moving receiver: |x - rx'| per pixel
          if (MODE == kRefract) {
            const float r0 = refr_time32(dxp(p).x - kc.ux2, dyp(p).x - kc.uy2, dzp(p).x - kc.uz2, zbr - kc.uz2,
                                         dzp(p).x - zbr, k1r, k2r);
            const float r1 = refr_time32(dxp(p).y - kc.ux2, dyp(p).y - kc.uy2, dzp(p).y - kc.uz2, zbr - kc.uz2,
                                         dzp(p).y - zbr, k1r, k2r);
            U = __fadd2_rn(make_float2(r0 - kc.a1, r1 - kc.a1), BT[p]);
          } else if (MODE == kExact) {
            const float2 r2 = __fadd2_rn(q, f2(kc.r2_r));
            const float den0 = leg_den(r2.x, kc.r_r);
            const float den1 = leg_den(r2.y, kc.r_r);
            if (MOTION) srr = __fadd2_rn(make_float2(den0, den1), f2(-kc.r_r));   // |x - rx'|
            if (WEIGHT) {
              const float2 dU = __fmul2_rn(__fmul2_rn(q, make_float2(rcp_approx(den0), rcp_approx(den1))), f2(kfs));
              U = __fadd2_rn(dU, BT[p]);
              wgt = __fmul2_rn(__fadd2_rn(BT[p], f2(rtk)), __ffma2_rn(dU, f2(inv_ks2), f2(rrk)));
            } else {
              U = __ffma2_rn(__fmul2_rn(q, make_float2(rcp_approx(den0), rcp_approx(den1))), f2(kfs), BT[p]);
            }
          } else {
            float2 h;
            if (MODE == kSeries4) {
              h = __ffma2_rn(f2(kc.a3), q, f2(kc.a2));
              h = __ffma2_rn(h, q, f2(kc.a1));
            } else {
              h = __ffma2_rn(f2(kc.a2), q, f2(kc.a1));
            }
            h = __ffma2_rn(h, q, f2(kc.a0));
            if (WEIGHT) {
              const float2 dU = __fmul2_rn(q, h);
              U = __fadd2_rn(dU, BT[p]);
              wgt = __fmul2_rn(__fadd2_rn(BT[p], f2(rtk)), __ffma2_rn(dU, f2(inv_ks2), f2(rrk)));
            } else {
              U = __ffma2_rn(q, h, BT[p]);
            }
          }
  #if SASBP_BININDEX
          if (MOTION) {   // moving receiver: U' = dU / (1 + w.v/c) ~ dU (kap0 + kg.d)
            float2 kap = __ffma2_rn(f2(kc.kgy), dyp(p), f2(kc.kap0));
            kap = __ffma2_rn(f2(kc.kgx), dxp(p), kap);
            if (HAS_DZ) kap = __ffma2_rn(f2(kc.kgz), dzp(p), kap);
            U = __fmul2_rn(U, kap);
          }
          const float2 T = __fadd2_rn(U, f2(urrv));            // exponent-aligned window coordinate V
  #else
          if (MOTION) {   // moving receiver: U = dU / (1 + w.v/c) ~ dU (kap0 + kg.d) + urr
            float2 kap = __ffma2_rn(f2(kc.kgy), dyp(p), f2(kc.kap0));
            kap = __ffma2_rn(f2(kc.kgx), dxp(p), kap);
            if (HAS_DZ) kap = __ffma2_rn(f2(kc.kgz), dzp(p), kap);
            if (MODE == kExact) {   // exact: kappa = |x - rx'| / (|x - rx'| + (u + d).v / c)
              const float2 dn = __fadd2_rn(srr, kap);
              kap = __fmul2_rn(srr, make_float2(rcp_approx(dn.x), rcp_approx(dn.y)));
            }
            U = __ffma2_rn(U, kap, f2(kc.urr));
          } else {
            U = __fadd2_rn(U, f2(kc.urr));                     // centred window coordinate
          }
          const float2 T = __fadd2_rn(U, f2(kMagic));          // rn(U) in the mantissa
  #endif
          const float2 ph = __ffma2_rn(U, f2(kph), f2(kc.phi0));
  #pragma unroll
          for (int s = 0; s < 2; ++s) {
            const float Us = s ? U.y : U.x;
            const float Ts = s ? T.y : T.x;
            const float phs = s ? ph.y : ph.x;
  #if SASBP_BININDEX
            uint32_t addr = ((uint32_t)__float_as_int(Ts) >> vsh & vmask) + (uint32_t)kc.woff;
  #else
            uint32_t addr = (uint32_t)__float_as_int(Ts) * 16u + (uint32_t)kc.woff;
  #endif
            if (MSK && masked && !SASBP_GATE_PRED) {   // gated-out pixel: read the zero cell
              const uint32_t mk = 0u - ((msk >> (2 * p + s)) & 1u);
              addr = (addr & mk) | (zcell & ~mk);
            }
            const float4 w = lds128(addr);
            float2 eh = __ffma2_rn(f2(Us), make_float2(w.z, w.w), make_float2(w.x, w.y));
            if (WEIGHT) eh = __fmul2_rn(eh, f2(s ? wgt.y : wgt.x));
            float sn, cs;
            __sincosf(phs, &sn, &cs);
            const float2 rot = make_float2(cs, sn);
            if (MSK && SASBP_GATE_PRED && !((msk >> (2 * p + s)) & 1u)) continue;   // gated out: no accumulate
            A[2 * p + s] = __ffma2_rn(f2(eh.x), rot, A[2 * p + s]);
            B[2 * p + s] = __ffma2_rn(f2(eh.y), rot, B[2 * p + s]);
          }
        }
      };
      if constexpr (GATE && !GIN) {
#if SASBP_GATE_SPLIT
        if (masked) pixels(std::true_type{}); else pixels(std::false_type{});
#else
        pixels(std::true_type{});
#endif
      } else {
        pixels(std::false_type{});
      }
    }
  }

#pragma unroll
  for (int k = 0; k < 2 * NP; ++k) {
    if (tm.valid(prm, k)) {
      float2* o = prm.image + ((size_t)tm.iz(k) * prm.ny + tm.iy(k)) * prm.nx + tm.ix(k);
      float2 v = make_float2(A[k].x - B[k].y, A[k].y + B[k].x);
      if (red_cta()) { atomicAdd(o, v); continue; }   // wave-tail partial (image zeroed by the launch)
      if (prm.accumulate) { const float2 a = *o; v.x += a.x; v.y += a.y; }
      *o = v;
    }
  }
}

// K3: count terms whose interpolation support meets the record, u in (-1, Ns).
// Same tiles and fp32 delay arithmetic as K2 (exact leg form), no echo traffic.  Gated counts use
// K2's own (tile, channel) cone classes: a culled channel counts nothing, an IN class needs no
// per-pixel test, only EDGE classes run the fp64 per-pixel gate (the transmit mask once per ping).
template <int KX, int KY, int KZ, int WY, int WZ>
__global__ void __launch_bounds__(32 * WY * WZ) count_kernel(const TdbpParams prm) {
  using TM = TileMap<KX, KY, KZ, WY, WZ>;
  constexpr int K = TM::K;
  static_assert(K <= 32, "pixel masks are 32-bit");
  constexpr int kCB = 32 * WY * WZ;   // channels per prologue batch: one per thread (the fp64
                                      // prologue is most of K3's work; 16 lanes of 128 left 7/8 idle)
  __shared__ ChanConst cc[kCB];
  const TM tm(prm);
  const int tid = threadIdx.x;
  double ct[3];
  tm.centre(prm, ct);
  float dx[K], dy[K], dz[K], dd[K];
  uint32_t okm = 0u;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    tm.offset(prm, k, dx[k], dy[k], dz[k]);
    dd[k] = dx[k] * dx[k] + dy[k] * dy[k] + dz[k] * dz[k];
    if (tm.valid(prm, k)) okm |= 1u << k;
  }
  const float Nsf = (float)prm.Ns;
  unsigned long long cnt = 0;
  int cur_ping = -1;
  uint32_t mtx = 0xFFFFFFFFu;
  for (int ch0 = prm.ch_lo; ch0 < prm.ch_hi; ch0 += kCB) {
    const int nb = min(kCB, prm.ch_hi - ch0);
    __syncthreads();
    if (tid < nb) cc[tid] = chan_prologue<true, true>(prm, ch0 + tid, ct, tid, 0u);
    __syncthreads();
    for (int c = 0; c < nb; ++c) {
      const ChanConst kc = cc[c];
      if (prm.gate && (kc.gate & 16)) continue;          // culled: the tile misses a cone
      uint32_t msk = okm;
      if (prm.gate) {
        if (kc.ping != cur_ping) {                       // transmit-cone mask, once per ping
          cur_ping = kc.ping;
          mtx = 0xFFFFFFFFu;
          if ((kc.gate & 3) == kGEdge) {
            double a[3], bb[3], x[3];
            ping_axes(prm, cur_ping, a, bb);
            mtx = 0u;
#pragma unroll
            for (int k = 0; k < K; ++k) {
              pixel_centre64(prm, tm.ix(k), tm.iy(k), tm.iz(k), x);
              if (in_fov_px(prm, x, prm.tx + 3 * cur_ping, a, bb)) mtx |= 1u << k;
            }
          }
        }
        msk &= mtx;
        if (((kc.gate >> 2) & 3) == kGEdge) {            // receive cone (bistatic)
          double a[3], bb[3], x[3];
          ping_axes(prm, kc.ping, a, bb);
#pragma unroll
          for (int k = 0; k < K; ++k) {
            if (!((msk >> k) & 1u)) continue;
            pixel_centre64(prm, tm.ix(k), tm.iy(k), tm.iz(k), x);
            if (!in_fov_px(prm, x, prm.rx + 3 * (size_t)(ch0 + c), a, bb)) msk &= ~(1u << k);
          }
        }
      }
      // the staged window [k_lo, k_lo + W] bounds every pixel's u (K2 interpolates from it): a window
      // wholly inside the record admits every pixel without a per-term test
      if (kc.klo >= 0 && kc.klo + prm.W + 1 <= prm.Ns) {
        cnt += (unsigned long long)__popc(msk);
        continue;
      }
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (!((msk >> k) & 1u)) continue;
        if (prm.refract) {   // counted with the fp64 refracted delay (off the clock)
          double x[3];
          pixel_centre64(prm, tm.ix(k), tm.iy(k), tm.iz(k), x);
          const double tau = refr_time64(x, prm.tx + 3 * kc.ping, prm.zb, prm.c, prm.c2) +
                             refr_time64(x, prm.rx + 3 * (size_t)(ch0 + c), prm.zb, prm.c, prm.c2);
          const double ua = (tau - prm.t0[kc.ping]) * prm.fs;
          cnt += (ua > -1.0 && ua < (double)prm.Ns) ? 1ull : 0ull;
          continue;
        }
        const float qt = fmaf(kc.tx2x, dx[k], fmaf(kc.tx2y, dy[k], fmaf(kc.tx2z, dz[k], dd[k])));
        const float qr = fmaf(kc.ux2, dx[k], fmaf(kc.uy2, dy[k], fmaf(kc.uz2, dz[k], dd[k])));
        const float rt = sqrtf(fmaxf(kc.r2_t + qt, 0.f)), rr = sqrtf(fmaxf(kc.r2_r + qr, 0.f));
        const float tk = kc.kap0 + kc.kgx * dx[k] + kc.kgy * dy[k] + kc.kgz * dz[k];
        const float kap = ((prm.vel || prm.nav) && prm.mode == kExact) ? rr / (rr + tk) : tk;
        const float du = (qt / fmaxf(rt + kc.r_t, 1e-30f) + qr / fmaxf(rr + kc.r_r, 1e-30f)) * (float)prm.k_s * kap;
        // absolute u = k_lo + 0.5 + Wh + (du + urr)
        const float ua = (float)kc.klo + 0.5f + (float)(prm.W >> 1) + (du + kc.urr);
        cnt += (ua > -1.f && ua < Nsf) ? 1ull : 0ull;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((tid & 31) == 0 && cnt) atomicAdd(prm.counter, cnt);
}

}  // namespace sasbp
