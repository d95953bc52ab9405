// conditioning.cu -- the input-conditioning kernels around K1/K2 (SURVEY §8(a) row a1 option and
// §8(f) NEXT-4):
//
//  * K1b sas_upsample (reading R19): band-limited xU upsampling by the 8-tap windowed sinc
//      out[U n + r] = sum_{m=-3}^{4} in[n + m] L(r/U - m),  L(s) = sinc(s) sinc(s/4), |s| < 4
//    ("8-tap windowed-sinc on the upsampled (x4) compressed series"; the paper is
//    silent on interpolation).  HBM-bound: 8 B read + 8U B written per input sample.  One CTA
//    stages a segment of 1024 input samples (+7 halo, zero-extended, R2) in shared memory; each
//    thread owns one input position, keeps its 8 taps in registers and writes its U outputs as
//    one contiguous 8U-byte run (a warp stores 256U contiguous bytes).  The U x 8 weights are
//    evaluated on the host in double precision from the definition and passed by value.
//
//  * K0 sas_baseband (reading R20): real passband -> complex baseband,
//      z[n] = x[n] exp(-j 2 pi fc (t0_p + n / fs_in)),  out[m] = sum_k h[k] z[m D + (Nh-1)/2 - k]
//    One CTA per (channel, run of MO outputs): the input span is mixed once into shared memory,
//    stored POLYPHASE (z_q[i] = z[i D + q]) so that, for a fixed tap, consecutive threads
//    (consecutive outputs) read consecutive words -- no bank conflicts for any decimation D.  The
//    carrier phase is reduced in fp64 (fc t0_p mod 1 on the host, n (fc / fs_in) mod 1 per
//    sample), so the ~1e4-cycle carrier phase never passes through fp32.
#include "sasbp.h"

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <vector>
#include <cuda_runtime.h>

extern "C" void sasbp_set_error(const char* msg);  // sasbp.cu: the thread-local sas_last_error buffer

namespace {

sas_status cond_fail(sas_status st, const char* what, cudaError_t e = cudaSuccess) {
  char buf[256];
  if (e != cudaSuccess) snprintf(buf, sizeof(buf), "%s: %s", what, cudaGetErrorString(e));
  else snprintf(buf, sizeof(buf), "%s", what);
  sasbp_set_error(buf);
  return st;
}

// ---------------------------------------------------------------- K1b: 8-tap xU upsampling

constexpr int kUpThreads = 256;
constexpr int kUpSeg = 1024;          // input samples per CTA
constexpr int kUpMax = 16;

struct UpWeights { float w[kUpMax][8]; };   // w[r][m + 3] = L(r/U - m)

__device__ __forceinline__ void st_cs_v4(float2* p, float2 a, float2 b) {
  // streaming store: the upsampled series is written once and read later by another kernel
  asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y)
               : "memory");
}

template <int UT>   // UT = U at compile time (1, 2, 4, 8), 0 = runtime U
__global__ void __launch_bounds__(kUpThreads) upsample_kernel(const float2* __restrict__ in, int Ns, int U_rt,
                                                              long long segs, const __grid_constant__ UpWeights W,
                                                              float2* __restrict__ out) {
  __shared__ float2 sx[kUpSeg + 8];
  const int U = UT ? UT : U_rt;
  const long long b = blockIdx.x;
  const long long ch = b / segs;
  const int n0 = (int)(b - ch * segs) * kUpSeg;
  const float2* x = in + ch * (long long)Ns;
  for (int i = threadIdx.x; i < kUpSeg + 7; i += kUpThreads) {   // x[n0 - 3 .. n0 + kUpSeg + 3]
    const int n = n0 - 3 + i;
    sx[i] = (n >= 0 && n < Ns) ? __ldcs(x + n) : make_float2(0.f, 0.f);
  }
  __syncthreads();
  float2* y = out + ch * (long long)Ns * U;
  for (int t = threadIdx.x; t < kUpSeg; t += kUpThreads) {
    const int n = n0 + t;
    if (n >= Ns) break;
    float2 tap[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) tap[m] = sx[t + m];
    float2* yo = y + (long long)n * U;
    if (UT >= 2) {
#pragma unroll
      for (int r = 0; r < (UT ? UT : 2); r += 2) {
        float2 a = make_float2(0.f, 0.f), c = make_float2(0.f, 0.f);
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          a.x = fmaf(W.w[r][m], tap[m].x, a.x); a.y = fmaf(W.w[r][m], tap[m].y, a.y);
          c.x = fmaf(W.w[r + 1][m], tap[m].x, c.x); c.y = fmaf(W.w[r + 1][m], tap[m].y, c.y);
        }
        st_cs_v4(yo + r, a, c);
      }
    } else {
      for (int r = 0; r < U; ++r) {
        float2 a = make_float2(0.f, 0.f);
#pragma unroll
        for (int m = 0; m < 8; ++m) { a.x = fmaf(W.w[r][m], tap[m].x, a.x); a.y = fmaf(W.w[r][m], tap[m].y, a.y); }
        __stcs(yo + r, a);
      }
    }
  }
}

// L(s) = sinc(s) sinc(s/4) for |s| < 4 (R19), in double precision
double lanczos4_host(double s) {
  const double pi = 3.141592653589793238462643383279;
  if (s == 0.0) return 1.0;
  if (std::fabs(s) >= 4.0) return 0.0;
  const double a = pi * s, b = pi * s * 0.25;
  return (std::sin(a) / a) * (std::sin(b) / b);
}

// ---------------------------------------------------------------- K0: basebanding

constexpr int kBbThreads = 256;
constexpr int kBbSmem = 48 * 1024;    // bytes of mixed input per CTA
constexpr int kBbMaxNh = 1023;

// carrier cycles at sample 0 of ping p, fc t0_p mod 1 (fp64; t0 == NULL -> 0)
__device__ __forceinline__ double bb_base(const double* __restrict__ t0, long long p, double fc) {
  if (!t0) return 0.0;
  const double v = fc * t0[p];
  return v - floor(v);
}

__global__ void __launch_bounds__(kBbThreads) baseband_kernel(const float* __restrict__ x, int E, int Nin, double kr,
                                                              double fc, const double* __restrict__ t0, const float* __restrict__ h,
                                                              int Nh, int D, int Nout, int MO, long long runs,
                                                              float2* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char bb_smem[];
  float* sh = reinterpret_cast<float*>(bb_smem);                            // taps [Nh] (padded to 4)
  float2* sz = reinterpret_cast<float2*>(bb_smem + ((Nh + 3) & ~3) * 4);     // polyphase z [D][Lq]
  const long long b = blockIdx.x;
  const long long ch = b / runs;
  const int m0 = (int)(b - ch * runs) * MO;
  const int half = (Nh - 1) >> 1;
  // span of input indices: n = m D + half - k, m in [m0, m0 + MO), k in [0, Nh)
  const int nlo = m0 * D + half - (Nh - 1);
  const int span = (MO - 1) * D + Nh;
  const int Lq = (span + D - 1) / D;          // samples per phase
  const float* xc = x + ch * (long long)Nin;
  const double bp = bb_base(t0, ch / E, fc);  // fc t0_p mod 1 (cycles)
  for (int k = threadIdx.x; k < Nh; k += kBbThreads) sh[k] = h[k];
  for (int i = threadIdx.x; i < span; i += kBbThreads) {
    const int n = nlo + i;
    float2 z = make_float2(0.f, 0.f);
    if (n >= 0 && n < Nin) {
      const float v = __ldcs(xc + n);
      double ph = fma((double)n, kr, bp);     // fc (t0_p + n / fs_in) mod 1, fp64
      ph -= rint(ph);                         // [-1/2, 1/2]
      float sn, cs;
      __sincosf(-6.283185307179586f * (float)ph, &sn, &cs);
      z = make_float2(v * cs, v * sn);
    }
    const int q = i % D;                      // polyphase: z_q[i / D]
    sz[q * Lq + i / D] = z;
  }
  __syncthreads();
  float2* yo = out + ch * (long long)Nout;
  for (int t = threadIdx.x; t < MO; t += kBbThreads) {
    const int m = m0 + t;
    if (m >= Nout) break;
    // tap k reads local input i = t D + j, j = Nh - 1 - k; with j = a D + q that is z_q[t + a]
    float ar = 0.f, ai = 0.f;
    for (int q = 0; q < D && q < Nh; ++q) {
      const float2* zq = sz + q * Lq + t;
#pragma unroll 4
      for (int j = q, a = 0; j < Nh; j += D, ++a) {
        const float2 z = zq[a];
        const float hk = sh[Nh - 1 - j];
        ar = fmaf(hk, z.x, ar);
        ai = fmaf(hk, z.y, ai);
      }
    }
    __stcs(yo + m, make_float2(ar, ai));
  }
}

// Register-blocked polyphase form (the default): each thread owns kBbR = 8 consecutive outputs.
// With j = a D + q the sum is  out[t] = sum_q sum_a hq[q][a] zq[q][t + a],  hq[q][a] =
// h[Nh - 1 - (a D + q)] (zero-padded to Apad taps per phase, a multiple of 8): per phase a
// 1-D convolution whose input window slides through registers -- per block of 8 taps a thread
// loads 8 new samples and 8 (broadcast) taps and issues 64 complex MACs as FFMA2.  The polyphase
// arrays are padded one sample per 8 (index i + i/8) so the warp's stride-8 window loads are
// conflict-free (stride 9 x 8 B).
constexpr int kBbR = 8;

__device__ __forceinline__ int bb_pad(int i) { return i + (i >> 3); }

__device__ __forceinline__ void bb_block(float2 (&acc)[kBbR], const float2 (&wa)[kBbR], const float2 (&wb)[kBbR],
                                         const float2* __restrict__ hq) {
#pragma unroll
  for (int aa = 0; aa < 8; ++aa) {
    const float2 hh = hq[aa];   // (h, h), same address for the whole warp
#pragma unroll
    for (int r = 0; r < kBbR; ++r) {
      const float2 z = (r + aa < 8) ? wa[r + aa] : wb[r + aa - 8];
      acc[r] = __ffma2_rn(hh, z, acc[r]);
    }
  }
}

template <int DT>   // DT = decimation at compile time (2, 4, 8: loops unrolled, all loads in flight), 0 = runtime
__global__ void __launch_bounds__(256) baseband_blocked_kernel(const float* __restrict__ x, int E, int Nin, double kr,
                                                               double fc, const double* __restrict__ t0p,
                                                               const float* __restrict__ h, int Nh, int D_rt, int Apad,
                                                               int Nout, int MO, long long runs, float2 rot1,
                                                               float2* __restrict__ out, int vec4) {
  const int D = DT ? DT : D_rt;
  extern __shared__ __align__(16) unsigned char bb_smem[];
  float2* hs = reinterpret_cast<float2*>(bb_smem);            // [D][Apad] (h, h)
  float2* sz = hs + (size_t)D * Apad + 2;                      // [D][LqP] padded polyphase input (2 slack
                                                               // slots before row 0: see the float4 staging)
  const long long b = blockIdx.x;
  const long long ch = b / runs;
  const int m0 = (int)(b - ch * runs) * MO;
  const int half = (Nh - 1) >> 1;
  const int nlo = m0 * D + half - (Nh - 1);    // local input i = n - nlo = t D + j
  const int Lq = MO + Apad;                     // samples per phase (+ slack for the last block)
  const int LqP = bb_pad(Lq) + 3;              // >= 3 slack slots after each row
  const float* xc = x + ch * (long long)Nin;
  const double bp = bb_base(t0p, ch / E, fc);
  for (int k = threadIdx.x; k < D * Apad; k += blockDim.x) {   // hq[q][a] = h[Nh - 1 - (a D + q)], zero padded
    const int q = k / Apad, a = k - q * Apad, j = a * D + q;
    const float hv = j < Nh ? h[Nh - 1 - j] : 0.f;
    hs[k] = make_float2(hv, hv);
  }
  // Staging, phase-inner: thread k-slots k = k0 + u blockDim (8 in flight), samples n = nlo + k D + q.
  // The carrier phasor exp(-j 2 pi fc t_n) is evaluated exactly (fp64 reduction + sincos) at
  // q = 0 and advanced by the fp32 rotation exp(-j 2 pi fc / fs_in) for q = 1..D-1, re-anchored
  // every 8 phases, so the error stays ~8 fp32 ulps.  No integer division anywhere.
  constexpr int kU = 8;
  const float2 rot = rot1;
  // full groups of kU slots per thread (unrolled, 8 loads in flight), then the Apad-slot tail.
  // Slot k0 + u B (B = blockDim) of phase q is sample nlo + (k0 + u B) D + q; its padded shared
  // position is bb_pad(k0) + u (B + B/8) (B is a multiple of 8).  Paired FP32 for the phasor
  // rotation (w <- w rot) and the mix (v w).
  const int Bd = blockDim.x;
  const float2 rotp = make_float2(-rot.y, rot.x);
  if (DT == 4 && vec4) {
    // D = 4, 16-byte aligned channel rows (vec4, checked on the host): aligned float4 loads
    // a = nlo - o + 4 k (o = nlo mod 4), kU = 8 per thread in flight (128 B, 4x the scalar path's
    // bytes per load).  Component j is local input i = 4 k + j - o, i.e. phase q = i & 3 of slot
    // i >> 2; the phasor is exact (fp64) at j = 0 and rotated for j = 1..3.  Loads wholly inside
    // 0..Nin-1 are one LDG.128, the few at the record edges are guarded scalars (zero outside).
    const int o = nlo & 3;
    const int a0 = nlo - o;
    const int nk = Lq + (o ? 1 : 0);           // float4s covering local inputs [0, 4 Lq)
    // kV = 9 float4s per thread per step: with 128 threads the 1024 + Apad + 1 float4s of a run
    // (Apad <= 16) take ONE step; with 8, 17 threads of warp 0 ran a second, almost empty step
    // that the other warps waited for at the barrier
    constexpr int kV = 9;
    for (int k0 = threadIdx.x; k0 < nk; k0 += kV * Bd) {
      float4 v[kV];
#pragma unroll
      for (int u = 0; u < kV; ++u) {
        const int k = k0 + u * Bd;
        const int a = a0 + 4 * k;
        v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (k < nk) {
          if (a >= 0 && a + 3 < Nin) {
            v[u] = __ldcs(reinterpret_cast<const float4*>(xc + a));
          } else {
            if (a >= 0 && a < Nin) v[u].x = __ldcs(xc + a);
            if (a + 1 >= 0 && a + 1 < Nin) v[u].y = __ldcs(xc + a + 1);
            if (a + 2 >= 0 && a + 2 < Nin) v[u].z = __ldcs(xc + a + 2);
            if (a + 3 >= 0 && a + 3 < Nin) v[u].w = __ldcs(xc + a + 3);
          }
        }
      }
      // component j of float4 k lands in phase row (j - o) & 3 at slot k + sj, sj = (j - o) >> 2
      // (0 or -1); for the slots of this thread's k = k0 + u Bd the padded position is
      // base_j + u (Bd + Bd/8) (Bd a multiple of 8).  The two components that fall outside slots
      // 0..Lq-1 (slot -1 of the first float4, slot Lq of the last) go to slack slots nobody reads
      // (2 before row 0, >= 3 after every row), so the stores need no per-component test.
      const int inc = Bd + (Bd >> 3);
      int base[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int sj = (j - o) >> 2;
        base[j] = ((j - o) & 3) * LqP + bb_pad(k0 + sj);
      }
#pragma unroll
      for (int u = 0; u < kV; ++u) {
        const int k = k0 + u * Bd;
        if (k >= nk) break;
        double ph = fma((double)(a0 + 4 * k), kr, bp);   // cycles at component 0, fp64
        ph -= rint(ph);
        float2 w;
        __sincosf(-6.283185307179586f * (float)ph, &w.y, &w.x);
        const float vv[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (j) w = __ffma2_rn(make_float2(w.y, w.y), rotp, __fmul2_rn(make_float2(w.x, w.x), rot));
          sz[base[j] + u * inc] = __fmul2_rn(make_float2(vv[j], vv[j]), w);
        }
      }
    }
  } else {
  const int Lfull = (Lq / (kU * (int)blockDim.x)) * (kU * (int)blockDim.x);
  const bool interior = nlo >= 0 && nlo + Lq * D <= Nin;   // no bounds checks needed (CTA-uniform)
  for (int k0 = threadIdx.x; k0 < Lfull; k0 += kU * Bd) {
    float2 w[kU];
    const float* xk = xc + nlo + k0 * D;
    float2* sk = sz + bb_pad(k0);
#pragma unroll
    for (int q = 0; q < (DT ? DT : D); ++q) {
      float v[kU];
      if (interior) {
#pragma unroll
        for (int u = 0; u < kU; ++u) v[u] = __ldcs(xk + u * Bd * D + q);
      } else {
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int n = nlo + (k0 + u * Bd) * D + q;
          v[u] = (n >= 0 && n < Nin) ? __ldcs(xc + n) : 0.f;
        }
      }
      if ((q & 7) == 0) {
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          double ph = fma((double)(nlo + (k0 + u * Bd) * D + q), kr, bp);   // cycles, fp64
          ph -= rint(ph);
          __sincosf(-6.283185307179586f * (float)ph, &w[u].y, &w[u].x);
        }
      } else {
#pragma unroll
        for (int u = 0; u < kU; ++u) w[u] = __ffma2_rn(make_float2(w[u].y, w[u].y), rotp, __fmul2_rn(make_float2(w[u].x, w[u].x), rot));
      }
      float2* sq = sk + q * LqP;
#pragma unroll
      for (int u = 0; u < kU; ++u) sq[u * (Bd + (Bd >> 3))] = __fmul2_rn(make_float2(v[u], v[u]), w[u]);
    }
  }
  for (int k = Lfull + threadIdx.x; k < Lq; k += blockDim.x) {
    for (int q = 0; q < D; ++q) {
      const int n = nlo + k * D + q;
      float2 z = make_float2(0.f, 0.f);
      if (n >= 0 && n < Nin) {
        double ph = fma((double)n, kr, bp);
        ph -= rint(ph);
        float sn, cs;
        __sincosf(-6.283185307179586f * (float)ph, &sn, &cs);
        const float v = __ldcs(xc + n);
        z = make_float2(v * cs, v * sn);
      }
      sz[q * LqP + bb_pad(k)] = z;
    }
  }
  }
  __syncthreads();
  const int t0 = threadIdx.x * kBbR;
  if (t0 >= MO || m0 + t0 >= Nout) return;
  float2 acc[kBbR];
#pragma unroll
  for (int r = 0; r < kBbR; ++r) acc[r] = make_float2(0.f, 0.f);
#pragma unroll
  for (int q = 0; q < (DT ? DT : D); ++q) {
    const float2* zq = sz + q * LqP;
    const float2* hq = hs + q * Apad;
    float2 wa[kBbR], wb[kBbR];
    // t0 and ab are multiples of 8, so bb_pad(t0 + ab + r) = bb_pad(t0 + ab) + r for r < 8
    const float2* z0 = zq + bb_pad(t0);
#pragma unroll
    for (int r = 0; r < kBbR; ++r) wa[r] = z0[r];
    for (int ab = 0; ab < Apad; ab += 16, z0 += 18) {
#pragma unroll
      for (int r = 0; r < kBbR; ++r) wb[r] = z0[9 + r];
      bb_block(acc, wa, wb, hq + ab);
      if (ab + 8 >= Apad) break;
#pragma unroll
      for (int r = 0; r < kBbR; ++r) wa[r] = z0[18 + r];
      bb_block(acc, wb, wa, hq + ab + 8);
    }
  }
  float2* yo = out + ch * (long long)Nout + m0 + t0;
  if (m0 + t0 + kBbR <= Nout && ((((uintptr_t)yo) & 15) == 0)) {
#pragma unroll
    for (int r = 0; r < kBbR; r += 2) st_cs_v4(yo + r, acc[r], acc[r + 1]);
  } else {
#pragma unroll
    for (int r = 0; r < kBbR; ++r)
      if (m0 + t0 + r < Nout) __stcs(yo + r, acc[r]);
  }
}

// ---------------------------------------------------------------- K0, complex-tap form (round 2, the default for D = 4)
//
// The mixer commutes with the FIR.  With w(n) = exp(-j 2 pi fc t_n), whose phase is linear in n,
// w(n_m - k) = w(n_m) exp(+j 2 pi kr k) (kr = fc / fs_in mod 1), so R20's
//   y[m] = sum_k h[k] x[n_m - k] w(n_m - k)  =  w(n_m) sum_k g[k] x[n_m - k],
//   g[k] = h[k] exp(+j 2 pi kr k),  n_m = m D + (Nh - 1) / 2 :
// the FIR runs on the REAL passband samples with complex taps (computed once per CTA, fp64 phase
// reduction), and one phasor per OUTPUT (exact at the thread's first output, fp32 rotation by
// exp(-j 2 pi kr D) for the next 7) replaces one per input sample.  No mixing pass, half the
// staged bytes (4-byte real samples), the same FFMA2 count per tap as the mixed form.  Staging:
// aligned float4 loads (D = 4, 16-byte aligned rows) de-interleaved into the D polyphase rows;
// each row keeps 8 samples per 12-word group so a thread's 8-sample window is two conflict-free
// LDS.128 (lane stride 12 words).
constexpr int kCtLead = 8;   // words of slack before row 0 (slot -1 of the first float4 lands at -5)
__host__ __device__ __forceinline__ int ct_pos(int i) { return (i >> 3) * 12 + (i & 7); }

__device__ __forceinline__ void ct_block(float2 (&acc)[kBbR], const float (&wa)[kBbR], const float (&wb)[kBbR],
                                         const float2* __restrict__ gq) {
#pragma unroll
  for (int aa = 0; aa < 8; ++aa) {
    const float2 g = gq[aa];   // complex tap, same address for the whole warp
#pragma unroll
    for (int r = 0; r < kBbR; ++r) {
      const float v = (r + aa < 8) ? wa[r + aa] : wb[r + aa - 8];
      acc[r] = __ffma2_rn(make_float2(v, v), g, acc[r]);
    }
  }
}

#ifndef BB_CTAP_MINB
#define BB_CTAP_MINB 8   // resident CTAs per SM the register allocation targets (64 registers; A/B config 4: 1.82 vs 1.94 ms at 7 CTAs/SM, 70 registers)
#endif
__global__ void __launch_bounds__(128, BB_CTAP_MINB) baseband_ctap_kernel(const float* __restrict__ x, int E, int Nin, double kr,
                                                            double fc, const double* __restrict__ t0p,
                                                            const float* __restrict__ h, int Nh, int Apad, int Nout,
                                                            int MO, long long runs, int RowW, float2 rotD,
                                                            float2* __restrict__ out) {
  constexpr int D = 4;
  extern __shared__ __align__(16) unsigned char bb_smem[];
  float2* gs = reinterpret_cast<float2*>(bb_smem);                 // [D][Apad] g_q[a] = g[Nh - 1 - (a D + q)]
  float* xs = reinterpret_cast<float*>(gs + (size_t)D * Apad) + kCtLead;   // [D][RowW] real polyphase rows
  const long long b = blockIdx.x;
  const long long ch = b / runs;
  const int m0 = (int)(b - ch * runs) * MO;
  const int half = (Nh - 1) >> 1;
  const int nlo = m0 * D + half - (Nh - 1);    // local input i = n - nlo = t D + j
  const int Lq = MO + Apad;
  const float* xc = x + ch * (long long)Nin;
  const double bp = bb_base(t0p, ch / E, fc);
  const int Bd = blockDim.x, tid = threadIdx.x;
  for (int k = tid; k < D * Apad; k += Bd) {
    const int q = k / Apad, a = k - q * Apad, j = a * D + q;
    float2 g = make_float2(0.f, 0.f);
    if (j < Nh) {
      const int kk = Nh - 1 - j;                 // tap index
      double ph = kr * (double)kk;               // cycles, fp64
      ph -= rint(ph);
      float sn, cs;
      __sincosf(6.283185307179586f * (float)ph, &sn, &cs);
      const float hv = h[kk];
      g = make_float2(hv * cs, hv * sn);
    }
    gs[k] = g;
  }
  // staging: float4 k covers local inputs 4 k - o .. 4 k - o + 3; component j -> row (j - o) & 3, slot k + sj
  const int o = nlo & 3;
  const int a0 = nlo - o;
  const int nk = Lq + (o ? 1 : 0);
  // the kernel runs 128 threads (host launch): slot k + 128 u sits 128 / 8 * 12 = 192 words after slot
  // k in a row, so each component's store address is one base per thread plus a constant offset
  constexpr int kV = 9, kThr = 128, kInc = kThr / 8 * 12;
  const bool interior = a0 >= 0 && a0 + 4 * nk <= Nin;   // CTA-uniform: no per-load bounds tests
  for (int k0 = tid; k0 < nk; k0 += kV * kThr) {
    float4 v[kV];
#pragma unroll
    for (int u = 0; u < kV; ++u) {
      const int k = k0 + u * kThr;
      const int a = a0 + 4 * k;
      v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (k < nk) {
        if (interior || (a >= 0 && a + 3 < Nin)) {
          v[u] = __ldcs(reinterpret_cast<const float4*>(xc + a));
        } else {
          if (a >= 0 && a < Nin) v[u].x = __ldcs(xc + a);
          if (a + 1 >= 0 && a + 1 < Nin) v[u].y = __ldcs(xc + a + 1);
          if (a + 2 >= 0 && a + 2 < Nin) v[u].z = __ldcs(xc + a + 2);
          if (a + 3 >= 0 && a + 3 < Nin) v[u].w = __ldcs(xc + a + 3);
        }
      }
    }
    float* base[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) base[j] = xs + ((j - o) & 3) * RowW + ct_pos(k0 + ((j - o) >> 2));
#pragma unroll
    for (int u = 0; u < kV; ++u) {
      if (k0 + u * kThr >= nk) break;
      base[0][u * kInc] = v[u].x;
      base[1][u * kInc] = v[u].y;
      base[2][u * kInc] = v[u].z;
      base[3][u * kInc] = v[u].w;
    }
  }
  __syncthreads();
  const int tt = tid * kBbR;
  if (tt >= MO || m0 + tt >= Nout) return;
  float2 acc[kBbR];
#pragma unroll
  for (int r = 0; r < kBbR; ++r) acc[r] = make_float2(0.f, 0.f);
#pragma unroll
  for (int q = 0; q < D; ++q) {
    const float* row = xs + q * RowW + ct_pos(tt);   // tt is a multiple of 8: group tt / 8
    const float2* gq = gs + q * Apad;
    float wa[kBbR], wb[kBbR];
    auto ld8 = [&](float (&w)[kBbR], const float* p) {
      const float4 lo = *reinterpret_cast<const float4*>(p), hi = *reinterpret_cast<const float4*>(p + 4);
      w[0] = lo.x; w[1] = lo.y; w[2] = lo.z; w[3] = lo.w; w[4] = hi.x; w[5] = hi.y; w[6] = hi.z; w[7] = hi.w;
    };
    ld8(wa, row);
    for (int ab = 0; ab < Apad; ab += 16, row += 24) {
      ld8(wb, row + 12);
      ct_block(acc, wa, wb, gq + ab);
      if (ab + 8 >= Apad) break;
      ld8(wa, row + 24);
      ct_block(acc, wb, wa, gq + ab + 8);
    }
  }
  // y[m] = w(n_m) acc, n_m = m D + half: exact phasor at the first output, rotated for the next 7
  double ph = fma((double)(m0 + tt) * D + half, kr, bp);
  ph -= rint(ph);
  float2 w;
  __sincosf(-6.283185307179586f * (float)ph, &w.y, &w.x);
  const float2 rotDp = make_float2(-rotD.y, rotD.x);
  float2* yo = out + ch * (long long)Nout + m0 + tt;
  float2 y[kBbR];
#pragma unroll
  for (int r = 0; r < kBbR; ++r) {
    if (r) w = __ffma2_rn(make_float2(w.y, w.y), rotDp, __fmul2_rn(make_float2(w.x, w.x), rotD));
    y[r] = __ffma2_rn(make_float2(acc[r].y, acc[r].y), make_float2(-w.y, w.x), __fmul2_rn(make_float2(acc[r].x, acc[r].x), w));
  }
  if (m0 + tt + kBbR <= Nout && ((((uintptr_t)yo) & 15) == 0)) {
#pragma unroll
    for (int r = 0; r < kBbR; r += 2) st_cs_v4(yo + r, y[r], y[r + 1]);
  } else {
#pragma unroll
    for (int r = 0; r < kBbR; ++r)
      if (m0 + tt + r < Nout) __stcs(yo + r, y[r]);
  }
}

cudaError_t set_bb_smem(int D, size_t smem) {
  auto kern = D == 2 ? baseband_blocked_kernel<2> : D == 4 ? baseband_blocked_kernel<4>
            : D == 8 ? baseband_blocked_kernel<8> : baseband_blocked_kernel<0>;
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

}  // namespace

// ---------------------------------------------------------------- C ABI

extern "C" sas_status sas_upsample_device(const void* in_dev, int32_t nch, int32_t Ns, int32_t U, void* out_dev,
                                          void* cuda_stream) {
  sasbp_set_error("");
  if (nch < 1 || Ns < 1) return cond_fail(SAS_E_INVALID, "nch and Ns must be >= 1");
  if (U < 1 || U > kUpMax) return cond_fail(SAS_E_INVALID, "U must be in 1..16");
  if (!in_dev || !out_dev) return cond_fail(SAS_E_INVALID, "NULL pointer");
  if ((((uintptr_t)in_dev) & 7) || (((uintptr_t)out_dev) & 15))
    return cond_fail(SAS_E_INVALID, "in_dev must be 8-byte and out_dev 16-byte aligned");
  if ((long double)nch * Ns * U > 4.0e15L) return cond_fail(SAS_E_INVALID, "nch*Ns*U too large");
  UpWeights W{};
  for (int r = 0; r < U; ++r)
    for (int m = -3; m <= 4; ++m) W.w[r][m + 3] = (float)lanczos4_host((double)r / U - m);
  const long long segs = (Ns + kUpSeg - 1) / kUpSeg;
  const long long blocks = segs * nch;
  if (blocks > 2147483647LL) return cond_fail(SAS_E_INVALID, "too many channels for one launch");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const float2* in = (const float2*)in_dev;
  float2* out = (float2*)out_dev;
  switch (U) {
    case 2: upsample_kernel<2><<<(unsigned)blocks, kUpThreads, 0, st>>>(in, Ns, U, segs, W, out); break;
    case 4: upsample_kernel<4><<<(unsigned)blocks, kUpThreads, 0, st>>>(in, Ns, U, segs, W, out); break;
    case 8: upsample_kernel<8><<<(unsigned)blocks, kUpThreads, 0, st>>>(in, Ns, U, segs, W, out); break;
    default: upsample_kernel<0><<<(unsigned)blocks, kUpThreads, 0, st>>>(in, Ns, U, segs, W, out); break;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cond_fail(SAS_E_CUDA, "upsample_kernel launch", e);
  return SAS_OK;
}

extern "C" sas_status sas_upsample(const float* in, int32_t nch, int32_t Ns, int32_t U, float* out) {
  sasbp_set_error("");
  if (!in || !out) return cond_fail(SAS_E_INVALID, "NULL pointer");
  if (nch < 1 || Ns < 1 || U < 1 || U > kUpMax) return cond_fail(SAS_E_INVALID, "nch, Ns >= 1 and U in 1..16 required");
  const size_t n = (size_t)nch * Ns;
  cudaStream_t st = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (e != cudaSuccess) return cond_fail(SAS_E_CUDA, "cudaStreamCreate", e);
  float2 *din = nullptr, *dout = nullptr;
  sas_status rs = SAS_OK;
  if (cudaMalloc(&din, n * sizeof(float2)) != cudaSuccess || cudaMalloc(&dout, n * U * sizeof(float2)) != cudaSuccess)
    rs = cond_fail(SAS_E_NOMEM, "cudaMalloc failed in sas_upsample");
  if (rs == SAS_OK && (e = cudaMemcpyAsync(din, in, n * sizeof(float2), cudaMemcpyHostToDevice, st)) != cudaSuccess)
    rs = cond_fail(SAS_E_CUDA, "H2D copy", e);
  if (rs == SAS_OK) rs = sas_upsample_device(din, nch, Ns, U, dout, st);
  if (rs == SAS_OK) {
    e = cudaMemcpyAsync(out, dout, n * U * sizeof(float2), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rs = cond_fail(SAS_E_CUDA, "D2H copy", e);
  }
  cudaStreamSynchronize(st);
  cudaFree(din);
  cudaFree(dout);
  cudaStreamDestroy(st);
  return rs;
}

// Fully asynchronous launch (all operands on the device): no host staging, no allocation.
static sas_status bb_launch(const float* x, int32_t P, int32_t E, int32_t Nin, double fs_in, double fc, const double* t0,
                            const float* h, int32_t Nh, int32_t D, int32_t Nout, float2* out, cudaStream_t st) {
  double kr = fc / fs_in;                     // cycles per input sample, mod 1
  kr -= std::floor(kr);
  // blocked polyphase kernel: 8 outputs per thread, threads = 256 / 128 / 64 / 32 so that the
  // padded polyphase arrays fit shared memory
  const int A = (Nh + D - 1) / D;             // taps per phase
  const int Apad = (A + 7) & ~7;
  // 128 threads (1024 outputs, ~37 KB of polyphase staging) per CTA: 6 CTAs/SM interleave their
  // stage and FIR phases better than 3 of 256 (A/B on config 2: 3.17 vs 3.65 ms)
  int threads = 128;
  if (const char* tv = getenv("SASBP_BB_THREADS")) {   // A/B knob: CTA size of the blocked kernel
    const int t = atoi(tv);
    if (t == 32 || t == 64 || t == 128 || t == 256) threads = t;
  }
  size_t smem = 0;
  for (; threads >= 32; threads >>= 1) {
    const long long MOb = (long long)threads * kBbR;
    const long long Lq = MOb + Apad;
    const long long LqP = Lq + (Lq >> 3) + 3;
    smem = ((size_t)D * Apad + (size_t)D * LqP + 2) * sizeof(float2);
    if (smem <= 200 * 1024) break;
  }
  const char* force = getenv("SASBP_BB_SIMPLE");
  cudaError_t e = cudaSuccess;
  const char* legacy = getenv("SASBP_BB_LEGACY");
  if (D == 4 && (Nin % 4) == 0 && (((uintptr_t)x) & 15) == 0 && !(force && force[0] == '1') &&
      !(legacy && legacy[0] == '1')) {
    // complex-tap kernel (128 threads, 1024 outputs per CTA)
    const int thr = 128;
    const int MOb = thr * kBbR;
    const int Lq = MOb + Apad;
    const int RowW = ((ct_pos(Lq) + 1 + 8) + 3) & ~3;   // >= 8 words of slack after the last slot
    const size_t csmem = (size_t)D * Apad * sizeof(float2) + ((size_t)kCtLead + (size_t)D * RowW + 4) * sizeof(float);
    const long long runs = (Nout + MOb - 1) / MOb;
    const long long blocks = runs * (long long)P * E;
    if (blocks > 2147483647LL) return cond_fail(SAS_E_INVALID, "too many channels for one launch");
    if (csmem <= 200 * 1024) {
      if (csmem > 48 * 1024)
        e = cudaFuncSetAttribute(baseband_ctap_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csmem);
      if (e == cudaSuccess) {
        const double aD = 2.0 * 3.141592653589793 * kr * D;
        baseband_ctap_kernel<<<(unsigned)blocks, thr, csmem, st>>>(
            x, E, Nin, kr, fc, t0, h, Nh, Apad, Nout, MOb, runs, RowW,
            make_float2((float)std::cos(aD), (float)-std::sin(aD)), out);
        e = cudaGetLastError();
      }
      if (e != cudaSuccess) return cond_fail(SAS_E_CUDA, "baseband_ctap_kernel", e);
      return SAS_OK;
    }
  }
  if (threads >= 32 && !(force && force[0] == '1')) {
    const int MOb = threads * kBbR;
    const long long runs = (Nout + MOb - 1) / MOb;
    const long long blocks = runs * (long long)P * E;
    if (blocks > 2147483647LL) return cond_fail(SAS_E_INVALID, "too many channels for one launch");
    e = set_bb_smem(D, smem);
    if (e == cudaSuccess) {
      auto kern = D == 2 ? baseband_blocked_kernel<2> : D == 4 ? baseband_blocked_kernel<4>
                : D == 8 ? baseband_blocked_kernel<8> : baseband_blocked_kernel<0>;
      // float4 staging: D = 4 and every channel row 16-byte aligned (SASBP_BB_VEC4=0 disables, A/B)
      const char* nv = getenv("SASBP_BB_VEC4");
      const int vec4 = (D == 4 && (Nin % 4) == 0 && (((uintptr_t)x) & 15) == 0 && !(nv && nv[0] == '0')) ? 1 : 0;
      kern<<<(unsigned)blocks, threads, smem, st>>>(
          x, E, Nin, kr, fc, t0, h, Nh, D, Apad, Nout, MOb, runs,
          make_float2((float)std::cos(2.0 * 3.141592653589793 * kr), (float)-std::sin(2.0 * 3.141592653589793 * kr)),
          out, vec4);
      e = cudaGetLastError();
    }
    if (e != cudaSuccess) return cond_fail(SAS_E_CUDA, "baseband_blocked_kernel", e);
    return SAS_OK;
  }
  // simple kernel (very large decimation): the mixed span (MO - 1) D + Nh fits kBbSmem bytes
  const int tap_bytes = ((Nh + 3) & ~3) * 4;
  const long long cap = (kBbSmem - tap_bytes) / 8;                      // complex samples
  long long MO = (cap - Nh) / D + 1;
  if (MO < 1) return cond_fail(SAS_E_UNSUPPORTED, "decimation too large for one CTA's staging buffer");
  MO = std::min<long long>(MO, 2048);
  MO = std::min<long long>(MO, Nout);
  const long long span = (MO - 1) * D + Nh;
  const long long Lq = (span + D - 1) / D;
  const size_t smem2 = (size_t)tap_bytes + (size_t)D * Lq * 8;
  const long long runs = (Nout + MO - 1) / MO;
  const long long blocks = runs * (long long)P * E;
  if (blocks > 2147483647LL) return cond_fail(SAS_E_INVALID, "too many channels for one launch");
  if (smem2 > 48 * 1024) e = cudaFuncSetAttribute(baseband_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
  if (e == cudaSuccess) {
    baseband_kernel<<<(unsigned)blocks, kBbThreads, smem2, st>>>(x, E, Nin, kr, fc, t0, h, Nh, D, Nout, (int)MO, runs, out);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) return cond_fail(SAS_E_CUDA, "baseband_kernel", e);
  return SAS_OK;
}

static sas_status bb_check(int32_t P, int32_t E, int32_t Nin, double fs_in, double fc, int32_t Nh, int32_t D,
                           int32_t Nout) {
  if (P < 1 || E < 1 || Nin < 1 || Nout < 1 || D < 1) return cond_fail(SAS_E_INVALID, "P, E, Nin, Nout, D must be >= 1");
  if (Nh < 1 || Nh > kBbMaxNh || (Nh % 2) == 0) return cond_fail(SAS_E_INVALID, "Nh must be odd and in 1..1023");
  if (!(std::isfinite(fs_in) && fs_in > 0) || !(std::isfinite(fc) && fc > 0))
    return cond_fail(SAS_E_INVALID, "fs_in and fc must be finite and > 0");
  if ((long double)P * E * ((long double)Nin + Nout) > 4.0e15L) return cond_fail(SAS_E_INVALID, "sizes too large");
  return SAS_OK;
}

extern "C" sas_status sas_baseband_device(const void* x_dev, int32_t P, int32_t E, int32_t Nin, double fs_in,
                                          double fc, const double* t0_dev, const float* h_dev, int32_t Nh, int32_t D,
                                          int32_t Nout, void* out_dev, void* cuda_stream) {
  sasbp_set_error("");
  sas_status st = bb_check(P, E, Nin, fs_in, fc, Nh, D, Nout);
  if (st != SAS_OK) return st;
  if (!x_dev || !h_dev || !out_dev) return cond_fail(SAS_E_INVALID, "NULL pointer");
  if ((((uintptr_t)x_dev) & 3) || (((uintptr_t)out_dev) & 7) || (((uintptr_t)t0_dev) & 7) || (((uintptr_t)h_dev) & 3))
    return cond_fail(SAS_E_INVALID, "misaligned pointer");
  return bb_launch((const float*)x_dev, P, E, Nin, fs_in, fc, t0_dev, h_dev, Nh, D, Nout, (float2*)out_dev,
                   (cudaStream_t)cuda_stream);
}

extern "C" sas_status sas_baseband(const float* x, int32_t P, int32_t E, int32_t Nin, double fs_in, double fc,
                                   const double* t0, const float* h, int32_t Nh, int32_t D, int32_t Nout, float* out) {
  sasbp_set_error("");
  if (!x || !h || !out) return cond_fail(SAS_E_INVALID, "NULL pointer");
  sas_status rs = bb_check(P, E, Nin, fs_in, fc, Nh, D, Nout);
  if (rs != SAS_OK) return rs;
  for (int32_t k = 0; k < Nh; ++k)
    if (!std::isfinite(h[k])) return cond_fail(SAS_E_INVALID, "non-finite FIR tap");
  if (t0)
    for (int32_t p = 0; p < P; ++p)
      if (!std::isfinite(t0[p])) return cond_fail(SAS_E_INVALID, "non-finite t0");
  const size_t nin = (size_t)P * E * Nin, nout = (size_t)P * E * Nout;
  cudaStream_t st = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (e != cudaSuccess) return cond_fail(SAS_E_CUDA, "cudaStreamCreate", e);
  float *dx = nullptr, *dh = nullptr;
  double* dt0 = nullptr;
  float2* dout = nullptr;
  if (cudaMalloc(&dx, nin * sizeof(float)) != cudaSuccess || cudaMalloc(&dout, nout * sizeof(float2)) != cudaSuccess ||
      cudaMalloc(&dh, (size_t)Nh * sizeof(float)) != cudaSuccess ||
      (t0 && cudaMalloc(&dt0, (size_t)P * sizeof(double)) != cudaSuccess))
    rs = cond_fail(SAS_E_NOMEM, "cudaMalloc failed in sas_baseband");
  if (rs == SAS_OK) {
    e = cudaMemcpyAsync(dx, x, nin * sizeof(float), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dh, h, (size_t)Nh * sizeof(float), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess && t0) e = cudaMemcpyAsync(dt0, t0, (size_t)P * sizeof(double), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) rs = cond_fail(SAS_E_CUDA, "H2D copy", e);
  }
  if (rs == SAS_OK) rs = bb_launch(dx, P, E, Nin, fs_in, fc, dt0, dh, Nh, D, Nout, dout, st);
  if (rs == SAS_OK) {
    e = cudaMemcpyAsync(out, dout, nout * sizeof(float2), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rs = cond_fail(SAS_E_CUDA, "D2H copy", e);
  }
  cudaStreamSynchronize(st);
  cudaFree(dx);
  cudaFree(dh);
  cudaFree(dt0);
  cudaFree(dout);
  cudaStreamDestroy(st);
  return rs;
}
