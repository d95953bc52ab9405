// rangecompress.cu -- K1, matched-filter range compression (the paper
// presumes compressed data; reading R14 in DESIGN.md):
//   out[ch][n] = sum_{m=0}^{Nr-1} raw[ch][n+m] * conj(replica[m]),  raw zero past Ns.
//
// FFT overlap-save path (Nr <= 2048): per CTA one block of L = 4096 input samples of one channel
// -> forward FFT -> times H[k] = conj(R[k]) / L (R = FFT of the zero-padded replica, one
// prep launch per call) -> inverse FFT -> the V = L - Nr + 1 alias-free outputs.  The FFT is a
// radix-16 Stockham in shared memory: 256 threads each own one 16-point butterfly per pass,
// 3 passes per transform; the first forward pass reads global memory directly, the last forward
// pass hands its registers straight to the first inverse pass (the spectrum product needs no
// reordering), the last inverse pass writes global memory; smem indices are padded by one
// complex per 16 so every pass is bank-conflict free.  Twiddles come from a 4096-entry table
// computed in double precision.  HBM traffic: the block inputs (L / V of the channel) + outputs.
//
// Direct path (2048 < Nr <= 8192): correlation in shared memory (FP32 complex MAC).
#include "sasbp.h"

#include <algorithm>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <cuda_runtime.h>

extern "C" void sasbp_set_error(const char* msg);  // sasbp.cu: the thread-local sas_last_error buffer

namespace {

// ---------------------------------------------------------------- direct correlation

constexpr int kRcThreads = 256;
constexpr int kRcOut = 4;                         // outputs per thread
constexpr int kRcTile = kRcThreads * kRcOut;      // outputs per CTA
constexpr int kRcMaxNr = 8192;

__global__ void __launch_bounds__(kRcThreads) rc_direct_kernel(const float2* __restrict__ raw, int Ns,
                                                               const float2* __restrict__ rep, int Nr, int lag0,
                                                               float2* __restrict__ out) {
  extern __shared__ float2 sm[];
  float2* sr = sm;            // replica [Nr], conjugated
  float2* sx = sm + Nr;       // input span [kRcTile + Nr - 1]
  const int ch = blockIdx.y;
  const int n0 = blockIdx.x * kRcTile;
  const float2* x = raw + (size_t)ch * Ns;
  for (int m = threadIdx.x; m < Nr; m += kRcThreads) {
    float2 r = rep[m];
    sr[m] = make_float2(r.x, -r.y);
  }
  const int span = kRcTile + Nr - 1;
  for (int i = threadIdx.x; i < span; i += kRcThreads) {
    const int n = n0 + lag0 + i;          // lag0 <= 0: the filter starts before lag 0 (whitening)
    sx[i] = (n >= 0 && n < Ns) ? x[n] : make_float2(0.f, 0.f);
  }
  __syncthreads();
  float ar[kRcOut], ai[kRcOut];
#pragma unroll
  for (int j = 0; j < kRcOut; ++j) { ar[j] = 0.f; ai[j] = 0.f; }
  const int t = threadIdx.x;
#pragma unroll 4
  for (int m = 0; m < Nr; ++m) {
    const float2 r = sr[m];
#pragma unroll
    for (int j = 0; j < kRcOut; ++j) {
      const float2 v = sx[t + j * kRcThreads + m];
      ar[j] = fmaf(v.x, r.x, ar[j]);
      ar[j] = fmaf(-v.y, r.y, ar[j]);
      ai[j] = fmaf(v.x, r.y, ai[j]);
      ai[j] = fmaf(v.y, r.x, ai[j]);
    }
  }
  float2* y = out + (size_t)ch * Ns;
#pragma unroll
  for (int j = 0; j < kRcOut; ++j) {
    int n = n0 + t + j * kRcThreads;
    if (n < Ns) y[n] = make_float2(ar[j], ai[j]);
  }
}

// ---------------------------------------------------------------- FFT overlap-save

constexpr int kL = 4096;          // FFT length
constexpr int kFT = 256;          // threads (one radix-16 butterfly each per pass)
constexpr int kPad = kL + kL / 16;

__device__ __forceinline__ int pad(int i) { return i + (i >> 4); }

#ifndef RC_PAIRED
#define RC_PAIRED 1   // complex arithmetic on the sm_100 paired FP32 path (FADD2 / FMUL2 / FFMA2)
#endif

// complex product; paired: a.x (b.x, b.y) + a.y (-b.y, b.x) -- FMUL2 + FFMA2 (+ one sign flip
// unless b is a constant)
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
#if RC_PAIRED
  return __ffma2_rn(make_float2(a.y, a.y), make_float2(-b.y, b.x), __fmul2_rn(make_float2(a.x, a.x), b));
#else
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
#endif
}

__device__ __forceinline__ float2 cadd(float2 a, float2 b) {
#if RC_PAIRED
  return __fadd2_rn(a, b);
#else
  return make_float2(a.x + b.x, a.y + b.y);
#endif
}
__device__ __forceinline__ float2 csub(float2 a, float2 b) {
#if RC_PAIRED
  return __fadd2_rn(a, make_float2(-b.x, -b.y));
#else
  return make_float2(a.x - b.x, a.y - b.y);
#endif
}

// radix-4 DFT in place; INV selects exp(+i) kernels
template <bool INV>
__device__ __forceinline__ void dft4(float2& x0, float2& x1, float2& x2, float2& x3) {
  const float2 t0 = cadd(x0, x2), t1 = csub(x0, x2);
  const float2 t2 = cadd(x1, x3);
  const float2 d = csub(x1, x3);
  const float2 t3 = INV ? make_float2(-d.y, d.x) : make_float2(d.y, -d.x);   // (+/- i) * d
  x0 = cadd(t0, t2);
  x2 = csub(t0, t2);
  x1 = cadd(t1, t3);
  x3 = csub(t1, t3);
}

// base-4 digit reversal of a 16-point index: sigma(4a + b) = 4b + a (an involution)
__host__ __device__ constexpr int sig(int n) { return 4 * (n & 3) + (n >> 2); }

// 16-point DFT in registers, n = 4a + b, k = c + 4d, no data movement: input element n is read
// from slot PIN ? sig(n) : n and output element k is left in slot PIN ? k : sig(k).
template <bool INV, bool PIN>
__device__ __forceinline__ void dft16(float2 v[16]) {
  const float s = INV ? 1.f : -1.f;
#define SL(n) (PIN ? sig(n) : (n))
#pragma unroll
  for (int b = 0; b < 4; ++b) dft4<INV>(v[SL(b)], v[SL(4 + b)], v[SL(8 + b)], v[SL(12 + b)]);
  // slot SL(4c + b) = Y[b][c]; twiddle W16^{bc}
  const float c1 = 0.92387953251128674f, s1 = 0.38268343236508978f, r2 = 0.70710678118654752f;
  const float2 w[10] = {make_float2(1.f, 0.f), make_float2(c1, s * s1), make_float2(r2, s * r2), make_float2(s1, s * c1),
                        make_float2(0.f, s * 1.f), make_float2(-s1, s * c1), make_float2(-r2, s * r2), make_float2(-c1, s * s1),
                        make_float2(-1.f, 0.f), make_float2(-c1, -s * s1)};
#pragma unroll
  for (int b = 1; b < 4; ++b)
#pragma unroll
    for (int c = 1; c < 4; ++c) v[SL(4 * c + b)] = cmul(v[SL(4 * c + b)], w[b * c]);
  // radix-4 over b: X[c + 4d] lands in slot SL(4c + d) = PIN ? (c + 4d) : sig(c + 4d)
#pragma unroll
  for (int c = 0; c < 4; ++c) dft4<INV>(v[SL(4 * c)], v[SL(4 * c + 1)], v[SL(4 * c + 2)], v[SL(4 * c + 3)]);
#undef SL
}

#ifndef RC_TW_RECUR
#define RC_TW_RECUR 1
#endif
#ifndef RC_MINB
#define RC_MINB 3   // 3 CTAs per SM: 80 registers (paired complex arithmetic), measured best of 2-4
#endif
// twiddle W_4096^m (forward sign) from the global table (L1 resident)
__device__ __forceinline__ float2 twid(const float2* __restrict__ tw, int m) { return __ldg(tw + m); }

// one Stockham pass on natural-order registers: twiddle, DFT16 (output left in sig order), store
template <bool INV, int NS>
__device__ __forceinline__ void pass_store(float2 v[16], float2* sm, const float2* __restrict__ tw, int j) {
  const int k = j & (NS - 1);
  float2 w1, wr;
  (void)w1; (void)wr;
  if (NS > 1) {
#pragma unroll
    for (int r = 1; r < 16; ++r) {
#if RC_TW_RECUR
      // w_r = w_1^r by recurrence (one table load per pass; ~r ulp of phase error)
      if (r == 1) { w1 = twid(tw, (k * (256 / NS)) & (kL - 1)); if (INV) w1.y = -w1.y; wr = w1; }
      else wr = cmul(wr, w1);
      v[r] = cmul(v[r], wr);
#else
      float2 w = twid(tw, (r * k * (256 / NS)) & (kL - 1));
      if (INV) w.y = -w.y;
      v[r] = cmul(v[r], w);
#endif
    }
  }
  dft16<INV, false>(v);
  const int base = (j - k) * 16 + k;
#pragma unroll
  for (int r = 0; r < 16; ++r) sm[pad(base + r * NS)] = v[sig(r)];
}

// last pass of a transform: result left in registers, element r in slot sig(r)
template <bool INV, int NS>
__device__ __forceinline__ void pass_regs(float2 v[16], const float2* __restrict__ tw, int j) {
  const int k = j & (NS - 1);
  float2 w1, wr;
  (void)w1; (void)wr;
#pragma unroll
  for (int r = 1; r < 16; ++r) {
#if RC_TW_RECUR
    if (r == 1) { w1 = twid(tw, (k * (256 / NS)) & (kL - 1)); if (INV) w1.y = -w1.y; wr = w1; }
    else wr = cmul(wr, w1);
    v[r] = cmul(v[r], wr);
#else
    float2 w = twid(tw, (r * k * (256 / NS)) & (kL - 1));
    if (INV) w.y = -w.y;
    v[r] = cmul(v[r], w);
#endif
  }
  dft16<INV, false>(v);
}

__device__ __forceinline__ void load_smem(float2 v[16], const float2* sm, int j) {
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = sm[pad(j + r * kFT)];
}

// forward FFT of the block whose element i = j + 256 r is ld(i); bin j + 256 r is left in slot sig(r)
template <class LD>
__device__ __forceinline__ void fft_forward_ld(float2 v[16], LD ld, float2* sm, const float2* __restrict__ tw, int j) {
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = ld(j + r * kFT);
  pass_store<false, 1>(v, sm, tw, j);
  __syncthreads();
  load_smem(v, sm, j);
  __syncthreads();
  pass_store<false, 16>(v, sm, tw, j);
  __syncthreads();
  load_smem(v, sm, j);
  pass_regs<false, 256>(v, tw, j);
}

// forward FFT of x[n0 .. n0+L) (zero outside 0..Ns-1)
__device__ __forceinline__ void fft_forward(float2 v[16], const float2* __restrict__ x, int n0, int Ns, float2* sm,
                                            const float2* __restrict__ tw, int j) {
  fft_forward_ld(v, [&](int i) {
    const int n = n0 + i;
    return ((unsigned)n < (unsigned)Ns) ? __ldg(x + n) : make_float2(0.f, 0.f);
  }, sm, tw, j);
}

__global__ void __launch_bounds__(kFT) rc_twiddle_kernel(float2* tw) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m < kL) {
    double s, c;
    sincospi(-2.0 * m / kL, &s, &c);
    tw[m] = make_float2((float)c, (float)s);
  }
}

// H[k] = conj(FFT_L(replica zero padded))[k] / L, stored in natural order
__global__ void __launch_bounds__(kFT) rc_prep_kernel(const float2* __restrict__ rep, int Nr, const float2* __restrict__ tw,
                                                      float2* __restrict__ H) {
  __shared__ float2 sm[kPad];
  const int j = threadIdx.x;
  float2 v[16];
  fft_forward(v, rep, 0, Nr, sm, tw, j);
  const float sc = 1.0f / kL;
#pragma unroll
  for (int r = 0; r < 16; ++r) H[j + r * kFT] = make_float2(v[sig(r)].x * sc, -v[sig(r)].y * sc);
}

// PACK = false: block blockIdx.x of channel blockIdx.y, outputs n0 .. n0 + V (records longer than
// the block).  PACK = true (short records, S = Ns + Nr - 1 <= L): the block holds kpb whole
// channels, channel c's span x[lag0 .. lag0 + S) at positions [c S, (c + 1) S) -- the Nr - 1 zeros
// after each record keep the circular correlation of one channel from reaching the next, so each
// output n < Ns at position c S + n is alias free (c S + n + Nr - 1 < (c + 1) S <= L).  The same
// transform then serves kpb channels instead of one (config 4: Ns = 1024, Nr = 160, 3 per block).
#ifndef RC_MINB_PACK
#define RC_MINB_PACK 2   // CTAs per SM for the packed-record instantiation: its index math spilled at 3
                         // (80 registers, 148 B of spills); 2 CTAs / 128 registers: config 4 2.29 -> 2.23 ms
#endif
template <bool PACK>
__global__ void __launch_bounds__(kFT, PACK ? RC_MINB_PACK : RC_MINB) rc_fft_kernel(const float2* __restrict__ raw, int Ns, int V, int lag0,
                                                        const float2* __restrict__ H, const float2* __restrict__ tw_g,
                                                        float2* __restrict__ out, long long nch, int S, int kpb,
                                                        uint32_t mS) {
  __shared__ float2 sm[kPad];
  const int j = threadIdx.x;
  const float2* tw = tw_g;
  float2 v[16];
  size_t ch = 0;
  int n0 = 0, kc = 0;
  if (PACK) {
    ch = (size_t)blockIdx.x * kpb;
    kc = (int)min((long long)kpb, nch - (long long)ch);   // channels in this block
    const float2* x = raw + ch * Ns;
    fft_forward_ld(v, [&](int i) {
      const int c = S == 1 ? i : (int)__umulhi((uint32_t)i, mS);   // i / S (exact: i S < 2^32; S = 1 has no 32-bit magic)
      const int n = i - c * S + lag0;
      return (c < kc && (unsigned)n < (unsigned)Ns) ? __ldg(x + (size_t)c * Ns + n) : make_float2(0.f, 0.f);
    }, sm, tw, j);
  } else {
    ch = blockIdx.y;
    n0 = blockIdx.x * V;
    fft_forward(v, raw + ch * Ns, n0 + lag0, Ns, sm, tw, j);
  }
  // spectrum product in registers (slot sig(r) holds bin j + 256 r)
#pragma unroll
  for (int r = 0; r < 16; ++r) v[sig(r)] = cmul(v[sig(r)], __ldg(H + j + r * kFT));
  // inverse FFT: its first pass (no twiddles) reads this very layout (PIN: input r in slot sig(r))
  dft16<true, true>(v);
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 16; ++r) sm[pad(j * 16 + r)] = v[r];
  __syncthreads();
  load_smem(v, sm, j);
  __syncthreads();
  pass_store<true, 16>(v, sm, tw, j);
  __syncthreads();
  load_smem(v, sm, j);
  pass_regs<true, 256>(v, tw, j);
  float2* y = out + ch * Ns;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const int i = j + r * kFT;
    if (PACK) {
      const int c = S == 1 ? i : (int)__umulhi((uint32_t)i, mS);
      const int n = i - c * S;
      if (c < kc && n < Ns) y[(size_t)c * Ns + n] = v[sig(r)];
    } else {
      const int n = n0 + i;
      if (i < V && n < Ns) y[n] = v[sig(r)];
    }
  }
}

// ---------------------------------------------------------------- FFT overlap-save, pipelined (round 2)
//
// The same transform as rc_fft_kernel (same blocks, same spectrum product, same outputs), with the
// block input staged through shared memory instead of loaded by each thread:
//  * persistent CTAs (RC_PIPE_MINB per SM) walk the blocks with a grid stride;
//  * each block's input lands in a staging buffer (RC_PIPE_NBUF of them, default 1) by 1D bulk
//    copies (cp.async.bulk global -> shared, completion counted on the buffer's mbarrier): a long
//    record's block window is one copy, a packed block's records one copy each, at their positions
//    c S - lag0;
//  * the copy of block t + NBUF is issued as soon as every thread has read block t's input, so it
//    streams in while block t is transformed (rc_fft_kernel issued its 16 loads per thread and
//    waited: 3.2 long-scoreboard stall cycles per issued instruction, 58 % issue);
//  * two exchange buffers in alternation (RC_PIPE_PP): a buffer is rewritten only after the barrier
//    that follows its last reads, so each exchange needs one barrier (4 per block instead of 8);
//  * the packed layout's zero gaps are written once per CTA (copies never touch them); a ragged
//    last block and long-record blocks at a channel edge zero their uncovered span after the wait;
//  * shared-memory indices are compile-time offsets from one base per pass (pad() distributes over
//    multiples of 16).
// Requires Ns even and a 16-byte aligned raw pointer (then every copy is 16-byte aligned: records
// start at even elements, windows at start = b V + lag0 with V even, and a buffer shift s = lag0 & 1
// gives the smem side the same parity); otherwise rc_fft_kernel runs.
#ifndef RC_PIPE_MINB
#define RC_PIPE_MINB 2
#endif
#ifndef RC_PIPE_NBUF
#define RC_PIPE_NBUF 1   // staging buffers per CTA (1: block t + 1 is copied while block t is transformed; A/B: 2 no faster)
#endif
constexpr int kNBuf = RC_PIPE_NBUF;
#ifndef RC_PIPE_PP
#define RC_PIPE_PP 1     // two exchange buffers in alternation (4 barriers per block instead of 8; A/B +0-2 %)
#endif
constexpr int kNX = RC_PIPE_PP ? 2 : 1;   // exchange buffers
constexpr int kBufE = kL + 8;   // staging buffer: block element i at index s + i, s in {0, 1}; +1 rounding

__device__ __forceinline__ uint32_t rc_smaddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void rc_bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void rc_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void rc_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void rc_fence_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// one Stockham pass as pass_store, shared indices as constant offsets: pad(base + r NS) =
// pad(base) + r (NS = 1: base is a multiple of 16) or pad(base) + r * 17 NS / 16 (NS multiple of 16)
template <bool INV, int NS>
__device__ __forceinline__ void pass_store_c(float2 v[16], float2* sm, const float2* __restrict__ tw, int j) {
  const int k = j & (NS - 1);
  if (NS > 1) {
    float2 w1 = twid(tw, (k * (256 / NS)) & (kL - 1));
    if (INV) w1.y = -w1.y;
    float2 wr = w1;
#pragma unroll
    for (int r = 1; r < 16; ++r) {
      if (r > 1) wr = cmul(wr, w1);
      v[r] = cmul(v[r], wr);
    }
  }
  dft16<INV, false>(v);
  float2* p = sm + pad((j - k) * 16 + k);
  constexpr int kStep = NS == 1 ? 1 : NS + NS / 16;
#pragma unroll
  for (int r = 0; r < 16; ++r) p[r * kStep] = v[sig(r)];
}
#ifndef RC_TW16
#define RC_TW16 0   // A/B knob: the NS = 16 passes take their twiddles from a per-CTA shared table
#endif
// NS = 16 pass with table twiddles: t16[r - 1][k] = (w, j w) for the forward sign and (conj w, j conj w)
// for the inverse, w = W_256^{r k}: v w = v.x (w) + v.y (j w) is one FMUL2 + one FFMA2, and no
// recurrence (the recurrence form spends 14 complex products per pass building w_r = w_1^r)
template <bool INV>
__device__ __forceinline__ void pass_store_t16(float2 v[16], float2* sm, const float4* __restrict__ t16, int j) {
  const int k = j & 15;
#pragma unroll
  for (int r = 1; r < 16; ++r) {
    const float4 t = t16[(r - 1) * 16 + k];
    v[r] = __ffma2_rn(make_float2(v[r].y, v[r].y), make_float2(t.z, t.w),
                      __fmul2_rn(make_float2(v[r].x, v[r].x), make_float2(t.x, t.y)));
  }
  dft16<INV, false>(v);
  float2* p = sm + pad((j - k) * 16 + k);
#pragma unroll
  for (int r = 0; r < 16; ++r) p[r * 17] = v[sig(r)];
}

// load_smem with constant offsets: pad(j + 256 r) = pad(j) + 272 r
__device__ __forceinline__ void load_smem_c(float2 v[16], const float2* sm, int j) {
  const float2* p = sm + pad(j);
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = p[r * (kFT + kFT / 16)];
}

struct RcPipeArgs {
  const float2* raw;   // [nch][Ns], 16-byte aligned, Ns even
  const float2* H;     // [kL] spectrum of the filter (rc_prep_kernel)
  const float2* tw;    // [kL] twiddles
  float2* out;         // [nch][Ns]
  long long nch;
  long long nblk;      // blocks
  int Ns, V, lag0;     // long records: V even (block b of a channel starts at bi V + lag0)
  int bpc;             // long records: blocks per channel
  int S, kpb;          // packed: record stride (even, >= Ns + Nr - 1) and records per block
  uint32_t mS;         // packed: i / S as a multiply-high
};

template <bool PACK>
__global__ void __launch_bounds__(kFT, RC_PIPE_MINB) rc_pipe_kernel(const __grid_constant__ RcPipeArgs a) {
  extern __shared__ __align__(128) unsigned char rc_dsm[];
  float2* buf = reinterpret_cast<float2*>(rc_dsm);          // [kNBuf][kBufE] staging
  float2* sm = buf + kNBuf * kBufE;                          // [kNX][kPad] exchange
  float2* sm2 = sm + (kNX - 1) * kPad;
  (void)sm2;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + kNX * kPad);   // [2]
  float4* t16 = reinterpret_cast<float4*>(bar + 2);                 // [2][15][16] (RC_TW16)
  (void)t16;
  const int j = threadIdx.x;
  const int s = a.lag0 & 1;
  const uint32_t bar0 = rc_smaddr(bar), bar1 = rc_smaddr(bar + 1);

  // block b -> copies into buffer kb (thread 0 only)
  auto issue = [&](long long b, int kb) {
    const uint32_t mb = kb ? bar1 : bar0;
    float2* dst = buf + kb * kBufE;
    if (PACK) {
      const long long ch = b * a.kpb;
      const int kc = (int)min((long long)a.kpb, a.nch - ch);
      const uint32_t bytes = (uint32_t)a.Ns * 8u;
      rc_expect(mb, bytes * (uint32_t)kc);
      for (int c = 0; c < kc; ++c)
        rc_bulk_g2s(rc_smaddr(dst + s + c * a.S - a.lag0), a.raw + (size_t)(ch + c) * a.Ns, bytes, mb);
    } else {
      const long long ch = b / a.bpc;
      const int start = (int)(b - ch * a.bpc) * a.V + a.lag0;
      const int i0 = max(0, -start), i1 = min(kL, a.Ns - start);
      const int cs = (s + i0) & ~1;
      int ce = (s + i1 + 1) & ~1;
      if (start + ce - s > a.Ns) ce -= 2;   // never read past the channel end (tail element loaded in the edge fix)
      const uint32_t bytes = ce > cs ? (uint32_t)(ce - cs) * 8u : 0u;
      rc_expect(mb, bytes);
      if (bytes) rc_bulk_g2s(rc_smaddr(dst + cs), a.raw + (size_t)ch * a.Ns + (start + cs - s), bytes, mb);
    }
  };

  // one-time: zero both staging buffers (the packed gaps stay zero), init the mbarriers
  for (int i = j; i < kNBuf * kBufE; i += kFT) buf[i] = make_float2(0.f, 0.f);
  if (RC_TW16) {
    for (int i = j; i < 2 * 15 * 16; i += kFT) {
      const int dir = i / 240, r = (i % 240) / 16 + 1, k = i % 16;
      float2 w = __ldg(a.tw + ((r * k * 16) & (kL - 1)));   // W_4096^{16 r k}, forward sign
      if (dir) w.y = -w.y;
      t16[i] = make_float4(w.x, w.y, -w.y, w.x);
    }
  }
  if (j == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  rc_fence_async();
  __syncthreads();
  const long long G = gridDim.x;
  if (j == 0) {
    if (blockIdx.x < a.nblk) issue(blockIdx.x, 0);
    if (kNBuf > 1 && blockIdx.x + G < a.nblk) issue(blockIdx.x + G, 1);
  }
  float2 v[16];
  int t = 0;
  for (long long b = blockIdx.x; b < a.nblk; b += G, ++t) {
    const int kb = kNBuf > 1 ? (t & 1) : 0;
    float2* in = buf + kb * kBufE;
    rc_wait(kb ? bar1 : bar0, (uint32_t)(kNBuf > 1 ? t >> 1 : t) & 1u);
    long long ch;
    int n0 = 0, kc = 0;
    if (PACK) {
      ch = b * a.kpb;
      kc = (int)min((long long)a.kpb, a.nch - ch);
      if (kc < a.kpb) {   // ragged last block: clear the slots of the missing records (stale data)
        for (int i = s + kc * a.S; i < s + kL; i += kFT) if (i + j < s + kL) in[i + j] = make_float2(0.f, 0.f);
        rc_fence_async();
        __syncthreads();
      }
    } else {
      ch = b / a.bpc;
      n0 = (int)(b - ch * a.bpc) * a.V;
      const int start = n0 + a.lag0;
      const int i0 = max(0, -start), i1 = min(kL, a.Ns - start);
      const bool fix = start + ((s + i1 + 1) & ~1) - s > a.Ns;   // issue() left the channel's last element out
      if (i0 > 0 || i1 < kL || fix) {   // channel edge: zero the span outside the record, copy the tail element
        for (int i = j; i < i0; i += kFT) in[s + i] = make_float2(0.f, 0.f);
        for (int i = i1 + j; i < kL; i += kFT) in[s + i] = make_float2(0.f, 0.f);
        if (j == 0 && fix) in[s + i1 - 1] = __ldg(a.raw + (size_t)ch * a.Ns + a.Ns - 1);
        rc_fence_async();
        __syncthreads();
      }
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = in[s + j + r * kFT];
#if RC_PIPE_PP
    // two exchange buffers X = sm, Y = sm2 alternate, so one barrier per exchange suffices: a buffer
    // is rewritten only after the barrier that follows its last reads
    pass_store_c<false, 1>(v, sm, a.tw, j);
    __syncthreads();   // every thread has read this input; X complete
    if (j == 0 && b + kNBuf * G < a.nblk) issue(b + kNBuf * G, kb);
    load_smem_c(v, sm, j);
    if (RC_TW16) pass_store_t16<false>(v, sm2, t16, j); else pass_store_c<false, 16>(v, sm2, a.tw, j);
    __syncthreads();
    load_smem_c(v, sm2, j);
    pass_regs<false, 256>(v, a.tw, j);
#pragma unroll
    for (int r = 0; r < 16; ++r) v[sig(r)] = cmul(v[sig(r)], __ldg(a.H + j + r * kFT));
    dft16<true, true>(v);
    {
      float2* p = sm + 17 * j;   // pad(16 j + r) = 17 j + r
#pragma unroll
      for (int r = 0; r < 16; ++r) p[r] = v[r];
    }
    __syncthreads();
    load_smem_c(v, sm, j);
    if (RC_TW16) pass_store_t16<true>(v, sm2, t16 + 240, j); else pass_store_c<true, 16>(v, sm2, a.tw, j);
    __syncthreads();
    load_smem_c(v, sm2, j);
    pass_regs<true, 256>(v, a.tw, j);
#else
    __syncthreads();   // every thread has read this input and is done with the previous block's exchange reads
    if (j == 0 && b + kNBuf * G < a.nblk) issue(b + kNBuf * G, kb);
    // forward FFT (bin j + 256 r left in slot sig(r))
    pass_store_c<false, 1>(v, sm, a.tw, j);
    __syncthreads();
    load_smem_c(v, sm, j);
    __syncthreads();
    if (RC_TW16) pass_store_t16<false>(v, sm, t16, j); else pass_store_c<false, 16>(v, sm, a.tw, j);
    __syncthreads();
    load_smem_c(v, sm, j);
    pass_regs<false, 256>(v, a.tw, j);
#pragma unroll
    for (int r = 0; r < 16; ++r) v[sig(r)] = cmul(v[sig(r)], __ldg(a.H + j + r * kFT));
    dft16<true, true>(v);
    __syncthreads();
    {
      float2* p = sm + 17 * j;   // pad(16 j + r) = 17 j + r
#pragma unroll
      for (int r = 0; r < 16; ++r) p[r] = v[r];
    }
    __syncthreads();
    load_smem_c(v, sm, j);
    __syncthreads();
    if (RC_TW16) pass_store_t16<true>(v, sm, t16 + 240, j); else pass_store_c<true, 16>(v, sm, a.tw, j);
    __syncthreads();
    load_smem_c(v, sm, j);
    pass_regs<true, 256>(v, a.tw, j);
#endif
    if (PACK) {
      float2* y = a.out + (size_t)ch * a.Ns;
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const int i = j + r * kFT;
        const int c = (int)__umulhi((uint32_t)i, a.mS);
        const int n = i - c * a.S;
        if (c < kc && n < a.Ns) __stcs(y + (size_t)c * a.Ns + n, v[sig(r)]);
      }
    } else {
      float2* y = a.out + (size_t)ch * a.Ns + n0;
      const int lim = min(a.V, a.Ns - n0);
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const int i = j + r * kFT;
        if (i < lim) __stcs(y + i, v[sig(r)]);
      }
    }
  }
}

sas_status rc_cuda_fail(const char* what, cudaError_t e) {
  char buf[256];
  snprintf(buf, sizeof(buf), "%s: %s", what, cudaGetErrorString(e));
  sasbp_set_error(buf);
  return SAS_E_CUDA;
}

// per-device twiddle table, built once
std::mutex g_tw_mu;
float2* g_tw[64] = {nullptr};

sas_status twiddles(float2** out, cudaStream_t st) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return rc_cuda_fail("cudaGetDevice", e);
  if (dev < 0 || dev >= 64) { sasbp_set_error("device index out of range"); return SAS_E_UNSUPPORTED; }
  std::lock_guard<std::mutex> lk(g_tw_mu);
  if (!g_tw[dev]) {
    float2* t = nullptr;
    e = cudaMalloc(&t, kL * sizeof(float2));
    if (e != cudaSuccess) { sasbp_set_error("cudaMalloc(twiddles) failed"); return SAS_E_NOMEM; }
    rc_twiddle_kernel<<<kL / kFT, kFT, 0, st>>>(t);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { cudaFree(t); return rc_cuda_fail("rc_twiddle_kernel", e); }
    g_tw[dev] = t;
  }
  *out = g_tw[dev];
  return SAS_OK;
}

}  // namespace

static sas_status rc_launch_direct(const float2* raw, long nch, int32_t Ns, const float2* rep, int32_t Nr, float2* out,
                                   cudaStream_t st, int lag0 = 0) {
  const size_t smem = sizeof(float2) * ((size_t)Nr + kRcTile + Nr - 1);
  cudaError_t e = cudaFuncSetAttribute(rc_direct_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return rc_cuda_fail("cudaFuncSetAttribute(rc_direct_kernel)", e);
  for (long c0 = 0; c0 < nch; c0 += 65535) {
    const unsigned n = (unsigned)((nch - c0) < 65535 ? (nch - c0) : 65535);
    dim3 grid((Ns + kRcTile - 1) / kRcTile, n);
    rc_direct_kernel<<<grid, kRcThreads, smem, st>>>(raw + c0 * Ns, Ns, rep, Nr, lag0, out + c0 * Ns);
    e = cudaGetLastError();
    if (e != cudaSuccess) return rc_cuda_fail("rc_direct_kernel launch", e);
  }
  return SAS_OK;
}

static sas_status rc_launch_fft(const float2* raw, long nch, int32_t Ns, const float2* rep, int32_t Nr, float2* out,
                                cudaStream_t st, int lag0 = 0) {
  float2* tw = nullptr;
  sas_status s = twiddles(&tw, st);
  if (s != SAS_OK) return s;
  float2* H = nullptr;
  cudaError_t e = cudaMallocAsync(&H, kL * sizeof(float2), st);
  if (e != cudaSuccess) return rc_cuda_fail("cudaMallocAsync(H)", e);
  rc_prep_kernel<<<1, kFT, 0, st>>>(rep, Nr, tw, H);
  e = cudaGetLastError();
  const int V = kL - Nr + 1;
  const int S = Ns + Nr - 1;             // a record's span including the Nr - 1 zeros after it
  const char* nopack = getenv("SASBP_RC_NOPACK");
  const bool pack = S <= kL / 2 && !(nopack && nopack[0] == '1');   // >= 2 whole records per transform
  const char* legacy = getenv("SASBP_RC_LEGACY");
  if (e == cudaSuccess && (Ns & 1) == 0 && ((uintptr_t)raw & 15) == 0 && !(legacy && legacy[0] == '1')) {
    RcPipeArgs a;
    a.raw = raw; a.H = H; a.tw = tw; a.out = out; a.nch = nch; a.Ns = Ns; a.lag0 = lag0;
    a.V = V & ~1;                        // even block stride: every window start has the parity of lag0
    a.bpc = (Ns + a.V - 1) / a.V;
    a.S = (S + 1) & ~1;                  // even record stride: every record starts at an even element
    a.kpb = kL / a.S;
    a.mS = 0xFFFFFFFFu / (uint32_t)a.S + 1u;
    a.nblk = pack ? (nch + a.kpb - 1) / a.kpb : nch * (long long)a.bpc;
    const size_t smem = ((size_t)kNBuf * kBufE + (size_t)kNX * kPad) * sizeof(float2) + 16 + (RC_TW16 ? 480 * 16 : 0);
    int dev = 0, nsm = 0, occ = 0;
    auto kern = pack ? rc_pipe_kernel<true> : rc_pipe_kernel<false>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kFT, smem);
    if (e == cudaSuccess) {
      const long long grid = std::min<long long>(a.nblk, (long long)std::max(occ, 1) * nsm);
      kern<<<(unsigned)grid, kFT, smem, st>>>(a);
      e = cudaGetLastError();
    }
    cudaFreeAsync(H, st);
    if (e != cudaSuccess) return rc_cuda_fail("rc_pipe_kernel launch", e);
    return SAS_OK;
  }
  if (pack) {
    const int kpb = kL / S;
    const uint32_t mS = 0xFFFFFFFFu / (uint32_t)S + 1u;   // i / S as a multiply-high
    const long long nblk = (nch + kpb - 1) / kpb;
    for (long long b0 = 0; b0 < nblk && e == cudaSuccess; b0 += 0x7FFFFFFFLL) {
      const long long nb = (nblk - b0) < 0x7FFFFFFFLL ? (nblk - b0) : 0x7FFFFFFFLL;
      rc_fft_kernel<true><<<(unsigned)nb, kFT, 0, st>>>(raw + b0 * kpb * Ns, Ns, V, lag0, H, tw, out + b0 * kpb * Ns,
                                                       nch - b0 * kpb, S, kpb, mS);
      e = cudaGetLastError();
    }
  } else {
    const unsigned blocks = (unsigned)((Ns + V - 1) / V);
    for (long c0 = 0; c0 < nch && e == cudaSuccess; c0 += 65535) {
      const unsigned n = (unsigned)((nch - c0) < 65535 ? (nch - c0) : 65535);
      rc_fft_kernel<false><<<dim3(blocks, n), kFT, 0, st>>>(raw + c0 * Ns, Ns, V, lag0, H, tw, out + c0 * Ns, nch, 0, 0, 0u);
      e = cudaGetLastError();
    }
  }
  cudaFreeAsync(H, st);
  if (e != cudaSuccess) return rc_cuda_fail("rc_fft_kernel launch", e);
  return SAS_OK;
}

static sas_status rc_check(int32_t P, int32_t E, int32_t Ns, int32_t Nr) {
  if (P < 1 || E < 1 || Ns < 1 || Nr < 1) {
    sasbp_set_error("P, E, Ns, Nr must be >= 1");
    return SAS_E_INVALID;
  }
  if (Nr > kRcMaxNr) {
    sasbp_set_error("replica longer than 8192 samples is not supported");
    return SAS_E_UNSUPPORTED;
  }
  if ((long double)P * E * Ns > 9.0e15L) { sasbp_set_error("P*E*Ns too large"); return SAS_E_INVALID; }
  return SAS_OK;
}

extern "C" sas_status sas_rangecompress_device(const void* raw_dev, int32_t P, int32_t E, int32_t Ns,
                                               const void* replica_dev, int32_t Nr, void* out_dev, void* cuda_stream) {
  sasbp_set_error("");
  sas_status s = rc_check(P, E, Ns, Nr);
  if (s != SAS_OK) return s;
  if (!raw_dev || !replica_dev || !out_dev) { sasbp_set_error("NULL pointer"); return SAS_E_INVALID; }
  const long nch = (long)P * E;
  const char* force = getenv("SASBP_RC_DIRECT");
  if (Nr <= kL / 2 && !(force && force[0] == '1'))
    return rc_launch_fft((const float2*)raw_dev, nch, Ns, (const float2*)replica_dev, Nr, (float2*)out_dev,
                         (cudaStream_t)cuda_stream);
  return rc_launch_direct((const float2*)raw_dev, nch, Ns, (const float2*)replica_dev, Nr, (float2*)out_dev,
                          (cudaStream_t)cuda_stream);
}

extern "C" sas_status sas_rangecompress(const float* raw, int32_t P, int32_t E, int32_t Ns, const float* replica,
                                        int32_t Nr, float* out) {
  sasbp_set_error("");
  sas_status s = rc_check(P, E, Ns, Nr);
  if (s != SAS_OK) return s;
  if (!raw || !replica || !out) { sasbp_set_error("NULL pointer"); return SAS_E_INVALID; }
  const size_t n = (size_t)P * E * Ns;
  float2 *draw = nullptr, *dout = nullptr, *drep = nullptr;
  cudaStream_t st = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (e != cudaSuccess) return rc_cuda_fail("cudaStreamCreate", e);
  sas_status rs = SAS_OK;
  if (cudaMalloc(&draw, n * sizeof(float2)) != cudaSuccess || cudaMalloc(&dout, n * sizeof(float2)) != cudaSuccess ||
      cudaMalloc(&drep, (size_t)Nr * sizeof(float2)) != cudaSuccess) {
    sasbp_set_error("cudaMalloc failed in sas_rangecompress");
    rs = SAS_E_NOMEM;
  }
  if (rs == SAS_OK) {
    e = cudaMemcpyAsync(draw, raw, n * sizeof(float2), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(drep, replica, (size_t)Nr * sizeof(float2), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) rs = rc_cuda_fail("H2D copy", e);
  }
  if (rs == SAS_OK) rs = sas_rangecompress_device(draw, P, E, Ns, drep, Nr, dout, st);
  if (rs == SAS_OK) {
    e = cudaMemcpyAsync(out, dout, n * sizeof(float2), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rs = rc_cuda_fail("D2H copy", e);
  }
  cudaStreamSynchronize(st);
  cudaFree(draw); cudaFree(dout); cudaFree(drep);
  cudaStreamDestroy(st);
  return rs;
}

// ---------------------------------------------------------------- spectral whitening (NEXT-4, R21)
//
// Eq. 9: G = h(1/(gamma mean P + P)) from the batch-mean M-point periodogram P (power
// gain, max G = 1); applied as the M-tap frequency-sampling FIR of amplitude sqrt(G) composed with
// the replica, q = conj(w) (x) r (Nr + M - 1 taps starting at lag 1 - M/2), so the whitened
// compression is ONE K1 pass with a longer filter and a negative start lag (exactly the cascade
// w * x then the matched filter: y[n] = sum_l x[n + l] conj(q[l])).
//
// Periodogram kernel: threads = (block slot, bin); each thread accumulates |X_b[k]|^2 over the
// blocks its slot visits (direct M-point DFT from a shared twiddle table, M^2 complex MACs per
// block); per-CTA partial sums go to a double accumulator with one atomic per bin.

namespace {

constexpr int kWhThreads = 256;
constexpr int kWhMaxM = 256;

__global__ void __launch_bounds__(kWhThreads) wh_periodogram_kernel(const float2* __restrict__ raw, int Ns, int M, int B,
                                                                    long long items, double* __restrict__ Pacc) {
  __shared__ float2 tw[kWhMaxM];
  __shared__ float2 xs[kWhThreads];
  __shared__ float red[kWhThreads];
  const int slots = kWhThreads / M;          // blocks processed together (M <= 256)
  const int s = threadIdx.x / M, k = threadIdx.x - (threadIdx.x / M) * M;
  for (int i = threadIdx.x; i < M; i += kWhThreads) {
    double sn, cs;
    sincospi(-2.0 * i / M, &sn, &cs);
    tw[i] = make_float2((float)cs, (float)sn);
  }
  float acc = 0.f;
  for (long long it0 = (long long)blockIdx.x * slots; it0 < items; it0 += (long long)gridDim.x * slots) {
    __syncthreads();
    if (s < slots) {   // stage slot s's block: sample n = k of item it0 + s
      const long long it = it0 + s;
      float2 v = make_float2(0.f, 0.f);
      if (it < items) {
        const long long ch = it / B;
        const int b = (int)(it - ch * B);
        const int n = b * M + k;
        if (n < Ns) v = __ldcs(raw + ch * (long long)Ns + n);
      }
      xs[s * M + k] = v;
    }
    __syncthreads();
    if (s < slots && it0 + s < items) {
      float re = 0.f, im = 0.f;
      int idx = 0;
      const float2* xb = xs + s * M;
      for (int n = 0; n < M; ++n) {
        const float2 w = tw[idx];
        const float2 x = xb[n];
        re = fmaf(x.x, w.x, fmaf(-x.y, w.y, re));
        im = fmaf(x.x, w.y, fmaf(x.y, w.x, im));
        idx += k;
        if (idx >= M) idx -= M;
      }
      acc = fmaf(re, re, fmaf(im, im, acc));
    }
  }
  red[threadIdx.x] = (s < slots) ? acc : 0.f;
  __syncthreads();
  if (threadIdx.x < M) {
    double t = 0.0;
    for (int q = 0; q < slots; ++q) t += (double)red[q * M + threadIdx.x];
    atomicAdd(Pacc + threadIdx.x, t);
  }
}

// Power-of-two M: radix-2 FFT per block in shared memory instead of the direct DFT.  A CTA takes
// 512 / M blocks per iteration; inputs land bit-reversed, log2 M in-place butterfly stages follow
// (thread = (block, butterfly t)), and thread (block, t) then holds bins t and t + M/2 of its
// block -- the same two bins every iteration, accumulated in registers.
__global__ void __launch_bounds__(kWhThreads) wh_periodogram_fft_kernel(const float2* __restrict__ raw, int Ns, int M,
                                                                        int logM, int B, long long items,
                                                                        double* __restrict__ Pacc) {
  __shared__ float2 tw[kWhMaxM / 2];
  __shared__ float2 xs[2 * kWhThreads];
  __shared__ float red[2 * kWhThreads];
  const int H = M >> 1;                       // butterflies per block
  const int nb = (2 * kWhThreads) / M;        // blocks per iteration
  const int blk = threadIdx.x / H, t = threadIdx.x - (threadIdx.x / H) * H;
  for (int i = threadIdx.x; i < H; i += kWhThreads) {
    double sn, cs;
    sincospi(-2.0 * i / M, &sn, &cs);
    tw[i] = make_float2((float)cs, (float)sn);
  }
  float a0 = 0.f, a1 = 0.f;
  for (long long it0 = (long long)blockIdx.x * nb; it0 < items; it0 += (long long)gridDim.x * nb) {
    __syncthreads();
    // load: element n of block slot s goes to position bitrev(n)
    for (int i = threadIdx.x; i < 2 * kWhThreads; i += kWhThreads) {
      const int s = i / M, n = i - (i / M) * M;
      const long long it = it0 + s;
      float2 v = make_float2(0.f, 0.f);
      if (it < items) {
        const long long ch = it / B;
        const int b = (int)(it - ch * B);
        const int idx = b * M + n;
        if (idx < Ns) v = __ldcs(raw + ch * (long long)Ns + idx);
      }
      xs[s * M + (int)(__brev((unsigned)n) >> (32 - logM))] = v;
    }
    __syncthreads();
    float2* xb = xs + blk * M;
    for (int half = 1, st = H; half < M; half <<= 1, st >>= 1) {   // twiddle stride st = M / (2 half)
      const int pos = t & (half - 1);
      const int i = ((t - pos) << 1) + pos, j = i + half;
      const float2 w = tw[pos * st];
      const float2 b = xb[j];
      const float2 bw = make_float2(fmaf(b.x, w.x, -b.y * w.y), fmaf(b.x, w.y, b.y * w.x));
      const float2 a = xb[i];
      xb[i] = make_float2(a.x + bw.x, a.y + bw.y);
      xb[j] = make_float2(a.x - bw.x, a.y - bw.y);
      __syncthreads();
    }
    if (it0 + blk < items) {
      const float2 u = xb[t], v = xb[t + H];
      a0 = fmaf(u.x, u.x, fmaf(u.y, u.y, a0));
      a1 = fmaf(v.x, v.x, fmaf(v.y, v.y, a1));
    }
  }
  red[2 * threadIdx.x] = a0;       // bin t
  red[2 * threadIdx.x + 1] = a1;   // bin t + H
  __syncthreads();
  if (threadIdx.x < M) {
    const int k = threadIdx.x, tt = k < H ? k : k - H, which = k < H ? 0 : 1;
    double s = 0.0;
    for (int q = 0; q < nb; ++q) s += (double)red[2 * (q * H + tt) + which];
    atomicAdd(Pacc + k, s);
  }
}

// M = 16 R (R = 1, 2, 4, 8, 16): register-resident FFT, R lanes per block.  Lane r of a group loads
// x[R i + r], i = 0..15 (the group reads 16 R contiguous samples per load step), does the 16-point
// DFT in registers (dft16), multiplies by W_M^{r k1}, and the groups transpose through shared
// memory so lane r finishes the S = 16/R length-R DFTs over r for k1 = r S .. r S + S - 1:
// X[k1 + 16 k2] = sum_r W_R^{r k2} W_M^{r k1} Y_r[k1].  Each lane then always holds the same 16
// bins, accumulated in registers across blocks; no barriers inside the loop.
template <int R>
__device__ __forceinline__ void dftR(float2 (&z)[R]) {
  if constexpr (R == 2) {
    const float2 a = z[0], b = z[1];
    z[0] = make_float2(a.x + b.x, a.y + b.y);
    z[1] = make_float2(a.x - b.x, a.y - b.y);
  } else if constexpr (R == 4) {
    dft4<false>(z[0], z[1], z[2], z[3]);
  } else if constexpr (R == 8) {
    // radix-2 x radix-4: n = 2 a + b; X[k] with k = c + 4 d
    float2 e[4] = {z[0], z[2], z[4], z[6]}, o[4] = {z[1], z[3], z[5], z[7]};
    dft4<false>(e[0], e[1], e[2], e[3]);
    dft4<false>(o[0], o[1], o[2], o[3]);
    const float r2 = 0.70710678118654752f;
    const float2 w[4] = {make_float2(1.f, 0.f), make_float2(r2, -r2), make_float2(0.f, -1.f), make_float2(-r2, -r2)};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float2 t = cmul(o[c], w[c]);
      z[c] = make_float2(e[c].x + t.x, e[c].y + t.y);
      z[c + 4] = make_float2(e[c].x - t.x, e[c].y - t.y);
    }
  } else if constexpr (R == 16) {
    float2 v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = z[i];
    dft16<false, false>(v);
#pragma unroll
    for (int k = 0; k < 16; ++k) z[k] = v[sig(k)];
  }
}

#ifndef WH_SWZ
#define WH_SWZ 1   // XOR-swizzled transpose + padded twiddle rows (0: the round-1 layout, for A/B)
#endif
#ifndef WH_MINB
#define WH_MINB 3   // 3 CTAs per SM (72 registers, twiddles in shared memory): A/B best of 2-4 without spills
#endif
template <int R>
__global__ void __launch_bounds__(kWhThreads, WH_MINB) wh_periodogram_reg_kernel(const float2* __restrict__ raw, int Ns, int B,
                                                                        long long items, double* __restrict__ Pacc) {
  constexpr int M = 16 * R, S = 16 / R, G = kWhThreads / R;   // G blocks per CTA iteration
  constexpr int GS = 17 * R;                                     // padded complex per group
  __shared__ float2 T[G * GS];
  __shared__ float red[M];
  constexpr int WR = WH_SWZ ? 17 : 16;
  __shared__ float2 wtab[R * WR];   // W_M^{r k1} at r * 17 + k1 (row pad: the R lanes of a group read
                                    // rows r in the same step -- conflict-free), shared (frees 32 registers)
  const int r = threadIdx.x % R, g = threadIdx.x / R;
  for (int k = threadIdx.x; k < M; k += kWhThreads) red[k] = 0.f;
  for (int i = threadIdx.x; i < R * 16; i += kWhThreads) {
    float sn, cs;
    sincospif(-2.0f * (float)((i >> 4) * (i & 15)) / (float)M, &sn, &cs);
    wtab[(i >> 4) * WR + (i & 15)] = make_float2(cs, sn);
  }
  __syncthreads();
  const float2* w = wtab + r * WR;
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = 0.f;
  for (long long it = (long long)blockIdx.x * G + g; it - g < items; it += (long long)gridDim.x * G) {
    float2 v[16];
    const bool live = it < items;
    long long ch = 0;
    int b = 0;
    if (live) { ch = it / B; b = (int)(it - ch * B); }
    const float2* xb = raw + ch * (long long)Ns + (long long)b * M;
    const int nmax = live ? Ns - b * M : 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int n = R * i + r;
      v[i] = n < nmax ? __ldcs(xb + n) : make_float2(0.f, 0.f);
    }
    if constexpr (R == 1) {
      dft16<false, false>(v);
#pragma unroll
      for (int k = 0; k < 16; ++k) acc[k] = fmaf(v[sig(k)].x, v[sig(k)].x, fmaf(v[sig(k)].y, v[sig(k)].y, acc[k]));
    } else {
      dft16<false, false>(v);
      __syncwarp();
      float2* Tg = T + g * GS;
#pragma unroll
      // Z_r[k1] at row k1, column r XOR (k1 / S): the reads below take column q of rows r S + s
      // (one row per lane r), which the swizzle spreads over R bank pairs; the writes (row k1,
      // all r) stay a permutation of the row -- no bank conflicts either way (GS = 17 R
      // separates the groups of a half-warp)
      for (int k1 = 0; k1 < 16; ++k1) Tg[k1 * R + (WH_SWZ ? (r ^ ((k1 / S) & (R - 1))) : r)] = cmul(v[sig(k1)], w[k1]);
      __syncwarp();
#pragma unroll
      for (int s = 0; s < S; ++s) {
        float2 z[R];
#pragma unroll
        for (int q = 0; q < R; ++q) z[q] = Tg[(r * S + s) * R + (WH_SWZ ? (q ^ r) : q)];
        dftR<R>(z);
#pragma unroll
        for (int k2 = 0; k2 < R; ++k2) acc[s * R + k2] = fmaf(z[k2].x, z[k2].x, fmaf(z[k2].y, z[k2].y, acc[s * R + k2]));
      }
    }
  }
  // lane r holds bins k = k1 + 16 k2 with k1 = r S + s (slot s R + k2); R = 1: bin k in slot k
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int k = (R == 1) ? i : (r * S + i / R) + 16 * (i % R);
    atomicAdd(red + k, acc[i]);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < M; k += kWhThreads) atomicAdd(Pacc + k, (double)red[k]);
}

__global__ void __launch_bounds__(kWhThreads) wh_gain_kernel(const double* __restrict__ Pacc, int M, double items,
                                                             double gamma, float* __restrict__ G) {
  __shared__ double g[kWhMaxM];
  __shared__ double mean_s, gmax_s;
  __shared__ int bad;
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int k = 0; k < M; ++k) m += Pacc[k] / items;
    mean_s = m / M;
    bad = 0;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < M; k += kWhThreads) {
    const double den = gamma * mean_s + Pacc[k] / items;
    if (!(den > 0)) bad = 1;
    g[k] = 1.0 / den;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double mx = 0.0;
    for (int k = 0; k < M; ++k) mx = fmax(mx, g[k]);
    gmax_s = mx;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < M; k += kWhThreads) G[k] = bad ? __int_as_float(0x7fc00000) : (float)(g[k] / gmax_s);
}

// q[l'] = sum_i conj(w[i]) r[l' + l0 + i], l' = 0 .. Nr + M - 2, l0 = 1 - M + M/2;
// w[i] = (1/M) sum_k sqrt(G[k]) exp(+j 2 pi k i / M), i = -M/2 .. M/2 - 1 (fp64)
__global__ void __launch_bounds__(kWhThreads) wh_compose_kernel(const float2* __restrict__ rep, int Nr,
                                                                const float* __restrict__ G, int M,
                                                                float2* __restrict__ q) {
  __shared__ double2 w[kWhMaxM];
  const int i0 = -(M / 2);
  for (int t = threadIdx.x; t < M; t += kWhThreads) {
    const int i = i0 + t;
    double re = 0.0, im = 0.0;
    for (int k = 0; k < M; ++k) {
      const int km = (int)((((long long)k * i) % M + M) % M);
      double sn, cs;
      sincospi(2.0 * km / M, &sn, &cs);
      const double a = sqrt((double)G[k]);
      re += a * cs;
      im += a * sn;
    }
    w[t] = make_double2(re / M, im / M);
  }
  __syncthreads();
  const int l0 = 1 - M + M / 2;
  const int Nq = Nr + M - 1;
  for (int lp = threadIdx.x; lp < Nq; lp += kWhThreads) {
    const int l = lp + l0;
    double re = 0.0, im = 0.0;
    for (int t = 0; t < M; ++t) {
      const int m = l + i0 + t;
      if (m < 0 || m >= Nr) continue;
      const float2 r = rep[m];
      const double2 c = w[t];                     // conj(w) * r
      re += c.x * r.x + c.y * r.y;
      im += c.x * r.y - c.y * r.x;
    }
    q[lp] = make_float2((float)re, (float)im);
  }
}

sas_status wh_check(long nch, int32_t Ns, int32_t M, double gamma) {
  if (nch < 1 || Ns < 1) { sasbp_set_error("nch and Ns must be >= 1"); return SAS_E_INVALID; }
  if (M < 1 || M > kWhMaxM || (M > 1 && (M & 1))) { sasbp_set_error("M must be 1 or even, <= 256"); return SAS_E_INVALID; }
  if (!(gamma >= 0) || !std::isfinite(gamma)) { sasbp_set_error("gamma must be finite and >= 0"); return SAS_E_INVALID; }
  return SAS_OK;
}

}  // namespace

extern "C" sas_status sas_whitening_gain_device(const void* raw_dev, int32_t nch, int32_t Ns, int32_t M, double gamma,
                                                float* G_dev, void* cuda_stream) {
  sasbp_set_error("");
  sas_status s = wh_check(nch, Ns, M, gamma);
  if (s != SAS_OK) return s;
  if (!raw_dev || !G_dev) { sasbp_set_error("NULL pointer"); return SAS_E_INVALID; }
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const int B = Ns / M > 0 ? Ns / M : 1;
  const long long items = (long long)nch * B;
  double* Pacc = nullptr;
  cudaError_t e = cudaMallocAsync(&Pacc, M * sizeof(double), st);
  if (e != cudaSuccess) return rc_cuda_fail("cudaMallocAsync(P)", e);
  e = cudaMemsetAsync(Pacc, 0, M * sizeof(double), st);
  const int slots = kWhThreads / M;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long grid = (items + slots - 1) / slots;
  grid = grid < (long long)sms * 8 ? grid : (long long)sms * 8;
  const bool pow2 = M >= 2 && (M & (M - 1)) == 0;
  const char* force = getenv("SASBP_WH_DFT");
  const char* force_rad2 = getenv("SASBP_WH_RADIX2");
  if (e == cudaSuccess && pow2 && M >= 16 && !(force && force[0] == '1') && !(force_rad2 && force_rad2[0] == '1')) {
    const int R = M / 16, Gb = kWhThreads / R;
    long long g3 = (items + Gb - 1) / Gb;
    g3 = g3 < (long long)sms * 8 ? g3 : (long long)sms * 8;
    const float2* rp = (const float2*)raw_dev;
    switch (R) {
      case 1: wh_periodogram_reg_kernel<1><<<(unsigned)g3, kWhThreads, 0, st>>>(rp, Ns, B, items, Pacc); break;
      case 2: wh_periodogram_reg_kernel<2><<<(unsigned)g3, kWhThreads, 0, st>>>(rp, Ns, B, items, Pacc); break;
      case 4: wh_periodogram_reg_kernel<4><<<(unsigned)g3, kWhThreads, 0, st>>>(rp, Ns, B, items, Pacc); break;
      case 8: wh_periodogram_reg_kernel<8><<<(unsigned)g3, kWhThreads, 0, st>>>(rp, Ns, B, items, Pacc); break;
      default: wh_periodogram_reg_kernel<16><<<(unsigned)g3, kWhThreads, 0, st>>>(rp, Ns, B, items, Pacc); break;
    }
    e = cudaGetLastError();
  } else if (e == cudaSuccess && pow2 && !(force && force[0] == '1')) {
    const int nb = 2 * kWhThreads / M;
    long long g2 = (items + nb - 1) / nb;
    g2 = g2 < (long long)sms * 8 ? g2 : (long long)sms * 8;
    int logM = 0;
    while ((1 << logM) < M) ++logM;
    wh_periodogram_fft_kernel<<<(unsigned)g2, kWhThreads, 0, st>>>((const float2*)raw_dev, Ns, M, logM, B, items, Pacc);
    e = cudaGetLastError();
  } else if (e == cudaSuccess) {
    wh_periodogram_kernel<<<(unsigned)grid, kWhThreads, 0, st>>>((const float2*)raw_dev, Ns, M, B, items, Pacc);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) {
    wh_gain_kernel<<<1, kWhThreads, 0, st>>>(Pacc, M, (double)items, gamma, G_dev);
    e = cudaGetLastError();
  }
  cudaFreeAsync(Pacc, st);
  if (e != cudaSuccess) return rc_cuda_fail("whitening gain kernels", e);
  return SAS_OK;
}

extern "C" sas_status sas_whitening_gain(const float* raw, int32_t nch, int32_t Ns, int32_t M, double gamma, float* G) {
  sasbp_set_error("");
  sas_status s = wh_check(nch, Ns, M, gamma);
  if (s != SAS_OK) return s;
  if (!raw || !G) { sasbp_set_error("NULL pointer"); return SAS_E_INVALID; }
  const size_t n = (size_t)nch * Ns;
  cudaStream_t st = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (e != cudaSuccess) return rc_cuda_fail("cudaStreamCreate", e);
  float2* draw = nullptr;
  float* dG = nullptr;
  sas_status rs = SAS_OK;
  if (cudaMalloc(&draw, n * sizeof(float2)) != cudaSuccess || cudaMalloc(&dG, M * sizeof(float)) != cudaSuccess) {
    sasbp_set_error("cudaMalloc failed in sas_whitening_gain");
    rs = SAS_E_NOMEM;
  }
  if (rs == SAS_OK && (e = cudaMemcpyAsync(draw, raw, n * sizeof(float2), cudaMemcpyHostToDevice, st)) != cudaSuccess)
    rs = rc_cuda_fail("H2D copy", e);
  if (rs == SAS_OK) rs = sas_whitening_gain_device(draw, nch, Ns, M, gamma, dG, st);
  if (rs == SAS_OK) {
    e = cudaMemcpyAsync(G, dG, M * sizeof(float), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rs = rc_cuda_fail("D2H copy", e);
  }
  if (rs == SAS_OK && !(G[0] == G[0])) { sasbp_set_error("all-zero batch: no spectrum to whiten"); rs = SAS_E_INVALID; }
  cudaStreamSynchronize(st);
  cudaFree(draw);
  cudaFree(dG);
  cudaStreamDestroy(st);
  return rs;
}

extern "C" sas_status sas_rangecompress_whitened_device(const void* raw_dev, int32_t P, int32_t E, int32_t Ns,
                                                        const void* replica_dev, int32_t Nr, const float* G_dev, int32_t M,
                                                        void* out_dev, void* cuda_stream) {
  sasbp_set_error("");
  if (M < 1 || M > kWhMaxM || (M > 1 && (M & 1))) { sasbp_set_error("M must be 1 or even, <= 256"); return SAS_E_INVALID; }
  const int Nq = Nr + M - 1;
  sas_status s = rc_check(P, E, Ns, Nq);
  if (s != SAS_OK) return s;
  if (!raw_dev || !replica_dev || !G_dev || !out_dev) { sasbp_set_error("NULL pointer"); return SAS_E_INVALID; }
  cudaStream_t st = (cudaStream_t)cuda_stream;
  float2* q = nullptr;
  cudaError_t e = cudaMallocAsync(&q, Nq * sizeof(float2), st);
  if (e != cudaSuccess) return rc_cuda_fail("cudaMallocAsync(q)", e);
  wh_compose_kernel<<<1, kWhThreads, 0, st>>>((const float2*)replica_dev, Nr, G_dev, M, q);
  e = cudaGetLastError();
  if (e != cudaSuccess) { cudaFreeAsync(q, st); return rc_cuda_fail("wh_compose_kernel", e); }
  const long nch = (long)P * E;
  const int lag0 = 1 - M + M / 2;
  const char* force = getenv("SASBP_RC_DIRECT");
  if (Nq <= kL / 2 && !(force && force[0] == '1'))
    s = rc_launch_fft((const float2*)raw_dev, nch, Ns, q, Nq, (float2*)out_dev, st, lag0);
  else
    s = rc_launch_direct((const float2*)raw_dev, nch, Ns, q, Nq, (float2*)out_dev, st, lag0);
  cudaFreeAsync(q, st);
  return s;
}

extern "C" sas_status sas_rangecompress_whitened(const float* raw, int32_t P, int32_t E, int32_t Ns, const float* replica,
                                                 int32_t Nr, const float* G, int32_t M, float* out) {
  sasbp_set_error("");
  if (!raw || !replica || !G || !out) { sasbp_set_error("NULL pointer"); return SAS_E_INVALID; }
  if (M < 1 || M > kWhMaxM || (M > 1 && (M & 1))) { sasbp_set_error("M must be 1 or even, <= 256"); return SAS_E_INVALID; }
  sas_status s = rc_check(P, E, Ns, Nr + M - 1);
  if (s != SAS_OK) return s;
  for (int k = 0; k < M; ++k)
    if (!(G[k] >= 0) || !std::isfinite(G[k])) { sasbp_set_error("G must be finite and >= 0"); return SAS_E_INVALID; }
  const size_t n = (size_t)P * E * Ns;
  float2 *draw = nullptr, *dout = nullptr, *drep = nullptr;
  float* dG = nullptr;
  cudaStream_t st = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (e != cudaSuccess) return rc_cuda_fail("cudaStreamCreate", e);
  sas_status rs = SAS_OK;
  if (cudaMalloc(&draw, n * sizeof(float2)) != cudaSuccess || cudaMalloc(&dout, n * sizeof(float2)) != cudaSuccess ||
      cudaMalloc(&drep, (size_t)Nr * sizeof(float2)) != cudaSuccess || cudaMalloc(&dG, (size_t)M * sizeof(float)) != cudaSuccess) {
    sasbp_set_error("cudaMalloc failed in sas_rangecompress_whitened");
    rs = SAS_E_NOMEM;
  }
  if (rs == SAS_OK) {
    e = cudaMemcpyAsync(draw, raw, n * sizeof(float2), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(drep, replica, (size_t)Nr * sizeof(float2), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dG, G, (size_t)M * sizeof(float), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) rs = rc_cuda_fail("H2D copy", e);
  }
  if (rs == SAS_OK) rs = sas_rangecompress_whitened_device(draw, P, E, Ns, drep, Nr, dG, M, dout, st);
  if (rs == SAS_OK) {
    e = cudaMemcpyAsync(out, dout, n * sizeof(float2), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rs = rc_cuda_fail("D2H copy", e);
  }
  cudaStreamSynchronize(st);
  cudaFree(draw); cudaFree(dout); cudaFree(drep); cudaFree(dG);
  cudaStreamDestroy(st);
  return rs;
}
