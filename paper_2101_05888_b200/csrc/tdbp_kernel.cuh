// tdbp_kernel.cuh -- the time-domain backprojection kernel (K2) for sm_100a.
//
// Computes, for every pixel of a CTA tile and every channel (ping p, element e), the term
//   ehat_{p,e}(u) * exp(+j 2 pi fc tau),  tau = (|x - tx_p| + |x - rx_{p,e}|)/c,  u = (tau - t0_p) fs
// of Eq. (eqn:backprojection)'s inversion ("integrate the time-series into
// the appropriate complex pixels" P:160) and accumulates it in registers.
//
// Design ("K2"):
//  * one CTA = one pixel tile (2D: 32x32, 3D: 16x8x8), 128 threads, K = 8 pixels per thread,
//    complex accumulators in registers across ALL channels; one image store per tile;
//  * channels are processed in batches of NB.  Per batch, a fp64 prologue computes for each
//    channel the tile-centre reference geometry (rows a2): r_ref per leg, the
//    window start k_lo, the window-relative reference index and the reference phase reduced
//    mod 2 pi -- so the ~1e5-rad carrier phase never passes through fp32 (range-relative);
//  * each channel's sample window [k_lo, k_lo + W] is staged in shared memory as
//    (mid, slope) float4 pairs: mid_j = (d[k_lo+j] + d[k_lo+j+1])/2, slope_j = d[k_lo+j+1]-d[k_lo+j],
//    zero outside 0..Ns-1 (reading R2) -> the lerp is one LDS.128 + 2 FFMA (row a4);
//  * per term (rows a3-a5), fp32 and tile-relative: q = 2u.d + |d|^2, dU = q h(q/r^2) with
//    h the 4-term series of (sqrt(1+eps)-1)/eps (or the exact form for near-field plans),
//    U' = dU_tx + dU_rx + u_ref', k = rn(U') via the 1.5*2^23 trick, beta = U' - k,
//    phase = U' * 2 pi fc/fs + phi0 -> MUFU sin/cos, 4 FFMA complex MAC.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sasbp {

constexpr int kThreads = 128;   // 4 warps
constexpr int kNB = 32;         // channels per batch

struct TdbpParams {
  const float2* echoes;   // [P*E][Ns]
  const double* tx;       // [P][3]
  const double* rx;       // [P*E][3]
  const double* t0;       // [P]
  float2* image;          // [nz][ny][nx]
  unsigned long long* counter;  // COUNT mode: in-window term total
  double origin[3], sx[3], sy[3], sz[3];
  double fc, fs, c;
  double hw;              // half window in samples: 2 * d_max * fs / c
  int P, E, Ns;
  int nx, ny, nz;
  int tiles_x, tiles_y, tiles_z;
  int W;                  // window slots per channel
  int accumulate;
};

// per-channel constants in shared memory (computed by the fp64 prologue)
struct __align__(16) ChanConst {
  float ux2, uy2, uz2, ir2;     // rx leg: 2 (c_T - rx), 1 / r_r^2
  float a0, a1, a2, a3;         // rx leg series coefficients * (fs/c) / r_r
  float urr, phi0, r_r, r2_r;   // window-relative ref index - 0.5; phase offset (rad); r_r; r_r^2
  float tx2x, tx2y, tx2z, r2_t; // tx leg: 2 (c_T - tx), r_t^2
  float r_t, kfs, pad0, pad1;   // r_t, fs/c
  int ping, woff, klo, pad2;    // ping index; LDS byte offset - MAGIC*16; window start
};

constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23: x + kMagic rounds x to an integer in the low bits
constexpr int kMagicBits = 0x4B400000;

__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
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

// fp64 prologue for one channel (row a2)
__device__ __forceinline__ void chan_prologue(const TdbpParams& prm, int ch, const double ct[3],
                                              int slot, uint32_t win_base, ChanConst* out) {
  const int p = ch / prm.E;
  const double* T = prm.tx + 3 * p;
  const double* R = prm.rx + 3 * (size_t)ch;
  double utx = ct[0] - T[0], uty = ct[1] - T[1], utz = ct[2] - T[2];
  double urx = ct[0] - R[0], ury = ct[1] - R[1], urz = ct[2] - R[2];
  double r_t = sqrt(utx * utx + uty * uty + utz * utz);
  double r_r = sqrt(urx * urx + ury * ury + urz * urz);
  double K = prm.fs / prm.c;
  double t0 = prm.t0[p];
  double Uref = (r_t + r_r) * K - t0 * prm.fs;          // absolute sample index at tile centre
  double klo_d = floor(Uref - prm.hw) - 2.0;
  int klo = (int)fmax(fmin(klo_d, 2.0e9), -2.0e9);
  double urr = Uref - (double)klo - 0.5;
  double cyc = prm.fc * (r_t + r_r) / prm.c;             // reference phase in cycles (fp64)
  double ph = cyc - urr * (prm.fc / prm.fs);
  ph -= floor(ph);
  ChanConst k;
  k.ux2 = (float)(2.0 * urx); k.uy2 = (float)(2.0 * ury); k.uz2 = (float)(2.0 * urz);
  double ir = 1.0 / r_r;
  k.ir2 = (float)(ir * ir);
  double g = K * ir;
  k.a0 = (float)(0.5 * g); k.a1 = (float)(-0.125 * g); k.a2 = (float)(0.0625 * g);
  k.a3 = (float)(-0.0390625 * g);
  k.urr = (float)urr;
  k.phi0 = (float)(6.283185307179586 * ph);
  k.r_r = (float)r_r; k.r2_r = (float)(r_r * r_r);
  k.tx2x = (float)(2.0 * utx); k.tx2y = (float)(2.0 * uty); k.tx2z = (float)(2.0 * utz);
  k.r2_t = (float)(r_t * r_t); k.r_t = (float)r_t; k.kfs = (float)K;
  k.pad0 = 0.f; k.pad1 = 0.f;
  k.ping = p;
  k.woff = (int)(win_base + (uint32_t)(slot * prm.W) * 16u - (uint32_t)kMagicBits * 16u);
  k.klo = klo;
  k.pad2 = 0;
  *out = k;
}

template <int KX, int KY, int KZ, int WY, int WZ, bool HAS_DZ, bool EXACT_RX, bool COUNT>
__global__ void __launch_bounds__(kThreads, 4) tdbp_kernel(const TdbpParams prm) {
  constexpr int K = KX * KY * KZ;
  constexpr int TX = 8 * KX, TY = 4 * KY * WY, TZ = KZ * WZ;
  extern __shared__ float4 smem[];
  ChanConst* cc = reinterpret_cast<ChanConst*>(smem);
  float4* win = smem + kNB * (sizeof(ChanConst) / 16);
  const uint32_t win_base = (uint32_t)__cvta_generic_to_shared(win);

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int lx = lane >> 2, ly = lane & 3;
  const int wy = warp % WY, wz = warp / WY;

  int b = blockIdx.x;
  const int tix = b % prm.tiles_x; b /= prm.tiles_x;
  const int tiy = b % prm.tiles_y; b /= prm.tiles_y;
  const int tiz = b;
  const int x0 = tix * TX, y0 = tiy * TY, z0 = tiz * TZ;

  // tile centre (fp64) -- reference point for the range-relative geometry
  const double cxr = x0 + 0.5 * (TX - 1), cyr = y0 + 0.5 * (TY - 1), czr = z0 + 0.5 * (TZ - 1);
  double ct[3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
    ct[a] = prm.origin[a] + cxr * prm.sx[a] + cyr * prm.sy[a] + czr * prm.sz[a];

  // per-pixel offsets from the tile centre (small, exact-ish in fp32)
  float dx[K], dy[K], dz[K], dd[K], acc_re[K], acc_im[K], btx[K];
  bool valid[K];
  unsigned cnt = 0;
#pragma unroll
  for (int kz = 0; kz < KZ; ++kz)
#pragma unroll
    for (int ky = 0; ky < KY; ++ky)
#pragma unroll
      for (int kx = 0; kx < KX; ++kx) {
        const int k = (kz * KY + ky) * KX + kx;
        const float rxi = (float)(lx + 8 * kx) - 0.5f * (TX - 1);
        const float ryi = (float)(ly + 4 * ky + 4 * KY * wy) - 0.5f * (TY - 1);
        const float rzi = (float)(kz + KZ * wz) - 0.5f * (TZ - 1);
        dx[k] = rxi * (float)prm.sx[0] + ryi * (float)prm.sy[0] + rzi * (float)prm.sz[0];
        dy[k] = rxi * (float)prm.sx[1] + ryi * (float)prm.sy[1] + rzi * (float)prm.sz[1];
        dz[k] = HAS_DZ ? rxi * (float)prm.sx[2] + ryi * (float)prm.sy[2] + rzi * (float)prm.sz[2] : 0.f;
        dd[k] = dx[k] * dx[k] + dy[k] * dy[k] + dz[k] * dz[k];
        acc_re[k] = 0.f; acc_im[k] = 0.f; btx[k] = 0.f;
        valid[k] = (x0 + lx + 8 * kx < prm.nx) && (y0 + ly + 4 * ky + 4 * KY * wy < prm.ny) &&
                   (z0 + kz + KZ * wz < prm.nz);
      }

  const float kph = (float)(6.283185307179586 * prm.fc / prm.fs);
  const int nch = prm.P * prm.E;
  const int W = prm.W;
  int cur_ping = -1;

  for (int ch0 = 0; ch0 < nch; ch0 += kNB) {
    const int nb = min(kNB, nch - ch0);
    __syncthreads();
    if (tid < nb) chan_prologue(prm, ch0 + tid, ct, tid, win_base, &cc[tid]);
    __syncthreads();
    // stage windows: slot j of channel c holds (mid, slope) of samples k_lo+j, k_lo+j+1
    for (int i = tid; i < nb * W; i += kThreads) {
      const int c = i / W, j = i - c * W;
      const int n = cc[c].klo + j;
      const float2* row = prm.echoes + (size_t)(ch0 + c) * prm.Ns;
      float2 d0 = make_float2(0.f, 0.f), d1 = make_float2(0.f, 0.f);
      if (n >= 0 && n < prm.Ns) d0 = __ldg(row + n);
      if (n + 1 >= 0 && n + 1 < prm.Ns) d1 = __ldg(row + n + 1);
      win[c * W + j] = make_float4(0.5f * (d0.x + d1.x), 0.5f * (d0.y + d1.y), d1.x - d0.x, d1.y - d0.y);
    }
    __syncthreads();

#pragma unroll 1
    for (int c = 0; c < nb; ++c) {
      const ChanConst kc = cc[c];
      if (kc.ping != cur_ping) {
        cur_ping = kc.ping;
        // transmit leg, exact range-relative form: dR = q / (sqrt(r^2 + q) + r)
#pragma unroll
        for (int k = 0; k < K; ++k) {
          float q = fmaf(kc.tx2x, dx[k], fmaf(kc.tx2y, dy[k], HAS_DZ ? fmaf(kc.tx2z, dz[k], dd[k]) : dd[k]));
          float r2 = kc.r2_t + q;
          float den = fmaf(r2, rsqrt_approx(r2), kc.r_t);
          btx[k] = q * rcp_approx(den) * kc.kfs;
        }
      }
#pragma unroll
      for (int k = 0; k < K; ++k) {
        float q = fmaf(kc.ux2, dx[k], fmaf(kc.uy2, dy[k], HAS_DZ ? fmaf(kc.uz2, dz[k], dd[k]) : dd[k]));
        float du;
        if (EXACT_RX) {
          float r2 = kc.r2_r + q;
          float den = fmaf(r2, rsqrt_approx(r2), kc.r_r);
          du = q * rcp_approx(den) * kc.kfs;
          du += btx[k];
        } else {
          float e = q * kc.ir2;
          float h = fmaf(fmaf(fmaf(kc.a3, e, kc.a2), e, kc.a1), e, kc.a0);
          du = fmaf(q, h, btx[k]);
        }
        const float U = du + kc.urr;   // window-relative sample index - 0.5
        if (COUNT) {
          // absolute u = k_lo + U + 0.5 in (-1, Ns): the term's support meets the record
          const float ua = (float)kc.klo + U + 0.5f;
          cnt += (valid[k] && ua > -1.f && ua < (float)prm.Ns) ? 1u : 0u;
        } else {
          const float T = U + kMagic;
          const float beta = U - (T - kMagic);
          const uint32_t addr = (uint32_t)__float_as_int(T) * 16u + (uint32_t)kc.woff;
          const float4 w = lds128(addr);
          const float er = fmaf(beta, w.z, w.x);
          const float ei = fmaf(beta, w.w, w.y);
          float sn, cs;
          __sincosf(fmaf(U, kph, kc.phi0), &sn, &cs);
          acc_re[k] = fmaf(er, cs, acc_re[k]);
          acc_re[k] = fmaf(-ei, sn, acc_re[k]);
          acc_im[k] = fmaf(er, sn, acc_im[k]);
          acc_im[k] = fmaf(ei, cs, acc_im[k]);
        }
      }
    }
  }

  if (COUNT) {
    // warp reduce then one atomic per warp
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) atomicAdd(prm.counter, (unsigned long long)cnt);
    return;
  }

#pragma unroll
  for (int kz = 0; kz < KZ; ++kz)
#pragma unroll
    for (int ky = 0; ky < KY; ++ky)
#pragma unroll
      for (int kx = 0; kx < KX; ++kx) {
        const int k = (kz * KY + ky) * KX + kx;
        const int ix = x0 + lx + 8 * kx;
        const int iy = y0 + ly + 4 * ky + 4 * KY * wy;
        const int iz = z0 + kz + KZ * wz;
        if (valid[k]) {
          float2* o = prm.image + ((size_t)iz * prm.ny + iy) * prm.nx + ix;
          float2 v = make_float2(acc_re[k], acc_im[k]);
          if (prm.accumulate) { float2 a = *o; v.x += a.x; v.y += a.y; }
          *o = v;
        }
      }
}

}  // namespace sasbp
