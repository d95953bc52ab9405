// k2_launch.cuh -- host-side launch templates of K2 (TDBP) and K3 (term counter).
//
// The kernel instantiations are spread over several translation units (k2_*.cu), one per
// (tile variant, gating, weighting) family, so nvcc builds them in parallel; sasbp.cu only sees
// the plain entry points declared at the bottom.
#pragma once
#include <cuda_runtime.h>

#include "tdbp_kernel.cuh"

#ifndef SASBP_ROTATE
#define SASBP_ROTATE 0
#endif

namespace sasbp {

// tile variants: 2D z-level plane, 2D with z components in the steps, 3D volume
enum K2Variant { kV2D = 0, kV2D_DZ = 1, kV3D = 2 };

struct K2Launch {
  bool tma;          // TMA row staging (else cp.async)
  bool axis;         // 3D grid with diagonal steps: compact per-pixel geometry (AXIS instantiations, TMA only)
  int mode;          // receive-leg mode (kSeries3 / kSeries4 / kExact); prm.refract selects kRefract
  bool count;        // K3 instead of K2
  cudaStream_t st;
  int* occ;          // out: resident CTAs per SM of the launched kernel
  int* split = nullptr;   // out: wave-tail split factor of the launch (1 = none)
  bool gsplit = false;    // gated: two launches -- IN pairs through a mask-free kernel, then the rest (A/B knob)
};

template <typename Kern>
cudaError_t launch_k(Kern kern, int threads, const TdbpParams& prm_in, const TmaDesc& tmap, size_t smem,
                     const K2Launch& L) {
  const unsigned blocks = (unsigned)prm_in.tiles_x * prm_in.tiles_y * prm_in.tiles_z;
  if (smem > 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  TdbpParams prm = prm_in;
  int per_sm = 0, dev = 0, sms = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem) == cudaSuccess &&
      cudaGetDevice(&dev) == cudaSuccess &&
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
    prm.resident = per_sm * sms;
  if (L.occ) *L.occ = per_sm;
  // Wave tail: with T tiles over R co-resident CTAs the last wave holds T mod R tiles and, tiles
  // being equal work, takes as long as a full one.  When it is at most half full, its tiles are
  // split in two channel halves (2 CTAs each, atomic float2 adds into the zeroed image), which
  // halves the tail's time (config 2 on 8 GPUs, image-shard: 3.46 waves -> 3.5 instead of 4).
  // Not for ACCUMULATE launches (I + a + b would depend on the order) or when disabled.
  prm.tail0 = (int)blocks;
  prm.tsplit = 1;
  unsigned grid = blocks;
  const int R = per_sm * sms;
  const char* nt = getenv("SASBP_NO_TAILSPLIT");
  if (SASBP_TAILSPLIT && !(nt && nt[0] == '1') && !prm.accumulate && R > 0 && prm.ch_hi - prm.ch_lo >= 2) {
    const unsigned tail = blocks % (unsigned)R;
    if (tail > 0 && 2 * tail <= (unsigned)R) {
      prm.tail0 = (int)(blocks - tail);
      prm.tsplit = 2;
      grid = blocks + tail;
      const size_t bytes = (size_t)prm.nx * prm.ny * prm.nz * sizeof(float2);
      cudaError_t e = cudaMemsetAsync(prm.image, 0, bytes, L.st);
      if (e != cudaSuccess) return e;
    }
  }
  if (L.split) *L.split = prm.tsplit;
#if !SASBP_ROTATE
  prm.resident = 0;
#endif
  kern<<<grid, threads, smem, L.st>>>(prm, tmap);
  return cudaGetLastError();
}

// one (tile shape, gating, weighting) family: TMA / cp.async x receive-leg modes x motion
template <int KX, int KY, int KZ, int WY, int WZ, bool DZ, bool GATE, bool WEIGHT>
cudaError_t launch_family(const TdbpParams& prm, const TmaDesc& tmap, const K2Launch& L) {
  const size_t smem = k2_smem_bytes(prm.W);
  const int nt = 32 * WY * WZ;
  if (L.count) {
    if (GATE || WEIGHT) return cudaErrorInvalidValue;   // counting lives in the dense family
    const unsigned blocks = (unsigned)prm.tiles_x * prm.tiles_y * prm.tiles_z;
    count_kernel<KX, KY, KZ, WY, WZ><<<blocks, nt, 0, L.st>>>(prm);
    return cudaGetLastError();
  }
  if (WEIGHT) {   // spreading weight (R18): stop-and-hop, straight rays only (checked on the host)
    if (prm.vel || prm.nav || prm.refract) return cudaErrorNotSupported;
    auto go = [&](auto kern) { return launch_k(kern, nt, prm, tmap, smem, L); };
    if constexpr (KZ > 1 || SASBP_AXIS2D) if (L.tma && L.axis) {   // compact geometry: 3D volumes only
      switch (L.mode) {
        case kSeries3: return go(tdbp_kernel<KX, KY, KZ, WY, WZ, DZ, kSeries3, true, GATE, false, true, WEIGHT>);
        case kSeries4: return go(tdbp_kernel<KX, KY, KZ, WY, WZ, DZ, kSeries4, true, GATE, false, true, WEIGHT>);
        default: return go(tdbp_kernel<KX, KY, KZ, WY, WZ, DZ, kExact, true, GATE, false, true, WEIGHT>);
      }
    }
    if (L.tma) {
      switch (L.mode) {
        case kSeries3: return go(tdbp_kernel<KX, KY, KZ, WY, WZ, DZ, kSeries3, true, GATE, false, false, WEIGHT>);
        case kSeries4: return go(tdbp_kernel<KX, KY, KZ, WY, WZ, DZ, kSeries4, true, GATE, false, false, WEIGHT>);
        default: return go(tdbp_kernel<KX, KY, KZ, WY, WZ, DZ, kExact, true, GATE, false, false, WEIGHT>);
      }
    }
    switch (L.mode) {
      case kSeries3: return go(tdbp_kernel<KX, KY, KZ, WY, WZ, DZ, kSeries3, false, GATE, false, false, WEIGHT>);
      case kSeries4: return go(tdbp_kernel<KX, KY, KZ, WY, WZ, DZ, kSeries4, false, GATE, false, false, WEIGHT>);
      default: return go(tdbp_kernel<KX, KY, KZ, WY, WZ, DZ, kExact, false, GATE, false, false, WEIGHT>);
    }
  }
  auto pick = [&](auto tma_tag, auto motion_tag, auto axis_tag) -> cudaError_t {
    constexpr bool T = decltype(tma_tag)::value;
    constexpr bool M = decltype(motion_tag)::value;
    constexpr bool AX = decltype(axis_tag)::value;
    if (prm.refract) {
      if (M) return cudaErrorNotSupported;   // rejected on the host before launch
      return launch_k(tdbp_kernel<KX, KY, KZ, WY, WZ, DZ, kRefract, T, GATE, false, AX>, nt, prm, tmap, smem, L);
    }
    if constexpr (GATE && !M && !WEIGHT) {
      if (L.gsplit) {
        // Two-launch gated form: the (tile, channel) pairs wholly inside the cone(s) run a kernel
        // without per-pixel masks (the dense loop), then the edge pairs accumulate with masks.  The
        // per-pixel terms and their order within each launch are those of the one-launch form.
        TdbpParams p1 = prm, p2 = prm;
        p1.gpart = 1;
        p2.gpart = 2;
        p2.accumulate = 1;
        K2Launch L2 = L;
        L2.occ = nullptr;
        L2.split = nullptr;
        cudaError_t e;
        switch (L.mode) {
          case kSeries3: e = launch_k(tdbp_kernel<KX, KY, KZ, WY, WZ, DZ, kSeries3, T, true, false, AX, false, true>, nt, p1, tmap, smem, L); break;
          case kSeries4: e = launch_k(tdbp_kernel<KX, KY, KZ, WY, WZ, DZ, kSeries4, T, true, false, AX, false, true>, nt, p1, tmap, smem, L); break;
          default: e = launch_k(tdbp_kernel<KX, KY, KZ, WY, WZ, DZ, kExact, T, true, false, AX, false, true>, nt, p1, tmap, smem, L); break;
        }
        if (e != cudaSuccess) return e;
        switch (L.mode) {
          case kSeries3: return launch_k(tdbp_kernel<KX, KY, KZ, WY, WZ, DZ, kSeries3, T, true, false, AX>, nt, p2, tmap, smem, L2);
          case kSeries4: return launch_k(tdbp_kernel<KX, KY, KZ, WY, WZ, DZ, kSeries4, T, true, false, AX>, nt, p2, tmap, smem, L2);
          default: return launch_k(tdbp_kernel<KX, KY, KZ, WY, WZ, DZ, kExact, T, true, false, AX>, nt, p2, tmap, smem, L2);
        }
      }
    }
    switch (L.mode) {
      case kSeries3: return launch_k(tdbp_kernel<KX, KY, KZ, WY, WZ, DZ, kSeries3, T, GATE, M, AX>, nt, prm, tmap, smem, L);
      case kSeries4: return launch_k(tdbp_kernel<KX, KY, KZ, WY, WZ, DZ, kSeries4, T, GATE, M, AX>, nt, prm, tmap, smem, L);
      default: return launch_k(tdbp_kernel<KX, KY, KZ, WY, WZ, DZ, kExact, T, GATE, M, AX>, nt, prm, tmap, smem, L);
    }
  };
  using TT = std::true_type;
  using FF = std::false_type;
  if constexpr (KZ > 1 || SASBP_AXIS2D)   // compact geometry: 3D volumes only
    if (L.tma && L.axis) return (prm.vel || prm.nav) ? pick(TT{}, TT{}, TT{}) : pick(TT{}, FF{}, TT{});
  if (L.tma) return (prm.vel || prm.nav) ? pick(TT{}, TT{}, FF{}) : pick(TT{}, FF{}, FF{});
  return (prm.vel || prm.nav) ? pick(FF{}, TT{}, FF{}) : pick(FF{}, FF{}, FF{});
}

// entry points, one per translation unit (k2_*.cu)
cudaError_t k2_launch_2d(const TdbpParams& prm, const TmaDesc& tmap, const K2Launch& L);        // dense + count
cudaError_t k2_launch_2d_gate(const TdbpParams& prm, const TmaDesc& tmap, const K2Launch& L);
cudaError_t k2_launch_2ddz(const TdbpParams& prm, const TmaDesc& tmap, const K2Launch& L);
cudaError_t k2_launch_2ddz_gate(const TdbpParams& prm, const TmaDesc& tmap, const K2Launch& L);
cudaError_t k2_launch_3d(const TdbpParams& prm, const TmaDesc& tmap, const K2Launch& L);
cudaError_t k2_launch_3d_gate(const TdbpParams& prm, const TmaDesc& tmap, const K2Launch& L);
cudaError_t k2_launch_2d_w(const TdbpParams& prm, const TmaDesc& tmap, const K2Launch& L);     // weighted (R18)
cudaError_t k2_launch_2ddz_w(const TdbpParams& prm, const TmaDesc& tmap, const K2Launch& L);
cudaError_t k2_launch_3d_w(const TdbpParams& prm, const TmaDesc& tmap, const K2Launch& L);

}  // namespace sasbp

// tile shapes of the variants (KX, KY, KZ, WY, WZ): 2D = 32 x 8*WY pixels, 3D = 16 x 8 x 8 voxels
#ifndef SASBP_WY2D
#define SASBP_WY2D 4
#endif
#ifndef SASBP_KX2D
#define SASBP_KX2D 4   // pixels per thread along x (even: x-adjacent pairs)
#endif
#ifndef SASBP_KY2D
#define SASBP_KY2D 2   // pixels per thread along y
#endif
#if SASBP_K4
#define SASBP_T2D 4, 1, 1, 8, 1
#else
#define SASBP_T2D SASBP_KX2D, SASBP_KY2D, 1, SASBP_WY2D, 1
#endif
#ifndef SASBP_KY3D
#define SASBP_KY3D 2   // voxels per thread along y (3D)
#endif
#ifndef SASBP_KZ3D
#define SASBP_KZ3D 4   // voxels per thread along z (3D): 2 x KY3D x KZ3D = 16 voxels per thread, tile 16 x 8 x 16
#endif
#ifndef SASBP_WZ3D
#define SASBP_WZ3D 4   // warps per 3D CTA, stacked along z
#endif
#define SASBP_T3D 2, SASBP_KY3D, SASBP_KZ3D, 1, SASBP_WZ3D
