// rangecompress.cu -- K1, matched-filter range compression (the paper
// presumes compressed data; reading R14 in DESIGN.md):
//   out[ch][n] = sum_{m=0}^{Nr-1} raw[ch][n+m] * conj(replica[m]),  raw zero past Ns.
//
// v0 design: direct correlation in shared memory (FP32 complex MAC), one CTA per
// (1024-output chunk, channel).  The replica and the chunk's input span (1024 + Nr - 1
// samples) are staged once in shared memory; each thread produces 4 outputs strided by 256
// so shared loads are conflict-free.  FFT-domain overlap-save is the planned HBM-bound
// replacement (K1).
#include "sasbp.h"

#include <cstdarg>
#include <cstdio>
#include <cuda_runtime.h>

namespace {

constexpr int kRcThreads = 256;
constexpr int kRcOut = 4;                         // outputs per thread
constexpr int kRcTile = kRcThreads * kRcOut;      // outputs per CTA
constexpr int kRcMaxNr = 8192;

__global__ void __launch_bounds__(kRcThreads) rc_direct_kernel(const float2* __restrict__ raw, int Ns,
                                                               const float2* __restrict__ rep, int Nr,
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
    int n = n0 + i;
    sx[i] = (n < Ns) ? x[n] : make_float2(0.f, 0.f);
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

}  // namespace

extern "C" void sasbp_set_error(const char* msg);  // sasbp.cu: the thread-local sas_last_error buffer

namespace {
sas_status rc_cuda_fail(const char* what, cudaError_t e) {
  char buf[256];
  snprintf(buf, sizeof(buf), "%s: %s", what, cudaGetErrorString(e));
  sasbp_set_error(buf);
  return SAS_E_CUDA;
}
}  // namespace

static sas_status rc_launch(const float2* raw, int32_t P, int32_t E, int32_t Ns, const float2* rep, int32_t Nr,
                            float2* out, cudaStream_t st) {
  const size_t smem = sizeof(float2) * ((size_t)Nr + kRcTile + Nr - 1);
  cudaError_t e = cudaFuncSetAttribute(rc_direct_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return rc_cuda_fail("cudaFuncSetAttribute(rc_direct_kernel)", e);
  dim3 grid((Ns + kRcTile - 1) / kRcTile, (unsigned)P * E);
  rc_direct_kernel<<<grid, kRcThreads, smem, st>>>(raw, Ns, rep, Nr, out);
  e = cudaGetLastError();
  if (e != cudaSuccess) return rc_cuda_fail("rc_direct_kernel launch", e);
  return SAS_OK;
}

static sas_status rc_check(int32_t P, int32_t E, int32_t Ns, int32_t Nr) {
  if (P < 1 || E < 1 || Ns < 1 || Nr < 1) {
    sasbp_set_error("P, E, Ns, Nr must be >= 1");
    return SAS_E_INVALID;
  }
  if (Nr > kRcMaxNr) {
    sasbp_set_error("replica longer than 8192 samples is not supported by the direct kernel");
    return SAS_E_UNSUPPORTED;
  }
  if ((long double)P * E > 65535.0L * 65535.0L) { sasbp_set_error("too many channels"); return SAS_E_INVALID; }
  return SAS_OK;
}

extern "C" sas_status sas_rangecompress_device(const void* raw_dev, int32_t P, int32_t E, int32_t Ns,
                                               const void* replica_dev, int32_t Nr, void* out_dev, void* cuda_stream) {
  sasbp_set_error("");
  sas_status s = rc_check(P, E, Ns, Nr);
  if (s != SAS_OK) return s;
  if (!raw_dev || !replica_dev || !out_dev) { sasbp_set_error("NULL pointer"); return SAS_E_INVALID; }
  if ((long)P * E > 65535) {
    // grid.y limit: split channel ranges
    const long nch = (long)P * E;
    for (long c0 = 0; c0 < nch; c0 += 65535) {
      int n = (int)((nch - c0) < 65535 ? (nch - c0) : 65535);
      s = rc_launch((const float2*)raw_dev + c0 * Ns, n, 1, Ns, (const float2*)replica_dev, Nr,
                    (float2*)out_dev + c0 * Ns, (cudaStream_t)cuda_stream);
      if (s != SAS_OK) return s;
    }
    return SAS_OK;
  }
  return rc_launch((const float2*)raw_dev, P, E, Ns, (const float2*)replica_dev, Nr, (float2*)out_dev,
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
  cudaFree(draw); cudaFree(dout); cudaFree(drep);
  cudaStreamDestroy(st);
  return rs;
}
