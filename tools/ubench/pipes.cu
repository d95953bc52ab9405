// Pipe-throughput microbenchmarks for the TDBP roofline.
// Measures, on the B200 it runs on, per-SM per-clock throughput of the
// instruction classes the backprojection inner loop is made of:
//   FFMA (3-register form), FFMA with an immediate, MUFU.SIN+MUFU.COS (__sinf/__cosf),
//   MUFU.RSQ (rsqrtf), LDS.128 (conflict-free), and a mixed "issue" probe.
// Output: one JSON line per probe on stdout.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

constexpr int CH = 8;        // independent chains per thread
constexpr int ITERS = 1 << 16;

// per block: SM clock64() at loop start / end, %smid, %globaltimer (ns) at start / end.  The
// per-SM throughput is taken over each SM's span [min start, max end] of clock64 (a per-SM
// counter; blocks of one SM need not start together), and the clock over the same span in ns.
__device__ unsigned long long g_c0[4096], g_c1[4096], g_n0[4096], g_n1[4096];
__device__ unsigned g_sm[4096];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t;
}
__device__ __forceinline__ unsigned smid() { unsigned s; asm volatile("mov.u32 %0, %smid;" : "=r"(s)); return s; }
__device__ __forceinline__ void rec(unsigned long long t0, unsigned long long t1, unsigned long long n0) {
  const unsigned long long n1 = gtimer();
  if (threadIdx.x == 0) {
    g_c0[blockIdx.x] = t0; g_c1[blockIdx.x] = t1; g_n0[blockIdx.x] = n0; g_n1[blockIdx.x] = n1;
    g_sm[blockIdx.x] = smid();
  }
}

__global__ void k_ffma(float* out, float a, float b) {
  float x[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) x[i] = threadIdx.x * 1e-3f + i;
  float y = a * 0.5f, z = b * 0.25f;
  unsigned long long n0 = gtimer(), t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = fmaf(x[i], y, z);
  }
  unsigned long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += x[i];
  if (s == 1234.5f) out[0] = s;
  rec(t0, t1, n0);
}

__global__ void k_ffma_imm(float* out, float a) {
  float x[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) x[i] = threadIdx.x * 1e-3f + i;
  float y = a * 0.5f;
  unsigned long long n0 = gtimer(), t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = fmaf(x[i], y, 0.7071f);
  }
  unsigned long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += x[i];
  if (s == 1234.5f) out[0] = s;
  rec(t0, t1, n0);
}

__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

__global__ void k_ffma2(float* out, float a, float b) {
  unsigned long long x[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    float2 v = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
    x[i] = *reinterpret_cast<unsigned long long*>(&v);
  }
  float2 yv = make_float2(a * 0.5f, a * 0.25f), zv = make_float2(b * 0.25f, b);
  unsigned long long y = *reinterpret_cast<unsigned long long*>(&yv), z = *reinterpret_cast<unsigned long long*>(&zv);
  unsigned long long n0 = gtimer(), t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = ffma2(x[i], y, z);
  }
  unsigned long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < CH; ++i) { float2 v = *reinterpret_cast<float2*>(&x[i]); s += v.x + v.y; }
  if (s == 1234.5f) out[0] = s;
  rec(t0, t1, n0);
}

// sin + cos of the same argument: 2 MUFU per chain step (+ FMUL.RZ + FADD)
__global__ void k_sincos(float* out, float a) {
  float x[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) x[i] = threadIdx.x * 1e-3f + i;
  unsigned long long n0 = gtimer(), t0 = clock64();
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = __sinf(x[i]) + __cosf(x[i]);
  }
  unsigned long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += x[i];
  if (s == 1234.5f) out[0] = s;
  rec(t0, t1, n0);
}

__global__ void k_rsqrt(float* out, float a) {
  float x[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) x[i] = threadIdx.x * 1e-3f + i + 1.f;
  unsigned long long n0 = gtimer(), t0 = clock64();
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = rsqrtf(x[i]);
  }
  unsigned long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += x[i];
  if (s == 1234.5f) out[0] = s;
  rec(t0, t1, n0);
}

__global__ void k_lds128(float* out, int stride) {
  __shared__ float4 buf[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  float4 acc = make_float4(0, 0, 0, 0);
  int idx[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) idx[i] = (threadIdx.x * stride + i * 37) & 1023;
  unsigned long long n0 = gtimer(), t0 = clock64();
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      float4 v = buf[idx[i]];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      idx[i] = (idx[i] + (int)v.x) & 1023;  // dependent address chain
    }
  }
  unsigned long long t1 = clock64();
  if (acc.x + acc.y + acc.z + acc.w == 1234.5f) out[0] = acc.x;
  rec(t0, t1, n0);
}

// integer ALU pipe: one LOP3 (xor3) per step (a chain of adds is folded by ptxas into IMAD/LEA,
// so no add probe)
template <int OP>
__global__ void k_int(float* out, unsigned y, unsigned z) {
  unsigned x[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) x[i] = threadIdx.x * 7u + i;
  unsigned long long n0 = gtimer(), t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      if (OP == 0) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[i]) : "r"(y), "r"(z));
      else asm volatile("add.u32 %0, %0, %1;" : "+r"(x[i]) : "r"(y));
    }
  }
  unsigned long long t1 = clock64();
  unsigned s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += x[i];
  if (s == 12345u) out[0] = (float)s;
  rec(t0, t1, n0);
}

template <typename F>
static int run(const char* name, F launch, int blocks, int threads, double ops_per_thread, int sms,
               int clk_khz) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  launch();  // warm
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  launch();
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms = 0; CK(cudaEventElapsedTime(&ms, e0, e1));
  static unsigned long long c0[4096], c1[4096], n0[4096], n1[4096];
  static unsigned sm[4096];
  CK(cudaMemcpyFromSymbol(c0, g_c0, sizeof(unsigned long long) * blocks));
  CK(cudaMemcpyFromSymbol(c1, g_c1, sizeof(unsigned long long) * blocks));
  CK(cudaMemcpyFromSymbol(n0, g_n0, sizeof(unsigned long long) * blocks));
  CK(cudaMemcpyFromSymbol(n1, g_n1, sizeof(unsigned long long) * blocks));
  CK(cudaMemcpyFromSymbol(sm, g_sm, sizeof(unsigned) * blocks));
  double total_ops = ops_per_thread * threads * (double)blocks;
  // per SM: ops of its blocks / (max end - min start) in its own clock64 cycles; clock = the same
  // span's cycles / its globaltimer ns.  Averaged over the SMs that ran blocks.
  double rate_sum = 0, ghz_sum = 0;
  int nsm = 0;
  for (int m = 0; m < 1024; ++m) {
    unsigned long long a = ~0ull, b = 0, na = ~0ull, nb = 0;
    int k = 0;
    for (int i = 0; i < blocks; ++i)
      if (sm[i] == (unsigned)m) {
        ++k; a = c0[i] < a ? c0[i] : a; b = c1[i] > b ? c1[i] : b;
        na = n0[i] < na ? n0[i] : na; nb = n1[i] > nb ? n1[i] : nb;
      }
    if (!k || b <= a || nb <= na) continue;
    rate_sum += ops_per_thread * threads * k / (double)(b - a);
    ghz_sum += (double)(b - a) / (double)(nb - na);
    ++nsm;
  }
  double per_sm_clk = nsm ? rate_sum / nsm : 0, eff_ghz = nsm ? ghz_sum / nsm : 0;
  printf("{\"probe\":\"%s\",\"blocks\":%d,\"threads\":%d,\"ms\":%.4f,\"Gops_per_s\":%.1f,"
         "\"ops_per_sm_per_clk\":%.2f,\"sm_clock_ghz\":%.3f,\"sms\":%d,\"max_clk_mhz\":%.0f}\n",
         name, blocks, threads, ms, total_ops / (ms * 1e-3) / 1e9, per_sm_clk, eff_ghz, sms,
         clk_khz / 1e3);
  return 0;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  int clk_khz = 0;
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  printf("{\"device\":\"%s\",\"sms\":%d,\"cc\":\"%d.%d\",\"clock_khz\":%d,\"smem_per_sm\":%zu,\"regs_per_sm\":%d}\n",
         prop.name, sms, prop.major, prop.minor, clk_khz, prop.sharedMemPerMultiprocessor,
         prop.regsPerMultiprocessor);
  float* out; CK(cudaMalloc(&out, 16));
  const int T = 256, B = sms * 4;  // 32 warps/SM, all co-resident
  if (run("ffma_3reg", [&] { k_ffma<<<B, T>>>(out, 1.0001f, 0.999f); }, B, T, (double)ITERS * CH, sms, clk_khz)) return 1;
  // FFMA2 (fma.rn.f32x2): count scalar FMAs (2 per instruction)
  if (run("ffma2_pairs", [&] { k_ffma2<<<B, T>>>(out, 1.0001f, 0.999f); }, B, T, (double)ITERS * CH * 2, sms, clk_khz)) return 1;
  if (run("ffma_imm", [&] { k_ffma_imm<<<B, T>>>(out, 1.0001f); }, B, T, (double)ITERS * CH, sms, clk_khz)) return 1;
  // sincos: count MUFU ops (2 per step)
  if (run("mufu_sin_cos", [&] { k_sincos<<<B, T>>>(out, 1.f); }, B, T, (double)(ITERS / 4) * CH * 2, sms, clk_khz)) return 1;
  if (run("mufu_rsq", [&] { k_rsqrt<<<B, T>>>(out, 1.f); }, B, T, (double)(ITERS / 4) * CH, sms, clk_khz)) return 1;
  // LDS.128: count 16-byte loads
  if (run("lds128", [&] { k_lds128<<<B, T>>>(out, 1); }, B, T, (double)(ITERS / 4) * CH, sms, clk_khz)) return 1;
  if (run("int_lop3", [&] { k_int<0><<<B, T>>>(out, 0x9e3779b9u, 0x7f4a7c15u); }, B, T, (double)ITERS * CH, sms, clk_khz)) return 1;
  CK(cudaGetLastError());
  return 0;
}
