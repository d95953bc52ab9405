// Minimal TMA row-load probe: [rows][cols] 8-byte elements, box {bw, 1}, negative x start.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

struct __align__(64) Desc { unsigned char b[128]; };

__global__ void k(const __grid_constant__ Desc d, int x, int y, int bw, unsigned long long* out) {
  __shared__ __align__(128) unsigned long long buf[256];
  __shared__ __align__(8) unsigned long long bar;
  uint32_t sb = (uint32_t)__cvta_generic_to_shared(buf), sbar = (uint32_t)__cvta_generic_to_shared(&bar);
  for (int i = threadIdx.x; i < 256; i += blockDim.x) buf[i] = 0xdeadbeefULL;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar), "r"(bw * 8) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(sb), "l"(&d), "r"(x), "r"(y), "r"(sbar) : "memory");
  }
  asm volatile("{\n .reg .pred p;\nW:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}\n" ::"r"(sbar) : "memory");
  for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char** argv) {
  int dtype = argc > 1 ? atoi(argv[1]) : (int)CU_TENSOR_MAP_DATA_TYPE_UINT64;
  int bw = argc > 2 ? atoi(argv[2]) : 26;
  int x = argc > 3 ? atoi(argv[3]) : -3;
  const int cols = 2048, rows = 256;
  unsigned long long* h = new unsigned long long[cols * rows];
  for (int i = 0; i < cols * rows; ++i) h[i] = i;
  unsigned long long *dbuf, *dout;
  cudaMalloc(&dbuf, 8ull * cols * rows); cudaMalloc(&dout, 8 * 256);
  cudaMemcpy(dbuf, h, 8ull * cols * rows, cudaMemcpyHostToDevice);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  Desc d;
  int elt = (dtype == CU_TENSOR_MAP_DATA_TYPE_FLOAT32) ? 4 : 8;
  int mult = 8 / elt;
  cuuint64_t dims[2] = {(cuuint64_t)cols * mult, (cuuint64_t)rows};
  cuuint64_t str[1] = {(cuuint64_t)cols * 8};
  cuuint32_t box[2] = {(cuuint32_t)(bw * mult), 1}, es[2] = {1, 1};
  CUresult r = enc((CUtensorMap*)&d, (CUtensorMapDataType)dtype, 2, dbuf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode dtype=%d bw=%d -> %d\n", dtype, bw, (int)r);
  k<<<1, 128>>>(d, x * mult, 5, bw, dout);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  if (e == cudaSuccess) {
    unsigned long long o[256];
    cudaMemcpy(o, dout, sizeof(o), cudaMemcpyDeviceToHost);
    for (int i = 0; i < 8; ++i) printf("%llx ", o[i]);
    printf("... expect row 5 starting at col %d (negatives -> 0)\n", x);
  }
  return 0;
}
