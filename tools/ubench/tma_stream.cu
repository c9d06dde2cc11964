// TMA streaming microbenchmark: the NN-sweep stage pattern (4-D boxes of a t-sliced SoA
// field) vs. contiguous 1-D bulk copies of the same bytes.  No compute: the ceiling the
// memory side of k_nn_tma can reach.  Build: nvcc -arch=sm_100a -lcuda tma_stream.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c)); }
__device__ __forceinline__ void expect(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory"); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  uint32_t d; do { asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(d) : "r"(sa(b)), "r"(ph) : "memory"); } while (!d); }
__device__ __forceinline__ void tma4(void* dst, const CUtensorMap* m, int a, int b, int c, int d, uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
    :: "r"(sa(dst)), "l"((uint64_t)m), "r"(a), "r"(b), "r"(c), "r"(d), "r"(sa(bar)) : "memory"); }
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t n, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(sa(dst)), "l"(src), "r"(n), "r"(sa(bar)) : "memory"); }

constexpr int NX = 64, NY = 64, NZ = 64, NT = 16, BY = 2, BZ = 2, NTHR = 256;
constexpr int NB = (NY / BY) * (NZ / BZ);

template <int MODE>
__global__ void k(const __grid_constant__ CUtensorMap mU, const float* U, int chunk_floats) {
  extern __shared__ __align__(128) unsigned char sm[];
  float* st = (float*)sm;
  const int SS = 72 * NTHR;
  uint64_t* full = (uint64_t*)(st + 2 * SS);
  uint64_t* empty = full + 2;
  if (threadIdx.x == 0) { mbar_init(&full[0], 1); mbar_init(&full[1], 1); mbar_init(&empty[0], NTHR); mbar_init(&empty[1], NTHR);
    asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  const long total = (long)NB * NT;
  const long w0 = total * blockIdx.x / gridDim.x, w1 = total * (blockIdx.x + 1) / gridDim.x;
  auto issue = [&](int s, long w) {
    const int blk = (int)(w / NT), t = (int)(w % NT);
    expect(&full[s], 72 * NTHR * 4);
    if (MODE == 0) {
      const int y0 = (blk % (NY / BY)) * BY, z0 = (blk / (NY / BY)) * BZ;
      for (int mu = 0; mu < 4; ++mu) tma4(st + s * SS + mu * 18 * NTHR, &mU, 0, y0, z0, t * 72 + mu * 18, &full[s]);
    } else {
      const float* src = U + ((long)t * NB + blk) * (long)chunk_floats;
      bulk(st + s * SS, src, 72 * NTHR * 4, &full[s]);
    }
  };
  long k = 0;
  if (threadIdx.x == 0) { if (w0 < w1) issue(0, w0); if (w0 + 1 < w1) issue(1, w0 + 1); }
  float acc = 0;
  for (long w = w0; w < w1; ++w, ++k) {
    const int s = k & 1;
    wait(&full[s], (k >> 1) & 1);
    acc += st[s * SS + threadIdx.x];
    arrive(&empty[s]);
    if (threadIdx.x == 0 && w + 2 < w1) { wait(&empty[s], (k >> 1) & 1); issue(s, w + 2); }
  }
  if (acc == 12345.f) printf("x");
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  size_t n = (size_t)NX * NY * NZ * NT * 72;
  float* U; cudaMalloc(&U, n * 4); cudaMemset(U, 0, n * 4);
  void* p; cudaDriverEntryPointQueryResult q; cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  Enc enc = (Enc)p;
  CUtensorMap m;
  cuuint64_t dims[4] = {NX, NY, NZ, (cuuint64_t)NT * 72};
  cuuint64_t str[3] = {NX * 4, NX * NY * 4, (cuuint64_t)NX * NY * NZ * 4};
  cuuint32_t box[4] = {NX, BY, BZ, 18}, es[4] = {1, 1, 1, 1};
  for (int promo = 0; promo < 4; ++promo) {
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, U, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, (CUtensorMapL2promotion)promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    size_t smem = 2 * 72 * NTHR * 4 + 64;
    cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int mode = 0; mode < 2; ++mode) {
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        if (mode == 0) k<0><<<148, NTHR, smem>>>(m, U, 0); else k<1><<<148, NTHR, smem>>>(m, U, 72 * NTHR);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double bytes = (double)NB * NT * 72 * NTHR * 4;
        if (rep == 2) printf("promo %d mode %s: %.3f ms  %.0f GB/s (%s)\n", promo, mode ? "bulk1d" : "tma4d", ms, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
