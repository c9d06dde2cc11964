// FP32 pipe microbenchmark (B200): exact scalar mul+add vs packed f32x2 variants.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b){ uint64_t d; asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b){ uint64_t d; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c){ uint64_t d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ uint64_t hide1(uint64_t a){ uint32_t lo=(uint32_t)a, l2; asm volatile("prmt.b32 %0, %1, 0, 0x3210;" : "=r"(l2) : "r"(lo)); return (a & 0xffffffff00000000ull) | l2; }

constexpr int CH = 8;
__global__ void k_scalar(float* out, int n, float x) {
  float acc[CH], p[CH];
  for (int c = 0; c < CH; ++c) { acc[c] = threadIdx.x + c; p[c] = x + c; }
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = __fadd_rn(acc[c], __fmul_rn(p[c], acc[c]));
  }
  float s = 0; for (int c = 0; c < CH; ++c) s += acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_packed_prmt(float* out, int n, float x) {
  uint64_t acc[CH], p[CH];
  for (int c = 0; c < CH; ++c) { float2 a = make_float2(threadIdx.x + c, c); float2 q = make_float2(x + c, x); acc[c] = *reinterpret_cast<uint64_t*>(&a); p[c] = *reinterpret_cast<uint64_t*>(&q); }
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = add2(acc[c], hide1(mul2(p[c], acc[c])));
  }
  float s = 0; for (int c = 0; c < CH; ++c) { float2 a = *reinterpret_cast<float2*>(&acc[c]); s += a.x + a.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// packed multiply, scalar adds: ptxas does not contract FMUL2 into a scalar FADD (exact arithmetic)
__global__ void k_mul2_sadd(float* out, int n, float x) {
  uint64_t acc[CH], p[CH];
  for (int c = 0; c < CH; ++c) { float2 a = make_float2(threadIdx.x + c, c); float2 q = make_float2(x + c, x); acc[c] = *reinterpret_cast<uint64_t*>(&a); p[c] = *reinterpret_cast<uint64_t*>(&q); }
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      uint64_t m = mul2(p[c], acc[c]);
      float lo = __fadd_rn(__uint_as_float(uint32_t(acc[c])), __uint_as_float(uint32_t(m)));
      float hi = __fadd_rn(__uint_as_float(uint32_t(acc[c] >> 32)), __uint_as_float(uint32_t(m >> 32)));
      acc[c] = uint64_t(__float_as_uint(lo)) | (uint64_t(__float_as_uint(hi)) << 32);
    }
  }
  float s = 0; for (int c = 0; c < CH; ++c) { float2 a = *reinterpret_cast<float2*>(&acc[c]); s += a.x + a.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_sfma(float* out, int n, float x) {
  float acc[CH], p[CH];
  for (int c = 0; c < CH; ++c) { acc[c] = threadIdx.x + c; p[c] = x + c; }
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fmaf(p[c], acc[c], acc[c]);
  }
  float s = 0; for (int c = 0; c < CH; ++c) s += acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_fma2(float* out, int n, float x) {
  uint64_t acc[CH], p[CH];
  for (int c = 0; c < CH; ++c) { float2 a = make_float2(threadIdx.x + c, c); float2 q = make_float2(x + c, x); acc[c] = *reinterpret_cast<uint64_t*>(&a); p[c] = *reinterpret_cast<uint64_t*>(&q); }
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma2(p[c], acc[c], acc[c]);
  }
  float s = 0; for (int c = 0; c < CH; ++c) { float2 a = *reinterpret_cast<float2*>(&acc[c]); s += a.x + a.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dscalar(double* out, int n, double x) {
  double acc[CH], p[CH];
  for (int c = 0; c < CH; ++c) { acc[c] = threadIdx.x + c; p[c] = x + c; }
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = __dadd_rn(acc[c], __dmul_rn(p[c], acc[c]));
  }
  double s = 0; for (int c = 0; c < CH; ++c) s += acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dfma(double* out, int n, double x) {
  double acc[CH], p[CH];
  for (int c = 0; c < CH; ++c) { acc[c] = threadIdx.x + c; p[c] = x + c; }
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(p[c], acc[c], acc[c]);
  }
  double s = 0; for (int c = 0; c < CH; ++c) s += acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class K, class T>
void run(const char* name, K k, T* out, int lanes_per_op_instr, int instrs_per_iter_per_chain) {
  int n = 4096; int blocks = 148 * 8, threads = 256;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k<<<blocks, threads>>>(out, n, (T)1e-7); cudaDeviceSynchronize();
  cudaEventRecord(a); k<<<blocks, threads>>>(out, n, (T)1e-7); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double warp_instr = double(blocks) * threads / 32 * n * CH * instrs_per_iter_per_chain;
  double lane_ops = double(blocks) * threads * n * CH * lanes_per_op_instr;  // (mul+add) pairs per lane
  printf("%-14s %8.3f ms  warp-instr/clk/SM(@1.965GHz) %.2f   mul+add lane-pairs/clk/SM %.1f\n", name, ms,
         warp_instr / (ms * 1e-3) / 148 / 1.965e9, lane_ops / (ms * 1e-3) / 148 / 1.965e9);
}

int main() {
  float* f; double* d; cudaMalloc(&f, 148 * 8 * 256 * 8); cudaMalloc(&d, 148 * 8 * 256 * 8);
  run("scalar f32", k_scalar, f, 1, 2);
  run("packed+prmt", k_packed_prmt, f, 2, 3);
  run("ffma2", k_fma2, f, 2, 1);
  run("fmul2+2 fadd", k_mul2_sadd, f, 2, 3);
  run("scalar ffma", k_sfma, f, 1, 1);
  run("scalar f64", k_dscalar, d, 1, 2);
  run("dfma", k_dfma, d, 1, 1);
  return 0;
}
