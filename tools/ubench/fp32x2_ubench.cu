// fp32x2_ubench.cu -- issue cost of the packed FP32 instructions of sm_100a
// (fma.rn.f32x2 -> FFMA2: two FP32 FMAs per lane per instruction) against
// scalar FFMA, per sub-partition, as a function of warps per scheduler.
// Question behind it: the FP32 flux kernels are issue bound (79 % of the
// issue slots, 43 % of them FP32 arithmetic); does packing two pair fluxes
// into f32x2 operations halve those slots, and at what pipe rate?
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA error %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)
__device__ __forceinline__ long long clk() {
  long long c; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)); return c;
}
typedef unsigned long long u64;
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 r; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r;
}
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
  u64 r; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r;
}
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
  u64 r; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r;
}
constexpr int R = 8;
// MODE 0: scalar FFMA x = fma(x, y, z)            (2 R chains per thread)
// MODE 1: FFMA2    x2 = fma2(x2, y2, z2)          (R packed chains = 2 R FMAs)
// MODE 2: FMUL2 / FADD2 alternating
// MODE 3: FFMA2 interleaved 1:1 with an independent IMAD (does the packed op free an issue slot?)
// MODE 4: scalar FFMA interleaved 1:2 with IMAD (same FP32 work, same integer work as MODE 3)
template <int MODE>
__global__ void k(float* out, long long* cyc, const float* in, int iters) {
  float x[2 * R], y[2 * R], z[2 * R];
  int n[R];
#pragma unroll
  for (int i = 0; i < 2 * R; ++i) {
    x[i] = in[threadIdx.x + 32 * i];
    y[i] = in[threadIdx.x + 32 * i + 1] * 1e-6f + 1.0f;
    z[i] = in[threadIdx.x + 32 * i + 2] * 1e-6f;
  }
#pragma unroll
  for (int i = 0; i < R; ++i) n[i] = threadIdx.x + i;
  u64 X[R], Y[R], Z[R];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    X[i] = (u64(__float_as_uint(x[2 * i + 1])) << 32) | __float_as_uint(x[2 * i]);
    Y[i] = (u64(__float_as_uint(y[2 * i + 1])) << 32) | __float_as_uint(y[2 * i]);
    Z[i] = (u64(__float_as_uint(z[2 * i + 1])) << 32) | __float_as_uint(z[2 * i]);
  }
  const long long t0 = clk();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int rep = 0; rep < 4; ++rep) {
      if (MODE == 0 || MODE == 4) {
#pragma unroll
        for (int i = 0; i < 2 * R; ++i) {
          x[i] = __fmaf_rn(x[i], y[(i + 3 * rep + 1) % (2 * R)], z[(i + 5 * rep + 2) % (2 * R)]);
          if (MODE == 4 && (i & 1)) n[i / 2] = n[i / 2] * 3 + it;
        }
      } else {
#pragma unroll
        for (int i = 0; i < R; ++i) {
          if (MODE == 1 || MODE == 3) X[i] = fma2(X[i], Y[(i + 3 * rep + 1) % R], Z[(i + 5 * rep + 2) % R]);
          if (MODE == 2) X[i] = (rep & 1) ? mul2(X[i], Y[(i + rep) % R]) : add2(X[i], Z[(i + rep) % R]);
          if (MODE == 3) n[i] = n[i] * 3 + it;
        }
      }
    }
  }
  const long long t1 = clk();
  float s = 0;
  int m = 0;
#pragma unroll
  for (int i = 0; i < 2 * R; ++i) s += x[i];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    s += __uint_as_float(unsigned(X[i])) + __uint_as_float(unsigned(X[i] >> 32));
    m += n[i];
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + float(m);
}
static float *d_out, *d_in; static long long* d_cyc;
template <int MODE> void run(const char* what, int fma_per_thread_iter) {
  for (int wps = 1; wps <= 4; ++wps) {
    const int iters = 512;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    k<MODE><<<148, wps * 128>>>(d_out, d_cyc, d_in, iters);
    CK(cudaEventRecord(e0));
    k<MODE><<<148, wps * 128>>>(d_out, d_cyc, d_in, iters);
    CK(cudaEventRecord(e1));
    CK(cudaDeviceSynchronize());
    long long c; CK(cudaMemcpy(&c, d_cyc, sizeof c, cudaMemcpyDeviceToHost));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    const double fmas = double(fma_per_thread_iter) * iters * 148.0 * wps * 128;
    printf("%-58s %d warps/scheduler: %7.3f cycles per FP32 FMA-lane-op per warp slot, %6.2f TFLOP/s\n", what, wps,
           double(c) / (double(fma_per_thread_iter) * iters) * 1.0, 2.0 * fmas / (ms * 1e-3) / 1e12);
  }
}
int main() {
  CK(cudaMalloc(&d_out, 148 * 512 * sizeof(float)));
  CK(cudaMalloc(&d_in, 4096 * sizeof(float)));
  CK(cudaMalloc(&d_cyc, 8));
  CK(cudaMemset(d_in, 0, 4096 * sizeof(float)));
  run<0>("scalar FFMA, 16 chains", 4 * 16);
  run<1>("FFMA2 (fma.rn.f32x2), 8 packed chains", 4 * 16);
  run<2>("FMUL2 / FADD2 alternating, 8 packed chains", 4 * 16);
  run<3>("FFMA2 + one IMAD per FFMA2", 4 * 16);
  run<4>("scalar FFMA + one IMAD per two FFMA", 4 * 16);
  return 0;
}
