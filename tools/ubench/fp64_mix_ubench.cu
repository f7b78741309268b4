// fp64_mix_ubench.cu -- can the FP64 pipe of sm_100a run at one instruction
// per two cycles per sub-partition when every instruction reads three
// DISTINCT register operands (as real flux code does), and with a
// DFMA/DMUL/DADD mix? 3 warps per sub-partition like the flux kernels.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA error %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)
__device__ __forceinline__ long long clk() {
  long long c; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)); return c;
}
// MODE 0: x[i] = fma(x[i], b, a)            (two shared operands)
// MODE 1: x[i] = fma(y[(i+3)%R], y[(i+7)%R], x[i])   three distinct registers
// MODE 2: like 1 but DFMA, DMUL, DADD in turn
// MODE 3: like 1 but results feed operands (rotating), closer to real dataflow
template <int R, int MODE>
__global__ void mix_kernel(double* out, long long* cyc, const double* in, int iters) {
  double x[R], y[R];
#pragma unroll
  for (int i = 0; i < R; ++i) { x[i] = in[i] + threadIdx.x; y[i] = in[R + i] * 1e-3 + 1.0; }
  const double a = in[0], b = in[1];
  long long t0 = clk();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int rep = 0; rep < 4; ++rep) {
#pragma unroll
      for (int i = 0; i < R; ++i) {
        if (MODE == 0) x[i] = __fma_rn(x[i], b, a);
        if (MODE == 1) x[i] = __fma_rn(y[(i + 3) % R], y[(i + 7) % R], x[i]);
        if (MODE == 2) {
          if ((i + rep) % 3 == 0) x[i] = __fma_rn(y[(i + 3) % R], y[(i + 7) % R], x[i]);
          else if ((i + rep) % 3 == 1) x[i] = __dmul_rn(x[i], y[(i + 5) % R]);
          else x[i] = __dadd_rn(x[i], y[(i + 2) % R]);
        }
        if (MODE == 3) x[i] = __fma_rn(x[(i + 5) % R], y[(i + 7) % R], x[(i + 11) % R]);
      }
    }
  }
  long long t1 = clk();
  double s = 0;
#pragma unroll
  for (int i = 0; i < R; ++i) s += x[i] + y[i];
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
static double *d_out, *d_in; static long long* d_cyc;
template <int R, int MODE> void run(int wps) {
  const int iters = 512;
  for (int rep = 0; rep < 2; ++rep) {
    mix_kernel<R, MODE><<<148, wps * 128>>>(d_out, d_cyc, d_in, iters);
    CK(cudaDeviceSynchronize());
  }
  long long c; CK(cudaMemcpy(&c, d_cyc, 8, cudaMemcpyDeviceToHost));
  const double n = double(wps) * iters * 4 * R;
  printf("mode %d regs %2d warps/smsp %d: %.3f cycles per FP64 instr per SMSP (pipe %.1f%%)\n", MODE, R, wps,
         c / n, 200.0 * n / c);
}
int main() {
  CK(cudaMalloc(&d_out, 148 * 1024 * 8)); CK(cudaMalloc(&d_cyc, 8)); CK(cudaMalloc(&d_in, 64 * 8));
  double h[64]; for (int i = 0; i < 64; ++i) h[i] = 1.0 + i * 1e-3;
  CK(cudaMemcpy(d_in, h, sizeof h, cudaMemcpyHostToDevice));
  for (int w : {1, 3}) {
    run<16, 0>(w); run<16, 1>(w); run<16, 2>(w); run<16, 3>(w);
    run<24, 1>(w); run<24, 2>(w); run<24, 3>(w);
  }
  return 0;
}
