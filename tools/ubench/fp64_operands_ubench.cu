// fp64_operands_ubench.cu -- cost of an FP64 instruction on sm_100a as a
// function of how many DISTINCT VECTOR-register source operands it reads
// (thread-varying values, so the compiler cannot move them to uniform
// registers or the constant bank). 3 warps per sub-partition, 12 independent
// accumulator chains per thread.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA error %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)
__device__ __forceinline__ long long clk() {
  long long c; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)); return c;
}
constexpr int R = 12;
// MODE 0: x = fma(x, y_i, z_i)      3 vector regs, all different per instruction
// MODE 1: x = fma(x, y_i, C)        2 vector regs + constant-bank operand
// MODE 2: x = fma(x, x, y_i)        2 distinct vector regs (x twice)
// MODE 3: x = x * y_i               DMUL, 2 vector regs
// MODE 4: x = x + y_i               DADD, 2 vector regs
// MODE 5: x = fma(y_i, z_i, x)      3 vector regs, accumulate form
// MODE 6: x = fma(y_0, z_i, x)      3 vector regs, first one shared by consecutive instr (reuse)
// MODE 7: x = fma(x, y_i, z_i) with FP32: FFMA 3 vector regs (control)
template <int MODE>
__global__ void op_kernel(double* out, long long* cyc, const double* in, double cst, int iters) {
  double x[R], y[R], z[R];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    x[i] = in[threadIdx.x + 32 * i];
    y[i] = in[threadIdx.x + 32 * i + 1] * 1e-9 + 1.0;
    z[i] = in[threadIdx.x + 32 * i + 2] * 1e-9;
  }
  long long t0 = clk();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int rep = 0; rep < 4; ++rep) {
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const int j = (i + rep * 5 + 1) % R, k = (i + rep * 7 + 3) % R;
        if (MODE == 0) x[i] = __fma_rn(x[i], y[j], z[k]);
        if (MODE == 1) x[i] = __fma_rn(x[i], y[j], cst);
        if (MODE == 2) x[i] = __fma_rn(x[i], x[i], z[k]);
        if (MODE == 3) x[i] = __dmul_rn(x[i], y[j]);
        if (MODE == 4) x[i] = __dadd_rn(x[i], z[k]);
        if (MODE == 5) x[i] = __fma_rn(y[j], z[k], x[i]);
        if (MODE == 6) x[i] = __fma_rn(y[rep], z[k], x[i]);
      }
    }
  }
  long long t1 = clk();
  double s = 0;
#pragma unroll
  for (int i = 0; i < R; ++i) s += x[i] + y[i] + z[i];
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
static double *d_out, *d_in; static long long* d_cyc;
template <int MODE> void run(const char* what) {
  const int iters = 512, wps = 3;
  for (int rep = 0; rep < 2; ++rep) {
    op_kernel<MODE><<<148, wps * 128>>>(d_out, d_cyc, d_in, 1.0000001, iters);
    CK(cudaDeviceSynchronize());
  }
  long long c; CK(cudaMemcpy(&c, d_cyc, 8, cudaMemcpyDeviceToHost));
  const double n = double(wps) * iters * 4 * R;
  printf("%-58s %.3f cycles per instruction per sub-partition\n", what, c / n);
}
int main() {
  CK(cudaMalloc(&d_out, 148 * 1024 * 8)); CK(cudaMalloc(&d_cyc, 8)); CK(cudaMalloc(&d_in, 4096 * 8));
  double h[4096]; for (int i = 0; i < 4096; ++i) h[i] = 1.0 + (i % 97) * 1e-3;
  CK(cudaMemcpy(d_in, h, sizeof h, cudaMemcpyHostToDevice));
  run<0>("DFMA x = fma(x, y, z)   3 distinct vector registers");
  run<1>("DFMA x = fma(x, y, c[]) 2 vector registers + constant");
  run<2>("DFMA x = fma(x, x, z)   2 distinct vector registers");
  run<3>("DMUL x = x * y          2 vector registers");
  run<4>("DADD x = x + z          2 vector registers");
  run<5>("DFMA x = fma(y, z, x)   3 distinct vector registers");
  run<6>("DFMA x = fma(y0, z, x)  3 vector registers, y0 reusable");
  return 0;
}
