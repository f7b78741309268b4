// fp64_mix2_ubench.cu -- which companion instructions cost the FP64 pipe
// issue bandwidth on sm_100a? One DFMA (two vector operands) plus ONE
// companion instruction per step, 3 warps per sub-partition, ILP 6.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA error %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)
__device__ __forceinline__ long long clk() {
  long long c; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)); return c;
}
constexpr int R = 6;
template <int MODE>
__global__ void k(double* out, long long* cyc, const double* in, int iters, int sh) {
  double x[R]; int a[R]; float f[R]; unsigned u[R];
  __shared__ double smem[512];
  smem[threadIdx.x & 511] = in[threadIdx.x & 255];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < R; ++i) { x[i] = in[threadIdx.x + i]; a[i] = threadIdx.x + i; f[i] = (float)x[i]; u[i] = a[i] * 7; }
  const double c1 = in[0], c2 = in[1];
  long long t0 = clk();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int rep = 0; rep < 8; ++rep) {
#pragma unroll
      for (int i = 0; i < R; ++i) {
        x[i] = __fma_rn(x[i], c1, c2);
        if (MODE == 1) asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(sh), "r"(rep));   // IMAD
        if (MODE == 2) asm volatile("add.s32 %0, %0, %1;" : "+r"(a[i]) : "r"(sh));                    // IADD3
        if (MODE == 3) asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(f[i]) : "f"(f[(i + 1) % R])); // FFMA
        if (MODE == 4) asm volatile("xor.b32 %0, %0, %1;" : "+r"(u[i]) : "r"(sh));                    // LOP3
        if (MODE == 5) asm volatile("{ .reg .pred p; setp.ne.s32 p, %2, 0; selp.b32 %0, %0, %1, p; }" : "+r"(a[i]) : "r"(sh), "r"(a[(i + 1) % R])); // ISETP + SEL
        if (MODE == 6) { double t; asm volatile("mov.f64 %0, %1;" : "=d"(t) : "d"(x[(i + 3) % R])); x[(i + 3) % R] = t; } // 64-bit move
        if (MODE == 7) x[i] += smem[(threadIdx.x + 32 * i + rep) & 511];                              // LDS + DADD
        if (MODE == 8) asm volatile("shl.b32 %0, %0, %1;" : "+r"(u[i]) : "r"(sh & 1));                 // SHF
      }
    }
  }
  long long t1 = clk();
  double s = 0;
#pragma unroll
  for (int i = 0; i < R; ++i) s += x[i] + a[i] + f[i] + u[i];
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
static double *d_out, *d_in; static long long* d_cyc;
template <int MODE> void run(const char* what) {
  const int iters = 256, wps = 3;
  for (int rep = 0; rep < 2; ++rep) { k<MODE><<<148, wps * 128>>>(d_out, d_cyc, d_in, iters, 3); CK(cudaDeviceSynchronize()); }
  long long c; CK(cudaMemcpy(&c, d_cyc, 8, cudaMemcpyDeviceToHost));
  const double n = double(wps) * iters * 8 * R;
  printf("DFMA + %-34s %.3f cycles per DFMA per sub-partition\n", what, c / n);
}
int main() {
  CK(cudaMalloc(&d_out, 148 * 1024 * 8)); CK(cudaMalloc(&d_cyc, 8)); CK(cudaMalloc(&d_in, 4096 * 8));
  double h[4096]; for (int i = 0; i < 4096; ++i) h[i] = 1.0 + (i % 97) * 1e-9;
  CK(cudaMemcpy(d_in, h, sizeof h, cudaMemcpyHostToDevice));
  run<0>("nothing"); run<1>("IMAD (integer multiply-add)"); run<2>("IADD"); run<3>("FFMA");
  run<4>("LOP3 (xor)"); run<5>("ISETP + SEL"); run<6>("64-bit register move"); run<7>("LDS.64 + DADD"); run<8>("SHL");
  return 0;
}
