// smem_ubench.cu -- how many shared-memory wavefronts does a warp-wide 64-bit
// access cost on sm_100a for the address patterns the flux kernels use?
// Prints SM cycles per warp-level LDS.64 (throughput, 16 warps per SM).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA error %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)
__device__ __forceinline__ long long clk() {
  long long c; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)); return c;
}
// idx[lane] = index (in doubles) lane reads; 16 independent loads per iteration
__global__ void lds_kernel(const int* idx, double* out, long long* cyc, int iters, int store) {
  extern __shared__ double sh[];
  for (int i = threadIdx.x; i < 6144; i += blockDim.x) sh[i] = i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int a = idx[lane];
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  long long t0 = clk();
  for (int it = 0; it < iters; ++it) {
    const int o = (it & 7) * 16;  // keeps alignment class (multiples of 128 B)
    if (!store) {
#pragma unroll
      for (int k = 0; k < 16; k += 4) {
        s0 += sh[a + o + k * 256];
        s1 += sh[a + o + (k + 1) * 256];
        s2 += sh[a + o + (k + 2) * 256];
        s3 += sh[a + o + (k + 3) * 256];
      }
    } else {
#pragma unroll
      for (int k = 0; k < 16; ++k) sh[a + o + k * 256] = s0 + k;
    }
  }
  long long t1 = clk();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3 + sh[threadIdx.x];
}
static int* d_idx; static double* d_out; static long long* d_cyc;
void run(const char* name, int (*f)(int), int store) {
  int h[32]; for (int l = 0; l < 32; ++l) h[l] = f(l);
  CK(cudaMemcpy(d_idx, h, sizeof h, cudaMemcpyHostToDevice));
  const int warps = 16, iters = 512;
  for (int rep = 0; rep < 2; ++rep) {
    lds_kernel<<<148, warps * 32, 6144 * 8>>>(d_idx, d_out, d_cyc, iters, store);
    CK(cudaDeviceSynchronize());
  }
  long long c; CK(cudaMemcpy(&c, d_cyc, 8, cudaMemcpyDeviceToHost));
  printf("%-44s %s: %.2f cycles per warp access\n", name, store ? "STS.64" : "LDS.64",
         (double)c / (double(warps) * iters * 16));
}
int main() {
  CK(cudaMalloc(&d_idx, 128)); CK(cudaMalloc(&d_out, 148 * 512 * 8)); CK(cudaMalloc(&d_cyc, 8));
  CK(cudaFuncSetAttribute(lds_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 6144 * 8));
  for (int st = 0; st < 2; ++st) {
    run("contiguous, 128B aligned", [](int l) { return l; }, st);
    run("contiguous, +8 B", [](int l) { return l + 1; }, st);
    run("contiguous, +72 B (k*25 doubles)", [](int l) { return l + 25; }, st);
    run("contiguous, +64 B", [](int l) { return l + 8; }, st);
    run("stride 5 doubles (x lines, PX=5)", [](int l) { return 5 * l; }, st);
    run("stride 5 doubles +1", [](int l) { return 5 * l + 1; }, st);
    run("y lines: x + 25 z (l = x + 5 z)", [](int l) { return (l % 5) + 25 * (l / 5); }, st);
    run("two runs: 25 aligned + 7 aligned (pad 32)", [](int l) { return l < 25 ? l : 160 + (l - 25); }, st);
    run("two runs: 25 + 7 contiguous elems (125 pitch)", [](int l) { return l < 25 ? l + 100 : 125 + (l - 25); }, st);
    run("stride 2 doubles", [](int l) { return 2 * l; }, st);
    run("stride 3 doubles", [](int l) { return 3 * l; }, st);
    run("stride 9 doubles", [](int l) { return 9 * l; }, st);
    run("stride 16 doubles (worst)", [](int l) { return 16 * l; }, st);
    run("broadcast", [](int) { return 3; }, st);
    run("permuted in aligned 256 B", [](int l) { return (l * 7) & 31; }, st);
    run("permuted in misaligned 256 B", [](int l) { return ((l * 7) & 31) + 3; }, st);
  }
  return 0;
}
