// fp64_ubench.cu -- micro-benchmarks of the sm_100a FP64 pipe that the volume
// kernel's design rests on (development aid, not part of the product):
//   A  dependent-issue latency of DFMA / DADD / DMUL / MUFU.RCP64H / LDS.64
//   B  DFMA throughput per SM sub-partition vs resident warps and ILP
//   C  DFMA issue alongside integer / FP32 / LDS instructions
//   D  instruction-cache capacity: straight-line DFMA bodies of growing size
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fp64_ubench fp64_ubench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA error %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ long long clk() {
  long long c; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)); return c;
}

enum Op { DFMA, DADD, DMUL, RCP, LDS };

template <int OP>
__global__ void latency_kernel(double* out, long long* cyc, double a, double b, int iters) {
  __shared__ double sh[64];
  sh[threadIdx.x & 63] = (double)((threadIdx.x * 8) & 511) ;
  __syncthreads();
  double x = a + threadIdx.x;
  long long idx = threadIdx.x & 63;
  long long t0 = clk();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 64; ++k) {
      if (OP == DFMA) x = __fma_rn(x, b, a);
      if (OP == DADD) x = __dadd_rn(x, a);
      if (OP == DMUL) x = __dmul_rn(x, b);
      if (OP == RCP) asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(x));
      if (OP == LDS) { idx = (long long)sh[idx & 63] >> 3; }
    }
  }
  long long t1 = clk();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = x + (double)idx;
}

// B/C: W warps per CTA (one CTA per SM), ILP independent chains
template <int ILP, int MIX>
__global__ void thr_kernel(double* out, long long* cyc, double a, double b, int iters) {
  __shared__ double sh[1024];
  sh[threadIdx.x] = a;
  __syncthreads();
  double x[ILP];
  int y = threadIdx.x; float z = (float)a; double w = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) x[i] = a + i + threadIdx.x;
  long long t0 = clk();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
#pragma unroll
      for (int i = 0; i < ILP; ++i) {
        x[i] = __fma_rn(x[i], b, a);
        if (MIX == 1) y = y * 3 + k;                 // integer
        if (MIX == 2) z = __fmaf_rn(z, z, 1.0f);     // FP32
        if (MIX == 3) w += sh[(threadIdx.x + k * 32 + i) & 1023]; // LDS + DADD
        if (MIX == 4) { y = y * 3 + k; z = __fmaf_rn(z, z, 1.0f); }
      }
    }
  }
  long long t1 = clk();
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += x[i];
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + y + z + w;
}

// D: straight-line body of UNR DFMAs over 8 chains (16 B per SASS instruction)
template <int UNR>
__global__ void __launch_bounds__(512) icache_kernel(double* out, long long* cyc, double a, double b, int iters) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = a + i + threadIdx.x;
  long long t0 = clk();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < UNR; ++k) x[k & 7] = __fma_rn(x[k & 7], b, a);
  }
  long long t1 = clk();
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

static double* d_out; static long long* d_cyc;

template <int OP> void run_lat(const char* name) {
  latency_kernel<OP><<<1, 32>>>(d_out, d_cyc, 1.0, 1.0000001, 64);
  CK(cudaDeviceSynchronize());
  latency_kernel<OP><<<1, 32>>>(d_out, d_cyc, 1.0, 1.0000001, 64);
  CK(cudaDeviceSynchronize());
  long long c; CK(cudaMemcpy(&c, d_cyc, 8, cudaMemcpyDeviceToHost));
  printf("A latency %-8s %.2f cycles/op\n", name, (double)c / (64.0 * 64));
}

template <int ILP, int MIX> void run_thr(int warps_per_smsp) {
  const int threads = warps_per_smsp * 4 * 32;
  const int iters = 256;
  thr_kernel<ILP, MIX><<<148, threads>>>(d_out, d_cyc, 1.0, 1.0000001, iters);
  CK(cudaDeviceSynchronize());
  thr_kernel<ILP, MIX><<<148, threads>>>(d_out, d_cyc, 1.0, 1.0000001, iters);
  CK(cudaDeviceSynchronize());
  long long c; CK(cudaMemcpy(&c, d_cyc, 8, cudaMemcpyDeviceToHost));
  const double dfma_per_smsp = (double)warps_per_smsp * iters * 16 * ILP;
  printf("B/C mix %d warps/smsp %d ilp %d : %.3f cycles per DFMA warp-instr per SMSP (pipe util %.1f%%)\n",
         MIX, warps_per_smsp, ILP, c / dfma_per_smsp, 100.0 * 2.0 * dfma_per_smsp / c);
}

template <int UNR> void run_ic(int warps_per_smsp) {
  const int threads = warps_per_smsp * 4 * 32;
  const int iters = (1 << 18) / UNR;
  icache_kernel<UNR><<<148, threads>>>(d_out, d_cyc, 1.0, 1.0000001, iters);
  CK(cudaDeviceSynchronize());
  icache_kernel<UNR><<<148, threads>>>(d_out, d_cyc, 1.0, 1.0000001, iters);
  CK(cudaDeviceSynchronize());
  long long c; CK(cudaMemcpy(&c, d_cyc, 8, cudaMemcpyDeviceToHost));
  const double n = (double)warps_per_smsp * iters * UNR;
  printf("D icache body %6.1f KB warps/smsp %d : %.3f cycles per DFMA per SMSP (pipe util %.1f%%)\n",
         UNR * 16.0 / 1024, warps_per_smsp, c / n, 200.0 * n / c);
}

int main() {
  CK(cudaMalloc(&d_out, 148 * 1024 * 8)); CK(cudaMalloc(&d_cyc, 64));
  run_lat<DFMA>("DFMA"); run_lat<DADD>("DADD"); run_lat<DMUL>("DMUL");
  run_lat<RCP>("RCP64H"); run_lat<LDS>("LDS+cvt");
  for (int w : {1, 2, 3, 4, 8}) {
    run_thr<1, 0>(w); run_thr<2, 0>(w); run_thr<4, 0>(w); run_thr<8, 0>(w);
  }
  for (int w : {3}) {
    run_thr<4, 1>(w); run_thr<4, 2>(w); run_thr<4, 3>(w); run_thr<4, 4>(w);
    run_thr<2, 1>(w); run_thr<2, 4>(w);
  }
  for (int w : {1, 3}) {
    run_ic<256>(w); run_ic<512>(w); run_ic<1024>(w); run_ic<2048>(w); run_ic<4096>(w);
    run_ic<8192>(w); run_ic<16384>(w);
  }
  return 0;
}
