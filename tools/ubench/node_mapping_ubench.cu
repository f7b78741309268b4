// node_mapping_ubench.cu -- the two thread mappings of the flux-differencing
// volume sweep (sweep_direction, kernels.hpp:154-249) side by side on sm_100a,
// N = 4 (NQ = 5), FP64, the product's own pair_flux (csrc/esdg_device.cuh):
//
//   line   thread per node LINE (what rhs_kernel does): the thread holds its
//          line's five nodes in registers, evaluates the ten unordered pairs,
//          updates both nodes of a pair in registers; x / y results go through
//          a shared slab (25 LDS + 25 STS per line and direction).
//   node   thread per NODE with the reference's Weighted schedule
//          (schedule.cpp:8-43: partners (i+1) % 5 and (i+2) % 5, every pair
//          once): the thread keeps its own node and five accumulators,
//          fetches the partner's nine values from shared memory, and hands
//          the partner's share c_ji (S - G b_i/b_j e_n) over through a
//          shared exchange array (5 STS, barrier, 5 LDS), two rounds per
//          direction.
//
// Both run the three directions on the same synthetic node values held in
// shared memory, repeatedly, with as many resident CTAs per SM as their
// registers and shared memory allow, and print SM cycles per element and the
// FP64 instructions they issue per element (from the source: 52 per pair in
// `line`, 57 in `node`), i.e. the fraction of the FP64 pipe's issue slots
// (one warp instruction per 2 cycles per sub-partition) each keeps busy.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false \
//        -I paper_2605_16684_b200/csrc -o tools/ubench/node_mapping_ubench tools/ubench/node_mapping_ubench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "esdg_device.cuh"

using namespace esdg_b200::dev;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA error %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)

constexpr int NQ = 5, N2 = 25, N3 = 125;

struct Coef {
  double negd[NQ * NQ];
  double cg;
};

// node values of one element: nine arrays of N3 doubles, plain SoA
__device__ __forceinline__ Node<double> load_node9(const double* v, int s, int dir) {
  Node<double> n;
  const int d1 = dir == 2 ? 0 : dir + 1, d2 = d1 == 2 ? 0 : d1 + 1;
  n.hr = v[0 * N3 + s];
  n.b = v[1 * N3 + s];
  n.hlr = v[2 * N3 + s];
  n.lb = v[3 * N3 + s];
  n.hphi = v[4 * N3 + s];
  n.hib = v[5 * N3 + s];
  n.hun = v[(6 + dir) * N3 + s];
  n.hut1 = v[(6 + d1) * N3 + s];
  n.hut2 = v[(6 + d2) * N3 + s];
  return n;
}

__device__ __forceinline__ void fill(double* vals, int n, int tid, int nthreads) {
  for (int i = tid; i < n; i += nthreads) {
    const int a = i / N3, s = i % N3;
    const double x = 1.0 + 0.01 * ((s * 37 + a * 11) % 17);
    vals[i] = a == 0 ? 0.5 * x : a == 1 ? 2e-6 * x : a == 2 ? 0.5 * log(x) : a == 3 ? log(2e-6 * x)
              : a == 4 ? 0.5 * 9.81 * (s / N2) : a == 5 ? 0.25e6 / x : 0.5 * (x - 1.05);
  }
}

// ---- line per thread: EPB elements, EPB * 25 threads ---------------------------
template <int EPB>
__global__ void __launch_bounds__(EPB* N2, 3) line_kernel(const __grid_constant__ Coef C, double* out,
                                                         int iters) {
  extern __shared__ double sh[];
  double* vals = sh;                 // [EPB][9][N3]
  double* slab = sh + EPB * 9 * N3;  // [EPB][5][N3]
  const int tid = threadIdx.x, e = tid / N2, l = tid % N2, l0 = l % NQ, l1 = l / NQ;
  for (int k = 0; k < EPB; ++k) fill(vals + k * 9 * N3, 9 * N3, tid, EPB * N2);
  for (int i = tid; i < EPB * 5 * N3; i += EPB * N2) slab[i] = 0.0;
  __syncthreads();
  const double* v = vals + e * 9 * N3;
  double* t = slab + e * 5 * N3;
  double accz[NQ][5];
  for (int it = 0; it < iters; ++it) {
#pragma unroll 1
    for (int dir = 0; dir < 3; ++dir) {
      const int base = dir == 0 ? NQ * l : (dir == 1 ? l0 + N2 * l1 : l);
      const int stride = dir == 0 ? 1 : (dir == 1 ? NQ : N2);
      Node<double> nd[NQ];
      double acc[NQ][5];
#pragma unroll
      for (int i = 0; i < NQ; ++i) {
        nd[i] = load_node9(v, base + i * stride, dir);
#pragma unroll
        for (int k = 0; k < 5; ++k) acc[i][k] = 0.0;
      }
#pragma unroll
      for (int i = 0; i < NQ; ++i)
#pragma unroll
        for (int j = 0; j < NQ; ++j) {
          if (j <= i) continue;
          const PairFlux<double> pf = pair_flux(nd[i], nd[j], C.cg);
          const double cij = C.negd[i * NQ + j], cji = C.negd[j * NQ + i];
          const double fni = fma_(pf.tg, nd[i].hib, pf.f[1]), fnj = fma_(-pf.tg, nd[j].hib, pf.f[1]);
          acc[i][0] = fma_(cij, pf.f[0], acc[i][0]);
          acc[i][1] = fma_(cij, fni, acc[i][1]);
          acc[i][2] = fma_(cij, pf.f[2], acc[i][2]);
          acc[i][3] = fma_(cij, pf.f[3], acc[i][3]);
          acc[i][4] = fma_(cij, pf.f[4], acc[i][4]);
          acc[j][0] = fma_(cji, pf.f[0], acc[j][0]);
          acc[j][1] = fma_(cji, fnj, acc[j][1]);
          acc[j][2] = fma_(cji, pf.f[2], acc[j][2]);
          acc[j][3] = fma_(cji, pf.f[3], acc[j][3]);
          acc[j][4] = fma_(cji, pf.f[4], acc[j][4]);
        }
      if (dir < 2) {
        double old[NQ][5];
#pragma unroll
        for (int i = 0; i < NQ; ++i)
#pragma unroll
          for (int k = 0; k < 5; ++k) old[i][k] = t[k * N3 + base + i * stride];
#pragma unroll
        for (int i = 0; i < NQ; ++i)
#pragma unroll
          for (int k = 0; k < 5; ++k) t[k * N3 + base + i * stride] = old[i][k] + acc[i][k];
        __syncthreads();
      } else {
#pragma unroll
        for (int i = 0; i < NQ; ++i)
#pragma unroll
          for (int k = 0; k < 5; ++k) accz[i][k] = acc[i][k];
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NQ; ++i)
#pragma unroll
    for (int k = 0; k < 5; ++k) s += accz[i][k] + t[k * N3 + l + i * N2];
  out[blockIdx.x * blockDim.x + tid] = s;
}

// ---- node per thread: EPB elements, EPB * 125 threads --------------------------
template <int EPB>
__global__ void __launch_bounds__(EPB* N3) node_kernel(const __grid_constant__ Coef C, double* out,
                                                        int iters) {
  extern __shared__ double sh[];
  double* vals = sh;                // [EPB][9][N3]
  double* xch = sh + EPB * 9 * N3;  // [EPB][5][N3] exchange array
  const int tid = threadIdx.x, e = tid / N3, s = tid % N3;
  const int c0 = s % NQ, c1 = (s / NQ) % NQ, c2 = s / N2;
  for (int k = 0; k < EPB; ++k) fill(vals + k * 9 * N3, 9 * N3, tid, EPB * N3);
  __syncthreads();
  const double* v = vals + e * 9 * N3;
  double* x = xch + e * 5 * N3;
  double acc[5] = {0, 0, 0, 0, 0};
  for (int it = 0; it < iters; ++it) {
#pragma unroll 1
    for (int dir = 0; dir < 3; ++dir) {
      const int i = dir == 0 ? c0 : (dir == 1 ? c1 : c2);
      const int stride = dir == 0 ? 1 : (dir == 1 ? NQ : N2);
      const Node<double> own = load_node9(v, s, dir);
      // own accumulators live in the rotated frame of the direction; un-rotate at the end
      double a[5] = {0, 0, 0, 0, 0};
#pragma unroll
      for (int o = 1; o <= NQ / 2; ++o) {
        const int j = i + o >= NQ ? i + o - NQ : i + o;
        const int sj = s + (j - i) * stride;
        const Node<double> pn = load_node9(v, sj, dir);
        // pair_flux is bitwise symmetric in its symmetric part and exactly
        // antisymmetric in tg, so either order gives the pair's one flux
        const PairFlux<double> pf = pair_flux(own, pn, C.cg);
        const double tg = pf.tg;
        const double cij = C.negd[i * NQ + j], cji = C.negd[j * NQ + i];
        const double fni = fma_(tg, own.hib, pf.f[1]), fnj = fma_(-tg, pn.hib, pf.f[1]);
        a[0] = fma_(cij, pf.f[0], a[0]);
        a[1] = fma_(cij, fni, a[1]);
        a[2] = fma_(cij, pf.f[2], a[2]);
        a[3] = fma_(cij, pf.f[3], a[3]);
        a[4] = fma_(cij, pf.f[4], a[4]);
        // the partner's share
        x[0 * N3 + sj] = cji * pf.f[0];
        x[1 * N3 + sj] = cji * fnj;
        x[2 * N3 + sj] = cji * pf.f[2];
        x[3 * N3 + sj] = cji * pf.f[3];
        x[4 * N3 + sj] = cji * pf.f[4];
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 5; ++k) a[k] += x[k * N3 + s];
        __syncthreads();
      }
      const int d1 = dir == 2 ? 0 : dir + 1, d2 = d1 == 2 ? 0 : d1 + 1;
      acc[0] += a[0];
      acc[1 + dir] += a[1];
      acc[1 + d1] += a[2];
      acc[1 + d2] += a[3];
      acc[4] += a[4];
    }
  }
  out[blockIdx.x * blockDim.x + tid] = acc[0] + acc[1] + acc[2] + acc[3] + acc[4];
}

template <class K>
void run(const char* name, K kern, int threads, int epb, size_t smem, const Coef& C, double* out, int fp64_per_pair) {
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  const int iters = 200, grid = 148 * per_sm;
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  kern<<<grid, threads, smem>>>(C, out, 4);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  kern<<<grid, threads, smem>>>(C, out, iters);
  CK(cudaEventRecord(b));
  CK(cudaDeviceSynchronize());
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  int clk_khz = 0;
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  const double elems_per_sm = double(per_sm) * epb * iters;
  const double cyc = ms * 1e-3 * clk_khz * 1e3 / elems_per_sm;  // SM cycles per element (3 directions)
  const double fp64 = 750.0 * fp64_per_pair;                     // thread instructions per element
  // 4 sub-partitions x 16 FP64 lanes: 64 thread instructions per SM cycle
  printf("%-6s %3d threads/CTA, %d CTA/SM (%2d warps/SM), %3d regs, %6.1f KB smem: %7.0f SM cycles/element, "
         "FP64 issue slots %4.1f %%\n",
         name, threads, per_sm, per_sm * ((threads + 31) / 32), fa.numRegs, smem / 1024.0, cyc,
         100.0 * fp64 / 64.0 / cyc);
}

int main() {
  Coef C;
  for (int i = 0; i < NQ * NQ; ++i) C.negd[i] = ((i / NQ) == (i % NQ)) ? 0.0 : 1.0 / (1 + (i % 7)) - 0.4;
  C.cg = 1.25;
  double* out;
  CK(cudaMalloc(&out, sizeof(double) * 148 * 16 * 1024));
  run("line", line_kernel<5>, 5 * N2, 5, sizeof(double) * 5 * 14 * N3, C, out, 52);
  run("node", node_kernel<1>, 1 * N3, 1, sizeof(double) * 1 * 14 * N3, C, out, 57);
  run("node", node_kernel<2>, 2 * N3, 2, sizeof(double) * 2 * 14 * N3, C, out, 57);
  run("node", node_kernel<4>, 4 * N3, 4, sizeof(double) * 4 * 14 * N3, C, out, 57);
  CK(cudaFree(out));
  return 0;
}
