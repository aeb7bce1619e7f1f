// Microbenchmark of the Jacobi inner (Gram-space) sweep alone: NCTA co-resident CTAs per
// SM each sweeping a 32x32 Hermitian Gram of a random 512x32 panel (cross sweep, as on
// a cross visit) -- cycles per sweep without the rest of the visit pipeline.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//   -I paper_1807_07914_b200/csrc -o tools/inner_bench tools/inner_bench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "bmps_jacobi.cuh"
using namespace bmps;

template <int W2>
__global__ void __launch_bounds__(256, 4)
inner_kernel(const double2* G0, int reps, int full, long long* cyc, int* nrot, double2* Gout, double2* Qout) {
  using C = JacCfg<W2>;
  extern __shared__ __align__(16) double2 sm[];
  double2* sG = sm;
  double2* sQ = sG + W2 * C::LDGG;
  double2* work = sQ + W2 * C::LDG;
  __shared__ InnerShared<W2> is;
  long long tot = 0;
  int nr = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int i = threadIdx.x; i < W2 * W2; i += blockDim.x)
      sG[(i % W2) + (i / W2) * C::LDGG] = G0[i];
    __syncthreads();
    const long long t0 = clock64();
    nr += jac_inner<W2>(sG, sQ, work, is, 4.0 * sqrt(512.0) * kEps, 1e-28, 1.0, full != 0, 1);
    __syncthreads();
    tot += clock64() - t0;
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) { *cyc = tot; *nrot = nr; }
  if (blockIdx.x == 0)
    for (int i = threadIdx.x; i < W2 * W2; i += blockDim.x) {
      Gout[i] = sG[(i % W2) + (i / W2) * C::LDGG];
      Qout[i] = sQ[(i % W2) + (i / W2) * C::LDG];
    }
}

int main(int argc, char** argv) {
  const int W2 = 32, R = 512;
  using C = JacCfg<W2>;
  std::vector<double2> P(R * W2), G(W2 * W2), Go(W2 * W2), Q(W2 * W2);
  srand(1);
  for (auto& x : P) x = make_double2(rand() / (double)RAND_MAX - 0.5, rand() / (double)RAND_MAX - 0.5);
  for (int i = 0; i < W2; ++i)
    for (int j = 0; j < W2; ++j) {
      double re = 0, im = 0;
      for (int k = 0; k < R; ++k) {
        const double2 a = P[k + i * R], b = P[k + j * R];
        re += a.x * b.x + a.y * b.y;
        im += a.x * b.y - a.y * b.x;
      }
      G[i + j * W2] = make_double2(re * 1e-3, im * 1e-3);
    }
  double2 *dG, *dO, *dQ; long long* dc; int* dn;
  cudaMalloc(&dG, sizeof(double2) * W2 * W2); cudaMalloc(&dO, sizeof(double2) * W2 * W2);
  cudaMalloc(&dQ, sizeof(double2) * W2 * W2);
  cudaMalloc(&dc, 8); cudaMalloc(&dn, 4);
  cudaMemcpy(dG, G.data(), sizeof(double2) * W2 * W2, cudaMemcpyHostToDevice);
  const size_t smem = sizeof(double2) * (W2 * C::LDGG + W2 * C::LDG + 8 * 64);
  cudaFuncSetAttribute(inner_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int reps = 200;
  for (int full = 0; full < 2; ++full)
    for (int ncta : {1, 2, 4}) {
      inner_kernel<32><<<148 * ncta, 256, smem>>>(dG, 2, full, dc, dn, dO, dQ);
      inner_kernel<32><<<148 * ncta, 256, smem>>>(dG, reps, full, dc, dn, dO, dQ);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      long long c; int n;
      cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&n, dn, 4, cudaMemcpyDeviceToHost);
#ifdef BMPS_PHASE_TIMERS
      {
        unsigned long long pc[24];
        cudaMemcpyFromSymbol(pc, g_phase_cycles, sizeof(pc));
        static unsigned long long prev[24];
        const double nb = (double)(pc[6] - prev[6]);
        printf("   batches %.0f: phase S %.0f, phase M %.0f cycles per batch (CTA 0.. all CTAs' thread 0)\n", nb,
               (pc[4] - prev[4]) / nb, (pc[5] - prev[5]) / nb);
        const double nr_ = (double)(pc[20] - prev[20]);
        if (nr_ > 0)
          printf("   per round (CTA 0, lane 0): shuffles %.0f, rotation %.0f, ballot+sync %.0f, updates+sync %.0f\n",
                 (pc[16] - prev[16]) / nr_, (pc[17] - prev[17]) / nr_, (pc[18] - prev[18]) / nr_, (pc[19] - prev[19]) / nr_);
        for (int i = 0; i < 24; ++i) prev[i] = pc[i];
      }
#endif
      const int rounds = full ? 31 : 16;
      printf("%s sweep, %d CTA/SM: %.0f cycles per sweep, %.0f per round (%d rounds), rotations/sweep %d\n",
             full ? "full " : "cross", ncta, (double)c / reps, (double)c / reps / rounds, rounds, n / reps);
    }
  // consistency: Q^H G0 Q == G_out, Q unitary
  cudaMemcpy(Go.data(), dO, sizeof(double2) * W2 * W2, cudaMemcpyDeviceToHost);
  cudaMemcpy(Q.data(), dQ, sizeof(double2) * W2 * W2, cudaMemcpyDeviceToHost);
  double err = 0, uerr = 0, gmax = 0;
  for (int i = 0; i < W2; ++i)
    for (int j = 0; j < W2; ++j) {
      double re = 0, im = 0, ur = 0, ui = 0;
      for (int k = 0; k < W2; ++k) {
        double tr = 0, ti = 0;
        for (int l = 0; l < W2; ++l) {
          const double2 g = G[k + l * W2], q = Q[l + j * W2];
          tr += g.x * q.x - g.y * q.y; ti += g.x * q.y + g.y * q.x;
        }
        const double2 qi = Q[k + i * W2];
        re += qi.x * tr + qi.y * ti; im += qi.x * ti - qi.y * tr;
        const double2 qj = Q[k + j * W2];
        ur += qi.x * qj.x + qi.y * qj.y; ui += qi.x * qj.y - qi.y * qj.x;
      }
      err = fmax(err, hypot(re - Go[i + j * W2].x, im - Go[i + j * W2].y));
      uerr = fmax(uerr, hypot(ur - (i == j), ui));
      gmax = fmax(gmax, hypot(G[i + j * W2].x, G[i + j * W2].y));
    }
  printf("max |Q^H G0 Q - G_out| / max|G0| = %.2e, max |Q^H Q - I| = %.2e\n", err / gmax, uerr);
  return 0;
}
