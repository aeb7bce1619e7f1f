// Does the Jacobi inner (Gram-space) sweep slow down because its scalar FP64 chains
// queue behind other warps' DMMA on the shared FP64 pipe of each SM sub-partition?
// (Measured with the round-by-round sweep of round 2's first sessions, profiles/
// r02_smsp_bench.txt: yes -- 2.1k cycles per round alone, 262k with DMMA warps of lower
// priority saturating the same sub-partitions, 15k from the highest warp ids, 3.7k when
// the sweep has a sub-partition to itself.)
// One 1024-thread CTA per SM: "rotation" warps run jac_inner on a 32x32 Gram while
// "math" warps run the apply pass's DMMA loop from shared memory. Placement of the
// rotation warps: spread over all four sub-partitions (wid < 8) or all on
// sub-partition 0 (wid % 4 == 0), with the math warps on the remaining warps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I include -I paper_1807_07914_b200/csrc \
//   -o tools/smsp_bench tools/smsp_bench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "bmps_jacobi.cuh"
using namespace bmps;

// PLACE 0: rotation warps wid 0..7; 1: wid % 4 == 0 (sub-partition 0); 2: wid 24..31
// (the highest warp ids: the scheduler arbitrates highest-wid-first); 3: wid % 4 == 3.
// GW warps per rotation group, 8 / GW groups each sweeping its own Gram.
template <int PLACE, int GW>
struct RotG {
  static constexpr int kN = GW * 32;
  BMPS_DEV static int rw() {
    return (PLACE & 1) ? (int)(threadIdx.x >> 7) : PLACE == 2 ? (int)(threadIdx.x >> 5) - 24 : (int)(threadIdx.x >> 5);
  }
  BMPS_DEV static bool mine() {
    const int wid = threadIdx.x >> 5;
    return PLACE == 1 ? (wid & 3) == 0 : PLACE == 3 ? (wid & 3) == 3 : PLACE == 2 ? wid >= 24 : wid < 8;
  }
  BMPS_DEV static int grp() { return rw() / GW; }
  BMPS_DEV static int tid() { return (rw() % GW) * 32 + (int)(threadIdx.x & 31); }
  BMPS_DEV static constexpr int n() { return kN; }
  BMPS_DEV static void sync() { __barrier_sync_count(1 + grp(), kN); }
  BMPS_DEV static int count(int p) {
    __shared__ int s_w[8];
    const unsigned bal = __ballot_sync(0xffffffffu, p != 0);
    if ((threadIdx.x & 31) == 0) s_w[rw()] = __popc(bal);
    sync();
    int r = 0;
    const int g0 = grp() * GW;
#pragma unroll
    for (int k = 0; k < GW; ++k) r += s_w[g0 + k];
    sync();
    return r;
  }
};

template <int PLACE, int GW>
__global__ void __launch_bounds__(1024, 1)
bench_kernel(const double2* G0, int reps, int math_on, int rot_on, long long* out) {
  using C = JacCfg<32>;
  using G = RotG<PLACE, GW>;
  constexpr int NG = 8 / GW;
  extern __shared__ __align__(16) double2 sm[];
  double2* sG = sm;                          // NG Grams
  double2* sQ = sG + NG * 32 * C::LDGG;      // NG Qs
  double2* sW = sQ + NG * 32 * C::LDG;       // inner-sweep workspaces (K_g, 8 x 64 per sweep)
  double2* sP = sW + NG * 8 * 64;            // math operand A (32 x 32 chunk)
  double2* sB = sP + C::BUF;                 // math operand B
  __shared__ InnerShared<32> rs[NG];
  __shared__ volatile int s_done;
  __shared__ long long s_rot_cyc[8], s_math_it[32], s_math_cyc[32];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) s_done = rot_on ? 0 : 0;
  for (int i = threadIdx.x; i < C::BUF; i += blockDim.x) {
    sP[i] = make_double2(1e-3 * (i % 17), 1e-3 * (i % 5));
    sB[i] = make_double2(1e-3 * (i % 13), 1e-3 * (i % 7));
  }
  __syncthreads();
  if (G::mine()) {
    if (!rot_on) return;
    double2* g = sG + G::grp() * 32 * C::LDGG;
    double2* q = sQ + G::grp() * 32 * C::LDG;
    long long tot = 0;
    for (int rep = 0; rep < reps; ++rep) {
      for (int i = G::tid(); i < 32 * 32; i += G::n()) g[(i % 32) + (i / 32) * C::LDGG] = G0[i];
      G::sync();
      const long long t0 = clock64();
      jac_inner<32, G>(g, q, sW + G::grp() * 8 * 64, rs[G::grp()], 4.0 * sqrt(512.0) * kEps, 1e-28, 1.0, false, 1);
      G::sync();
      tot += clock64() - t0;
    }
    if (G::tid() == 0) s_rot_cyc[G::grp()] = tot;
    G::sync();
    if (G::tid() == 0) atomicAdd((int*)&s_done, 1);
    // report by the first rotation thread once every group is done
    if (G::grp() == 0 && G::tid() == 0) {
      while (s_done < NG) { }
      long long m = 0;
      for (int k = 0; k < NG; ++k) m = max(m, s_rot_cyc[k]);
      out[blockIdx.x * 4 + 0] = m;
    }
    return;
  }
  if (!math_on) return;
  // math warps: the apply pass's inner loop (two 8x8 output tiles, k = 32, 3-product DMMA)
  const int kr = lane & 3, rc = lane >> 2;
  double acc[2][kZ3];
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int z = 0; z < kZ3; ++z) acc[u][z] = 0.0;
  long long it = 0;
  const long long t0 = clock64();
  const int mi = wid & 3;
  for (;;) {
    if (rot_on ? (s_done >= NG) : (it >= (long long)reps * 40)) break;
#pragma unroll 2
    for (int k4 = 0; k4 < 8; ++k4) {
      const int k = k4 * 4 + kr;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const double2 a = sP[mi * 8 + rc + k * C::RCP];
        const double2 b = sB[k + (((wid >> 2) & 1) * 16 + u * 8 + rc) * C::RCP];
        zmma3(acc[u], a, b);
      }
    }
    ++it;
  }
  const long long t1 = clock64();
  double s = 0;
  for (int u = 0; u < 2; ++u) s += z3_get(acc[u], 0).x + z3_get(acc[u], 1).y;
  if (s == 1.2345e-300) out[3] = 1;
  if (lane == 0) { s_math_it[wid] = it; s_math_cyc[wid] = t1 - t0; }
  __syncwarp();
  // last math warp to finish does not know the others; let warp with the highest id report its own view
  if (lane == 0) {
    atomicAdd((unsigned long long*)&out[blockIdx.x * 4 + 1], (unsigned long long)it);
    atomicMax((unsigned long long*)&out[blockIdx.x * 4 + 2], (unsigned long long)(t1 - t0));
  }
}

template <int PLACE, int GW>
void run(const char* name, const double2* dG, int math_on, int rot_on, int nblocks) {
  using C = JacCfg<32>;
  constexpr int NG = 8 / GW;
  const size_t smem = sizeof(double2) * (NG * 32 * C::LDGG + NG * 32 * C::LDG + NG * 8 * 64 + 2 * C::BUF);
  cudaFuncSetAttribute(bench_kernel<PLACE, GW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  long long* d;
  cudaMalloc(&d, 8 * 4 * nblocks);
  const int reps = 100;
  for (int pass = 0; pass < 2; ++pass) {
    cudaMemset(d, 0, 8 * 4 * nblocks);
    bench_kernel<PLACE, GW><<<nblocks, 1024, smem>>>(dG, reps, math_on, rot_on, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
  }
  std::vector<long long> h(4 * nblocks);
  cudaMemcpy(h.data(), d, 8 * 4 * nblocks, cudaMemcpyDeviceToHost);
  const double rot_round = rot_on ? (double)h[0] / reps / 16 : 0.0;
  // per math iteration one warp issues 48 DMMA; SM peak = 4 DMMA per 16 cycles
  const double dmma = (double)h[1] * 48.0;
  const double frac = h[2] ? dmma / ((double)h[2] * 0.25) : 0.0;
  printf("%-44s rot %6.0f cyc/round (%d sweeps in flight)   math DMMA %5.1f%% of SM peak\n", name,
         rot_round, rot_on ? NG : 0, 100.0 * frac);
  cudaFree(d);
}

int main(int argc, char** argv) {
  const int nblocks = argc > 1 ? atoi(argv[1]) : 1;
  const int W2 = 32, R = 512;
  std::vector<double2> P(R * W2), Gm(W2 * W2);
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
      Gm[i + j * W2] = make_double2(re * 1e-3, im * 1e-3);
    }
  double2* dG;
  cudaMalloc(&dG, sizeof(double2) * W2 * W2);
  cudaMemcpy(dG, Gm.data(), sizeof(double2) * W2 * W2, cudaMemcpyHostToDevice);
  printf("blocks %d (one 1024-thread CTA per SM)\n", nblocks);
  run<0, 8>("spread rot (8 warps), math idle", dG, 0, 1, nblocks);
  run<1, 8>("SMSP0 rot (8 warps), math idle", dG, 0, 1, nblocks);
  run<0, 8>("math only, 24 warps on 4 SMSPs", dG, 1, 0, nblocks);
  run<1, 8>("math only, 24 warps on SMSP 1-3", dG, 1, 0, nblocks);
  run<0, 8>("spread rot (8 warps) + math 24 warps", dG, 1, 1, nblocks);
  run<1, 8>("SMSP0 rot (8 warps) + math SMSP 1-3", dG, 1, 1, nblocks);
  run<2, 8>("spread rot (warps 24-31) + math 24 warps", dG, 1, 1, nblocks);
  run<3, 8>("SMSP3 rot (8 warps) + math SMSP 0-2", dG, 1, 1, nblocks);
  run<0, 4>("spread rot 2 x 4 warps + math", dG, 1, 1, nblocks);
  run<2, 4>("spread rot 2 x 4 warps (24-31) + math", dG, 1, 1, nblocks);
  run<3, 4>("SMSP3 rot 2 x 4 warps + math SMSP 0-2", dG, 1, 1, nblocks);
  run<1, 4>("SMSP0 rot 2 x 4 warps + math SMSP 1-3", dG, 1, 1, nblocks);
  run<1, 4>("SMSP0 rot 2 x 4 warps, math idle", dG, 0, 1, nblocks);
  return 0;
}
