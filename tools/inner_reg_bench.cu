// Prototype for round 2: the Jacobi inner (Gram-space) cross sweep with
// G and Q register-resident in one 4-warp group, against the shared-memory jac_inner
// of the kernel. One CTA, a 32x32 Hermitian Gram of a random 512x32 panel, cycles per
// cross round, and a consistency check of the result.
//
// Layout: warp g, lane c (= column c). I-rows p = 4g..4g+3 (GI[u] = G[p, c]) and the
// J-rows paired with them in round rho, jr = 16 + (p + rho) mod 16 (GJ[u] = G[jr, c]);
// Q rows 8g..8g+7 (QR[k] = Q[8g + k, c]). Per round: pivots by shuffles, every lane
// computes its warp's 4 rotations (same jacobi_rotation as the kernel), row rotations
// inside the thread, the 16 pairs' parameters through shared memory (barrier 1),
// column rotations of G and Q by lane shuffles, then the J rows advance by one pair
// (a register move, one shared exchange with the next warp: barrier 2).
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I include -I paper_1807_07914_b200/csrc \
//   -o tools/inner_reg_bench tools/inner_reg_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "bmps_jacobi.cuh"
using namespace bmps;

constexpr int W2 = 32, w = 16;
#ifndef ONE_ROT_PER_LANE
#define ONE_ROT_PER_LANE 1
#endif

BMPS_DEV double2 shfl2(double2 v, int src) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

__global__ void __launch_bounds__(128) reg_inner_kernel(const double2* G0, int reps, long long* cyc,
                                                        int* nrot, double2* Gout, double2* Qout) {
  __shared__ double s_c[w], s_s[w];
  __shared__ double2 s_e[w];
  __shared__ int s_act[w];
  __shared__ double2 s_x[4][32];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const double tol = 4.0 * sqrt(512.0) * kEps, noise2 = 1e-28, fro = 1.0;
  long long tot = 0;
  int nr = 0;
  double2 GI[4], GJ[4], QR[8];
  for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      GI[u] = G0[(4 * g + u) + lane * W2];
      GJ[u] = G0[(16 + 4 * g + u) + lane * W2];
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) QR[k] = make_double2(8 * g + k == lane ? 1.0 : 0.0, 0.0);
    __syncthreads();
    const long long t0 = clock64();
    for (int rho = 0; rho < w; ++rho) {
      // 1. this warp's 4 rotations (every lane computes them)
      double cu[4], su[4];
      double2 eu[4];
      int au[4];
#if ONE_ROT_PER_LANE
      // pivots of all 4 pairs to every lane, then lane group u = lane / 8 computes
      // rotation u only and lanes 0, 8, 16, 24 broadcast the parameters
      double pa[4], pb[4];
      double2 pg[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int p = 4 * g + u, jr = 16 + (p + rho) % 16;
        pa[u] = __shfl_sync(0xffffffffu, GI[u].x, p);
        pb[u] = __shfl_sync(0xffffffffu, GJ[u].x, jr);
        pg[u] = shfl2(GI[u], jr);
      }
      const int grp = lane >> 3;
      const double a = grp == 0 ? pa[0] : grp == 1 ? pa[1] : grp == 2 ? pa[2] : pa[3];
      const double b = grp == 0 ? pb[0] : grp == 1 ? pb[1] : grp == 2 ? pb[2] : pb[3];
      const double2 gg = grp == 0 ? pg[0] : grp == 1 ? pg[1] : grp == 2 ? pg[2] : pg[3];
      double c = 1.0, s = 0.0;
      double2 e = make_double2(1.0, 0.0);
      int ract = jacobi_rotation(a, b, gg, tol, noise2, fro, c, s, e);
      if (!ract) {
        c = 1.0;
        s = 0.0;
        e = make_double2(1.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        cu[u] = __shfl_sync(0xffffffffu, c, 8 * u);
        su[u] = __shfl_sync(0xffffffffu, s, 8 * u);
        eu[u] = shfl2(e, 8 * u);
        au[u] = __shfl_sync(0xffffffffu, ract, 8 * u);
      }
      if ((lane & 7) == 0) {
        const int p = 4 * g + grp;
        s_c[p] = c;
        s_s[p] = s;
        s_e[p] = e;
        s_act[p] = ract;
      }
#else
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int p = 4 * g + u, jr = 16 + (p + rho) % 16;
        const double a = __shfl_sync(0xffffffffu, GI[u].x, p);
        const double b = __shfl_sync(0xffffffffu, GJ[u].x, jr);
        const double2 gg = shfl2(GI[u], jr);
        double c = 1.0, s = 0.0;
        double2 e = make_double2(1.0, 0.0);
        au[u] = jacobi_rotation(a, b, gg, tol, noise2, fro, c, s, e);
        if (!au[u]) {
          c = 1.0;
          s = 0.0;
          e = make_double2(1.0, 0.0);
        }
        cu[u] = c;
        su[u] = s;
        eu[u] = e;
        if (lane == 0) {
          s_c[p] = c;
          s_s[p] = s;
          s_e[p] = e;
          s_act[p] = au[u];
        }
      }
#endif
      // 2. row rotations, inside the thread: G[p,:], G[jr,:] <- J^H [G[p,:]; G[jr,:]]
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (!au[u]) continue;
        const double2 se = cscale(eu[u], su[u]), ce = cscale(eu[u], cu[u]);
        const double2 ni = cms(GI[u], cu[u], se, GJ[u]);
        const double2 nj = cma(GI[u], su[u], ce, GJ[u]);
        GI[u] = ni;
        GJ[u] = nj;
      }
      __barrier_sync_count(1, 128);
      // 3. column rotations of G and Q: lane c pairs with its column's partner
      const int q = lane < w ? lane : (lane - w - rho + 2 * w) % w;
      const int partner = lane < w ? w + (lane + rho) % w : q;
      const int act = s_act[q];
      const double cq = s_c[q], sq = s_s[q];
      const double2 eq = s_e[q];
      const double2 se = cscale(eq, sq), ce = cscale(eq, cq);
      const bool iside = lane < w;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double2 yi = shfl2(GI[u], partner), yj = shfl2(GJ[u], partner);
        if (act) {
          GI[u] = iside ? cmsc(GI[u], cq, se, yi) : cmac(yi, sq, ce, GI[u]);
          GJ[u] = iside ? cmsc(GJ[u], cq, se, yj) : cmac(yj, sq, ce, GJ[u]);
        }
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const double2 y = shfl2(QR[k], partner);
        if (act) QR[k] = iside ? cmsc(QR[k], cq, se, y) : cmac(y, sq, ce, QR[k]);
      }
      if (threadIdx.x == 0)
        for (int p = 0; p < w; ++p) nr += s_act[p];
      // 4. the J rows advance by one pair: GJ[u] <- GJ[u+1], GJ[3] <- next warp's GJ[0]
      s_x[g][lane] = GJ[0];
#pragma unroll
      for (int u = 0; u < 3; ++u) GJ[u] = GJ[u + 1];
      __barrier_sync_count(1, 128);
      GJ[3] = s_x[(g + 1) & 3][lane];
    }
    __syncthreads();
    tot += clock64() - t0;
  }
  if (threadIdx.x == 0) {
    *cyc = tot;
    *nrot = nr;
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    Gout[(4 * g + u) + lane * W2] = GI[u];
    Gout[(16 + 4 * g + u) + lane * W2] = GJ[u];
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) Qout[(8 * g + k) + lane * W2] = QR[k];
}

// The kernel's shared-memory inner sweep (CtaGrp, 256 threads) on the same Gram.
__global__ void smem_inner_kernel(const double2* G0, int reps, long long* cyc, int* nrot, double2* Gout,
                                  double2* Qout) {
  using C = JacCfg<W2>;
  __shared__ double2 sG[W2 * C::LDGG];
  __shared__ double2 sQ[W2 * C::LDG];
  __shared__ RotShared rs;
  long long tot = 0;
  int nr = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int i = threadIdx.x; i < W2 * W2; i += blockDim.x) sG[(i % W2) + (i / W2) * C::LDGG] = G0[i];
    __syncthreads();
    const long long t0 = clock64();
    nr += jac_inner<W2>(sG, sQ, rs, 4.0 * sqrt(512.0) * kEps, 1e-28, 1.0, false, 1);
    __syncthreads();
    tot += clock64() - t0;
  }
  if (threadIdx.x == 0) {
    *cyc = tot;
    *nrot = nr;
  }
  for (int i = threadIdx.x; i < W2 * W2; i += blockDim.x) {
    Gout[i] = sG[(i % W2) + (i / W2) * C::LDGG];
    Qout[i] = sQ[(i % W2) + (i / W2) * C::LDG];
  }
}

int main() {
  const int R = 512;
  std::vector<double2> P(R * W2), G(W2 * W2);
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
  double2 *dG, *dGa, *dQa, *dGb, *dQb;
  long long* dc;
  int* dn;
  cudaMalloc(&dG, sizeof(double2) * W2 * W2);
  cudaMalloc(&dGa, sizeof(double2) * W2 * W2);
  cudaMalloc(&dQa, sizeof(double2) * W2 * W2);
  cudaMalloc(&dGb, sizeof(double2) * W2 * W2);
  cudaMalloc(&dQb, sizeof(double2) * W2 * W2);
  cudaMalloc(&dc, 8);
  cudaMalloc(&dn, 4);
  cudaMemcpy(dG, G.data(), sizeof(double2) * W2 * W2, cudaMemcpyHostToDevice);
  const int reps = 200;
  long long c;
  int n;
  smem_inner_kernel<<<1, 256>>>(dG, 2, dc, dn, dGa, dQa);
  smem_inner_kernel<<<1, 256>>>(dG, reps, dc, dn, dGa, dQa);
  cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(&n, dn, 4, cudaMemcpyDeviceToHost);
  printf("shared-memory inner (256 thr): %.0f cycles per cross round, rotations/sweep %d\n",
         (double)c / reps / w, n / reps);
  reg_inner_kernel<<<1, 128>>>(dG, 2, dc, dn, dGb, dQb);
  reg_inner_kernel<<<1, 128>>>(dG, reps, dc, dn, dGb, dQb);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(&n, dn, 4, cudaMemcpyDeviceToHost);
  printf("register inner   (128 thr): %.0f cycles per cross round, rotations/sweep %d\n",
         (double)c / reps / w, n / reps);
  // consistency: G' = Q^H G0 Q for the register version; distance to the shared version
  std::vector<double2> Ga(W2 * W2), Qa(W2 * W2), Gb(W2 * W2), Qb(W2 * W2);
  cudaMemcpy(Ga.data(), dGa, sizeof(double2) * W2 * W2, cudaMemcpyDeviceToHost);
  cudaMemcpy(Qa.data(), dQa, sizeof(double2) * W2 * W2, cudaMemcpyDeviceToHost);
  cudaMemcpy(Gb.data(), dGb, sizeof(double2) * W2 * W2, cudaMemcpyDeviceToHost);
  cudaMemcpy(Qb.data(), dQb, sizeof(double2) * W2 * W2, cudaMemcpyDeviceToHost);
  double gmax = 0, dab = 0, cons = 0, offa = 0, offb = 0;
  for (int i = 0; i < W2 * W2; ++i) gmax = fmax(gmax, hypot(G[i].x, G[i].y));
  for (int i = 0; i < W2; ++i)
    for (int j = 0; j < W2; ++j) {
      const double2 a = Ga[i + j * W2], b = Gb[i + j * W2];
      dab = fmax(dab, hypot(a.x - b.x, a.y - b.y));
      if (i < w && j >= w) {
        offa = fmax(offa, hypot(a.x, a.y));
        offb = fmax(offb, hypot(b.x, b.y));
      }
      // (Q^H G0 Q)_{ij}
      double re = 0, im = 0;
      for (int k = 0; k < W2; ++k)
        for (int l = 0; l < W2; ++l) {
          const double2 qk = Qb[k + i * W2], g0 = G[k + l * W2], ql = Qb[l + j * W2];
          // conj(qk) * g0 * ql
          const double tr = qk.x * g0.x + qk.y * g0.y, ti = qk.x * g0.y - qk.y * g0.x;
          re += tr * ql.x - ti * ql.y;
          im += tr * ql.y + ti * ql.x;
        }
      cons = fmax(cons, hypot(re - b.x, im - b.y));
    }
  printf("max|G0| %.3e; |G_reg - G_smem| %.2e; |Q^H G0 Q - G_reg| %.2e; max cross |G_IJ| smem %.2e reg %.2e\n",
         gmax, dab, cons, offa, offb);
  return 0;
}
