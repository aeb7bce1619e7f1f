// Microbenchmark of the Jacobi inner (Gram-space) sweep alone: one CTA per
// launch, a 32x32 Hermitian Gram from a random 512x32 panel, cross rounds
// (as on a cross visit) -- cycles per round without the rest of the pipeline.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I include -I paper_1807_07914_b200/csrc \
//   -o tools/inner_bench tools/inner_bench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "bmps_jacobi.cuh"
using namespace bmps;

template <int W2>
__global__ void inner_kernel(const double2* G0, int reps, long long* cyc, int* nrot, double2* Gout, double2* Qout) {
  using C = JacCfg<W2>;
  __shared__ double2 sG[W2 * C::LDGG];
  __shared__ double2 sQ[W2 * C::LDG];
  __shared__ RotShared rs;
  long long tot = 0;
  int nr = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int i = threadIdx.x; i < W2 * W2; i += blockDim.x)
      sG[(i % W2) + (i / W2) * C::LDGG] = G0[i];
    __syncthreads();
    const long long t0 = clock64();
    nr += jac_inner<W2>(sG, sQ, rs, 4.0 * sqrt(512.0) * kEps, 1e-28, 1.0, false, 1);
    __syncthreads();
    tot += clock64() - t0;
  }
  if (threadIdx.x == 0) { *cyc = tot; *nrot = nr; }
  for (int i = threadIdx.x; i < W2 * W2; i += blockDim.x) {
    Gout[i] = sG[(i % W2) + (i / W2) * C::LDGG];
    Qout[i] = sQ[(i % W2) + (i / W2) * C::LDG];
  }
}


// Configurable copy of jac_inner's cross path: MODE bit0 = G update, bit1 = Q update
template <int W2, int MODE>
__device__ int inner_var(double2* sG, double2* sQ, RotShared& rs, double tol, double noise2, double fro) {
  using C = JacCfg<W2>;
  constexpr int w = W2 / 2;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < W2 * W2; idx += blockDim.x) {
    const int i = idx % W2, j = idx / W2;
    sQ[i + j * C::LDG] = make_double2(i == j ? 1.0 : 0.0, 0.0);
  }
  int any = 0;
  int pq_q = (int)((sqrtf(8.0f * (float)tid + 1.0f) - 1.0f) * 0.5f);
  const int pq_p = tid - pq_q * (pq_q + 1) / 2;
  for (int rho = 0; rho < w; ++rho) {
    int act = 0;
    if (tid < w) {
      const int i = tid, j = w + (tid + rho) % w;
      double c = 1.0, s = 0.0;
      double2 e = make_double2(1.0, 0.0);
      act = jacobi_rotation(sG[i + i * C::LDGG].x, sG[j + j * C::LDGG].x, sG[i + j * C::LDGG], tol, noise2, fro, c, s, e);
      if (!act) { c = 1.0; s = 0.0; e = make_double2(1.0, 0.0); }
      rs.i[tid] = i; rs.j[tid] = j; rs.act[tid] = act; rs.c[tid] = c; rs.s[tid] = s; rs.e[tid] = e;
      rs.se[tid] = cscale(e, s); rs.ce[tid] = cscale(e, c);
    }
    const int nact = __syncthreads_count(act);
    any += nact;
    if (nact == 0) continue;
    if (MODE & 1) {
      for (int idx = tid; idx < w * (w + 1) / 2; idx += blockDim.x) {
        const int q = (MODE & 256) ? pq_q : (int)((sqrtf(8.0f * (float)idx + 1.0f) - 1.0f) * 0.5f);
        const int p = (MODE & 256) ? pq_p : idx - q * (q + 1) / 2;
        if (!(MODE & 16) && !(rs.act[p] | rs.act[q])) continue;
        const int ip = (MODE & 32) ? p : rs.i[p], jp = (MODE & 32) ? w + (p + rho) % w : rs.j[p];
        const int iq = (MODE & 32) ? q : rs.i[q], jq = (MODE & 32) ? w + (q + rho) % w : rs.j[q];
        const double cp = rs.c[p], sp = rs.s[p], cq = rs.c[q], sq = rs.s[q];
        const double2 sep = rs.se[p], cep = rs.ce[p], seq = rs.se[q], ceq = rs.ce[q];
        double2 g00, g01, g10, g11;
        if (MODE & 64) {
          g00 = make_double2(ip, iq); g01 = make_double2(ip, jq); g10 = make_double2(jp, iq); g11 = make_double2(jp, jq);
        } else {
          g00 = sG[ip + iq * C::LDGG]; g01 = sG[ip + jq * C::LDGG];
          g10 = sG[jp + iq * C::LDGG]; g11 = sG[jp + jq * C::LDGG];
        }
        const double2 r00 = cmsc(g00, cq, seq, g01), r01 = cmac(g00, sq, ceq, g01);
        const double2 r10 = cmsc(g10, cq, seq, g11), r11 = cmac(g10, sq, ceq, g11);
        double2 n00 = cms(r00, cp, sep, r10), n01 = cms(r01, cp, sep, r11);
        double2 n10 = cma(r00, sp, cep, r10), n11 = cma(r01, sp, cep, r11);
        if (MODE & 8) { n00 = g00; n01 = g01; n10 = g10; n11 = g11; }
        if (MODE & 128) {
          if (n00.x == 12345.0 && n01.y == 1.0 && n10.x == 3.0 && n11.y == 2.0) sG[0] = n00;
          continue;
        }
        sG[ip + iq * C::LDGG] = n00; sG[ip + jq * C::LDGG] = n01;
        sG[jp + iq * C::LDGG] = n10; sG[jp + jq * C::LDGG] = n11;
        if (!(MODE & 4) && p != q) {
          sG[iq + ip * C::LDGG] = cconj(n00); sG[jq + ip * C::LDGG] = cconj(n01);
          sG[iq + jp * C::LDGG] = cconj(n10); sG[jq + jp * C::LDGG] = cconj(n11);
        }
      }
    }
    if (MODE & 2) {
      for (int idx = tid; idx < W2 * w; idx += blockDim.x) {
        const int k = idx % W2, q = idx / W2;
        if (!rs.act[q]) continue;
        const int iq = rs.i[q], jq = rs.j[q];
        const double cq = rs.c[q], sq = rs.s[q];
        const double2 qi = sQ[k + iq * C::LDG], qj = sQ[k + jq * C::LDG];
        sQ[k + iq * C::LDG] = cmsc(qi, cq, rs.se[q], qj);
        sQ[k + jq * C::LDG] = cmac(qi, sq, rs.ce[q], qj);
      }
    }
    __syncthreads();
  }
  return any;
}

template <int W2, int MODE>
__global__ void var_kernel(const double2* G0, int reps, long long* cyc, int* nrot) {
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
    nr += inner_var<W2, MODE>(sG, sQ, rs, 4.0 * sqrt(512.0) * kEps, 1e-28, 1.0);
    __syncthreads();
    tot += clock64() - t0;
  }
  if (threadIdx.x == 0) { *cyc = tot; *nrot = nr; }
}

int main() {
  const int W2 = 32, R = 512;
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
  double2 *dG, *dO, *dQ, *dO2, *dQ2; long long* dc; int* dn;
  cudaMalloc(&dG, sizeof(double2) * W2 * W2); cudaMalloc(&dO, sizeof(double2) * W2 * W2);
  cudaMalloc(&dQ, sizeof(double2) * W2 * W2); cudaMalloc(&dO2, sizeof(double2) * W2 * W2);
  cudaMalloc(&dQ2, sizeof(double2) * W2 * W2);
  cudaMalloc(&dc, 8); cudaMalloc(&dn, 4);
  cudaMemcpy(dG, G.data(), sizeof(double2) * W2 * W2, cudaMemcpyHostToDevice);
  const int reps = 200;
  inner_kernel<32><<<1, 256>>>(dG, 2, dc, dn, dO, dQ);
  inner_kernel<32><<<1, 256>>>(dG, reps, dc, dn, dO, dQ);
  long long c; int n;
  cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&n, dn, 4, cudaMemcpyDeviceToHost);
  printf("cross inner sweep: %.0f cycles per sweep, %.0f per round (16 rounds), rotations/sweep %d\n",
         (double)c / reps, (double)c / reps / 16, n / reps);
  const char* names[13] = {"rotations only", "+G", "+Q", "+G+Q", "G nomirror", "G nomath", "G noact", "G arith idx", "G all three",
                           "G noloads", "G nostores", "G pq hoisted", "G nold nost"};
  for (int mode = 0; mode < 13; ++mode) {
    if (mode == 0) var_kernel<32, 0><<<1, 256>>>(dG, reps, dc, dn);
    if (mode == 1) var_kernel<32, 1><<<1, 256>>>(dG, reps, dc, dn);
    if (mode == 2) var_kernel<32, 2><<<1, 256>>>(dG, reps, dc, dn);
    if (mode == 3) var_kernel<32, 3><<<1, 256>>>(dG, reps, dc, dn);
    if (mode == 4) var_kernel<32, 1 | 4><<<1, 256>>>(dG, reps, dc, dn);
    if (mode == 5) var_kernel<32, 1 | 8><<<1, 256>>>(dG, reps, dc, dn);
    if (mode == 6) var_kernel<32, 1 | 16><<<1, 256>>>(dG, reps, dc, dn);
    if (mode == 7) var_kernel<32, 1 | 32><<<1, 256>>>(dG, reps, dc, dn);
    if (mode == 8) var_kernel<32, 1 | 4 | 16 | 32><<<1, 256>>>(dG, reps, dc, dn);
    if (mode == 9) var_kernel<32, 1 | 64><<<1, 256>>>(dG, reps, dc, dn);
    if (mode == 10) var_kernel<32, 1 | 128><<<1, 256>>>(dG, reps, dc, dn);
    if (mode == 11) var_kernel<32, 1 | 256><<<1, 256>>>(dG, reps, dc, dn);
    if (mode == 12) var_kernel<32, 1 | 64 | 128><<<1, 256>>>(dG, reps, dc, dn);
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&n, dn, 4, cudaMemcpyDeviceToHost);
    printf("variant %-15s: %.0f cycles per round (rot/sweep %d)\n", names[mode], (double)c / reps / 16, n / reps);
  }
  return 0;
}
