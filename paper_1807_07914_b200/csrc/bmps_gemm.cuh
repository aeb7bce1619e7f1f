// Batched complex128 GEMM tile engine on FP64 tensor cores (DMMA m8n8k4).
//
// One CTA (256 threads = 8 warps arranged 2 x 4) computes a 64 x 64 complex
// tile of C = A * B, staging K in chunks of 16 through shared memory. The
// operand element loaders, problem shape and epilogue are supplied by an Op
// type so the same engine serves the theta contraction, the SVD split and the
// environment transfers (shapes are read on the device, so no host sync is
// needed between a producer and this consumer):
//
//   struct Op {
//     static constexpr bool kAKMajor;   // A(i,k) contiguous in k (else in i)
//     static constexpr bool kBKMajor;   // B(k,j) contiguous in k (else in j)
//     __device__ bool begin(int item, int& M, int& N, int& K);
//     __device__ double2 a(int i, int k) const;
//     __device__ double2 b(int k, int j) const;
//     __device__ void store(int i, int j, double2 v) const;
//   };
#pragma once
#include "bmps_common.cuh"

namespace bmps {

constexpr int kTile = 64;
constexpr int kKC = 16;
// padded row of the k-major staging tiles, in 16-byte elements (2 would make the DMMA
// fragment loads conflict-free but the k-major operand stores 2-way: measured no gain)
#ifndef BMPS_GEMM_PAD
#define BMPS_GEMM_PAD 1
#endif
constexpr int kLds = kTile + BMPS_GEMM_PAD;
#ifndef BMPS_GEMM_MINB
#define BMPS_GEMM_MINB 2
#endif

// Chunk k0 of both operands, global -> registers (4 + 4 elements per thread), and
// registers -> the k-major staging tiles. Split so that the main loop can have chunk
// k + 1's global loads in flight while chunk k is multiplied (gemm_mainloop).
template <class Op>
BMPS_DEV void gemm_fetch_chunk(const Op& op, double2 (&ra)[4], double2 (&rb)[4], int M, int N, int K,
                               int m0, int n0, int k0, int tid) {
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int kk = Op::kAKMajor ? (tid & 15) : (tid >> 6) + 4 * it;
    const int i = Op::kAKMajor ? (tid >> 4) + 16 * it : (tid & 63);
    const int gi = m0 + i, gk = k0 + kk;
    ra[it] = (gi < M && gk < K) ? op.a(gi, gk) : make_double2(0.0, 0.0);
  }
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int kk = Op::kBKMajor ? (tid & 15) : (tid >> 6) + 4 * it;
    const int j = Op::kBKMajor ? (tid >> 4) + 16 * it : (tid & 63);
    const int gj = n0 + j, gk = k0 + kk;
    rb[it] = (gj < N && gk < K) ? op.b(gk, gj) : make_double2(0.0, 0.0);
  }
}

template <class Op>
BMPS_DEV void gemm_stage_chunk(double2 (*sA)[kLds], double2 (*sB)[kLds], const double2 (&ra)[4],
                               const double2 (&rb)[4], int tid) {
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int kk = Op::kAKMajor ? (tid & 15) : (tid >> 6) + 4 * it;
    const int i = Op::kAKMajor ? (tid >> 4) + 16 * it : (tid & 63);
    sA[kk][i] = ra[it];
  }
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int kk = Op::kBKMajor ? (tid & 15) : (tid >> 6) + 4 * it;
    const int j = Op::kBKMajor ? (tid >> 4) + 16 * it : (tid & 63);
    sB[kk][j] = rb[it];
  }
}

// acc[mi][ni][4]: warp tile 32 x 16 = 4 x 2 DMMA tiles; (re0, re1, im0, im1). The 4-product
// form here: 8 tiles x 6 accumulators of the 3-product form cost occupancy (measured slower).
BMPS_DEV void gemm_mma_chunk(double (&acc)[4][2][4], const double2 (*sA)[kLds],
                             const double2 (*sB)[kLds], int wm, int wn, int lane) {
  const int kr = lane & 3, rc = lane >> 2;
#pragma unroll
  for (int k4 = 0; k4 < kKC / 4; ++k4) {
    double2 a[4], b[2];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) a[mi] = sA[k4 * 4 + kr][wm * 32 + mi * 8 + rc];
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) b[ni] = sB[k4 * 4 + kr][wn * 16 + ni * 8 + rc];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) zmma(acc[mi][ni], a[mi], b[ni]);
  }
}

// acc += A[m0.., :] B[:, n0..] over all of K: the next chunk's operands travel from global
// memory to registers while the staged chunk is on the tensor pipe (the loop used to expose
// one global round trip per 16-deep chunk); same arithmetic in the same order.
template <class Op>
BMPS_DEV void gemm_mainloop(const Op& op, double (&acc)[4][2][4], double2 (*sA)[kLds],
                            double2 (*sB)[kLds], int M, int N, int K, int m0, int n0, int tid) {
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;
  double2 ra[4], rb[4];
  gemm_fetch_chunk(op, ra, rb, M, N, K, m0, n0, 0, tid);
  for (int k0 = 0; k0 < K; k0 += kKC) {
    gemm_stage_chunk<Op>(sA, sB, ra, rb, tid);
    __syncthreads();
    if (k0 + kKC < K) gemm_fetch_chunk(op, ra, rb, M, N, K, m0, n0, k0 + kKC, tid);
    gemm_mma_chunk(acc, sA, sB, wm, wn, lane);
    __syncthreads();
  }
}

template <class Op>
__global__ void __launch_bounds__(256, BMPS_GEMM_MINB) gemm_kernel(Op op) {
  __shared__ __align__(16) double2 sA[kKC][kLds];
  __shared__ __align__(16) double2 sB[kKC][kLds];
  int M, N, K;
  if (!op.begin(blockIdx.z, M, N, K)) return;
  const int m0 = blockIdx.x * kTile, n0 = blockIdx.y * kTile;
  if (m0 >= M || n0 >= N) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;
  double acc[4][2][4];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[mi][ni][q] = 0.0;
  gemm_mainloop(op, acc, sA, sB, M, N, K, m0, n0, tid);
  const int rr = lane >> 2, cc = (lane & 3) * 2;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = m0 + wm * 32 + mi * 8 + rr, j = n0 + wn * 16 + ni * 8 + cc + h;
        if (i < M && j < N) op.store(i, j, make_double2(acc[mi][ni][h], acc[mi][ni][2 + h]));
      }
}

}  // namespace bmps
