// Dense statevector backend (R:src/mpsqvm/dense.py) on sm_100a -- the GPU
// counterpart of the reference's SVD-free cross-check simulator (SURVEY §8(f)
// row 4). A state is complex128 [2^n] in HBM, flat index with qubit 0 as the
// HIGH bit (dense.py:23), i.e. qubit q is bit (n - 1 - q).
//
// Every kernel here is HBM-bound integer-indexed streaming (no GEMM shape):
//   dense_1q / dense_2q : one pass over the state per gate, each thread owning
//                         the 2 (4) amplitudes a gate mixes; consecutive threads
//                         touch consecutive addresses for every target bit, so
//                         loads/stores are coalesced; grid-stride over a wave of
//                         148 x 8 CTAs.
//   dense_run_smem      : n <= 12 (64 KB): one CTA per state keeps the whole
//                         state in shared memory and applies the full gate list
//                         (the batched VQE-sweep / small-circuit case, where a
//                         per-gate launch would be launch-bound).
//   dense_expect        : <psi|P|psi> for Pauli strings as one fused pass,
//                         sum_i conj(psi_i) (-i)^{nY} (-1)^{popc(i & zy)} psi_{i ^ x},
//                         deterministic two-level reduction (fixed block order).
//   dense_tree_*        : heap of marginal probabilities (node (k, v) = total
//                         |psi|^2 of the states whose top k bits are v) for the
//                         sequential conditional sampler (dense.py:88-110).
#pragma once
#include "bmps_common.cuh"

namespace bmps {

struct DenseGate2 {
  double2 m[4];   // row-major 2x2
};
struct DenseGate4 {
  double2 m[16];  // row-major 4x4, [2a+b][2s+t], a/s on the first qubit (gates.py:3-4)
};

constexpr int kDenseSmemQubits = 12;  // 2^12 x 16 B = 64 KB of shared memory per state
constexpr int kDenseMaxQubits = 33;   // 2^33 x 16 B = 128 GB of the 180 GB HBM

// insert a zero bit at position b of t
BMPS_DEV unsigned long long ins0(unsigned long long t, int b) {
  return ((t >> b) << (b + 1)) | (t & ((1ull << b) - 1ull));
}

__global__ void __launch_bounds__(256) dense_init_kernel(double2* a, int S, unsigned long long N) {
  const unsigned long long total = N * (unsigned long long)S;
  for (unsigned long long i = blockIdx.x * 256ull + threadIdx.x; i < total; i += gridDim.x * 256ull)
    a[i] = make_double2(i % N == 0 ? 1.0 : 0.0, 0.0);
}

__global__ void __launch_bounds__(256) dense_1q_kernel(double2* a, int n, int q, DenseGate2 g) {
  const int b = n - 1 - q;
  const unsigned long long half = 1ull << (n - 1), bit = 1ull << b;
  for (unsigned long long t = blockIdx.x * 256ull + threadIdx.x; t < half; t += gridDim.x * 256ull) {
    const unsigned long long i0 = ins0(t, b), i1 = i0 | bit;
    const double2 x = a[i0], y = a[i1];
    a[i0] = cfma(g.m[1], y, cmul(g.m[0], x));
    a[i1] = cfma(g.m[3], y, cmul(g.m[2], x));
  }
}

__global__ void __launch_bounds__(256) dense_2q_kernel(double2* a, int n, int q1, int q2,
                                                       DenseGate4 g) {
  const int b1 = n - 1 - q1, b2 = n - 1 - q2;
  const int lo = min(b1, b2), hi = max(b1, b2);
  const unsigned long long quarter = 1ull << (n - 2), m1 = 1ull << b1, m2 = 1ull << b2;
  for (unsigned long long t = blockIdx.x * 256ull + threadIdx.x; t < quarter; t += gridDim.x * 256ull) {
    const unsigned long long base = ins0(ins0(t, lo), hi);
    const unsigned long long idx[4] = {base, base | m2, base | m1, base | m1 | m2};
    double2 x[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) x[k] = a[idx[k]];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      double2 acc = cmul(g.m[4 * r], x[0]);
#pragma unroll
      for (int k = 1; k < 4; ++k) acc = cfma(g.m[4 * r + k], x[k], acc);
      a[idx[r]] = acc;
    }
  }
}

// Whole gate list on one shared-memory resident state per CTA (n <= 12).
// ops[s][k] = (arity, q1, q2); mats[s][k] = 16 complex (2x2 gates use the first 4).
__global__ void __launch_bounds__(512) dense_run_smem_kernel(double2* amps, int n, const int* ops,
                                                             const double2* mats, int nops) {
  extern __shared__ __align__(16) double2 dsm[];
  const int s = blockIdx.x;
  const int N = 1 << n;
  double2* a = amps + (size_t)s * N;
  for (int i = threadIdx.x; i < N; i += blockDim.x) dsm[i] = a[i];
  __syncthreads();
  const int* op = ops + (size_t)s * nops * 3;
  const double2* mt = mats + (size_t)s * nops * 16;
  for (int k = 0; k < nops; ++k) {
    const int ar = op[3 * k], q1 = op[3 * k + 1], q2 = op[3 * k + 2];
    const double2* g = mt + (size_t)k * 16;
    if (ar == 1) {
      const int b = n - 1 - q1;
      const double2 g0 = g[0], g1 = g[1], g2 = g[2], g3 = g[3];
      for (int t = threadIdx.x; t < N / 2; t += blockDim.x) {
        const int i0 = (int)ins0(t, b), i1 = i0 | (1 << b);
        const double2 x = dsm[i0], y = dsm[i1];
        dsm[i0] = cfma(g1, y, cmul(g0, x));
        dsm[i1] = cfma(g3, y, cmul(g2, x));
      }
    } else {
      const int b1 = n - 1 - q1, b2 = n - 1 - q2;
      const int lo = min(b1, b2), hi = max(b1, b2);
      for (int t = threadIdx.x; t < N / 4; t += blockDim.x) {
        const int base = (int)ins0(ins0(t, lo), hi);
        const int idx[4] = {base, base | (1 << b2), base | (1 << b1), base | (1 << b1) | (1 << b2)};
        double2 x[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) x[j] = dsm[idx[j]];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          double2 acc = cmul(g[4 * r], x[0]);
#pragma unroll
          for (int j = 1; j < 4; ++j) acc = cfma(g[4 * r + j], x[j], acc);
          dsm[idx[r]] = acc;
        }
      }
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < N; i += blockDim.x) a[i] = dsm[i];
}

// Partial sums of sum_i conj(psi_i) sign(i) psi_{i ^ x} per (block, string);
// masks[2k] = x mask (X and Y positions), masks[2k+1] = sign mask (Z and Y).
constexpr int kDenseExpBlocks = 296;   // 2 waves of 148 SMs
__global__ void __launch_bounds__(256) dense_expect_partial_kernel(
    const double2* amps, int n, const int* state_idx, const unsigned long long* masks,
    double2* partial) {
  const int k = blockIdx.y;
  const unsigned long long N = 1ull << n;
  const double2* a = amps + (size_t)state_idx[k] * N;
  const unsigned long long xm = masks[2 * k], zm = masks[2 * k + 1];
  double2 acc = make_double2(0.0, 0.0);
  for (unsigned long long i = blockIdx.x * 256ull + threadIdx.x; i < N; i += gridDim.x * 256ull) {
    const double2 u = a[i], v = a[i ^ xm];
    const double2 t = cmul(cconj(u), v);
    if (__popcll(i & zm) & 1) acc = csub(acc, t);
    else acc = cadd(acc, t);
  }
  __shared__ double2 red[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 t = red[0];
    for (int w = 1; w < 8; ++w) t = cadd(t, red[w]);
    partial[(size_t)k * gridDim.x + blockIdx.x] = t;
  }
}

// out[k] = (-i)^{ny[k]} * sum_b partial[k][b] (fixed order: deterministic)
__global__ void dense_expect_final_kernel(const double2* partial, int nblk, const int* ny, int K,
                                          double2* out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  double2 t = make_double2(0.0, 0.0);
  for (int b = 0; b < nblk; ++b) t = cadd(t, partial[(size_t)k * nblk + b]);
  switch (ny[k] & 3) {
    case 1: t = make_double2(t.y, -t.x); break;    // * (-i)
    case 2: t = make_double2(-t.x, -t.y); break;   // * (-1)
    case 3: t = make_double2(-t.y, t.x); break;    // * (+i)
    default: break;
  }
  out[k] = t;
}

// Marginal-probability heap: tree[2^k + v] for level k, tree[2^n + i] = |psi_i|^2.
__global__ void __launch_bounds__(256) dense_tree_leaves_kernel(const double2* a, int n,
                                                                double* tree) {
  const unsigned long long N = 1ull << n;
  for (unsigned long long i = blockIdx.x * 256ull + threadIdx.x; i < N; i += gridDim.x * 256ull)
    tree[N + i] = cabs2(a[i]);
}

// Level k of the heap from level k + 1 (one launch per level).
__global__ void __launch_bounds__(256) dense_tree_level_kernel(double* tree, int k) {
  const unsigned long long M = 1ull << k;
  for (unsigned long long v = blockIdx.x * 256ull + threadIdx.x; v < M; v += gridDim.x * 256ull)
    tree[M + v] = tree[2 * (M + v)] + tree[2 * (M + v) + 1];
}

// One thread per shot: walk the heap with the host-drawn uniforms (one per qubit
// per shot, in qubit order -- dense.py:100-108), p0 = P(0) / (P(0) + P(1)).
__global__ void __launch_bounds__(256) dense_sample_kernel(const double* tree, int n,
                                                           const double* u, int shots,
                                                           unsigned long long* out) {
  const int s = blockIdx.x * 256 + threadIdx.x;
  if (s >= shots) return;
  unsigned long long node = 1;
  for (int k = 0; k < n; ++k) {
    const double p0v = tree[2 * node], p1v = tree[2 * node + 1];
    const double total = p0v + p1v;
    const double p0 = total > 0 ? p0v / total : 0.5;
    node = 2 * node + (u[(size_t)s * n + k] < p0 ? 0 : 1);
  }
  out[s] = node - (1ull << n);
}

}  // namespace bmps
