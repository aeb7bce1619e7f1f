// libbmps: B200-native (sm_100a) MPS hot path behind the C ABI of include/bmps.h.
//
// Kernels: K1 apply_1q, K2 theta, K3 block Jacobi SVD,
// K4 finalize + split, K5 environment transfers, K6 amplitudes, plus init and
// in-order stats. All complex128/float64; GEMM-shaped work (theta, Gram,
// rotation apply, split, transfers) runs on FP64 tensor cores (DMMA).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <cstdio>
#include <string>
#include <vector>

#include "bmps.h"
#include "bmps_dense.cuh"
#include "bmps_update.cuh"

using namespace bmps;

namespace {

constexpr int kNumSMs = 148;

// Process-wide data (no numerical state): a statistic, and per-device caches of
// kernel attributes / occupancy filled once under a mutex. Every tunable of a
// call arrives in its bmps_params.
std::atomic<unsigned long long> g_launches{0};  // kernels launched through this library

constexpr int kMaxDevices = 64;
struct DevCache {
  bool attrs = false;        // dynamic shared-memory attributes set
  int sms = 0;               // multiprocessor count
  int jac_slots[4] = {0, 0, 0, 0};  // resident dynamic-Jacobi CTAs (W2 16 / 32 / 64 / ws)
  int cl_per_sm = 0;         // resident 4-CTA cluster-Jacobi CTAs per SM
};
std::mutex g_cache_mu;
DevCache g_cache[kMaxDevices];

int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d < 0 || d >= kMaxDevices ? 0 : d;
}

// ---------------------------------------------------------------------------
// init: product state |0...0> (mps.py:55-66)
// ---------------------------------------------------------------------------
__global__ void init_kernel(StateView sv, int S, double* trunc_err, long long* entries,
                            long long* peak, int* mbs, int* status, int* status_bond) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = sv.n;
  if (g < S * (n + 1)) {
    const int s = g / (n + 1), b = g % (n + 1);
    sv.dimv(s)[b] = 1;
    sv.bond(s, b)[0] = 1.0;
    if (b < n) {
      double2* t = sv.site(s, b);
      t[0] = make_double2(1.0, 0.0);        // (l=0, p=0, r=0)
      t[sv.cap] = make_double2(0.0, 0.0);   // (l=0, p=1, r=0)
    }
  }
  if (g < S) {
    trunc_err[g] = 0.0;
    entries[g] = 2LL * n;
    peak[g] = 2LL * n;
    mbs[g] = 1;
    status[g] = 0;
    status_bond[g] = -1;
  }
}

// ---------------------------------------------------------------------------
// K1: Gamma[l,s,r] <- sum_t G[s,t] Gamma[l,t,r] (mps.py:88-92), coalesced over r.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) apply1q_kernel(StateView sv, const int* items,
                                                      const double2* gates) {
  const int item = blockIdx.y;
  const int s = items[2 * item], q = items[2 * item + 1];
  const int* d = sv.dimv(s);
  const int dl = d[q], dr = d[q + 1], cap = sv.cap;
  const double2 g00 = gates[4 * (size_t)item + 0], g01 = gates[4 * (size_t)item + 1];
  const double2 g10 = gates[4 * (size_t)item + 2], g11 = gates[4 * (size_t)item + 3];
  double2* t = sv.site(s, q);
  const int total = dl * dr;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    const int l = idx / dr, r = idx % dr;
    double2* p0 = t + (size_t)(2 * l) * cap + r;
    double2* p1 = p0 + cap;
    const double2 a = *p0, b = *p1;
    *p0 = cadd(cmul(g00, a), cmul(g01, b));
    *p1 = cadd(cmul(g10, a), cmul(g11, b));
  }
}

// ---------------------------------------------------------------------------
// K6: <bits|psi> = [1] T_0[:, b_0, :] ... T_{n-1}[:, b_{n-1}, :] (mps.py:172-179),
// T_k = Gamma_k lam_{k+1}. A CTA takes a group of up to kAmpGroup consecutive
// bitstrings; when they belong to one state (the usual call: a state's bitstrings
// listed together) every Gamma element is loaded once for the whole group (both
// physical slices, each bitstring picks its own), which divides the L2 traffic of
// this L2-bound kernel by the group size. Each bitstring's row sum runs over l in
// order, as in the one-bitstring-per-CTA form, so results do not depend on the
// grouping. Mixed-state groups are walked one bitstring at a time.
// ---------------------------------------------------------------------------
#ifndef BMPS_AMP_VEC
#define BMPS_AMP_VEC 2048   // group x cap bound (vector buffers 2 x 16 B x BMPS_AMP_VEC)
#endif
#ifndef BMPS_AMP_GROUP
#define BMPS_AMP_GROUP 8
#endif
constexpr int kAmpGroup = BMPS_AMP_GROUP;
#ifndef BMPS_AMP_UNROLL
#define BMPS_AMP_UNROLL 4
#endif
constexpr int kAmpUnroll = BMPS_AMP_UNROLL;

BMPS_DEV void amplitude_group(const StateView& sv, int s, const unsigned char* const* bb, int nb,
                              double2* vbuf, double2* out_first) {
  const int n = sv.n, cap = sv.cap, tid = threadIdx.x;
  const int* d = sv.dimv(s);
  double2* cur = vbuf;                      // [nb][cap]
  double2* nxt = vbuf + (size_t)nb * cap;   // [nb][cap]
  if (tid < nb) cur[(size_t)tid * cap] = make_double2(1.0, 0.0);
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    const int dl = d[k], dr = d[k + 1];
    const double2* t = sv.site(s, k);
    const double* lam = sv.bond(s, k + 1);
    int drp = 1;
    while (drp < dr) drp <<= 1;
    // ng thread groups share the bitstrings (group q takes j = q, q + ng, ...)
    const int ng = drp >= (int)blockDim.x ? 1 : min(nb, (int)blockDim.x / drp);
    const int q = tid / drp;
    unsigned mask = 0;   // bit j: bitstring q + j*ng reads slice 1
#pragma unroll
    for (int j = 0; j < kAmpGroup; ++j) {
      const int jj = q + j * ng;
      if (jj < nb && bb[jj][k]) mask |= 1u << j;
    }
    for (int r = (ng > 1 ? tid % drp : tid); r < dr && q < ng; r += (ng > 1 ? dr + 1 : (int)blockDim.x)) {
      double2 acc[kAmpGroup];
#pragma unroll
      for (int j = 0; j < kAmpGroup; ++j) acc[j] = make_double2(0.0, 0.0);
      // BMPS_AMP_UNROLL rows per step, their loads issued together (memory-level parallelism)
      int l = 0;
      for (; l + kAmpUnroll <= dl; l += kAmpUnroll) {
        double2 t0[kAmpUnroll], t1[kAmpUnroll];
#pragma unroll
        for (int u = 0; u < kAmpUnroll; ++u) {
          t0[u] = t[(size_t)(2 * (l + u)) * cap + r];
          t1[u] = t[(size_t)(2 * (l + u) + 1) * cap + r];
        }
#pragma unroll
        for (int u = 0; u < kAmpUnroll; ++u)
#pragma unroll
          for (int j = 0; j < kAmpGroup; ++j) {
            const int jj = q + j * ng;
            if (jj < nb)
              acc[j] = cfma(cur[(size_t)jj * cap + l + u], (mask >> j) & 1u ? t1[u] : t0[u], acc[j]);
          }
      }
      for (; l < dl; ++l) {
        const double2 t0 = t[(size_t)(2 * l) * cap + r];
        const double2 t1 = t[(size_t)(2 * l + 1) * cap + r];
#pragma unroll
        for (int j = 0; j < kAmpGroup; ++j) {
          const int jj = q + j * ng;
          if (jj < nb) acc[j] = cfma(cur[(size_t)jj * cap + l], (mask >> j) & 1u ? t1 : t0, acc[j]);
        }
      }
      const double lr = lam[r];
#pragma unroll
      for (int j = 0; j < kAmpGroup; ++j) {
        const int jj = q + j * ng;
        if (jj < nb) nxt[(size_t)jj * cap + r] = cscale(acc[j], lr);
      }
    }
    __syncthreads();
    double2* tmp = cur;
    cur = nxt;
    nxt = tmp;
  }
  if (tid < nb) out_first[tid] = cur[(size_t)tid * cap];
  __syncthreads();
}

__global__ void __launch_bounds__(256) amplitude_kernel(StateView sv, const int* state_idx,
                                                        const unsigned char* bits, int count, int group,
                                                        double2* out) {
  extern __shared__ __align__(16) double2 vbuf[];  // 2 * group * cap
  const int i0 = blockIdx.x * group, nb = min(group, count - i0);
  const int s = state_idx[i0];
  bool same = true;
  for (int j = 1; j < nb; ++j) same &= state_idx[i0 + j] == s;
  const unsigned char* bb[kAmpGroup];
#pragma unroll
  for (int j = 0; j < kAmpGroup; ++j) bb[j] = bits + (size_t)(i0 + min(j, nb - 1)) * sv.n;
  if (same) {
    amplitude_group(sv, s, bb, nb, vbuf, out + i0);
  } else {
    for (int j = 0; j < nb; ++j) amplitude_group(sv, state_idx[i0 + j], bb + j, 1, vbuf, out + i0 + j);
  }
}

// ---------------------------------------------------------------------------
// Sequential conditional sampling (mps.py:206-237): per shot, left to right,
// w_b = vec @ T_k[:, b, :], p0 = |w0|^2 / (|w0|^2 + |w1|^2) (0.5 if both
// vanish), bit 0 iff u < p0 with the host's pre-drawn uniform u (one per qubit
// per shot, in qubit order), vec <- w_bit (unnormalised, like the reference).
// One CTA per shot.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) sample_kernel(StateView sv, const int* state_idx,
                                                     const double* uniforms, unsigned char* bits) {
  extern __shared__ __align__(16) double2 sbuf[];  // cur[cap], w0[cap], w1[cap]
  __shared__ double red[2][8];
  const int shot = blockIdx.x, s = state_idx[shot], n = sv.n, cap = sv.cap;
  const int* d = sv.dimv(s);
  double2* cur = sbuf;
  double2* w0 = sbuf + cap;
  double2* w1 = sbuf + 2 * cap;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) cur[0] = make_double2(1.0, 0.0);
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    const int dl = d[k], dr = d[k + 1];
    const double2* t = sv.site(s, k);
    const double* lam = sv.bond(s, k + 1);
    double p0 = 0.0, p1 = 0.0;
    for (int r = tid; r < dr; r += blockDim.x) {
      double2 a0 = make_double2(0.0, 0.0), a1 = make_double2(0.0, 0.0);
      for (int l = 0; l < dl; ++l) {
        a0 = cfma(cur[l], t[(size_t)(2 * l) * cap + r], a0);
        a1 = cfma(cur[l], t[(size_t)(2 * l + 1) * cap + r], a1);
      }
      a0 = cscale(a0, lam[r]);
      a1 = cscale(a1, lam[r]);
      w0[r] = a0;
      w1[r] = a1;
      p0 += cabs2(a0);
      p1 += cabs2(a1);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      p0 += __shfl_xor_sync(0xffffffffu, p0, o);
      p1 += __shfl_xor_sync(0xffffffffu, p1, o);
    }
    if (lane == 0) {
      red[0][warp] = p0;
      red[1][warp] = p1;
    }
    __syncthreads();
    double t0 = 0.0, t1 = 0.0;
    for (int i = 0; i < 8; ++i) {
      t0 += red[0][i];
      t1 += red[1][i];
    }
    const double total = t0 + t1;
    const double pz = total > 0.0 ? t0 / total : 0.5;
    const int bit = uniforms[(size_t)shot * n + k] < pz ? 0 : 1;
    if (tid == 0) bits[(size_t)shot * n + k] = (unsigned char)bit;
    const double2* src = bit ? w1 : w0;
    for (int r = tid; r < dr; r += blockDim.x) cur[r] = src[r];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// MpsState.conditional_prob_zero (mps.py:206-214) for one (state, site):
// w_b = prefix @ T_k[:, b, :] (T_k = Gamma_k lam_{k+1}), p_b = <w_b, w_b>. One CTA;
// p0, p1 summed per thread in r order, then over threads in a fixed tree.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) conditional_kernel(StateView sv, int s, int k,
                                                          const double2* prefix, double2* w0,
                                                          double2* w1, double* p01) {
  __shared__ double red[2][256];
  const int tid = threadIdx.x, cap = sv.cap;
  const int* d = sv.dimv(s);
  const int dl = d[k], dr = d[k + 1];
  const double2* t = sv.site(s, k);
  const double* lam = sv.bond(s, k + 1);
  double p0 = 0.0, p1 = 0.0;
  for (int r = tid; r < dr; r += blockDim.x) {
    double2 a0 = make_double2(0.0, 0.0), a1 = make_double2(0.0, 0.0);
    for (int l = 0; l < dl; ++l) {
      a0 = cfma(prefix[l], t[(size_t)(2 * l) * cap + r], a0);
      a1 = cfma(prefix[l], t[(size_t)(2 * l + 1) * cap + r], a1);
    }
    a0 = cscale(a0, lam[r]);
    a1 = cscale(a1, lam[r]);
    w0[r] = a0;
    w1[r] = a1;
    p0 += cabs2(a0);
    p1 += cabs2(a1);
  }
  red[0][tid] = p0;
  red[1][tid] = p1;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (tid < o) {
      red[0][tid] += red[0][tid + o];
      red[1][tid] += red[1][tid + o];
    }
    __syncthreads();
  }
  if (tid == 0) {
    p01[0] = red[0][0];
    p01[1] = red[1][0];
  }
}

// ---------------------------------------------------------------------------
// K5: environment transfers (mps.py:196-204 reassociated into two GEMMs).
//   prep : OT[b,s,q] = sum_t O[s,t] Gamma[b,t,q] lam[q]   (Pauli O)
//   left : F = E_k @ OT (dl x 2dr);   E_{k+1} = T^H F  (T as (2dl x dr))
//   right: F = OT @ R^T (2dl x dr);   R_k = conj(T) F^T (T, F as (dl x 2dr))
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) env_prep_kernel(StateView sv, const int* state_idx,
                                                       const int* site, const unsigned char* pauli,
                                                       double2* ot, size_t ot_stride) {
  const int it = blockIdx.y;
  const int s = state_idx[it], k = site[it], op = pauli[it], cap = sv.cap;
  const int* d = sv.dimv(s);
  const int dl = d[k], dr = d[k + 1];
  const double2* g = sv.site(s, k);
  const double* lam = sv.bond(s, k + 1);
  double2* o = ot + (size_t)it * ot_stride;
  const int total = dl * dr;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    const int b = idx / dr, q = idx % dr;
    const double2 t0 = cscale(g[(size_t)(2 * b) * cap + q], lam[q]);
    const double2 t1 = cscale(g[(size_t)(2 * b + 1) * cap + q], lam[q]);
    double2 o0, o1;
    switch (op) {
      case 1: o0 = t1; o1 = t0; break;                                   // X
      case 2: o0 = make_double2(t1.y, -t1.x); o1 = make_double2(-t0.y, t0.x); break;  // Y: -i t1, i t0
      case 3: o0 = t0; o1 = make_double2(-t1.x, -t1.y); break;           // Z
      default: o0 = t0; o1 = t1; break;                                  // I
    }
    o[(size_t)(2 * b) * cap + q] = o0;
    o[(size_t)(2 * b + 1) * cap + q] = o1;
  }
}

struct EnvOpBase {
  StateView sv;
  const int* state_idx;
  const int* site;
  int dl, dr, cap;
  BMPS_DEV void dims_of(int item) {
    const int s = state_idx[item], k = site[item];
    const int* d = sv.dimv(s);
    dl = d[k];
    dr = d[k + 1];
    cap = sv.cap;
  }
};

// left GEMM1: F[a, (s,q)] = sum_b E[a,b] OT[b,s,q];  F stored as (2a+s)*cap + q
struct EnvL1 : EnvOpBase {
  static constexpr bool kAKMajor = true, kBKMajor = false;
  const double2* env;
  const double2* ot;
  double2* f;
  size_t env_stride, ot_stride;
  const int* env_idx;   // optional: item i reads environment env_idx[i]
  const double2 *e_, *o_;
  double2* f_;
  BMPS_DEV bool begin(int item, int& M, int& N, int& K) {
    dims_of(item);
    e_ = env + (size_t)(env_idx ? env_idx[item] : item) * env_stride;
    o_ = ot + (size_t)item * ot_stride;
    f_ = f + (size_t)item * ot_stride;
    M = dl;
    N = 2 * dr;
    K = dl;
    return true;
  }
  BMPS_DEV double2 a(int i, int k) const { return e_[(size_t)i * cap + k]; }
  // GEMM column j = 2q + s (interleaved, no integer division in the loaders)
  BMPS_DEV double2 b(int k, int j) const { return o_[(size_t)(2 * k + (j & 1)) * cap + (j >> 1)]; }
  BMPS_DEV void store(int i, int j, double2 v) const {
    f_[(size_t)(2 * i + (j & 1)) * cap + (j >> 1)] = v;
  }
};

// left GEMM2: E'[r,q] = sum_{(a,s)} conj(Gamma[(a,s),r] lam[r]) F[(a,s),q]
struct EnvL2 : EnvOpBase {
  static constexpr bool kAKMajor = false, kBKMajor = false;
  const double2* f;
  double2* out;
  size_t ot_stride, env_stride;
  const int* env_idx;   // optional: item i writes environment env_idx[i]
  const double2* g_;
  const double* lam_;
  const double2* f_;
  double2* o_;
  BMPS_DEV bool begin(int item, int& M, int& N, int& K) {
    dims_of(item);
    const int s = state_idx[item], k = site[item];
    g_ = sv.site(s, k);
    lam_ = sv.bond(s, k + 1);
    f_ = f + (size_t)item * ot_stride;
    o_ = out + (size_t)(env_idx ? env_idx[item] : item) * env_stride;
    M = dr;
    N = dr;
    K = 2 * dl;
    return true;
  }
  BMPS_DEV double2 a(int i, int k) const { return cconj(cscale(g_[(size_t)k * cap + i], lam_[i])); }
  BMPS_DEV double2 b(int k, int j) const { return f_[(size_t)k * cap + j]; }
  BMPS_DEV void store(int i, int j, double2 v) const { o_[(size_t)i * cap + j] = v; }
};

// right GEMM1: F[(b,s), r] = sum_q OT[(b,s),q] R[r,q]
struct EnvR1 : EnvOpBase {
  static constexpr bool kAKMajor = true, kBKMajor = true;
  const double2* env;
  const double2* ot;
  double2* f;
  size_t env_stride, ot_stride;
  const int* env_idx;   // optional: item i reads environment env_idx[i]
  const double2 *e_, *o_;
  double2* f_;
  BMPS_DEV bool begin(int item, int& M, int& N, int& K) {
    dims_of(item);
    e_ = env + (size_t)(env_idx ? env_idx[item] : item) * env_stride;
    o_ = ot + (size_t)item * ot_stride;
    f_ = f + (size_t)item * ot_stride;
    M = 2 * dl;
    N = dr;
    K = dr;
    return true;
  }
  BMPS_DEV double2 a(int i, int k) const { return o_[(size_t)i * cap + k]; }
  BMPS_DEV double2 b(int k, int j) const { return e_[(size_t)j * cap + k]; }
  BMPS_DEV void store(int i, int j, double2 v) const { f_[(size_t)i * cap + j] = v; }
};

// right GEMM2: R'[a,b] = sum_{(s,r)} conj(Gamma[a,s,r] lam[r]) F[(b,s), r]
struct EnvR2 : EnvOpBase {
  static constexpr bool kAKMajor = true, kBKMajor = true;
  const double2* f;
  double2* out;
  size_t ot_stride, env_stride;
  const int* env_idx;   // optional: item i writes environment env_idx[i]
  const double2* g_;
  const double* lam_;
  const double2* f_;
  double2* o_;
  BMPS_DEV bool begin(int item, int& M, int& N, int& K) {
    dims_of(item);
    const int s = state_idx[item], k = site[item];
    g_ = sv.site(s, k);
    lam_ = sv.bond(s, k + 1);
    f_ = f + (size_t)item * ot_stride;
    o_ = out + (size_t)(env_idx ? env_idx[item] : item) * env_stride;
    M = dl;
    N = dl;
    K = 2 * dr;
    return true;
  }
  // GEMM depth k = 2r + s (interleaved, no integer division in the loaders)
  BMPS_DEV double2 a(int i, int k) const {
    const int s = k & 1, r = k >> 1;
    return cconj(cscale(g_[(size_t)(2 * i + s) * cap + r], lam_[r]));
  }
  BMPS_DEV double2 b(int k, int j) const {
    const int s = k & 1, r = k >> 1;
    return f_[(size_t)(2 * j + s) * cap + r];
  }
  BMPS_DEV void store(int i, int j, double2 v) const { o_[(size_t)i * cap + j] = v; }
};

__global__ void __launch_bounds__(256) env_close_kernel(const int* dims, int n, int cap,
                                                        const int* state_idx, const int* bond,
                                                        const double2* el, size_t l_stride,
                                                        const int* l_idx, const double2* er,
                                                        size_t r_stride, const int* r_idx,
                                                        double2* out) {
  const int it = blockIdx.x;
  const int D = dims[(size_t)state_idx[it] * (n + 1) + bond[it]];
  const double2* a = el + (size_t)(l_idx ? l_idx[it] : it) * l_stride;
  const double2* b = er + (size_t)(r_idx ? r_idx[it] : it) * r_stride;
  double2 acc = make_double2(0.0, 0.0);
  for (int idx = threadIdx.x; idx < D * D; idx += blockDim.x) {
    const int i = idx / D, j = idx % D;
    acc = cfma(a[(size_t)i * cap + j], b[(size_t)i * cap + j], acc);
  }
  __shared__ double2 red[256];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] = cadd(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[it] = red[0];
}

// Fused Pauli-string sweep for small bonds (cap <= kSweepCap): one CTA per
// (state, string) item walks the string's support lo..hi with the environment
// resident in shared memory and closes it against the cached right environment
// R_{hi+1}: the same contraction as the K5 GEMM pair (mps.py:196-204 reassociated:
// F = E (O T), E' = T^H F, T = Gamma lambda), in one launch for every string instead
// of three launches plus gathers per site. CUDA-core FP64: the blocks are at most
// 32 x 64 x 32, far below a DMMA tile's worth of reuse.
constexpr int kSweepCap = 32;
__global__ void __launch_bounds__(256) pauli_sweep_kernel(StateView sv, const int* state_idx,
                                                          const int* env_idx,
                                                          const unsigned char* codes,
                                                          const int* lo, const int* hi,
                                                          const double2* lenv,
                                                          const double2* renv,
                                                          size_t env_stride, double2* out) {
  extern __shared__ __align__(16) double2 ssw[];
  double2* sE = ssw;                                 // [kSweepCap][kSweepCap]
  double2* sF = sE + kSweepCap * kSweepCap;          // [2 kSweepCap][kSweepCap]
  double2* sT = sF + 2 * kSweepCap * kSweepCap;      // [2 kSweepCap][kSweepCap]
  __shared__ double2 red[8];
  const int it = blockIdx.x, tid = threadIdx.x, n = sv.n, cap = sv.cap;
  const int s = state_idx[it];
  const int* d = sv.dimv(s);
  const int l0 = lo[it], h0 = hi[it];
  const size_t ebase = (size_t)env_idx[it] * env_stride;
  {
    const int D = d[l0];
    const double2* L = lenv + ebase + (size_t)l0 * cap * cap;
    for (int idx = tid; idx < D * D; idx += blockDim.x)
      sE[(idx / D) * kSweepCap + idx % D] = L[(size_t)(idx / D) * cap + idx % D];
  }
  __syncthreads();
  for (int k = l0; k <= h0; ++k) {
    const int dl = d[k], dr = d[k + 1], op = codes[(size_t)it * n + k];
    const double2* g = sv.site(s, k);
    const double* lam = sv.bond(s, k + 1);
    for (int idx = tid; idx < 2 * dl * dr; idx += blockDim.x) {
      const int row = idx / dr, q = idx % dr;   // row = 2b + t
      sT[row * kSweepCap + q] = cscale(g[(size_t)row * cap + q], lam[q]);
    }
    __syncthreads();
    // F[(a,s), q] = sum_b E[a,b] (O T)[b,s,q]
    for (int idx = tid; idx < 2 * dl * dr; idx += blockDim.x) {
      const int as = idx / dr, q = idx % dr, a = as >> 1, so = as & 1;
      const int t = (op == 1 || op == 2) ? so ^ 1 : so;
      double2 acc = make_double2(0.0, 0.0);
      for (int b = 0; b < dl; ++b) acc = cfma(sE[a * kSweepCap + b], sT[(2 * b + t) * kSweepCap + q], acc);
      if (op == 2) acc = so == 0 ? make_double2(acc.y, -acc.x) : make_double2(-acc.y, acc.x);  // -i, +i
      else if (op == 3 && so == 1) acc = make_double2(-acc.x, -acc.y);
      sF[as * kSweepCap + q] = acc;
    }
    __syncthreads();
    // E'[r,q] = sum_{(a,s)} conj(T[(a,s), r]) F[(a,s), q]
    for (int idx = tid; idx < dr * dr; idx += blockDim.x) {
      const int r = idx / dr, q = idx % dr;
      double2 acc = make_double2(0.0, 0.0);
      for (int as = 0; as < 2 * dl; ++as)
        acc = cfma(cconj(sT[as * kSweepCap + r]), sF[as * kSweepCap + q], acc);
      sE[r * kSweepCap + q] = acc;
    }
    __syncthreads();
  }
  const int bond = h0 >= l0 ? h0 + 1 : l0;
  const int D = d[bond];
  const double2* R = renv + ebase + (size_t)bond * cap * cap;
  double2 acc = make_double2(0.0, 0.0);
  for (int idx = tid; idx < D * D; idx += blockDim.x) {
    const int i = idx / D, j = idx % D;
    acc = cfma(sE[i * kSweepCap + j], R[(size_t)i * cap + j], acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
  }
  if ((tid & 31) == 0) red[tid >> 5] = acc;
  __syncthreads();
  if (tid == 0) {
    double2 t = red[0];
    for (int w = 1; w < 8; ++w) t = cadd(t, red[w]);
    out[it] = t;
  }
}

// All identity environments of a state in one CTA (small bonds, cap <= kSweepCap):
// direction 0 writes L_1..L_n from L_0 = [[1]] (E' = T^H (E T)), direction 1 writes
// R_{n-1}..R_0 from R_n = [[1]] (R' = conj(T) (T R^T)^T) -- the identity-Pauli case
// of K5, with the environment kept in shared memory across the whole chain.
__global__ void __launch_bounds__(256) env_sweep_kernel(StateView sv, const int* states,
                                                        int direction, double2* env,
                                                        size_t env_stride) {
  extern __shared__ __align__(16) double2 ssw[];
  double2* sE = ssw;
  double2* sF = sE + kSweepCap * kSweepCap;
  double2* sT = sF + 2 * kSweepCap * kSweepCap;
  const int it = blockIdx.x, tid = threadIdx.x, n = sv.n, cap = sv.cap;
  const int s = states[it];
  const int* d = sv.dimv(s);
  double2* e = env + (size_t)it * env_stride;
  if (tid == 0) sE[0] = make_double2(1.0, 0.0);
  __syncthreads();
  for (int step = 0; step < n; ++step) {
    const int k = direction == 0 ? step : n - 1 - step;
    const int dl = d[k], dr = d[k + 1];
    const double2* g = sv.site(s, k);
    const double* lam = sv.bond(s, k + 1);
    for (int idx = tid; idx < 2 * dl * dr; idx += blockDim.x) {
      const int row = idx / dr, q = idx % dr;
      sT[row * kSweepCap + q] = cscale(g[(size_t)row * cap + q], lam[q]);
    }
    __syncthreads();
    if (direction == 0) {
      for (int idx = tid; idx < 2 * dl * dr; idx += blockDim.x) {   // F[(a,s),q] = sum_b E[a,b] T[(b,s),q]
        const int as = idx / dr, q = idx % dr, a = as >> 1, so = as & 1;
        double2 acc = make_double2(0.0, 0.0);
        for (int b = 0; b < dl; ++b) acc = cfma(sE[a * kSweepCap + b], sT[(2 * b + so) * kSweepCap + q], acc);
        sF[as * kSweepCap + q] = acc;
      }
      __syncthreads();
      double2* out = e + (size_t)(k + 1) * cap * cap;
      for (int idx = tid; idx < dr * dr; idx += blockDim.x) {       // E'[r,q] = sum conj(T[as,r]) F[as,q]
        const int r = idx / dr, q = idx % dr;
        double2 acc = make_double2(0.0, 0.0);
        for (int as = 0; as < 2 * dl; ++as)
          acc = cfma(cconj(sT[as * kSweepCap + r]), sF[as * kSweepCap + q], acc);
        sE[r * kSweepCap + q] = acc;
        out[(size_t)r * cap + q] = acc;
      }
    } else {
      for (int idx = tid; idx < 2 * dl * dr; idx += blockDim.x) {   // F[(b,s),r] = sum_q T[(b,s),q] R[r,q]
        const int bs = idx / dr, r = idx % dr;
        double2 acc = make_double2(0.0, 0.0);
        for (int q = 0; q < dr; ++q) acc = cfma(sT[bs * kSweepCap + q], sE[r * kSweepCap + q], acc);
        sF[bs * kSweepCap + r] = acc;
      }
      __syncthreads();
      double2* out = e + (size_t)k * cap * cap;
      for (int idx = tid; idx < dl * dl; idx += blockDim.x) {       // R'[a,b] = sum_{s,r} conj(T[(a,s),r]) F[(b,s),r]
        const int a = idx / dl, b = idx % dl;
        double2 acc = make_double2(0.0, 0.0);
        for (int so = 0; so < 2; ++so)
          for (int r = 0; r < dr; ++r)
            acc = cfma(cconj(sT[(2 * a + so) * kSweepCap + r]), sF[(2 * b + so) * kSweepCap + r], acc);
        sE[a * kSweepCap + b] = acc;
        out[(size_t)a * cap + b] = acc;
      }
    }
    __syncthreads();
  }
}

__global__ void init_active_kernel(int* active, int nitems) {
  if (threadIdx.x == 0) *active = nitems;
}

__global__ void item_info_kernel(const ItemMeta* meta, int nitems, int* sweeps, int* keep) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nitems) return;
  if (sweeps) sweeps[i] = meta[i].sweeps;
  if (keep) keep[i] = meta[i].keep;
}

// workspace layout for bmps_apply_2q
struct Ws {
  ItemMeta* meta;
  double* sig;
  int* perm;
  int* counter;
  double2* M0;
  double2* X;
  double2* Y;
  double2* Z;
  double2* aux;
  JacSched* sched;
  double2* gcache;
  size_t gcache_stride;
  int* pairlog;
  int nbcap;
  size_t pairlog_stride;
  size_t mat_stride;
  size_t aux_stride;
  int maxp;
  int sig_stride;
  double* fro_part;   // per item: theta's per-CTA ||M||_F^2 partials
  int fro_stride;
};

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

size_t ws_layout(int cap, int nitems, char* base, Ws* ws) {
  const size_t mat_stride = (size_t)4 * cap * cap;
  const int sig_stride = 2 * cap;
  size_t off = 0;
  const size_t o_meta = off;
  off = align256(off + sizeof(ItemMeta) * (size_t)nitems);
  const size_t o_sig = off;
  off = align256(off + sizeof(double) * (size_t)sig_stride * nitems);
  const size_t o_perm = off;
  off = align256(off + sizeof(int) * (size_t)sig_stride * nitems);
  const size_t o_cnt = off;
  off = align256(off + 256);
  const size_t o_m0 = off;
  off = align256(off + sizeof(double2) * mat_stride * nitems);
  const size_t o_x = off;
  off = align256(off + sizeof(double2) * mat_stride * nitems);
  const size_t o_y = off;
  off = align256(off + sizeof(double2) * mat_stride * nitems);
  const size_t o_z = off;
  off = align256(off + sizeof(double2) * (size_t)(2 * cap) * (2 * cap) * nitems);
  const int maxp = (2 * cap + kQrNb - 1) / kQrNb;
  const size_t aux_stride = qr_aux_stride(maxp);
  const size_t o_aux = off;
  off = align256(off + sizeof(double2) * aux_stride * nitems);
  const size_t o_sched = off;
  off = align256(off + sizeof(JacSched) * (size_t)nitems);
  const size_t gcache_stride = std::max((size_t)((2 * cap + 15) / 16 + 1) * 256,
                                        (size_t)((2 * cap + 31) / 32 + 1) * 1024);
  const size_t o_gc = off;
  off = align256(off + sizeof(double2) * gcache_stride * nitems);
  const int nbcap = (2 * cap + 7) / 8 + 1;   // blocks of the narrowest panel (8 columns), even
  const size_t pairlog_stride = (size_t)nbcap + (size_t)nbcap * nbcap;
  const size_t o_pl = off;
  off = align256(off + sizeof(int) * pairlog_stride * nitems);
  const int tpd = (cap + 31) / 32;
  const int fro_stride = tpd * tpd;
  const size_t o_fro = off;
  off = align256(off + sizeof(double) * (size_t)fro_stride * nitems);
  if (ws && base) {
    ws->meta = (ItemMeta*)(base + o_meta);
    ws->sig = (double*)(base + o_sig);
    ws->perm = (int*)(base + o_perm);
    ws->counter = (int*)(base + o_cnt);
    ws->M0 = (double2*)(base + o_m0);
    ws->X = (double2*)(base + o_x);
    ws->Y = (double2*)(base + o_y);
    ws->Z = (double2*)(base + o_z);
    ws->aux = (double2*)(base + o_aux);
    ws->sched = (JacSched*)(base + o_sched);
    ws->gcache = (double2*)(base + o_gc);
    ws->gcache_stride = gcache_stride;
    ws->pairlog = (int*)(base + o_pl);
    ws->nbcap = nbcap;
    ws->pairlog_stride = pairlog_stride;
    ws->aux_stride = aux_stride;
    ws->maxp = maxp;
    ws->mat_stride = mat_stride;
    ws->sig_stride = sig_stride;
    ws->fro_part = (double*)(base + o_fro);
    ws->fro_stride = fro_stride;
  }
  return off;
}

// Dynamic shared-memory attributes and occupancy figures of this device, set /
// measured once per device (cudaFuncSetAttribute is per device).
constexpr int kSweepCapSmem = (int)(sizeof(double2) * 5 * 32 * 32);
const DevCache& device_cache() {
  const int dev = current_device();
  std::lock_guard<std::mutex> lock(g_cache_mu);
  DevCache& dc = g_cache[dev];
  if (dc.attrs) return dc;
  cudaFuncSetAttribute(theta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kThetaSmem);
  cudaFuncSetAttribute(qr_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kQrUpdateSmem);
  cudaFuncSetAttribute(qr_panel_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(sizeof(double2) * kQrNb * kQrPanelSmemRows));
  cudaFuncSetAttribute(qr_panel_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(sizeof(double2) * kQrNb * qr_small_ld(kQrSmallRows)));
  cudaFuncSetAttribute(dq_apply_q1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kQ1Smem);
  cudaFuncSetAttribute(qr_panel_cluster_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(sizeof(double2) * kQrNb * kQrClusterRows));
  cudaFuncSetAttribute(qr_panel_cluster_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(sizeof(double2) * kQrNb * kQrClusterRows));
  cudaFuncSetAttribute(qr_panel_cluster_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(sizeof(double2) * kQrNb * kQrClusterRows));
  cudaFuncSetAttribute(jacobi_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)JacCfg<32>::kSmem);
  cudaFuncSetAttribute(jacobi_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)JacCfg<64>::kSmem);
  cudaFuncSetAttribute(jacobi_dynamic_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)JacCfg<32>::kSmem);
  cudaFuncSetAttribute(jacobi_dynamic_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)JacCfg<64>::kSmem);
  cudaFuncSetAttribute(jacobi_dynamic_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)JacCfg<16>::kSmem);
  cudaFuncSetAttribute(jacobi_cluster_kernel<32, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)ClCfg<32>::kSmem);
  cudaFuncSetAttribute(jacobi_cluster_kernel<32, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)ClCfg<32>::kSmem);
  cudaFuncSetAttribute(amplitude_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * BMPS_AMP_VEC);
  cudaFuncSetAttribute(sample_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(3 * 1024 * sizeof(double2)));
  cudaFuncSetAttribute(pauli_sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSweepCapSmem);
  cudaFuncSetAttribute(env_sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSweepCapSmem);
  cudaFuncSetAttribute(dense_run_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(sizeof(double2) << kDenseSmemQubits));
  cudaDeviceGetAttribute(&dc.sms, cudaDevAttrMultiProcessorCount, dev);
  if (dc.sms <= 0) dc.sms = kNumSMs;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_dynamic_kernel<16>, 256, JacCfg<16>::kSmem);
  dc.jac_slots[0] = std::max(1, per_sm) * dc.sms;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_dynamic_kernel<32>, 256, JacCfg<32>::kSmem);
  dc.jac_slots[1] = std::max(1, per_sm) * dc.sms;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_dynamic_kernel<64>, 256, JacCfg<64>::kSmem);
  dc.jac_slots[2] = std::max(1, per_sm) * dc.sms;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&dc.cl_per_sm, jacobi_cluster_kernel<32, 4>, 256,
                                                ClCfg<32>::kSmem);
  dc.cl_per_sm = std::max(dc.cl_per_sm, 1);
  cudaGetLastError();
  dc.attrs = true;
  return dc;
}

int32_t launch_status() {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "libbmps: launch failed: %s\n", cudaGetErrorString(e));
    return BMPS_E_LAUNCH;
  }
  return BMPS_OK;
}

StateView make_view(double* gamma, double* lam, int32_t* dims, int n, int cap) {
  StateView sv;
  sv.gamma = (double2*)gamma;
  sv.lam = lam;
  sv.dims = dims;
  sv.n = n;
  sv.cap = cap;
  return sv;
}

// Test hook kernel of bmps_debug_inner_sweep: jac_inner on one 32 x 32 Gram.
__global__ void __launch_bounds__(256) inner_sweep_test_kernel(const double2* gin, double2* gout,
                                                              double2* qout, int full, double tol,
                                                              double noise2, double fro, int max_inner,
                                                              int* nrot) {
  constexpr int W2 = 32;
  using C = JacCfg<W2>;
  extern __shared__ __align__(16) double2 tsm[];
  double2* sG = tsm;
  double2* sQ = sG + W2 * C::LDGG;
  double2* work = sQ + W2 * C::LDG;
  __shared__ InnerShared<W2> is;
  for (int i = threadIdx.x; i < W2 * W2; i += blockDim.x) sG[(i % W2) + (i / W2) * C::LDGG] = gin[i];
  __syncthreads();
  const int n = jac_inner<W2>(sG, sQ, work, is, tol, noise2, fro, full != 0, max_inner);
  __syncthreads();
  for (int i = threadIdx.x; i < W2 * W2; i += blockDim.x) {
    gout[i] = sG[(i % W2) + (i / W2) * C::LDGG];
    qout[i] = sQ[(i % W2) + (i / W2) * C::LDG];
  }
  if (threadIdx.x == 0) *nrot = n;
}

}  // namespace

extern "C" {

int32_t bmps_version(void) { return 2; }

uint64_t bmps_launch_count(void) { return g_launches.load(); }

int32_t bmps_build_flags(void) {
#ifdef BMPS_EXPERIMENTAL
  return 1;
#else
  return 0;
#endif
}

void bmps_default_params(bmps_params* p) {
  if (!p) return;
  *p = bmps_params{};
  p->tol_factor = 4.0;
  p->max_sweeps = 60;
  p->max_inner = 1;
  p->qr_min_cols = 65;
  p->jacobi_mode = 4;
  p->block_w2 = 32;
  p->double_qr = 1;
  p->col_sort = 1;
  p->gram_cache = 1;
  p->pair_skip = 1;
  p->jac_cluster = -1;
  p->jac_per_sm = 0;
  p->jac_ws = 0;
  p->tma_staging = 0;
  p->cluster_size = 8;
  p->qr_cluster = 1;
  p->n_svd_events = 0;
  p->svd_events = nullptr;
  p->svd_events_used = nullptr;
  p->thr_a = 3e-2;
  p->thr_b = 3e-3;
  p->thr_a_sweeps = 2;
  p->thr_b_sweeps = 5;
  p->thr_auto = 1;
  p->qr_small = -1;
  p->visits_hint = 0;
}

// Development aid: cumulative Jacobi phase cycles (builds with -DBMPS_PHASE_TIMERS only).
int32_t bmps_phase_cycles(uint64_t* out4) {
#ifdef BMPS_PHASE_TIMERS
  cudaMemcpyFromSymbol(out4, g_phase_cycles, 24 * sizeof(unsigned long long));
  return BMPS_OK;
#else
  (void)out4;
  return BMPS_E_ARG;
#endif
}

// Development aid: per-warp phase-B trace of the inner sweep (-DBMPS_PHASE_TIMERS only):
// out = 64 rounds x 8 warps x {start, own work done, barrier released, rotations}.
int32_t bmps_inner_trace(uint64_t* out, int32_t n) {
#ifdef BMPS_PHASE_TIMERS
  if (!out || n < 64 * 8 * 4) return BMPS_E_ARG;
  cudaMemcpyFromSymbol(out, g_inner_trace, sizeof(unsigned long long) * 64 * 8 * 4);
  return BMPS_OK;
#else
  (void)out; (void)n;
  return BMPS_E_ARG;
#endif
}

// Test hook: one inner (Gram-space) sweep of the W2 = 32 visit on a caller-supplied Gram.
int32_t bmps_debug_inner_sweep(const double* gram_in, double* gram_out, double* q_out,
                               int32_t full, double tol, double noise2, double fro,
                               int32_t max_inner, int32_t* nrot, void* stream) {
  if (!gram_in || !gram_out || !q_out || !nrot || max_inner < 1) return BMPS_E_ARG;
  constexpr int W2 = 32;
  using C = JacCfg<W2>;
  const size_t smem = sizeof(double2) * (size_t)(W2 * C::LDGG + W2 * C::LDG + 12 * 64);
  // per call: the attribute is per device and this is a test hook, not a hot path
  cudaFuncSetAttribute(inner_sweep_test_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  inner_sweep_test_kernel<<<1, 256, smem, (cudaStream_t)stream>>>(
      (const double2*)gram_in, (double2*)gram_out, (double2*)q_out, full, tol, noise2, fro, max_inner, nrot);
  ++g_launches;
  return launch_status();
}

const char* bmps_status_string(int32_t code) {
  switch (code) {
    case BMPS_OK: return "ok";
    case BMPS_E_ARG: return "invalid argument";
    case BMPS_E_LAUNCH: return "kernel launch failed";
    case BMPS_E_WORKSPACE: return "workspace too small";
    case BMPS_S_SVD_FAILED: return "SVD failed (Jacobi did not converge)";
    case BMPS_S_ALL_TRUNCATED: return "all singular values truncated";
    case BMPS_S_CAPACITY: return "bond dimension exceeds allocated capacity";
    default: return "unknown status";
  }
}

int32_t bmps_init_product(double* gamma, double* lam, int32_t* dims, double* trunc_err,
                          int64_t* entries, int64_t* peak, int32_t* max_bond_seen,
                          int32_t* status, int32_t* status_bond, int32_t S, int32_t n,
                          int32_t cap, void* stream) {
  if (S < 1 || n < 1 || cap < 1 || !gamma || !lam || !dims) return BMPS_E_ARG;
  StateView sv = make_view(gamma, lam, dims, n, cap);
  const int total = std::max(S * (n + 1), S);
  init_kernel<<<(total + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
      sv, S, trunc_err, (long long*)entries, (long long*)peak, max_bond_seen, status, status_bond);
  ++g_launches;
  return launch_status();
}

int32_t bmps_apply_1q(double* gamma, const int32_t* dims, int32_t S, int32_t n, int32_t cap,
                      const int32_t* items, const double* gates, int32_t nitems, void* stream) {
  if (nitems == 0) return BMPS_OK;
  if (nitems < 0 || S < 1 || n < 1 || cap < 1) return BMPS_E_ARG;
  StateView sv = make_view(gamma, nullptr, (int32_t*)dims, n, cap);
  const int per_item = std::min(std::max((cap * cap + 255) / 256, 1), 64);
  dim3 grid(per_item, nitems);
  apply1q_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(sv, items, (const double2*)gates);
  ++g_launches;
  return launch_status();
}

size_t bmps_apply_2q_workspace_bytes(int32_t cap, int32_t nitems) {
  return ws_layout(cap, nitems, nullptr, nullptr);
}

int32_t bmps_apply_2q(double* gamma, double* lam, int32_t* dims, int32_t S, int32_t n,
                      int32_t cap, const int32_t* items, const double* gates, int32_t nitems,
                      bmps_policy policy, bmps_update_record* log, const int32_t* log_index,
                      void* workspace, size_t workspace_bytes, int32_t dim_bound,
                      const bmps_params* params, void* stream) {
  if (nitems == 0) return BMPS_OK;
  if (nitems < 0 || S < 1 || n < 2 || cap < 1 || cap > 1024 || !log || !log_index)
    return BMPS_E_ARG;
  if (workspace_bytes < ws_layout(cap, nitems, nullptr, nullptr)) return BMPS_E_WORKSPACE;
  bmps_params P;
  if (params) P = *params;
  else bmps_default_params(&P);
  if (!(P.tol_factor > 0) || P.max_sweeps < 1 || P.max_inner < 1 || P.qr_min_cols < 1 ||
      !(P.block_w2 == 0 || P.block_w2 == 16 || P.block_w2 == 32 || P.block_w2 == 64) ||
      !(P.jac_cluster == -1 || P.jac_cluster == 0 || P.jac_cluster == 2 || P.jac_cluster == 4) ||
      P.jac_per_sm < 0 || P.jac_per_sm > 8 || P.cluster_size < 1 || P.cluster_size > 16 ||
      !(P.jacobi_mode == 0 || P.jacobi_mode == 1 || P.jacobi_mode == 4 || P.jacobi_mode == 2 ||
        P.jacobi_mode == 3) ||
      P.jac_ws != 0 || !(P.thr_a >= 0) || !(P.thr_b >= 0) || P.thr_a_sweeps < 0 ||
      P.thr_b_sweeps < 0 || P.thr_b_sweeps >= P.max_sweeps || P.qr_small < -1 || P.qr_small > 1 || P.visits_hint < 0 || (P.n_svd_events > 0 && (!P.svd_events || !P.svd_events_used)))
    return BMPS_E_ARG;
#ifndef BMPS_EXPERIMENTAL
  if (P.tma_staging || P.jacobi_mode == 2 || P.jacobi_mode == 3) return BMPS_E_ARG;
#endif
  const bool timed = P.n_svd_events > 0;
  if (timed && *P.svd_events_used >= P.n_svd_events) return BMPS_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const DevCache& dc = device_cache();
  Ws ws;
  ws_layout(cap, nitems, (char*)workspace, &ws);
  StateView sv = make_view(gamma, lam, dims, n, cap);
  if (dim_bound <= 0 || dim_bound > cap) dim_bound = cap;

  // K2 theta; ||M||_F^2 from per-CTA partials summed in a fixed order (bit-deterministic)
  cudaMemsetAsync(ws.meta, 0, sizeof(ItemMeta) * (size_t)nitems, st);
  const int tpd = (dim_bound + 31) / 32;
  theta_kernel<<<dim3(tpd * tpd, nitems), 256, kThetaSmem, st>>>(
      sv, items, (const double2*)gates, ws.meta, ws.M0, ws.X, ws.mat_stride, tpd, P.qr_min_cols,
      P.double_qr, P.col_sort, ws.fro_part, ws.fro_stride);
  ++g_launches;
  fro_reduce_kernel<<<nitems, 32, 0, st>>>(ws.meta, ws.fro_part, ws.fro_stride, tpd * tpd);
  ++g_launches;
  int32_t rc = launch_status();
  if (rc) return rc;
  cudaEvent_t ev_end = nullptr;
  if (timed) {
    const int k = (*P.svd_events_used)++;
    cudaEventRecord((cudaEvent_t)P.svd_events[2 * k], st);
    ev_end = (cudaEvent_t)P.svd_events[2 * k + 1];
  }
  const int cmax0 = 2 * dim_bound;
  if (P.col_sort && P.double_qr && cmax0 >= P.qr_min_cols) {
    dq_colsort_kernel<<<nitems, 512, 0, st>>>(ws.meta, ws.M0, ws.X, ws.mat_stride);
    ++g_launches;
    if ((rc = launch_status())) return rc;
  }

  // K3a Householder QR preconditioner (items with c >= qr_min_cols)
  const int cmax = 2 * dim_bound;
  if (cmax >= P.qr_min_cols) {
    QrArgs qa;
    qa.meta = ws.meta;
    qa.X = ws.X;
    qa.Y = ws.Y;
    qa.Z = ws.Z;
    qa.aux = ws.aux;
    qa.mat_stride = ws.mat_stride;
    qa.aux_stride = ws.aux_stride;
    qa.maxp = ws.maxp;
    const int npanels = (cmax + kQrNb - 1) / kQrNb;
    for (int second = 0; second <= (P.double_qr ? 1 : 0); ++second) {
      qa.second = second;
      for (int p = 0; p < npanels; ++p) {
        qa.panel = p;
        // rows of this panel: the first QR works on r x c (r <= 2 dim_bound), the second on c x c
        const int prow = cmax - p * kQrNb;
        // shared-memory panels run one CTA per SM (up to 229 KB): worth it while the
        // batch fits one wave, or when the panel is small enough for two per SM
        if (prow > kQrPanelSmemRows && P.qr_cluster && 2 * nitems <= dc.sms) {
          // tall panel, few items: row slices over a cluster, each resident in its CTA's
          // shared memory (measured: cfg3 / cfg5 -1.5% time; with hundreds of items one
          // CTA per item streaming from L2 keeps more SMs busy: bench 917 vs 909 updates/s)
          const int cs = prow <= 2 * kQrClusterRows ? 2 : prow <= 4 * kQrClusterRows ? 4 : 8;
          const int sl = (prow + cs - 1) / cs;
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(nitems * cs, 1, 1);
          cfg.blockDim = dim3(512, 1, 1);
          cfg.dynamicSmemBytes = sizeof(double2) * kQrNb * sl;
          cfg.stream = st;
          cudaLaunchAttribute attr[1];
          attr[0].id = cudaLaunchAttributeClusterDimension;
          attr[0].val.clusterDim.x = cs;
          attr[0].val.clusterDim.y = 1;
          attr[0].val.clusterDim.z = 1;
          cfg.attrs = attr;
          cfg.numAttrs = 1;
          const cudaError_t e = cs == 2 ? cudaLaunchKernelEx(&cfg, qr_panel_cluster_kernel<2>, qa)
                              : cs == 4 ? cudaLaunchKernelEx(&cfg, qr_panel_cluster_kernel<4>, qa)
                                        : cudaLaunchKernelEx(&cfg, qr_panel_cluster_kernel<8>, qa);
          if (e != cudaSuccess) {
            fprintf(stderr, "libbmps: cluster QR panel launch failed: %s\n", cudaGetErrorString(e));
            return BMPS_E_LAUNCH;
          }
        } else if (kQrNb == 32 && prow <= kQrSmallRows &&
                   (P.qr_small > 0 || (P.qr_small < 0 && nitems > dc.sms))) {
          // short panel: 128 threads, two barriers per column step, three CTAs per SM
          qr_panel_small_kernel<<<nitems, 128, sizeof(double2) * kQrNb * qr_small_ld(std::max(prow, 32)), st>>>(qa);
        } else if (prow <= kQrPanelSmemRows && (nitems <= dc.sms || prow <= 150 * 32 / kQrNb)) {
          qr_panel_kernel<true><<<nitems, 512, sizeof(double2) * kQrNb * prow, st>>>(qa);
        } else {
          qr_panel_kernel<false><<<nitems, 512, 0, st>>>(qa);
        }
        ++g_launches;
        const int trail = cmax - (p + 1) * kQrNb;
        if (trail > 0) {
          qr_update_kernel<<<dim3((trail + kQrChunk - 1) / kQrChunk, nitems), 256, kQrUpdateSmem,
                             st>>>(qa);
          ++g_launches;
        }
      }
      qr_form_y_kernel<<<dim3(std::min(64, (cmax * cmax + 255) / 256), nitems), 256, 0, st>>>(qa);
      ++g_launches;
    }
    if ((rc = launch_status())) return rc;
  }

  // K3b Jacobi SVD
  JacArgs ja;
  ja.meta = ws.meta;
  ja.X = ws.X;
  ja.Y = ws.Y;
  ja.Z = ws.Z;
  ja.mat_stride = ws.mat_stride;
  ja.round = 0;
  ja.max_sweeps = P.max_sweeps;
  ja.max_inner = P.max_inner;
  ja.tol_factor = P.tol_factor;
  ja.sched = ws.sched;
  ja.active = ws.counter;
  ja.nitems = nitems;
  ja.tma = P.tma_staging;
  ja.gcache = P.gram_cache ? ws.gcache : nullptr;
  ja.gcache_stride = ws.gcache_stride;
  ja.pairlog = P.pair_skip ? ws.pairlog : nullptr;
  ja.nbcap = ws.nbcap;
  ja.thr_a = P.thr_a;
  ja.thr_b = P.thr_b;
  ja.thr_a_sweeps = P.thr_a_sweeps;
  ja.thr_b_sweeps = P.thr_b_sweeps;
  if (cmax <= 64) {
    ja.persistent = 1;
    if (cmax <= 32)
      jacobi_kernel<32><<<dim3(1, nitems), 256, JacCfg<32>::kSmem, st>>>(ja);
    else
      jacobi_kernel<64><<<dim3(1, nitems), 256, JacCfg<64>::kSmem, st>>>(ja);
    ++g_launches;
    if ((rc = launch_status())) return rc;
  } else {
    const int nbmax = (cmax + 15) / 16 + ((cmax + 15) / 16 & 1);
    const int cl_mode = P.jacobi_mode == 0 ? 4 : P.jacobi_mode;
    if (cl_mode == 4) {
      cudaMemsetAsync(ws.sched, 0, sizeof(JacSched) * (size_t)nitems, st);
      if (P.pair_skip)
        cudaMemsetAsync(ws.pairlog, 0xff, sizeof(int) * ws.pairlog_stride * (size_t)nitems, st);
      init_active_kernel<<<1, 32, 0, st>>>(ws.counter, nitems);
      ++g_launches;
      // panel width by the tunable (default 32). 16 (8-column blocks) quadruples the
      // visits per round for small batches, but each visit keeps most of a 32-wide
      // visit's latency: one cfg3 brick layer (16 items) ran 36 -> 41 ms, so the auto
      // mode (0: 16 when nitems x visits < CTA slots) is off by default
      int wi = P.block_w2 == 64 ? 2 : P.block_w2 == 16 ? 0 : 1;
      if (P.block_w2 == 0) wi = (long long)nitems * (nbmax / 2) < dc.jac_slots[1] ? 0 : 1;
      int slots = dc.jac_slots[wi];
      // small batches: one visit per cluster of CTAs (row split), see jacobi_cluster_kernel
      // (auto: when a round's visits fit the co-resident clusters; a visit on a cluster
      // of CS CTAs finishes sooner, but CS x fewer visits are in flight)
      int csize = 0;
      // vis_est = the caller's estimate of the visits one round really has
      // (bmps_params.visits_hint, from per-item bond bounds), else the bound items x blocks / 2
      const long long vis_est = P.visits_hint > 0 ? P.visits_hint : (long long)nitems * (nbmax / 2);
      // Row-split cluster visits (jacobi_cluster_kernel) only when forced (jac_cluster 2 / 4):
      // per-layer A/B timings (tools/cfg3_layer_times.py, profiles/r02_cluster_rule_ab.log)
      // showed that what they bought was fewer visits per SM, which the grid rule below gives
      // the single-CTA visits directly -- config 3's layers 32-35 ms on pairs vs 31-33 ms at
      // one CTA per SM, config 1's 8-item layers 2.56 ms on 4-CTA clusters vs 2.45 ms
      if (wi == 1 && !P.tma_staging && P.jac_cluster > 0) csize = P.jac_cluster;
      // CTAs per SM by the visits a round has: by the layer times below, two visits sharing an
      // SM each take about twice as long as one alone (cause not isolated: L2 hit rate and
      // DRAM reads are the same, profiles/r02_per_sm_mechanism.log), so below the throughput
      // regime fewer, faster CTAs win -- a round is as slow as its slowest visit.
      // Measured (chi = 256 steady-state layers, ms per layer at 1 / 2 / 3 / 4 CTAs per SM;
      // profiles/r02_per_sm_ab.log, r02_cfg3_layer_times.log): ~290 visits per round (config
      // 3) 31-33 / 32-35 / - / 37-41; 528 visits: 52.5 / 41.9 / 44.2 / 47.1; 780: 72.5 / 55.5
      // / 51.5 / 53.1; 1040: 92.7 / 70.2 / 63.5 / 62.2. The best count is ceil(visits / 2.2
      // SMs): one CTA slot per ~2.2 visits of the round, the occupancy maximum from ~1000.
      if (P.jac_per_sm > 0) {
        slots = std::min(slots, P.jac_per_sm * dc.sms);
      } else if (csize == 0 && wi == 1) {
        const long long k = (10LL * vis_est + 22LL * dc.sms - 1) / (22LL * dc.sms);
        if (k * dc.sms < slots) slots = (int)std::max(1LL, k) * dc.sms;
      }
      const int vis = wi == 2 ? std::max(1, (cmax + 63) / 64)
                    : wi == 1 ? nbmax / 2
                              : (cmax + 15) / 16;
      const int grid = std::min(slots, nitems * vis);
      // threshold sweeps trade a fraction of a sweep for fewer applies: a gain when the
      // launch is throughput-bound, a loss when a round's visits do not even fill the
      // resident CTAs and the item's sweep count is what the layer waits for
      if (P.thr_auto && (long long)nitems * vis < slots) ja.thr_a_sweeps = ja.thr_b_sweeps = 0;
      if (csize > 0) {
        const int nclusters = std::max(1, std::min(nitems * (nbmax / 2), dc.cl_per_sm * dc.sms / csize));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(nclusters * csize, 1, 1);
        cfg.blockDim = dim3(256, 1, 1);
        cfg.dynamicSmemBytes = ClCfg<32>::kSmem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = csize;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        const cudaError_t e = csize == 4 ? cudaLaunchKernelEx(&cfg, jacobi_cluster_kernel<32, 4>, ja)
                                         : cudaLaunchKernelEx(&cfg, jacobi_cluster_kernel<32, 2>, ja);
        if (e != cudaSuccess) {
          fprintf(stderr, "libbmps: cluster Jacobi launch failed: %s\n", cudaGetErrorString(e));
          return BMPS_E_LAUNCH;
        }
      }
      else if (wi == 2)
        jacobi_dynamic_kernel<64><<<grid, 256, JacCfg<64>::kSmem, st>>>(ja);
      else if (wi == 1)
        jacobi_dynamic_kernel<32><<<grid, 256, JacCfg<32>::kSmem, st>>>(ja);
      else
        jacobi_dynamic_kernel<16><<<grid, 256, JacCfg<16>::kSmem, st>>>(ja);
      ++g_launches;
      if ((rc = launch_status())) return rc;
    } else if (cl_mode == 1) {
      ja.persistent = 1;
      jacobi_kernel<32><<<dim3(1, nitems), 256, JacCfg<32>::kSmem, st>>>(ja);
      ++g_launches;
      if ((rc = launch_status())) return rc;
    }
#ifdef BMPS_EXPERIMENTAL
    else if (cl_mode == 3) {
      ja.persistent = 2;
      const int csize = std::min(P.cluster_size, nbmax / 2);
      if (csize > 8)
        cudaFuncSetAttribute(jacobi_kernel<32>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(csize, nitems, 1);
      cfg.blockDim = dim3(256, 1, 1);
      cfg.dynamicSmemBytes = JacCfg<32>::kSmem;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = csize;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      cudaError_t e = cudaLaunchKernelEx(&cfg, jacobi_kernel<32>, ja);
      ++g_launches;
      if (e != cudaSuccess) {
        fprintf(stderr, "libbmps: cluster launch failed: %s\n", cudaGetErrorString(e));
        return BMPS_E_LAUNCH;
      }
      if ((rc = launch_status())) return rc;
    } else {
      // development variant: one launch per Jacobi round, a fixed number of sweeps
      // (no host polling inside the ABI); items converge by their own flags
      ja.persistent = 0;
      for (int sweep = 0; sweep < P.max_sweeps; ++sweep) {
        for (int rho = 0; rho < nbmax - 1; ++rho) {
          ja.round = rho;
          jacobi_kernel<32><<<dim3(nbmax / 2, nitems), 256, JacCfg<32>::kSmem, st>>>(ja);
          ++g_launches;
        }
        sweep_end_kernel<<<(nitems + 127) / 128, 128, 0, st>>>(ws.meta, nitems, P.max_sweeps,
                                                               ws.counter);
        ++g_launches;
        if ((rc = launch_status())) return rc;
      }
    }
#endif
  }

  // K3c double-QR epilogue: L = Q1 [Z sorted; 0] for the kept columns
  if (P.double_qr && cmax >= P.qr_min_cols) {
    dq_sort_kernel<<<nitems, 512, 0, st>>>(ws.meta, ws.Z, ws.Y, ws.mat_stride, ws.sig,
                                           ws.sig_stride, policy.cutoff, policy.max_bond,
                                           policy.relative);
    ++g_launches;
    QrArgs qa;
    qa.meta = ws.meta;
    qa.X = ws.X;
    qa.Y = ws.Y;
    qa.Z = ws.Z;
    qa.aux = ws.aux;
    qa.mat_stride = ws.mat_stride;
    qa.aux_stride = ws.aux_stride;
    qa.maxp = ws.maxp;
    qa.second = 0;
    const int kq = policy.max_bond > 0 ? std::min(policy.max_bond, cmax) : cmax;
    for (int p = (cmax + kQrNb - 1) / kQrNb - 1; p >= 0; --p) {
      qa.panel = p;
      dq_apply_q1_kernel<<<dim3((kq + kQrChunk - 1) / kQrChunk, nitems), 256, kQ1Smem, st>>>(qa);
      ++g_launches;
    }
    if ((rc = launch_status())) return rc;
  }

  if (timed) cudaEventRecord(ev_end, st);
  // K4 finalize + split
  finalize_kernel<<<nitems, 512, 0, st>>>(sv, items, ws.meta, ws.X, ws.Y, ws.mat_stride, ws.sig,
                                          ws.perm, ws.sig_stride, policy.cutoff, policy.max_bond,
                                          policy.relative, log, log_index);
  ++g_launches;
  if ((rc = launch_status())) return rc;
  const int kb = policy.max_bond > 0 ? std::min(policy.max_bond, cap) : cap;
  {
    SplitOp<false> sop;
    sop.sv = sv;
    sop.items = items;
    sop.meta = ws.meta;
    sop.M0 = ws.M0;
    sop.X = ws.X;
    sop.Yq = ws.Y;
    sop.mat_stride = ws.mat_stride;
    sop.sig_ws = ws.sig;
    sop.perm_ws = ws.perm;
    sop.sig_stride = ws.sig_stride;
    dim3 sgrid((cmax + 63) / 64, (std::min(kb, cmax) + 63) / 64, nitems);
    gemm_kernel<SplitOp<false>><<<sgrid, 256, 0, st>>>(sop);
    ++g_launches;
    if (cmax >= P.qr_min_cols) {
      SplitOp<true> pop;
      pop.sv = sv;
      pop.items = items;
      pop.meta = ws.meta;
      pop.M0 = ws.M0;
      pop.X = ws.X;
      pop.Yq = ws.Y;
      pop.mat_stride = ws.mat_stride;
      pop.sig_ws = ws.sig;
      pop.perm_ws = ws.perm;
      pop.sig_stride = ws.sig_stride;
      gemm_kernel<SplitOp<true>><<<sgrid, 256, 0, st>>>(pop);
      ++g_launches;
    }
  }
  return launch_status();
}

int32_t bmps_stats_replay(const bmps_update_record* log, const int32_t* ranges, int32_t nranges,
                          double* trunc_err, int64_t* entries, int64_t* peak,
                          int32_t* max_bond_seen, int32_t* status, int32_t* status_bond,
                          double* bond_err, int32_t n, double* min_margin, double* min_gap,
                          void* stream) {
  if (nranges == 0) return BMPS_OK;
  if (nranges < 0 || !log || !ranges || (bond_err && n < 2)) return BMPS_E_ARG;
  stats_replay_kernel<<<(nranges + 127) / 128, 128, 0, (cudaStream_t)stream>>>(
      log, ranges, nranges, trunc_err, (long long*)entries, (long long*)peak, max_bond_seen,
      status, status_bond, bond_err, n, min_margin, min_gap);
  ++g_launches;
  return launch_status();
}

int32_t bmps_apply_2q_sweeps(const void* workspace, int32_t nitems, int32_t* sweeps,
                             void* stream) {
  if (nitems <= 0) return BMPS_OK;
  const ItemMeta* meta = (const ItemMeta*)workspace;  // meta sits at offset 0
  item_info_kernel<<<(nitems + 127) / 128, 128, 0, (cudaStream_t)stream>>>(meta, nitems, sweeps,
                                                                           nullptr);
  ++g_launches;
  return launch_status();
}

int32_t bmps_amplitudes(const double* gamma, const double* lam, const int32_t* dims, int32_t S,
                        int32_t n, int32_t cap, const int32_t* state_idx, const uint8_t* bits,
                        int32_t count, double* out, void* stream) {
  if (count == 0) return BMPS_OK;
  if (count < 0 || S < 1 || n < 1 || cap < 1) return BMPS_E_ARG;
  StateView sv = make_view((double*)gamma, (double*)lam, (int32_t*)dims, n, cap);
  // bitstrings per CTA: up to kAmpGroup, vectors (2 x group x cap) within 32 x BMPS_AMP_VEC bytes
  const int group = max(1, min(kAmpGroup, BMPS_AMP_VEC / cap));
  const size_t smem = 2 * (size_t)group * cap * sizeof(double2);
  device_cache();
  amplitude_kernel<<<(count + group - 1) / group, 256, smem, (cudaStream_t)stream>>>(
      sv, state_idx, bits, count, group, (double2*)out);
  ++g_launches;
  return launch_status();
}

int32_t bmps_sample(const double* gamma, const double* lam, const int32_t* dims, int32_t S,
                    int32_t n, int32_t cap, const int32_t* state_idx, const double* uniforms,
                    int32_t shots, uint8_t* bits, void* stream) {
  if (shots == 0) return BMPS_OK;
  if (shots < 0 || S < 1 || n < 1 || cap < 1) return BMPS_E_ARG;
  StateView sv = make_view((double*)gamma, (double*)lam, (int32_t*)dims, n, cap);
  const size_t smem = 3 * (size_t)cap * sizeof(double2);
  device_cache();
  sample_kernel<<<shots, 256, smem, (cudaStream_t)stream>>>(sv, state_idx, uniforms, bits);
  ++g_launches;
  return launch_status();
}

int32_t bmps_conditional(const double* gamma, const double* lam, const int32_t* dims, int32_t S,
                         int32_t n, int32_t cap, int32_t state, int32_t site, const double* prefix,
                         double* w0, double* w1, double* p01, void* stream) {
  if (S < 1 || n < 1 || cap < 1 || state < 0 || state >= S || site < 0 || site >= n || !prefix ||
      !w0 || !w1 || !p01)
    return BMPS_E_ARG;
  StateView sv = make_view((double*)gamma, (double*)lam, (int32_t*)dims, n, cap);
  conditional_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(sv, state, site, (const double2*)prefix,
                                                         (double2*)w0, (double2*)w1, p01);
  ++g_launches;
  return launch_status();
}

int32_t bmps_env_transfer(const double* gamma, const double* lam, const int32_t* dims, int32_t S,
                          int32_t n, int32_t cap, const int32_t* state_idx, const int32_t* site,
                          const uint8_t* pauli, int32_t direction, const double* env_in,
                          int64_t in_stride, const int32_t* in_idx, double* env_out,
                          int64_t out_stride, const int32_t* out_idx, double* scratch,
                          int32_t count, void* stream) {
  if (count == 0) return BMPS_OK;
  if (count < 0 || S < 1 || n < 1 || cap < 1 || (direction != 0 && direction != 1))
    return BMPS_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  StateView sv = make_view((double*)gamma, (double*)lam, (int32_t*)dims, n, cap);
  const size_t ot_stride = (size_t)2 * cap * cap;
  double2* ot = (double2*)scratch;
  double2* f = ot + ot_stride * count;
  const int per_item = std::min(std::max((cap * cap + 255) / 256, 1), 64);
  env_prep_kernel<<<dim3(per_item, count), 256, 0, st>>>(sv, state_idx, site, pauli, ot, ot_stride);
  ++g_launches;
  int32_t rc = launch_status();
  if (rc) return rc;
  const int t1 = (cap + 63) / 64, t2 = (2 * cap + 63) / 64;
  if (direction == 0) {
    EnvL1 g1;
    g1.sv = sv; g1.state_idx = state_idx; g1.site = site;
    g1.env = (const double2*)env_in; g1.ot = ot; g1.f = f;
    g1.env_stride = (size_t)in_stride; g1.ot_stride = ot_stride; g1.env_idx = in_idx;
    gemm_kernel<EnvL1><<<dim3(t1, t2, count), 256, 0, st>>>(g1);
    ++g_launches;
    if ((rc = launch_status())) return rc;
    EnvL2 g2;
    g2.sv = sv; g2.state_idx = state_idx; g2.site = site;
    g2.f = f; g2.out = (double2*)env_out; g2.ot_stride = ot_stride; g2.env_stride = (size_t)out_stride;
    g2.env_idx = out_idx;
    gemm_kernel<EnvL2><<<dim3(t1, t1, count), 256, 0, st>>>(g2);
    ++g_launches;
  } else {
    EnvR1 g1;
    g1.sv = sv; g1.state_idx = state_idx; g1.site = site;
    g1.env = (const double2*)env_in; g1.ot = ot; g1.f = f;
    g1.env_stride = (size_t)in_stride; g1.ot_stride = ot_stride; g1.env_idx = in_idx;
    gemm_kernel<EnvR1><<<dim3(t2, t1, count), 256, 0, st>>>(g1);
    ++g_launches;
    if ((rc = launch_status())) return rc;
    EnvR2 g2;
    g2.sv = sv; g2.state_idx = state_idx; g2.site = site;
    g2.f = f; g2.out = (double2*)env_out; g2.ot_stride = ot_stride; g2.env_stride = (size_t)out_stride;
    g2.env_idx = out_idx;
    gemm_kernel<EnvR2><<<dim3(t1, t1, count), 256, 0, st>>>(g2);
    ++g_launches;
  }
  return launch_status();
}

int32_t bmps_pauli_sweep(const double* gamma, const double* lam, const int32_t* dims, int32_t S,
                         int32_t n, int32_t cap, const int32_t* state_idx, const int32_t* env_idx,
                         const uint8_t* codes, const int32_t* lo, const int32_t* hi,
                         const double* env_l, const double* env_r, int64_t env_stride,
                         int32_t count, double* out, void* stream) {
  if (count == 0) return BMPS_OK;
  if (count < 0 || S < 1 || n < 1 || cap < 1 || cap > kSweepCap || !env_l || !env_r || !out)
    return BMPS_E_ARG;
  StateView sv = make_view((double*)gamma, (double*)lam, (int32_t*)dims, n, cap);
  constexpr size_t smem = sizeof(double2) * 5 * kSweepCap * kSweepCap;
  device_cache();
  pauli_sweep_kernel<<<count, 256, smem, (cudaStream_t)stream>>>(
      sv, state_idx, env_idx, codes, lo, hi, (const double2*)env_l, (const double2*)env_r,
      (size_t)env_stride, (double2*)out);
  ++g_launches;
  return launch_status();
}

int32_t bmps_env_sweep(const double* gamma, const double* lam, const int32_t* dims, int32_t S,
                       int32_t n, int32_t cap, const int32_t* states, int32_t count,
                       int32_t direction, double* env, int64_t env_stride, void* stream) {
  if (count == 0) return BMPS_OK;
  if (count < 0 || S < 1 || n < 1 || cap < 1 || cap > kSweepCap || !env ||
      (direction != 0 && direction != 1))
    return BMPS_E_ARG;
  StateView sv = make_view((double*)gamma, (double*)lam, (int32_t*)dims, n, cap);
  constexpr size_t smem = sizeof(double2) * 5 * kSweepCap * kSweepCap;
  device_cache();
  env_sweep_kernel<<<count, 256, smem, (cudaStream_t)stream>>>(sv, states, direction,
                                                               (double2*)env, (size_t)env_stride);
  ++g_launches;
  return launch_status();
}

int32_t bmps_env_close(const int32_t* dims, int32_t n, int32_t cap, const int32_t* state_idx,
                       const int32_t* bond, const double* env_l, int64_t l_stride,
                       const int32_t* l_idx, const double* env_r, int64_t r_stride,
                       const int32_t* r_idx, int32_t count, double* out, void* stream) {
  if (count == 0) return BMPS_OK;
  if (count < 0 || n < 1 || cap < 1) return BMPS_E_ARG;
  env_close_kernel<<<count, 256, 0, (cudaStream_t)stream>>>(
      dims, n, cap, state_idx, bond, (const double2*)env_l, (size_t)l_stride, l_idx,
      (const double2*)env_r, (size_t)r_stride, r_idx, (double2*)out);
  ++g_launches;
  return launch_status();
}

// ---- dense statevector backend (R:src/mpsqvm/dense.py) ---------------------

namespace {
int dense_grid(unsigned long long work) {
  const unsigned long long b = (work + 255) / 256;
  return (int)std::max(1ull, std::min(b, (unsigned long long)kNumSMs * 8));
}
}  // namespace

int32_t bmps_dense_init(double* amps, int32_t S, int32_t n, void* stream) {
  if (!amps || S < 1 || n < 1 || n > kDenseMaxQubits) return BMPS_E_ARG;
  const unsigned long long N = 1ull << n;
  dense_init_kernel<<<dense_grid(N * S), 256, 0, (cudaStream_t)stream>>>((double2*)amps, S, N);
  ++g_launches;
  return launch_status();
}

int32_t bmps_dense_apply_1q(double* amps, int32_t n, int32_t q, const double* gate_host,
                            void* stream) {
  if (!amps || !gate_host || n < 1 || n > kDenseMaxQubits || q < 0 || q >= n) return BMPS_E_ARG;
  DenseGate2 g;
  for (int k = 0; k < 4; ++k) g.m[k] = make_double2(gate_host[2 * k], gate_host[2 * k + 1]);
  dense_1q_kernel<<<dense_grid(1ull << (n - 1)), 256, 0, (cudaStream_t)stream>>>(
      (double2*)amps, n, q, g);
  ++g_launches;
  return launch_status();
}

int32_t bmps_dense_apply_2q(double* amps, int32_t n, int32_t q1, int32_t q2,
                            const double* gate_host, void* stream) {
  if (!amps || !gate_host || n < 2 || n > kDenseMaxQubits || q1 < 0 || q1 >= n || q2 < 0 ||
      q2 >= n || q1 == q2)
    return BMPS_E_ARG;
  DenseGate4 g;
  for (int k = 0; k < 16; ++k) g.m[k] = make_double2(gate_host[2 * k], gate_host[2 * k + 1]);
  dense_2q_kernel<<<dense_grid(1ull << (n - 2)), 256, 0, (cudaStream_t)stream>>>(
      (double2*)amps, n, q1, q2, g);
  ++g_launches;
  return launch_status();
}

int32_t bmps_dense_run_smem(double* amps, int32_t S, int32_t n, const int32_t* ops,
                            const double* mats, int32_t nops, void* stream) {
  if (nops == 0) return BMPS_OK;
  if (!amps || !ops || !mats || S < 1 || n < 1 || n > kDenseSmemQubits || nops < 0) return BMPS_E_ARG;
  const size_t smem = sizeof(double2) << n;
  device_cache();
  dense_run_smem_kernel<<<S, 512, smem, (cudaStream_t)stream>>>((double2*)amps, n, ops,
                                                                (const double2*)mats, nops);
  ++g_launches;
  return launch_status();
}

size_t bmps_dense_expect_workspace_bytes(int32_t count) {
  return sizeof(double2) * (size_t)kDenseExpBlocks * (size_t)std::max(count, 0);
}

int32_t bmps_dense_expect(const double* amps, int32_t S, int32_t n, const int32_t* state_idx,
                          const uint64_t* masks, const int32_t* ny, int32_t count,
                          void* workspace, size_t workspace_bytes, double* out, void* stream) {
  if (count == 0) return BMPS_OK;
  if (!amps || !state_idx || !masks || !ny || !out || S < 1 || n < 1 || n > kDenseMaxQubits ||
      count < 0)
    return BMPS_E_ARG;
  if (workspace_bytes < bmps_dense_expect_workspace_bytes(count)) return BMPS_E_WORKSPACE;
  const unsigned long long N = 1ull << n;
  const int nblk = (int)std::min<unsigned long long>(kDenseExpBlocks, (N + 255) / 256);
  cudaStream_t st = (cudaStream_t)stream;
  dense_expect_partial_kernel<<<dim3(nblk, count), 256, 0, st>>>(
      (const double2*)amps, n, state_idx, (const unsigned long long*)masks, (double2*)workspace);
  ++g_launches;
  dense_expect_final_kernel<<<(count + 127) / 128, 128, 0, st>>>((const double2*)workspace, nblk,
                                                                  ny, count, (double2*)out);
  ++g_launches;
  return launch_status();
}

int32_t bmps_dense_prob_tree(const double* amps, int32_t n, double* tree, void* stream) {
  if (!amps || !tree || n < 1 || n > kDenseMaxQubits) return BMPS_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  dense_tree_leaves_kernel<<<dense_grid(1ull << n), 256, 0, st>>>((const double2*)amps, n, tree);
  ++g_launches;
  for (int k = n - 1; k >= 0; --k) {
    dense_tree_level_kernel<<<dense_grid(1ull << k), 256, 0, st>>>(tree, k);
    ++g_launches;
  }
  return launch_status();
}

int32_t bmps_dense_sample(const double* tree, int32_t n, const double* uniforms, int32_t shots,
                          uint64_t* out, void* stream) {
  if (shots == 0) return BMPS_OK;
  if (!tree || !uniforms || !out || n < 1 || n > kDenseMaxQubits || shots < 0) return BMPS_E_ARG;
  dense_sample_kernel<<<(shots + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
      tree, n, uniforms, shots, (unsigned long long*)out);
  ++g_launches;
  return launch_status();
}

}  // extern "C"
