// Householder QR preconditioner for the one-sided Jacobi SVD (Drmac-Veselic).
//
// X0 = Q R (r x c, r >= c). One-sided Jacobi then runs on Y = R^H (c x c),
// whose columns are far closer to orthogonal than X0's when the spectrum is
// graded: on chi=256 steady-state theta matrices of config 3 the sweep count
// drops from 16-47 to 8-11 (numpy model of this exact block ordering). Q is
// never formed: with Y V_Y = U_Y Sigma, the right singular vectors of X0 are
// U_Y (= normalised final columns of Y) and the left ones are X0 V Sigma^-1,
// recovered by the split GEMM.
//
// Blocked right-looking Householder, panels of kQrNb columns:
//   qr_panel_kernel  (1 CTA / item): factor the panel in place, build T of the
//                    compact WY form  P_b...P_1 = I - V T^H V^H;
//   qr_update_kernel (1 CTA / item / 64 trailing columns): A <- A - V T^H V^H A;
//   qr_form_y_kernel : Y = R^H (lower triangular, ld = c).
// P_k = I - conj(tau_k) v_k v_k^H with v_k[k] = 1 (LAPACK zlarfg convention:
// H_k^H x = beta e_1, beta real).
#pragma once
#include <cooperative_groups.h>

#include "bmps_common.cuh"

namespace bmps {

#ifndef BMPS_QR_NB
#define BMPS_QR_NB 32
#endif
#ifndef BMPS_QR_CHUNK
#define BMPS_QR_CHUNK 64
#endif
constexpr int kQrNb = BMPS_QR_NB;   // panel width (16 or 32)
constexpr int kQrChunk = BMPS_QR_CHUNK;  // trailing columns per CTA (32 or 64)
static_assert(kQrNb == 16 || kQrNb == 32, "panel width");
static_assert(kQrChunk == 32 || kQrChunk == 64, "chunk width");
constexpr int kWT = kQrNb / 8;      // 8x8 row tiles of W = V^H A
constexpr int kCT = kQrChunk / 8;   // 8x8 column tiles of the chunk
constexpr int kNU = kWT * kCT / 8;  // W column tiles per warp (one row tile)
constexpr int kWPR = kCT / kNU;     // warps per W row tile
constexpr int kWU = kQrNb * kQrChunk / 256;  // W entries per thread

// T (upper triangular, row-major T[x * kQrNb + y]) of the compact WY form from tau
// and the strict upper part of S = V^H V (S[z * lds + y]): T_yy = tau_y,
// T[0:y, y] = -tau_y T[0:y, 0:y] S[0:y, y]. Run by one warp, lane = row x: a lane
// only reads back entries of its own row, so the y recurrence needs no barrier.
BMPS_DEV void build_t(double2* T, const double2* S, int lds, const double2* tau, int nbp) {
  const int lane = threadIdx.x & 31;
  for (int y = 0; y < kQrNb; ++y) {
    double2 v = make_double2(0.0, 0.0);
    if (y < nbp) {
      const double2 ty = tau[y];
      if (lane < y) {
        double2 acc = make_double2(0.0, 0.0);
        for (int z = lane; z < y; ++z) acc = cfma(T[lane * kQrNb + z], S[z * lds + y], acc);
        v = cmul(make_double2(-ty.x, -ty.y), acc);
      } else if (lane == y) {
        v = ty;
      }
    }
    if (lane < kQrNb) T[lane * kQrNb + y] = v;
  }
}

struct QrArgs {
  ItemMeta* meta;
  double2* X;        // working copy of X0 (r x c, ld r): overwritten by V (below diag) and R
  double2* Y;        // Jacobi input Y = R^H (c x c, ld c)
  double2* Z;        // double-QR Jacobi input Z = R2^H (c x c, ld c)
  double2* aux;      // per item: [tau1 2048][T 256][tau2 2048][T 256]
  size_t mat_stride;
  size_t aux_stride;
  int panel;
  int second;        // 0: QR of X (r x c); 1: QR of Y = R1^H (c x c), double-QR items only
  int maxp;          // panel capacity: the first QR keeps the T of every panel (reused by Q1)
};

// aux per item: [tau1: 2048][T1: maxp x kQrNb^2][tau2: 2048][T2: kQrNb^2]
BMPS_HOSTDEV inline size_t qr_aux_stride(int maxp) {
  return (size_t)2 * 2048 + (size_t)(maxp + 1) * kQrNb * kQrNb;
}
BMPS_DEV double2* qr_tslot(const QrArgs& a, double2* tau) {
  return tau + 2048 + (a.second ? 0 : (size_t)a.panel * kQrNb * kQrNb);
}

// matrix, rows and tau/T base of the pass
BMPS_DEV bool qr_pass(const QrArgs& a, int item, double2*& A, int& rows, double2*& tau) {
  const ItemMeta* m = a.meta + item;
  if (!m->precond || (a.second && !m->dq)) return false;
  A = (a.second ? a.Y : a.X) + (size_t)item * a.mat_stride;
  rows = a.second ? m->c : m->r;
  tau = a.aux + (size_t)item * a.aux_stride +
        (a.second ? 2048 + (size_t)a.maxp * kQrNb * kQrNb : 0);
  return true;
}

BMPS_DEV double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < nw; ++i) t += red[i];
  return t;
}

// S = V^H V of a factored panel (Householder vectors below the diagonal of A's
// columns j0..j1-1, rows [j0, r), global memory) and the T factor of its compact WY
// form. 512 threads.
BMPS_DEV void panel_build_t(const double2* A, int r, int j0, int j1, const double2* tau, double2* T) {
  __shared__ double2 s_S[kQrNb][kQrNb];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // V^H V on DMMA (v_k[k] = 1, zero above k): 32-row chunks of V
  // staged in shared memory, warp w accumulates 8x8 tile (w / 4, w % 4)
  const int nbp = j1 - j0;
  {
    __shared__ double2 sVc[32][kQrNb + 1];
    double sacc[4] = {0.0, 0.0, 0.0, 0.0};
    const int kr = lane & 3, rc = lane >> 2;
    const int ti = warp >> 2, tj = warp & 3;   // 512 threads: 16 warps cover 4 x 4 tiles
    const bool own = ti < kQrNb / 8 && tj < kQrNb / 8;
    // chunk loader: element i of the 32-row chunk at rb (each thread owns the same
    // elements of every chunk: 32 x kQrNb <= 2 x 512); the next chunk is loaded into
    // registers while the current one is multiplied
    constexpr int kPer = (32 * kQrNb + 511) / 512;
    auto vload = [&](int rb, int u) -> double2 {
      const int i = tid + u * 512;
      const int row = i % 32, p = i / 32;
      const int gr = rb + row, k = j0 + p;
      double2 v = make_double2(0.0, 0.0);
      if (i < 32 * kQrNb && p < nbp && gr < r) {
        if (gr == k) v = make_double2(1.0, 0.0);
        else if (gr > k) v = A[(size_t)k * r + gr];
      }
      return v;
    };
    double2 vnext[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) vnext[u] = vload(j0, u);
    for (int rb = j0; rb < r; rb += 32) {
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int i = tid + u * 512;
        if (i < 32 * kQrNb) sVc[i % 32][i / 32] = vnext[u];
      }
#pragma unroll
      for (int u = 0; u < kPer; ++u) vnext[u] = rb + 32 < r ? vload(rb + 32, u) : make_double2(0.0, 0.0);
      __syncthreads();
      if (own) {
#pragma unroll
        for (int k4 = 0; k4 < 8; ++k4) {
          const int k = k4 * 4 + kr;
          zmma(sacc, cconj(sVc[k][ti * 8 + rc]), sVc[k][tj * 8 + rc]);
        }
      }
      __syncthreads();
    }
    if (own) {
#pragma unroll
      for (int h = 0; h < 2; ++h)
        s_S[ti * 8 + rc][tj * 8 + kr * 2 + h] = make_double2(sacc[h], sacc[2 + h]);
    }
    __syncthreads();
  }
  if (warp == 0) build_t(T, &s_S[0][0], kQrNb, tau + j0, nbp);
}

// SMEM = true: the panel's rows [j0, r) are staged in shared memory for the
// factorization (every column step then costs shared-memory instead of L2
// round trips: ~4x faster for these latency-bound launches); the arithmetic and
// its order are identical to the global-memory version. Used when
// (r - j0) x kQrNb x 16 B fits (kQrPanelSmemRows).
constexpr int kQrPanelSmemRows = 384 * 32 / kQrNb;   // 384 x 32 x 16 B + 33 KB static <= 227 KB
#ifndef BMPS_QR_PANEL_U
#define BMPS_QR_PANEL_U 4
#endif
// row strides per batch of the per-column loops (4 measured best of 4 / 8 / 16)
constexpr int kQrPanelU = BMPS_QR_PANEL_U;
template <bool SMEM>
__global__ void __launch_bounds__(512) qr_panel_kernel(QrArgs a) {
  __shared__ double red[16];
  extern __shared__ __align__(16) double2 spanel[];
  const int item = blockIdx.x;
  const ItemMeta* m = a.meta + item;
  double2* A;
  double2* tau;
  int r;
  if (!qr_pass(a, item, A, r, tau)) return;
  const int c = m->c;
  const int j0 = a.panel * kQrNb;
  if (j0 >= c) return;
  const int j1 = min(j0 + kQrNb, c);
  double2* T = qr_tslot(a, tau);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ldp = r - j0;   // staged column k holds rows j0.. at spanel[(k - j0) * ldp]
  if (SMEM) {
    for (int idx = tid; idx < (j1 - j0) * ldp; idx += blockDim.x) {
      const int kk = idx / ldp, i = idx % ldp;
      spanel[idx] = A[(size_t)(j0 + kk) * r + j0 + i];
    }
    __syncthreads();
  }
  // column k of the panel, indexed by global row (>= j0)
  auto colp = [&](int k) -> double2* {
    return SMEM ? spanel + (size_t)(k - j0) * ldp - j0 : A + (size_t)k * r;
  };
  for (int k = j0; k < j1; ++k) {
    double2* col = colp(k);
    double s = 0.0;
#pragma unroll 4
    for (int i = k + 1 + tid; i < r; i += blockDim.x) s += cabs2(col[i]);
    const double xnorm2 = block_sum(s, red);
    const double2 alpha = col[k];
    double2 t = make_double2(0.0, 0.0);
    double2 scale = make_double2(0.0, 0.0);
    double beta = alpha.x;
    if (xnorm2 > 0.0 || alpha.y != 0.0) {
      const double nrm = sqrt(cabs2(alpha) + xnorm2);
      beta = alpha.x >= 0.0 ? -nrm : nrm;
      t = make_double2((beta - alpha.x) / beta, -alpha.y / beta);  // tau = (beta - alpha) / beta
      const double2 d = make_double2(alpha.x - beta, alpha.y);       // 1 / (alpha - beta)
      const double inv = 1.0 / cabs2(d);
      scale = make_double2(d.x * inv, -d.y * inv);
    }
    __syncthreads();
#pragma unroll 4
    for (int i = k + 1 + tid; i < r; i += blockDim.x) col[i] = cmul(col[i], scale);
    if (tid == 0) {
      col[k] = make_double2(beta, 0.0);
      tau[k] = t;
    }
    __syncthreads();
    // apply P_k = I - conj(tau) v v^H to panel columns k+1 .. j1-1 (one warp per column)
    for (int jj = k + 1 + warp; jj < j1 && (t.x != 0.0 || t.y != 0.0); jj += blockDim.x >> 5) {
      double2* cj = colp(jj);
      // four row strides per iteration, loads issued together (tall panels run from
      // L2: one dependent round trip per stride otherwise); interleaved partial sums
      constexpr int U = kQrPanelU;
      double2 wp[U];
#pragma unroll
      for (int u = 0; u < U; ++u) wp[u] = make_double2(0.0, 0.0);
      if (lane == 0) wp[0] = cj[k];
      int i = k + 1 + lane;
      for (; i + 32 * (U - 1) < r; i += 32 * U) {
        double2 av[U], bv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          av[u] = col[i + 32 * u];
          bv[u] = cj[i + 32 * u];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) wp[u] = cfma(cconj(av[u]), bv[u], wp[u]);
      }
      for (; i < r; i += 32) wp[0] = cfma(cconj(col[i]), cj[i], wp[0]);
#pragma unroll
      for (int h = U / 2; h > 0; h >>= 1)
#pragma unroll
        for (int u = 0; u < h; ++u) wp[u] = cadd(wp[u], wp[u + h]);
      double2 w = wp[0];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        w.x += __shfl_xor_sync(0xffffffffu, w.x, o);
        w.y += __shfl_xor_sync(0xffffffffu, w.y, o);
      }
      const double2 f = cmul(cconj(t), w);
      if (lane == 0) cj[k] = csub(cj[k], f);
      i = k + 1 + lane;
      for (; i + 32 * (U - 1) < r; i += 32 * U) {
        double2 av[U], bv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          av[u] = col[i + 32 * u];
          bv[u] = cj[i + 32 * u];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) cj[i + 32 * u] = csub(bv[u], cmul(av[u], f));
      }
      for (; i < r; i += 32) cj[i] = csub(cj[i], cmul(col[i], f));
    }
    __syncthreads();
  }
  if (SMEM) {
    for (int idx = tid; idx < (j1 - j0) * ldp; idx += blockDim.x) {
      const int kk = idx / ldp, i = idx % ldp;
      A[(size_t)(j0 + kk) * r + j0 + i] = spanel[idx];
    }
    __syncthreads();
  }
  panel_build_t(A, r, j0, j1, tau, T);
}

// Short panels (rows [j0, r) <= kQrSmallRows) of large batches -- config 4's 128-column
// items, and the last panels of every taller matrix: 128 threads, thread i = row j0 + i,
// the panel in shared memory (column kk at spanel[kk * ldp], ldp odd: 64.5 KB at 128 rows,
// three CTAs per SM instead of two of the 512-thread kernel with its 33 KB of static buffers,
// more for shorter panels). A step has two barriers instead of five: each warp keeps the
// reflector's rows in registers for its <= 8 trailing columns, and the warp that updates
// column k + 1 also returns that column's ||x[k+2:]||^2 for the next step. Measured on
// config 4 (4096 items per launch): 0.72 -> 0.45 ms per panel launch, evolution -5.3%; what
// is left is the shared-memory traffic of the column updates (each step streams the
// trailing panel through the SM's one 128 B/clk port) next to the scalar FP64 issue. Same Householder
// algorithm (zlarfg convention) with fixed-order reductions; S = V^H V comes from the staged
// panel on DMMA, and T is built by warp 0 as in panel_build_t.
constexpr int kQrSmallRows = 128;
BMPS_HOSTDEV inline int qr_small_ld(int rows) { return ((rows + 3) & ~3) + 1; }
__global__ void __launch_bounds__(128) qr_panel_small_kernel(QrArgs a) {
  extern __shared__ __align__(16) double2 spanel[];
  __shared__ double red[4];
  __shared__ double s_next;
  const int item = blockIdx.x;
  const ItemMeta* m = a.meta + item;
  double2* A;
  double2* tau;
  int r;
  if (!qr_pass(a, item, A, r, tau)) return;
  const int c = m->c;
  const int j0 = a.panel * kQrNb;
  if (j0 >= c) return;
  const int j1 = min(j0 + kQrNb, c), nbp = j1 - j0;
  double2* T = qr_tslot(a, tau);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rows = r - j0;               // <= kQrSmallRows (host dispatch)
  const int ldp = qr_small_ld(rows);     // rows [rows, ldp - 1) stay zero for the DMMA pass
  const double2 zero = make_double2(0.0, 0.0);
#pragma unroll 8
  for (int kk = 0; kk < kQrNb; ++kk)
    if (tid < ldp) spanel[kk * ldp + tid] = (kk < nbp && tid < rows) ? A[(size_t)(j0 + kk) * r + j0 + tid] : zero;
  __syncthreads();
  for (int kk = 0; kk < nbp; ++kk) {
    double2* col = spanel + kk * ldp;
    const double2 x = tid < rows ? col[tid] : zero;
    double xnorm2;
    if (kk == 0) {
      double s = tid > kk ? cabs2(x) : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) red[warp] = s;
      __syncthreads();
      xnorm2 = (red[0] + red[1]) + (red[2] + red[3]);
    } else {
      xnorm2 = s_next;   // left by the warp that updated this column in step kk - 1
    }
    const double2 alpha = col[kk];
    double2 t = zero, scale = zero;
    double beta = alpha.x;
    if (xnorm2 > 0.0 || alpha.y != 0.0) {
      const double nrm = sqrt(cabs2(alpha) + xnorm2);
      beta = alpha.x >= 0.0 ? -nrm : nrm;
      t = make_double2((beta - alpha.x) / beta, -alpha.y / beta);
      const double2 d = make_double2(alpha.x - beta, alpha.y);
      const double inv = 1.0 / cabs2(d);
      scale = make_double2(d.x * inv, -d.y * inv);
    }
    __syncthreads();   // every thread has read alpha (and s_next) before they change
    if (tid > kk && tid < rows) col[tid] = cmul(x, scale);
    if (tid == kk) {
      col[kk] = make_double2(beta, 0.0);
      tau[j0 + kk] = t;
    }
    __syncthreads();
    const bool reflect = t.x != 0.0 || t.y != 0.0;
    // v (unit entry at row kk, zero above) for this lane's rows lane + 32 u
    double2 vv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int row = lane + 32 * u;
      vv[u] = row == kk ? make_double2(1.0, 0.0) : (row > kk && row < rows) ? col[row] : zero;
    }
    // four of the warp's columns per pass (j4, j4 + 4, j4 + 8, j4 + 12): their loads,
    // dot products and the five shuffle stages of the reductions overlap -- one column at
    // a time left a step's ~8 columns per warp as 8 serial latency chains
    for (int j4 = kk + 1 + warp; j4 < nbp; j4 += 16) {
      double2 b[4][4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int jq = j4 + 4 * q;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int row = lane + 32 * u;
          b[q][u] = (jq < nbp && row < rows) ? spanel[jq * ldp + row] : zero;
        }
      }
      if (reflect) {
        double2 w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          w[q] = zero;
#pragma unroll
          for (int u = 0; u < 4; ++u) w[q] = cfma(cconj(vv[u]), b[q][u], w[q]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            w[q].x += __shfl_xor_sync(0xffffffffu, w[q].x, o);
            w[q].y += __shfl_xor_sync(0xffffffffu, w[q].y, o);
          }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int jq = j4 + 4 * q;
          const double2 f = cmul(cconj(t), w[q]);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int row = lane + 32 * u;
            b[q][u] = csub(b[q][u], cmul(vv[u], f));
            if (jq < nbp && row >= kk && row < rows) spanel[jq * ldp + row] = b[q][u];
          }
        }
      }
      if (j4 == kk + 1) {
        // the next step's ||x[kk+2:]||^2 from the updated entries (warp 0 owns column kk + 1)
        double s = 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) s += (lane + 32 * u > kk + 1) ? cabs2(b[0][u]) : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) s_next = s;
      }
    }
    __syncthreads();
  }
  // write the factored panel back; then V (unit diagonal, zero above) stays staged for S
#pragma unroll 8
  for (int kk = 0; kk < nbp; ++kk) {
    if (tid < rows) A[(size_t)(j0 + kk) * r + j0 + tid] = spanel[kk * ldp + tid];
    if (tid <= kk) spanel[kk * ldp + tid] = make_double2(tid == kk ? 1.0 : 0.0, 0.0);
  }
  __syncthreads();
  {
    // S = V^H V: warp w accumulates the tile row w (panel columns 8 w ..), all four tile columns
    const int kr = lane & 3, rc = lane >> 2;
    double sacc[4][4];
#pragma unroll
    for (int tj = 0; tj < 4; ++tj)
#pragma unroll
      for (int q = 0; q < 4; ++q) sacc[tj][q] = 0.0;
    const int nk4 = (rows + 3) >> 2;
    for (int k4 = 0; k4 < nk4; ++k4) {
      const int row = k4 * 4 + kr;
      const double2 av = cconj(spanel[(warp * 8 + rc) * ldp + row]);
#pragma unroll
      for (int tj = 0; tj < 4; ++tj) zmma(sacc[tj], av, spanel[(tj * 8 + rc) * ldp + row]);
    }
    __syncthreads();   // the panel is dead: S takes its place
#pragma unroll
    for (int tj = 0; tj < 4; ++tj)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        spanel[(warp * 8 + rc) * kQrNb + tj * 8 + kr * 2 + h] = make_double2(sacc[tj][h], sacc[tj][2 + h]);
    __syncthreads();
  }
  if (warp == 0) build_t(T, spanel, kQrNb, tau + j0, nbp);
}

// Tall panels (rows [j0, r) beyond kQrPanelSmemRows): one thread-block cluster of CS
// CTAs per item, CTA q staging the contiguous row slice q of the panel in its own
// shared memory (<= kQrClusterRows rows, 128 KB), so no column step ever goes to L2
// -- one CTA streaming a 2048-row panel from L2 reached ~75 GB/s and left 100 of
// 148 SMs idle on config 5's ~50-item layers. Per column step k (2 cluster barriers):
//   1. every CTA writes its partial ||x[k+1:]||^2 to shared memory; barrier; every
//      CTA sums the CS partials in rank order (bit-identical in all CTAs) and reads
//      alpha = x[k] from the owner of row k through DSMEM -> the same reflector
//      (beta, tau, scale) everywhere;
//   2. each CTA scales its rows, then writes its partial dots v^H x_j of the panel's
//      remaining columns; barrier; rank-ordered sums -> f_j = conj(tau) w_j, and
//      each CTA updates its own rows.
// Same Householder algorithm as qr_panel_kernel (zlarfg convention); the
// reductions run in a different, fixed order (deterministic). Rank 0 then forms
// S = V^H V and T from the written-back panel.
constexpr int kQrClusterRows = 256;
template <int CS>
__global__ void __launch_bounds__(512, 1) qr_panel_cluster_kernel(QrArgs a) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double red[16];
  __shared__ double2 part[kQrNb + 1];   // [0].x: norm partial; [1 + t]: dot partial of column k + 1 + t
  extern __shared__ __align__(16) double2 spanel[];
  const int rank = (int)cl.block_rank();
  const int item = blockIdx.x / CS;
  const ItemMeta* m = a.meta + item;
  double2* A;
  double2* tau;
  int r;
  const bool active = qr_pass(a, item, A, r, tau);
  const int c = active ? m->c : 0;
  const int j0 = a.panel * kQrNb;
  // inactive items still take part in every cluster barrier (all CTAs of a cluster agree)
  const bool work = active && j0 < c;
  const int j1 = work ? min(j0 + kQrNb, c) : j0;
  const int rows = work ? r - j0 : 0;
  const int sl = (rows + CS - 1) / CS;            // rows per slice
  const int lo = j0 + rank * sl, hi = min(j0 + (rank + 1) * sl, j0 + rows);   // my rows [lo, hi)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // staged column k holds my rows at spanel[(k - j0) * sl + (i - lo)]
  for (int idx = tid; idx < (j1 - j0) * sl; idx += blockDim.x) {
    const int kk = idx / sl, i = lo + idx % sl;
    if (i < hi) spanel[idx] = A[(size_t)(j0 + kk) * r + i];
  }
  __syncthreads();
  auto colp = [&](int k) -> double2* { return spanel + (size_t)(k - j0) * sl - lo; };
  for (int k = j0; k < j1; ++k) {
    double2* col = colp(k);
    const int owner = (k - j0) / sl;
    double s = 0.0;
    for (int i = max(k + 1, lo) + tid; i < hi; i += blockDim.x) s += cabs2(col[i]);
    s = block_sum(s, red);
    if (tid == 0) part[0] = make_double2(s, 0.0);
    cl.sync();
    double xnorm2 = 0.0;
#pragma unroll
    for (int q = 0; q < CS; ++q) xnorm2 += cl.map_shared_rank(part, q)[0].x;
    // x[k] in the owner's slice (its rows start at j0 + owner * sl)
    const double2 alpha =
        cl.map_shared_rank(spanel, owner)[(size_t)(k - j0) * sl + (k - (j0 + owner * sl))];
    double2 t = make_double2(0.0, 0.0);
    double2 scale = make_double2(0.0, 0.0);
    double beta = alpha.x;
    if (xnorm2 > 0.0 || alpha.y != 0.0) {
      const double nrm = sqrt(cabs2(alpha) + xnorm2);
      beta = alpha.x >= 0.0 ? -nrm : nrm;
      t = make_double2((beta - alpha.x) / beta, -alpha.y / beta);
      const double2 d = make_double2(alpha.x - beta, alpha.y);
      const double inv = 1.0 / cabs2(d);
      scale = make_double2(d.x * inv, -d.y * inv);
    }
    for (int i = max(k + 1, lo) + tid; i < hi; i += blockDim.x) col[i] = cmul(col[i], scale);
    __syncthreads();   // every CTA has read the owner's alpha (cluster barrier below orders the write)
    const bool rot = t.x != 0.0 || t.y != 0.0;
    // partial dots of the reflector with columns k+1 .. j1-1 (one warp per column)
    for (int jj = k + 1 + warp; jj < j1; jj += blockDim.x >> 5) {
      const double2* cj = colp(jj);
      double2 w = make_double2(0.0, 0.0);
      if (rot) {
        if (lane == 0 && owner == rank) w = cj[k];
        for (int i = max(k + 1, lo) + lane; i < hi; i += 32) w = cfma(cconj(col[i]), cj[i], w);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          w.x += __shfl_xor_sync(0xffffffffu, w.x, o);
          w.y += __shfl_xor_sync(0xffffffffu, w.y, o);
        }
      }
      if (lane == 0) part[1 + (jj - k - 1)] = w;
    }
    cl.sync();   // partial dots visible; the owner's alpha read by everyone
    if (owner == rank && tid == 0) {
      col[k] = make_double2(beta, 0.0);
      tau[k] = t;
    }
    for (int jj = k + 1 + warp; jj < j1 && rot; jj += blockDim.x >> 5) {
      double2 w = make_double2(0.0, 0.0);
#pragma unroll
      for (int q = 0; q < CS; ++q) w = cadd(w, cl.map_shared_rank(part, q)[1 + (jj - k - 1)]);
      const double2 f = cmul(cconj(t), w);
      double2* cj = colp(jj);
      if (lane == 0 && owner == rank) cj[k] = csub(cj[k], f);
      for (int i = max(k + 1, lo) + lane; i < hi; i += 32) cj[i] = csub(cj[i], cmul(col[i], f));
    }
    // part[] is rewritten in the next step only after its first cluster barrier, which
    // every CTA reaches after finishing these reads; local rows need a CTA barrier
    __syncthreads();
  }
  for (int idx = tid; idx < (j1 - j0) * sl; idx += blockDim.x) {
    const int kk = idx / sl, i = lo + idx % sl;
    if (i < hi) A[(size_t)(j0 + kk) * r + i] = spanel[idx];
  }
  __threadfence();
  cl.sync();   // the whole panel is back in global memory
  if (rank == 0 && work) panel_build_t(A, r, j0, j1, tau, qr_tslot(a, tau));
}

// Compact-WY application to one 64-column chunk of A (rows [j0, r), ld r):
//   W = V^H A (kQrNb x 64) -> W <- T^H W (TH) or T W -> A <- A - V W,
// V = the panel's Householder vectors (columns j0.., unit diagonal implied, zero
// above) stored below the diagonal of Vm (ld r). Both products on DMMA; row blocks
// of kQrRB stream through two cp.async stages (zero-filled beyond r / the chunk),
// and the first block of the second pass is in flight during the T product.
#ifndef BMPS_QR_RB
#define BMPS_QR_RB 8   // rows per staged block of the WY apply
#endif
constexpr int kQrRB = BMPS_QR_RB;
// row strides in 16-byte elements: = 2 mod 8 makes the DMMA fragment loads of the k
// loops (lanes: k = 4 consecutive rows x 2 consecutive columns) conflict-free
// (+1 padding gave 2-way conflicts); pass 2's V fragments stay 2-way
#ifndef BMPS_QR_PAD
#define BMPS_QR_PAD 2
#endif
constexpr int kQrLdA = kQrChunk + BMPS_QR_PAD;
constexpr int kQrLdV = kQrNb + BMPS_QR_PAD;
#ifndef BMPS_QR_Q1_RB
#define BMPS_QR_Q1_RB 16   // row block of the Q1 epilogue's WY apply (measured: 16 beats 8 there)
#endif
constexpr int kQ1RB = BMPS_QR_Q1_RB;
BMPS_HOSTDEV constexpr int qr_stage(int rb) { return rb * (kQrLdV + kQrLdA); }
BMPS_HOSTDEV constexpr size_t wy_apply_smem(int rb) {
  return (size_t)(2 * qr_stage(rb) + kQrNb * kQrLdA + kQrNb * kQrNb) * sizeof(double2);
}
constexpr int kQrStage = qr_stage(kQrRB);
constexpr size_t kQrUpdateSmem = wy_apply_smem(kQrRB);

template <int RB>
BMPS_DEV void wy_issue(double2* smem, int b, const double2* Vm, const double2* A, int r, int j0,
                       int nbp, int c0, int nc) {
  double2* sV = smem + (b & 1) * qr_stage(RB);
  double2* sA = sV + RB * kQrLdV;
  const int rb = j0 + b * RB;
  for (int i = threadIdx.x; i < RB * kQrNb; i += blockDim.x) {
    const int row = i % RB, p = i / RB;
    const int gr = rb + row, k = j0 + p;
    double2* dst = sV + row * kQrLdV + p;
    if (p < nbp && gr > k && gr < r) cp_async16(dst, Vm + (size_t)k * r + gr, true);
    else *dst = make_double2(p < nbp && gr == k ? 1.0 : 0.0, 0.0);
  }
  for (int i = threadIdx.x; i < RB * kQrChunk; i += blockDim.x) {
    const int row = i % RB, q = i / RB;
    const int gr = rb + row;
    const bool ok = gr < r && q < nc;
    cp_async16(sA + row * kQrLdA + q, ok ? A + (size_t)(c0 + q) * r + gr : A, ok);
  }
  cp_async_commit();
}

template <bool TH, int RB>
BMPS_DEV void wy_apply(double2* smem, const double2* Vm, double2* A, int r, int j0, int nbp,
                       int c0, int nc) {
  double2* sW = smem + 2 * qr_stage(RB);  // [kQrNb][kQrLdA]
  const double2* sT = sW + kQrNb * kQrLdA;  // [kQrNb][kQrNb], filled by the caller
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kr = lane & 3, rc = lane >> 2;
  const int nblk = (r - j0 + RB - 1) / RB;
  // pass 1: W = V^H A; warp -> W row tile warp / kWPR, kNU column tiles
  double acc[kNU][kZ3];
#pragma unroll
  for (int u = 0; u < kNU; ++u)
#pragma unroll
    for (int q = 0; q < kZ3; ++q) acc[u][q] = 0.0;
  const int tr = warp / kWPR, tc0 = (warp % kWPR) * kNU;
  wy_issue<RB>(smem, 0, Vm, A, r, j0, nbp, c0, nc);
  for (int b = 0; b < nblk; ++b) {
    if (b + 1 < nblk) {
      wy_issue<RB>(smem, b + 1, Vm, A, r, j0, nbp, c0, nc);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double2* sV = smem + (b & 1) * qr_stage(RB);
    const double2* sA = sV + RB * kQrLdV;
#pragma unroll
    for (int k4 = 0; k4 < RB / 4; ++k4) {
      const int k = k4 * 4 + kr;
      const double2 av = cconj(sV[k * kQrLdV + tr * 8 + rc]);
#pragma unroll
      for (int u = 0; u < kNU; ++u) zmma3(acc[u], av, sA[k * kQrLdA + (tc0 + u) * 8 + rc]);
    }
    __syncthreads();
  }
  wy_issue<RB>(smem, 0, Vm, A, r, j0, nbp, c0, nc);  // pass 2's first block, in flight below
#pragma unroll
  for (int u = 0; u < kNU; ++u)
#pragma unroll
    for (int h = 0; h < 2; ++h)
      sW[(tr * 8 + rc) * kQrLdA + (tc0 + u) * 8 + kr * 2 + h] = z3_get(acc[u], h);
  __syncthreads();
  double2 wt[kWU];
#pragma unroll
  for (int u = 0; u < kWU; ++u) {
    const int idx = tid + u * 256;
    const int p = idx / kQrChunk, q = idx % kQrChunk;
    double2 sacc = make_double2(0.0, 0.0);
    if (TH) {
      for (int z = 0; z <= p; ++z) sacc = cfma(cconj(sT[z * kQrNb + p]), sW[z * kQrLdA + q], sacc);
    } else {
      for (int z = p; z < kQrNb; ++z) sacc = cfma(sT[p * kQrNb + z], sW[z * kQrLdA + q], sacc);
    }
    wt[u] = sacc;
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kWU; ++u) {
    const int idx = tid + u * 256;
    sW[(idx / kQrChunk) * kQrLdA + idx % kQrChunk] = wt[u];
  }
  // pass 2: A -= V W; a RB x kQrChunk block = (RB / 8) x kCT tiles, kOU per warp
  constexpr int kOU = (RB / 8) * kCT / 8;   // output column tiles per warp
  const int orow = warp / (kCT / kOU), oc0 = (warp % (kCT / kOU)) * kOU;
  for (int b = 0; b < nblk; ++b) {
    if (b + 1 < nblk) {
      wy_issue<RB>(smem, b + 1, Vm, A, r, j0, nbp, c0, nc);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double2* sV = smem + (b & 1) * qr_stage(RB);
    const double2* sA = sV + RB * kQrLdV;
    double oacc[kOU][kZ3];
#pragma unroll
    for (int u = 0; u < kOU; ++u)
#pragma unroll
      for (int q = 0; q < kZ3; ++q) oacc[u][q] = 0.0;
#pragma unroll
    for (int k4 = 0; k4 < kQrNb / 4; ++k4) {
      const int k = k4 * 4 + kr;
      const double2 av = sV[(orow * 8 + rc) * kQrLdV + k];
#pragma unroll
      for (int u = 0; u < kOU; ++u) zmma3(oacc[u], av, sW[k * kQrLdA + (oc0 + u) * 8 + rc]);
    }
    const int rb = j0 + b * RB;
#pragma unroll
    for (int u = 0; u < kOU; ++u)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int row = orow * 8 + rc, q = (oc0 + u) * 8 + kr * 2 + h;
        const int gr = rb + row;
        if (gr < r && q < nc)
          A[(size_t)(c0 + q) * r + gr] =
              csub(sA[row * kQrLdA + q], z3_get(oacc[u], h));
      }
    __syncthreads();
  }
}

// A[:, chunk] <- A - V T^H (V^H A[:, chunk]) for the 64 trailing columns of this CTA.
__global__ void __launch_bounds__(256) qr_update_kernel(QrArgs a) {
  extern __shared__ __align__(16) double2 qsm[];
  const int item = blockIdx.y;
  const ItemMeta* m = a.meta + item;
  double2* A;
  double2* tauw;
  int r;
  if (!qr_pass(a, item, A, r, tauw)) return;
  const int c = m->c;
  const int j0 = a.panel * kQrNb;
  const int j1 = min(j0 + kQrNb, c);
  const int nbp = j1 - j0;
  const int c0 = j1 + blockIdx.x * kQrChunk;
  if (c0 >= c || nbp <= 0) return;
  double2* sT = qsm + 2 * kQrStage + kQrNb * kQrLdA;
  const double2* T = qr_tslot(a, tauw);
  for (int i = threadIdx.x; i < kQrNb * kQrNb; i += blockDim.x) sT[i] = T[i];
  wy_apply<true, kQrRB>(qsm, A, A, r, j0, nbp, c0, min(kQrChunk, c - c0));
}

// Y = R^H (c x c, ld c): Y[i][j] = conj(R[j][i]) for j <= i, else 0.
__global__ void __launch_bounds__(256) qr_form_y_kernel(QrArgs a) {
  const int item = blockIdx.y;
  const ItemMeta* m = a.meta + item;
  double2* Aw;
  double2* tau;
  int r;
  if (!qr_pass(a, item, Aw, r, tau)) return;
  const int c = m->c;
  const double2* A = Aw;
  double2* Y = (a.second ? a.Z : a.Y) + (size_t)item * a.mat_stride;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < c * c; idx += gridDim.x * blockDim.x) {
    const int i = idx % c, j = idx / c;   // Y row i, col j
    Y[(size_t)i + (size_t)j * c] = j <= i ? cconj(A[(size_t)j + (size_t)i * r]) : make_double2(0.0, 0.0);
  }
}

// ---------------------------------------------------------------------------
// Double-QR path: after the Jacobi on Z = R2^H, L = Q1 [Z sorted; 0] are the
// left singular vectors of X0 scaled by sigma (exactly what Jacobi on X0 would
// produce), so finalize/split run their ordinary (non-preconditioned) path on L.
// ---------------------------------------------------------------------------

// Static column pivoting ahead of the first QR (double-QR items): X[:, j] =
// X0[:, p(j)] with p ordering the columns of X0 by descending norm (ties by
// index). On cfg3 steady-state theta this cuts the Jacobi from 9.8 to 8.8 sweeps
// (numpy model of this exact block ordering; QR with full column pivoting: 8.6).
// The permutation needs no undoing: X0 P = Q1 R1 leaves Q1 -- and hence the
// left singular vectors L = Q1 [Z; 0] the double-QR path returns -- unchanged
// in meaning, and the split reads the unpermuted X0.
__global__ void __launch_bounds__(512) dq_colsort_kernel(const ItemMeta* meta, const double2* M0,
                                                         double2* X, size_t mat_stride) {
  __shared__ double snrm[2048];
  __shared__ int sidx[2048];
  const int item = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const ItemMeta* m = meta + item;
  if (!m->dq) return;
  const int r = m->r, c = m->c;
  const double2* x0 = M0 + (size_t)item * mat_stride;
  double2* x = X + (size_t)item * mat_stride;
  int P2 = 1;
  while (P2 < c) P2 <<= 1;
  for (int j = warp; j < P2; j += 16) {
    double acc = 0.0;
    if (j < c)
      for (int i = lane; i < r; i += 32) acc += cabs2(x0[(size_t)i + (size_t)j * r]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      snrm[j] = j < c ? acc : -1.0;
      sidx[j] = j;
    }
  }
  __syncthreads();
  for (int k = 2; k <= P2; k <<= 1) {
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      for (int t = tid; t < P2; t += blockDim.x) {
        const int u = t ^ jj;
        if (u > t) {
          const double st = snrm[t], su = snrm[u];
          const int it = sidx[t], iu = sidx[u];
          const bool u_first = su > st || (su == st && iu < it);
          const bool t_first = st > su || (st == su && it < iu);
          if (((t & k) == 0) ? u_first : t_first) {
            snrm[t] = su;
            snrm[u] = st;
            sidx[t] = iu;
            sidx[u] = it;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int j = warp; j < c; j += 16) {
    const double2* src = x0 + (size_t)sidx[j] * r;
    double2* dst = x + (size_t)j * r;
    for (int i = lane; i < r; i += 32) dst[i] = src[i];
  }
}

// sigma_j = ||z_j||, sort descending, keep (policy), L[:, k] = [Z[:, perm k]; 0]
// into the Y buffer (r x c, ld r). Marks the item as "result in Y, rows r".
__global__ void __launch_bounds__(512) dq_sort_kernel(ItemMeta* meta, const double2* Zb,
                                                      double2* Yb, size_t mat_stride,
                                                      double* sig_ws, int sig_stride,
                                                      double cutoff, int max_bond, int relative) {
  __shared__ double ssig[2048];
  __shared__ int sidx[2048];
  const int item = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  ItemMeta* m = meta + item;
  if (!m->dq || m->status) return;
  const int r = m->r, c = m->c;
  const double2* z = Zb + (size_t)item * mat_stride;
  double2* L = Yb + (size_t)item * mat_stride;
  int P2 = 1;
  while (P2 < c) P2 <<= 1;
  for (int j = warp; j < P2; j += 16) {
    double acc = 0.0;
    if (j < c)
      for (int i = lane; i < c; i += 32) acc += cabs2(z[(size_t)i + (size_t)j * c]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      ssig[j] = j < c ? sqrt(acc) : -1.0;
      sidx[j] = j;
    }
  }
  __syncthreads();
  for (int k = 2; k <= P2; k <<= 1) {
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      for (int t = tid; t < P2; t += blockDim.x) {
        const int u = t ^ jj;
        if (u > t) {
          const double st = ssig[t], su = ssig[u];
          const int it = sidx[t], iu = sidx[u];
          const bool u_first = su > st || (su == st && iu < it);
          const bool t_first = st > su || (st == su && it < iu);
          if (((t & k) == 0) ? u_first : t_first) {
            ssig[t] = su;
            ssig[u] = st;
            sidx[t] = iu;
            sidx[u] = it;
          }
        }
      }
      __syncthreads();
    }
  }
  if (tid == 0) {
    int keep;
    if (cutoff > 0.0) {
      const double thr = cutoff * (relative ? ssig[0] : 1.0);
      keep = 0;
      for (int k = 0; k < c; ++k) keep += ssig[k] >= thr ? 1 : 0;
    } else {
      keep = c;
    }
    keep = max(keep, 1);
    if (max_bond > 0) keep = min(keep, max_bond);
    m->keep_pre = keep;
    m->precond = 0;
    m->msel = 1;
    m->jrows = r;
  }
  double* sg = sig_ws + (size_t)item * sig_stride;
  for (int k = tid; k < c; k += blockDim.x) sg[k] = ssig[k];
  for (int idx = tid; idx < r * c; idx += blockDim.x) {
    const int i = idx % r, k = idx / r;
    L[(size_t)i + (size_t)k * r] =
        i < c ? z[(size_t)i + (size_t)sidx[k] * c] : make_double2(0.0, 0.0);
  }
}

// L[:, 0:keep] <- (I - V T V^H) L for the panel's Householder block (V from the
// first QR, stored below the diagonal of X; T rebuilt from tau1). Called for the
// panels in reverse order so that L <- H_1 ... H_c L = Q1 L.
constexpr size_t kQ1Smem = wy_apply_smem(kQ1RB);

__global__ void __launch_bounds__(256) dq_apply_q1_kernel(QrArgs a) {
  extern __shared__ __align__(16) double2 qsm[];
  double2* sT = qsm + 2 * qr_stage(kQ1RB) + kQrNb * kQrLdA;  // [kQrNb][kQrNb]
  const int item = blockIdx.y;
  const ItemMeta* m = a.meta + item;
  if (!m->dq || !m->msel || m->status) return;
  const int r = m->r, c = m->c, keep = m->keep_pre;
  const int j0 = a.panel * kQrNb;
  if (j0 >= c) return;
  const int j1 = min(j0 + kQrNb, c);
  const int nbp = j1 - j0;
  const int c0 = blockIdx.x * kQrChunk;
  if (c0 >= keep) return;
  const double2* V = a.X + (size_t)item * a.mat_stride;      // Householder vectors of QR 1
  const double2* T = a.aux + (size_t)item * a.aux_stride + 2048 + (size_t)a.panel * kQrNb * kQrNb;
  double2* Lm = a.Y + (size_t)item * a.mat_stride;
  for (int i = threadIdx.x; i < kQrNb * kQrNb; i += blockDim.x) sT[i] = T[i];  // T1 of this panel
  __syncthreads();
  wy_apply<false, kQ1RB>(qsm, V, Lm, r, j0, nbp, c0, min(kQrChunk, keep - c0));
}

}  // namespace bmps
