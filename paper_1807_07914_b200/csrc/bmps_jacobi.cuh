// K3 block one-sided (Hestenes) Jacobi SVD, Gram-based, on FP64 tensor cores.
//
// X (r x c, column-major, r >= c) is orthogonalised in place by unitary column
// rotations, X <- X V. Columns are grouped in blocks of w = W2/2. A visit of
// the block pair (I, J):
//   1. Gram  G = P^H P of the panel P = [X_I X_J] (r x W2) on DMMA, the panel
//      streamed through shared memory in 64-row chunks with cp.async double
//      buffering (chunk k+1 lands while chunk k feeds the tensor cores);
//   2. one cyclic Jacobi sweep on G in shared memory, accumulating Q: the full
//      round robin over all W2 columns on the first tournament round of an
//      outer sweep, the w cross rounds (i in I, j in J) otherwise. Each round
//      updates G <- J^H G J as independent 2x2 blocks (one thread per block)
//      and Q <- Q J, two barriers per round;
//   3. P <- P Q on DMMA, streamed the same way, only if a rotation happened.
// Block pairs follow a round-robin tournament over the nb column blocks; an
// item has converged when a whole outer sweep performed no rotation. The
// rotation test (pair_needs_rotation) is relative for dominant columns and
// absolute (tol * ||M||_F) for small ones.
// V is not accumulated: the split recovers the other singular vectors from the
// preserved X0 by a GEMM (SplitOp).
#pragma once
#include <cooperative_groups.h>

#include "bmps_common.cuh"

namespace bmps {

#ifndef BMPS_JAC_MINB
#define BMPS_JAC_MINB 4   // resident Jacobi CTAs per SM the register budget is sized for
#endif

#ifdef BMPS_PHASE_TIMERS
// cycles spent in [0] Gram pass, [1] inner sweep (incl. check), [2] apply pass, [3] visits
__device__ unsigned long long g_phase_cycles[8];
#define BMPS_TICK(var) const long long var = clock64()
#define BMPS_ACC(slot, t0, t1) \
  if (threadIdx.x == 0) atomicAdd(&g_phase_cycles[slot], (unsigned long long)((t1) - (t0)))
#else
#define BMPS_TICK(var)
#define BMPS_ACC(slot, t0, t1)
#endif

template <int W2>
struct JacCfg {
  static constexpr int RC = 32;                 // rows per staged chunk
  // W2 = 32: the Gram lives in staging buffer 1 during the inner sweep (it is dead
  // before the apply streams into that buffer), so a CTA needs 53 KB and 4 fit per SM.
  static constexpr bool G_IN_BUF = W2 == 32;
  static constexpr int RCP = G_IN_BUF ? RC + 2 : RC + 4;  // padded chunk column (bank spread)
  static constexpr int LDG = W2 + 4;            // padded Q column
  static constexpr int LDGG = G_IN_BUF ? RCP : W2 + 4;  // Gram column (fits a buffer)
  static constexpr int NBUF = 2;                // double-buffered chunks
  static constexpr int NT = W2 / 8;             // 8x8 tiles per Gram dimension
  static constexpr int UT = NT * (NT + 1) / 2;  // upper-triangle Gram tiles
  static constexpr int GT = UT / 8;             // whole upper tiles per warp
  static constexpr int GREM = UT - 8 * GT;      // leftover tiles, split over k
  static constexpr int GSPLIT = GREM ? 8 / GREM : 1;  // warps sharing one leftover tile
  static constexpr int AT = (RC / 8) * NT / 8;  // apply tiles per warp
  static constexpr int BUF = RCP * W2;          // one staging buffer (complex elements)
  static constexpr size_t kSmem =
      (size_t)(W2 * LDG + (G_IN_BUF ? 0 : W2 * LDGG) + NBUF * BUF) * sizeof(double2);
  static_assert(!G_IN_BUF || (W2 * LDGG <= BUF && NBUF == 2), "Gram must fit staging buffer 1");
};

// Per-item scheduling word of the dynamic (persistent, work-claiming) mode.
struct JacSched {
  unsigned long long ticket;  // (round << 32) | next visit index to claim
  int done;                   // visits of the current round completed
  int dirty;                  // any rotation in the current sweep
  int pad[4];
};

struct JacArgs {
  ItemMeta* meta;
  double2* X;
  double2* Y;
  double2* Z;        // double-QR items: Jacobi on Z = R2^H
  size_t mat_stride;
  int round;
  int persistent;
  int max_sweeps;
  int max_inner;
  double tol_factor;
  JacSched* sched;   // dynamic mode
  int* active;       // dynamic mode: items not yet converged
  int nitems;
  int tma;           // stage panels with TMA bulk copies (else cp.async)
  double2* gcache;   // per item: rotated 16x16 intra-block Grams (nullptr: off)
  size_t gcache_stride;
  int* pairlog;      // per item: [nbcap] last rotation round of each block, then
                     // [nbcap x nbcap] round of the last clean check of each block pair
                     // (-1: none / rotated since); nullptr: no skipping
  int nbcap;
};

struct RotShared {
  double c[32], s[32];
  double2 e[32];
  double2 se[32], ce[32];   // s e, c e
  int i[32], j[32], act[32];
};

// ---- TMA bulk copies (cp.async.bulk) with mbarrier completion -------------
BMPS_DEV unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
BMPS_DEV void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
BMPS_DEV void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
BMPS_DEV void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      " @!P bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
BMPS_DEV void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
BMPS_DEV void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
BMPS_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
BMPS_DEV void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
BMPS_DEV void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
BMPS_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// Staging state of a CTA: one mbarrier per chunk buffer and its phase bits.
struct JacStage {
  unsigned long long* bar;  // [2] in shared memory
  unsigned phase;           // bit b = parity to wait for on buffer b
};

BMPS_DEV void stage_init(unsigned long long* bar) {
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
}

template <int W2>
BMPS_DEV int panel_col(int p, int I, int J) {
  constexpr int w = W2 / 2;
  return p < w ? I * w + p : J * w + (p - w);
}

// Asynchronous (cp.async, zero-filled) load of rows [row0, row0+RC) of the panel.
// With RC = W2 = 32 and 256 threads each thread owns row `lane` of panel columns
// warp, warp+8, warp+16, warp+24 (a warp moves one 512-byte column segment).
template <int W2>
BMPS_DEV void jac_issue_chunk(double2* buf, const double2* X, int r, int c, int row0, int I, int J) {
  using C = JacCfg<W2>;
  if (C::RC == 32) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int row = row0 + lane;
#pragma unroll
    for (int u = 0; u < W2 / 8; ++u) {
      const int p = warp + 8 * u, col = panel_col<W2>(p, I, J);
      const bool ok = row < r && col < c;
      cp_async16(buf + lane + p * C::RCP, ok ? X + (size_t)row + (size_t)col * r : X, ok);
    }
  } else {
    for (int idx = threadIdx.x; idx < C::RC * W2; idx += blockDim.x) {
      const int m = idx % C::RC, p = idx / C::RC;
      const int row = row0 + m, col = panel_col<W2>(p, I, J);
      const bool ok = row < r && col < c;
      cp_async16(buf + m + p * C::RCP, ok ? X + (size_t)row + (size_t)col * r : X, ok);
    }
  }
  cp_async_commit();
}

template <int W2>
BMPS_DEV void jac_store_chunk(const double2* buf, double2* X, int r, int c, int row0, int I, int J) {
  using C = JacCfg<W2>;
  if (C::RC == 32) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int row = row0 + lane;
    if (row < r) {
#pragma unroll
      for (int u = 0; u < W2 / 8; ++u) {
        const int p = warp + 8 * u, col = panel_col<W2>(p, I, J);
        if (col < c) X[(size_t)row + (size_t)col * r] = buf[lane + p * C::RCP];
      }
    }
  } else {
    for (int idx = threadIdx.x; idx < C::RC * W2; idx += blockDim.x) {
      const int m = idx % C::RC, p = idx / C::RC;
      const int row = row0 + m, col = panel_col<W2>(p, I, J);
      if (row < r && col < c) X[(size_t)row + (size_t)col * r] = buf[m + p * C::RCP];
    }
  }
}

// TMA version of the chunk load (all threads call): rows beyond r and columns
// beyond c are zero-filled with ordinary stores; warp 0 arms the buffer's
// mbarrier and issues one bulk copy per valid panel column (rows are
// contiguous in the column-major matrix).
template <int W2>
BMPS_DEV void jac_issue_bulk(double2* buf, JacStage& st, int b, const double2* X, int r, int c,
                             int row0, int I, int J) {
  using C = JacCfg<W2>;
  const int nv = min(C::RC, r - row0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (nv < C::RC || panel_col<W2>(W2 - 1, I, J) >= c) {
    for (int idx = threadIdx.x; idx < C::RC * W2; idx += blockDim.x) {
      const int m = idx % C::RC, p = idx / C::RC;
      if (m >= nv || panel_col<W2>(p, I, J) >= c) buf[m + p * C::RCP] = make_double2(0.0, 0.0);
    }
  }
  if (warp == 0) {
    bulk_wait_read0();  // an earlier bulk store out of this buffer must have read it
    fence_proxy_async();
    int nvalid = 0;
    for (int p = 0; p < W2; ++p) nvalid += panel_col<W2>(p, I, J) < c ? 1 : 0;
    if (lane == 0) mbar_expect_tx(st.bar + b, (unsigned)(nvalid * nv * 16));
    __syncwarp();
    for (int p = lane; p < W2; p += 32) {
      const int col = panel_col<W2>(p, I, J);
      if (col < c) bulk_g2s(buf + p * C::RCP, X + (size_t)row0 + (size_t)col * r, (unsigned)(nv * 16), st.bar + b);
    }
  }
}

BMPS_DEV void jac_wait_bulk(JacStage& st, int b) {
  mbar_wait(st.bar + b, (st.phase >> b) & 1u);
  st.phase ^= 1u << b;
}

// TMA version of the chunk store: the buffer was written with ordinary stores
// (caller synchronised); warp 0 issues one bulk copy per valid column.
template <int W2>
BMPS_DEV void jac_store_bulk(const double2* buf, double2* X, int r, int c, int row0, int I, int J) {
  using C = JacCfg<W2>;
  const int nv = min(C::RC, r - row0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {
    fence_proxy_async();
    for (int p = lane; p < W2; p += 32) {
      const int col = panel_col<W2>(p, I, J);
      if (col < c) bulk_s2g(X + (size_t)row0 + (size_t)col * r, buf + p * C::RCP, (unsigned)(nv * 16));
    }
    bulk_commit();
  }
}

// Make every bulk store of this CTA complete and visible (before other CTAs
// or later kernels read the matrix).
BMPS_DEV void jac_flush_bulk() {
  if ((threadIdx.x >> 5) == 0) bulk_wait0();
  __syncthreads();
  __threadfence();
}

// Upper-triangle Gram tile t -> (ti, tj), ti <= tj.
template <int NT>
BMPS_DEV void upper_tile(int t, int& ti, int& tj) {
  ti = 0;
  while (t >= NT - ti) {
    t -= NT - ti;
    ++ti;
  }
  tj = ti + t;
}

// G += P^H P over one staged chunk (rows beyond nrows are zero-filled), upper
// triangle only: each warp owns GT whole tiles plus a 1/GSPLIT k-slice of one
// leftover tile (slot GT of acc), so the 8 warps carry equal DMMA work.
template <int W2>
BMPS_DEV void jac_gram_chunk(double (&acc)[JacCfg<W2>::GT + 1][kZ3], const double2* sP, int nrows) {
  using C = JacCfg<W2>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int kr = lane & 3, rc = lane >> 2;
  const int nk4 = (nrows + 3) >> 2;
#pragma unroll
  for (int u = 0; u < C::GT; ++u) {
    int ti, tj;
    upper_tile<C::NT>(warp * C::GT + u, ti, tj);
    for (int k4 = 0; k4 < nk4; ++k4) {
      const int k = k4 * 4 + kr;
      zmma3(acc[u], cconj(sP[k + (ti * 8 + rc) * C::RCP]), sP[k + (tj * 8 + rc) * C::RCP]);
    }
  }
  if (C::GREM && warp / C::GSPLIT < C::GREM) {
    int ti, tj;
    upper_tile<C::NT>(8 * C::GT + warp / C::GSPLIT, ti, tj);
    const int part = warp % C::GSPLIT;
    const int k0 = part * nk4 / C::GSPLIT, k1 = (part + 1) * nk4 / C::GSPLIT;
    for (int k4 = k0; k4 < k1; ++k4) {
      const int k = k4 * 4 + kr;
      zmma3(acc[C::GT], cconj(sP[k + (ti * 8 + rc) * C::RCP]), sP[k + (tj * 8 + rc) * C::RCP]);
    }
  }
}

// Scatter the Gram accumulators into sG (both triangles); scratch holds the
// k-split partials of the leftover tiles (8 warps x 64 complex).
template <int W2>
BMPS_DEV void jac_gram_store(const double (&acc)[JacCfg<W2>::GT + 1][kZ3], double2* sG, double2* scratch) {
  using C = JacCfg<W2>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rr = lane >> 2, cc = (lane & 3) * 2;
#pragma unroll
  for (int u = 0; u < C::GT; ++u) {
    int ti, tj;
    upper_tile<C::NT>(warp * C::GT + u, ti, tj);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i = ti * 8 + rr, j = tj * 8 + cc + h;
      const double2 v = z3_get(acc[u], h);
      sG[i + j * C::LDGG] = v;
      if (ti != tj) sG[j + i * C::LDGG] = cconj(v);
    }
  }
  if (C::GREM) {
#pragma unroll
    for (int h = 0; h < 2; ++h)
      scratch[warp * 64 + rr * 8 + cc + h] = z3_get(acc[C::GT], h);
    __syncthreads();
    for (int idx = threadIdx.x; idx < C::GREM * 64; idx += blockDim.x) {
      const int t = idx / 64, e = idx % 64;
      double2 v = make_double2(0.0, 0.0);
      for (int p = 0; p < C::GSPLIT; ++p) v = cadd(v, scratch[(t * C::GSPLIT + p) * 64 + e]);
      int ti, tj;
      upper_tile<C::NT>(8 * C::GT + t, ti, tj);
      const int i = ti * 8 + e / 8, j = tj * 8 + e % 8;
      sG[i + j * C::LDGG] = v;
      if (ti != tj) sG[j + i * C::LDGG] = cconj(v);
    }
  }
}

// Cross-block Gram only (G_IJ, w x w with w = W2/2). W2 = 32: 4 tiles, warp w
// accumulates tile w/2 over half of the chunk's k range (acc[0]); W2 = 64: 16
// tiles, two whole tiles per warp (acc[0], acc[1]).
template <int W2>
BMPS_DEV void jac_gram_chunk_cross(double (&acc)[JacCfg<W2>::GT + 1][kZ3], const double2* sP,
                                   int nrows) {
  using C = JacCfg<W2>;
  constexpr int NTc = W2 / 16, CT = NTc * NTc;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int kr = lane & 3, rc = lane >> 2;
  const int nk4 = (nrows + 3) >> 2;
  if (CT >= 8) {
    constexpr int TPW = CT >= 8 ? CT / 8 : 1;
    for (int k4 = 0; k4 < nk4; ++k4) {
      const int k = k4 * 4 + kr;
#pragma unroll
      for (int u = 0; u < TPW; ++u) {
        const int t = warp * TPW + u, ti = t / NTc, tj = NTc + t % NTc;
        zmma3(acc[u], cconj(sP[k + (ti * 8 + rc) * C::RCP]), sP[k + (tj * 8 + rc) * C::RCP]);
      }
    }
  } else {
    constexpr int KS = CT < 8 ? 8 / CT : 1;   // warps sharing one tile (k-split)
    const int t = warp / KS, part = warp % KS;
    const int ti = t / NTc, tj = NTc + t % NTc;
    const int k0 = part * nk4 / KS, k1 = (part + 1) * nk4 / KS;
    for (int k4 = k0; k4 < k1; ++k4) {
      const int k = k4 * 4 + kr;
      zmma3(acc[0], cconj(sP[k + (ti * 8 + rc) * C::RCP]), sP[k + (tj * 8 + rc) * C::RCP]);
    }
  }
}

// sG <- [[cache_I, G_IJ], [G_IJ^H, cache_J]] (scratch: 8 warps x 64 partials).
template <int W2>
BMPS_DEV void jac_gram_store_cross(const double (&acc)[JacCfg<W2>::GT + 1][kZ3], double2* sG,
                                   double2* scratch, const double2* cI, const double2* cJ) {
  using C = JacCfg<W2>;
  constexpr int w = W2 / 2, NTc = W2 / 16, CT = NTc * NTc;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rr = lane >> 2, cc = (lane & 3) * 2;
  for (int idx = threadIdx.x; idx < w * w; idx += blockDim.x) {
    const int i = idx % w, j = idx / w;
    sG[i + j * C::LDGG] = cI[i + j * w];
    sG[(w + i) + (w + j) * C::LDGG] = cJ[i + j * w];
  }
  if (CT >= 8) {
    constexpr int TPW = CT >= 8 ? CT / 8 : 1;
#pragma unroll
    for (int u = 0; u < TPW; ++u) {
      const int t = warp * TPW + u, ti = t / NTc, tj = NTc + t % NTc;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = ti * 8 + rr, j = tj * 8 + cc + h;
        const double2 v = z3_get(acc[u], h);
        sG[i + j * C::LDGG] = v;
        sG[j + i * C::LDGG] = cconj(v);
      }
    }
    return;
  }
#pragma unroll
  for (int h = 0; h < 2; ++h)
    scratch[warp * 64 + rr * 8 + cc + h] = z3_get(acc[0], h);
  __syncthreads();
  constexpr int KS = CT < 8 ? 8 / CT : 1;
  for (int idx = threadIdx.x; idx < CT * 64; idx += blockDim.x) {
    const int t = idx / 64, e = idx % 64;
    double2 v = scratch[(KS * t) * 64 + e];
    for (int k = 1; k < KS; ++k) v = cadd(v, scratch[(KS * t + k) * 64 + e]);
    const int i = (t / NTc) * 8 + e / 8, j = w + (t % NTc) * 8 + e % 8;
    sG[i + j * C::LDGG] = v;
    sG[j + i * C::LDGG] = cconj(v);
  }
}

template <int W2>
BMPS_DEV void jac_cache_store(const double2* sG, double2* cI, double2* cJ) {
  using C = JacCfg<W2>;
  constexpr int w = W2 / 2;
  for (int idx = threadIdx.x; idx < w * w; idx += blockDim.x) {
    const int i = idx % w, j = idx / w;
    cI[i + j * w] = sG[i + j * C::LDGG];
    cJ[i + j * w] = sG[(w + i) + (w + j) * C::LDGG];
  }
}

// acc = P_chunk (RC x W2) * Q (W2 x W2). Warp w owns output tiles
// t = w*AT .. w*AT+AT-1 in row-major (tile row mi = t / NT, tile col nj = t % NT).
template <int W2>
BMPS_DEV void jac_apply_mma(double (&acc)[JacCfg<W2>::AT][kZ3], const double2* sP, const double2* sQ) {
  using C = JacCfg<W2>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int kr = lane & 3, rc = lane >> 2;
#pragma unroll
  for (int u = 0; u < C::AT; ++u)
#pragma unroll
    for (int q = 0; q < kZ3; ++q) acc[u][q] = 0.0;
#pragma unroll 2
  for (int k4 = 0; k4 < W2 / 4; ++k4) {
    const int k = k4 * 4 + kr;
#pragma unroll
    for (int u = 0; u < C::AT; ++u) {
      const int t = warp * C::AT + u, mi = t / C::NT, nj = t % C::NT;
      const double2 a = sP[mi * 8 + rc + k * C::RCP];
      const double2 b = sQ[k + (nj * 8 + rc) * C::LDG];
      zmma3(acc[u], a, b);
    }
  }
}

template <int W2>
BMPS_DEV void jac_apply_writeback(const double (&acc)[JacCfg<W2>::AT][kZ3], double2* sP) {
  using C = JacCfg<W2>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int kr = lane & 3, rc = lane >> 2;
#pragma unroll
  for (int u = 0; u < C::AT; ++u)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int t = warp * C::AT + u, mi = t / C::NT, nj = t % C::NT;
      const int m = mi * 8 + rc, nn = nj * 8 + kr * 2 + h;
      sP[m + nn * C::RCP] = z3_get(acc[u], h);
    }
}

// Write the apply accumulators straight to the matrix in global memory (each
// store instruction covers 8 rows x 8 columns of a DMMA tile).
template <int W2>
BMPS_DEV void jac_apply_store_global(const double (&acc)[JacCfg<W2>::AT][kZ3], double2* X, int r,
                                     int c, int row0, int I, int J) {
  using C = JacCfg<W2>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int kr = lane & 3, rc = lane >> 2;
#pragma unroll
  for (int u = 0; u < C::AT; ++u)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int t = warp * C::AT + u, mi = t / C::NT, nj = t % C::NT;
      const int row = row0 + mi * 8 + rc, col = panel_col<W2>(nj * 8 + kr * 2 + h, I, J);
      if (row < r && col < c)
        X[(size_t)row + (size_t)col * r] = z3_get(acc[u], h);
    }
}

// Pairing of inner round rho: full round robin over W2 columns, or cross
// pairs (p, w + (p + rho) mod w) between the two blocks of the panel.
template <int W2>
BMPS_DEV void inner_pair(bool full, int rho, int p, int& i, int& j) {
  constexpr int w = W2 / 2;
  if (full) {
    tourney_pair(W2, rho, p, i, j);
  } else {
    i = p;
    j = w + (p + rho) % w;
  }
}

// One (or more) cyclic Jacobi sweeps on the W2 x W2 Gram, accumulating Q.
// Returns the number of rotations of the first sweep (block-uniform).
template <int W2>
BMPS_DEV int jac_inner(double2* sG, double2* sQ, RotShared& rs, double tol, double noise2,
                       double fro, bool full, int max_inner) {
  using C = JacCfg<W2>;
  constexpr int w = W2 / 2;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < W2 * W2; idx += blockDim.x) {
    const int i = idx % W2, j = idx / W2;
    sQ[i + j * C::LDG] = make_double2(i == j ? 1.0 : 0.0, 0.0);
  }
  int first = 0;
  const int rounds = full ? W2 - 1 : w;
  for (int it = 0; it < max_inner; ++it) {
    int any = 0;
    for (int rho = 0; rho < rounds; ++rho) {
      BMPS_TICK(tr0);
      int act = 0;
      if (tid < w) {
        int i, j;
        inner_pair<W2>(full, rho, tid, i, j);
        double c = 1.0, s = 0.0;
        double2 e = make_double2(1.0, 0.0);
        act = jacobi_rotation(sG[i + i * C::LDGG].x, sG[j + j * C::LDGG].x, sG[i + j * C::LDGG], tol,
                              noise2, fro, c, s, e);
        if (!act) {
          c = 1.0;
          s = 0.0;
          e = make_double2(1.0, 0.0);
        }
        rs.i[tid] = i;
        rs.j[tid] = j;
        rs.act[tid] = act;
        rs.c[tid] = c;
        rs.s[tid] = s;
        rs.e[tid] = e;
        rs.se[tid] = cscale(e, s);
        rs.ce[tid] = cscale(e, c);
      }
      const int nact = __syncthreads_count(act);
      BMPS_TICK(tr1);
      BMPS_ACC(4, tr0, tr1);
      BMPS_ACC(6, 0, 1);
      any += nact;
      if (nact == 0) continue;
      // G <- J^H G J as independent 2x2 blocks (p <= q computed, (q, p) mirrored);
      // Q <- Q J
      for (int idx = tid; idx < w * (w + 1) / 2; idx += blockDim.x) {
        const int q = (int)((sqrtf(8.0f * (float)idx + 1.0f) - 1.0f) * 0.5f);
        const int p = idx - q * (q + 1) / 2;
        if (!(rs.act[p] | rs.act[q])) continue;  // identity on both sides
        const int ip = rs.i[p], jp = rs.j[p], iq = rs.i[q], jq = rs.j[q];
        const double cp = rs.c[p], sp = rs.s[p], cq = rs.c[q], sq = rs.s[q];
        const double2 sep = rs.se[p], cep = rs.ce[p], seq = rs.se[q], ceq = rs.ce[q];
        const double2 g00 = sG[ip + iq * C::LDGG], g01 = sG[ip + jq * C::LDGG];
        const double2 g10 = sG[jp + iq * C::LDGG], g11 = sG[jp + jq * C::LDGG];
        // right: [x_iq, x_jq] <- [x_iq, x_jq] [[cq, sq], [-sq e_q*, cq e_q*]]
        const double2 r00 = cmsc(g00, cq, seq, g01);
        const double2 r01 = cmac(g00, sq, ceq, g01);
        const double2 r10 = cmsc(g10, cq, seq, g11);
        const double2 r11 = cmac(g10, sq, ceq, g11);
        // left: rows ip, jp by J_p^H = [[cp, -sp e_p], [sp, cp e_p]]
        const double2 n00 = cms(r00, cp, sep, r10);
        const double2 n01 = cms(r01, cp, sep, r11);
        const double2 n10 = cma(r00, sp, cep, r10);
        const double2 n11 = cma(r01, sp, cep, r11);
        sG[ip + iq * C::LDGG] = n00;
        sG[ip + jq * C::LDGG] = n01;
        sG[jp + iq * C::LDGG] = n10;
        sG[jp + jq * C::LDGG] = n11;
        if (p != q) {
          sG[iq + ip * C::LDGG] = cconj(n00);
          sG[jq + ip * C::LDGG] = cconj(n01);
          sG[iq + jp * C::LDGG] = cconj(n10);
          sG[jq + jp * C::LDGG] = cconj(n11);
        }
      }
      for (int idx = tid; idx < W2 * w; idx += blockDim.x) {
        const int k = idx % W2, q = idx / W2;
        if (!rs.act[q]) continue;
        const int iq = rs.i[q], jq = rs.j[q];
        const double cq = rs.c[q], sq = rs.s[q];
        const double2 qi = sQ[k + iq * C::LDG], qj = sQ[k + jq * C::LDG];
        sQ[k + iq * C::LDG] = cmsc(qi, cq, rs.se[q], qj);
        sQ[k + jq * C::LDG] = cmac(qi, sq, rs.ce[q], qj);
      }
      __syncthreads();
      BMPS_TICK(tr2);
      BMPS_ACC(5, tr1, tr2);
    }
    if (it == 0) first = any;
    if (!any) break;
  }
  return first;
}

// One block-pair visit; returns true if any rotation was applied. If
// `resident`, the whole panel (r <= RC) already sits in buffer 0 and is
// neither loaded nor stored here. W2 = 32 streams the panel with TMA bulk
// copies (double buffered, mbarrier completion); W2 = 64 with cp.async.
template <int W2>
BMPS_DEV bool jac_visit(double2* X, int r, int c, int I, int J, double tol, double noise2,
                        double fro, bool full, int max_inner, bool resident, double2* sG,
                        double2* sQ, double2* sP, RotShared& rs, JacStage& st, bool tma,
                        double2* gcache = nullptr, bool inner_regs = false) {
  using C = JacCfg<W2>;
  BMPS_TICK(tv0);
  const int nch = (r + C::RC - 1) / C::RC;
  const bool bulk = !resident && tma;
  // cross visits reuse the rotated intra-block Grams cached by earlier visits
  const bool cross_gram = gcache != nullptr && !full && !resident;
  double2* cI = gcache ? gcache + (size_t)I * (W2 / 2) * (W2 / 2) : nullptr;
  double2* cJ = gcache ? gcache + (size_t)J * (W2 / 2) * (W2 / 2) : nullptr;
  double gacc[C::GT + 1][kZ3];
#pragma unroll
  for (int u = 0; u < C::GT + 1; ++u)
#pragma unroll
    for (int q = 0; q < kZ3; ++q) gacc[u][q] = 0.0;
  if (resident) {
    jac_gram_chunk<W2>(gacc, sP, r);
  } else if (bulk) {
    __syncthreads();
    jac_issue_bulk<W2>(sP, st, 0, X, r, c, 0, I, J);
    for (int k = 0; k < nch; ++k) {
      const int b = k & 1;
      if (k + 1 < nch) jac_issue_bulk<W2>(sP + (b ^ 1) * C::BUF, st, b ^ 1, X, r, c, (k + 1) * C::RC, I, J);
      jac_wait_bulk(st, b);
      __syncthreads();
      if (cross_gram) jac_gram_chunk_cross<W2>(gacc, sP + b * C::BUF, min(C::RC, r - k * C::RC));
      else jac_gram_chunk<W2>(gacc, sP + b * C::BUF, min(C::RC, r - k * C::RC));
      __syncthreads();
    }
  } else {
    __syncthreads();
    jac_issue_chunk<W2>(sP, X, r, c, 0, I, J);
    for (int k = 0; k < nch; ++k) {
      double2* cur = sP + (k % C::NBUF) * C::BUF;
      if (C::NBUF == 2 && k + 1 < nch) {
        jac_issue_chunk<W2>(sP + ((k + 1) % 2) * C::BUF, X, r, c, (k + 1) * C::RC, I, J);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      if (cross_gram) jac_gram_chunk_cross<W2>(gacc, cur, min(C::RC, r - k * C::RC));
      else jac_gram_chunk<W2>(gacc, cur, min(C::RC, r - k * C::RC));
      __syncthreads();
      if (C::NBUF == 1 && k + 1 < nch) jac_issue_chunk<W2>(sP, X, r, c, (k + 1) * C::RC, I, J);
    }
  }
  BMPS_TICK(tv1);
  BMPS_ACC(0, tv0, tv1);
  // k-split partials need 8 warps x 64 complex: Q's space, or (W2 = 16) staging buffer 1,
  // whose last chunk every warp has consumed by now
  double2* scratch = W2 * C::LDG >= 512 ? sQ : sP + C::BUF;
  if (cross_gram) jac_gram_store_cross<W2>(gacc, sG, scratch, cI, cJ);
  else jac_gram_store<W2>(gacc, sG, scratch);
  __syncthreads();
  const bool staged = nch == 1;  // single chunk still in buffer 0 from the Gram pass
  // prefetch the first apply chunk so its load overlaps the inner sweep
  if (!resident && !staged) {
    if (bulk) jac_issue_bulk<W2>(sP, st, 0, X, r, c, 0, I, J);
    else jac_issue_chunk<W2>(sP, X, r, c, 0, I, J);
  }
  // fast path: one parallel test of every pair the inner sweep would visit
  int need = 0;
  {
    constexpr int w = W2 / 2;
    const int npairs = full ? W2 * W2 : w * w;
    for (int idx = threadIdx.x; idx < npairs && !need; idx += blockDim.x) {
      int i, j;
      if (full) {
        i = idx % W2;
        j = idx / W2;
        if (i >= j) continue;
      } else {
        i = idx % w;
        j = w + idx / w;
      }
      need = jacobi_needs(sG[i + i * C::LDGG].x, sG[j + j * C::LDGG].x, sG[i + j * C::LDGG], tol,
                          noise2, fro);
    }
  }
  const int nrot = __syncthreads_or(need) ? jac_inner<W2>(sG, sQ, rs, tol, noise2, fro, full, max_inner)
                                          : 0;
  BMPS_TICK(tv2);
  BMPS_ACC(1, tv1, tv2);
  BMPS_ACC(3, 0, 1);
  if (gcache != nullptr && !resident && (full || nrot > 0)) jac_cache_store<W2>(sG, cI, cJ);
  if (C::G_IN_BUF) __syncthreads();  // sG (buffer 1) is read before the apply refills it
  if (nrot == 0) {
    if (!resident && !staged) {
      if (bulk) jac_wait_bulk(st, 0);
      else cp_async_wait<0>();
    }
    return false;
  }
  double aacc[C::AT][kZ3];
  if (resident) {
    jac_apply_mma<W2>(aacc, sP, sQ);
    __syncthreads();
    jac_apply_writeback<W2>(aacc, sP);
    __syncthreads();
    return true;
  }
  if (bulk) {
    for (int k = 0; k < nch; ++k) {
      const int b = k & 1;
      double2* cur = sP + b * C::BUF;
      if (!staged && k + 1 < nch) {
        const int row1 = (k + 1) * C::RC;
        if (r - row1 < C::RC || panel_col<W2>(W2 - 1, I, J) >= c) {
          // the issue zero-fills: the bulk store out of that buffer must be done reading
          if ((threadIdx.x >> 5) == 0) bulk_wait_read0();
          __syncthreads();
        }
        jac_issue_bulk<W2>(sP + (b ^ 1) * C::BUF, st, b ^ 1, X, r, c, row1, I, J);
      }
      if (!staged) jac_wait_bulk(st, b);
      __syncthreads();
      jac_apply_mma<W2>(aacc, cur, sQ);
      __syncthreads();
      jac_apply_writeback<W2>(aacc, cur);
      __syncthreads();
      jac_store_bulk<W2>(cur, X, r, c, k * C::RC, I, J);
    }
    jac_flush_bulk();
    return true;
  }

  // cp.async re-stream: load chunk k+1 while chunk k is multiplied and stored
  for (int k = 0; k < nch; ++k) {
    double2* cur = sP + (k % C::NBUF) * C::BUF;
    if (!staged) {
      if (C::NBUF == 2 && k + 1 < nch) {
        jac_issue_chunk<W2>(sP + ((k + 1) % 2) * C::BUF, X, r, c, (k + 1) * C::RC, I, J);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
    }
    __syncthreads();
    jac_apply_mma<W2>(aacc, cur, sQ);
    jac_apply_store_global<W2>(aacc, X, r, c, k * C::RC, I, J);
    __syncthreads();  // every warp is done reading `cur` before it is refilled
    if (C::NBUF == 1 && !staged && k + 1 < nch) jac_issue_chunk<W2>(sP, X, r, c, (k + 1) * C::RC, I, J);
  }
  BMPS_TICK(tv3);
  BMPS_ACC(2, tv2, tv3);
  return true;
}

template <int W2>
BMPS_DEV void jac_load_resident(double2* sP, const double2* X, int r, int c) {
  jac_issue_chunk<W2>(sP, X, r, c, 0, 0, 1);
  cp_async_wait<0>();
  __syncthreads();
}

template <int W2>
__global__ void __launch_bounds__(256, (W2 <= 32) ? BMPS_JAC_MINB : 1) jacobi_kernel(JacArgs args) {
  using C = JacCfg<W2>;
  extern __shared__ __align__(16) double2 jsm[];
  double2* sQ = jsm;
  double2* sP = sQ + W2 * C::LDG;
  double2* sG = C::G_IN_BUF ? sP + C::BUF : sP + C::NBUF * C::BUF;
  __shared__ RotShared rs;
  __shared__ unsigned long long jbar[2];
  const int item = blockIdx.y;
  ItemMeta* m = args.meta + item;
  if (m->conv) return;
  JacStage st{jbar, 0u};
  stage_init(jbar);
  const int r = m->jrows, c = m->c;
  double2* X = (m->dq ? args.Z : m->precond ? args.Y : args.X) + (size_t)item * args.mat_stride;
  double2* gc = args.gcache ? args.gcache + (size_t)item * args.gcache_stride : nullptr;
  constexpr int w = W2 / 2;
  int nb = (c + w - 1) / w;
  nb += nb & 1;
  const double tol = args.tol_factor * sqrt((double)r) * kEps;
  const double noise2 = kNoiseRel * kNoiseRel * m->fro2;
  const double fro = sqrt(m->fro2);
  if (nb == 2) {
    // single panel: the whole matrix is one visit, iterated to convergence
    if (blockIdx.x != 0) return;
    const bool resident = r <= C::RC;
    if (resident) jac_load_resident<W2>(sP, X, r, c);
    int sweep = 0;
    bool clean = false;
    for (; sweep < args.max_sweeps; ++sweep) {
      if (!jac_visit<W2>(X, r, c, 0, 1, tol, noise2, fro, true, 64, resident, sG, sQ, sP, rs, st, args.tma)) {
        clean = true;
        break;
      }
    }
    if (resident) {
      __syncthreads();
      jac_store_chunk<W2>(sP, X, r, c, 0, 0, 1);
    }
    if (threadIdx.x == 0) {
      m->sweeps = sweep;
      m->conv = 1;
      if (!clean) m->status = BMPS_S_SVD_FAILED;
    }
    return;
  }
  if (args.persistent == 2) {
    // one thread-block cluster per item; rounds separated by cluster barriers,
    // the sweep's dirty flag OR-reduced in rank 0's shared memory (DSMEM)
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    __shared__ int sflag[2];
    const int rank = (int)cl.block_rank(), P = (int)cl.num_blocks();
    if (threadIdx.x < 2) sflag[threadIdx.x] = 0;
    cl.sync();
    int* flag0 = cl.map_shared_rank(sflag, 0);
    int sweep = 0;
    bool clean = false;
    for (; sweep < args.max_sweeps; ++sweep) {
      bool any = false;
      for (int rho = 0; rho < nb - 1; ++rho) {
        for (int v = rank; v < nb / 2; v += P) {
          int I, J;
          tourney_pair(nb, rho, v, I, J);
          any |= jac_visit<W2>(X, r, c, I, J, tol, noise2, fro, rho == 0, args.max_inner, false, sG,
                               sQ, sP, rs, st, args.tma, gc);
        }
        __threadfence();
        cl.sync();
      }
      if (any && threadIdx.x == 0) atomicOr(flag0 + (sweep & 1), 1);
      cl.sync();
      const int dirty = *((volatile int*)(flag0 + (sweep & 1)));
      if (rank == 0 && threadIdx.x == 0) sflag[(sweep + 1) & 1] = 0;
      if (!dirty) {
        clean = true;
        break;
      }
    }
    if (rank == 0 && threadIdx.x == 0) {
      m->sweeps = sweep;
      m->conv = 1;
      if (!clean) m->status = BMPS_S_SVD_FAILED;
    }
    cl.sync();
    return;
  }
  if (args.persistent) {
    if (blockIdx.x != 0) return;
    int sweep = 0;
    bool clean = false;
    for (; sweep < args.max_sweeps; ++sweep) {
      bool any = false;
      for (int rho = 0; rho < nb - 1; ++rho)
        for (int v = 0; v < nb / 2; ++v) {
          int I, J;
          tourney_pair(nb, rho, v, I, J);
          any |= jac_visit<W2>(X, r, c, I, J, tol, noise2, fro, rho == 0, args.max_inner, false, sG,
                               sQ, sP, rs, st, args.tma, gc);
        }
      if (!any) {
        clean = true;
        break;
      }
    }
    if (threadIdx.x == 0) {
      m->sweeps = sweep;
      m->conv = 1;
      if (!clean) m->status = BMPS_S_SVD_FAILED;
    }
    return;
  }
  const int v = blockIdx.x, rho = args.round;
  if (v >= nb / 2 || rho >= nb - 1) return;
  int I, J;
  tourney_pair(nb, rho, v, I, J);
  if (jac_visit<W2>(X, r, c, I, J, tol, noise2, fro, rho == 0, args.max_inner, false, sG, sQ, sP,
                    rs, st, args.tma, gc) &&
      threadIdx.x == 0)
    atomicOr(&m->flag, 1);
}

// Dynamic mode: a persistent grid (one wave of resident CTAs) claims block-pair
// visits from any item whose current tournament round still has unclaimed
// visits. The CTA finishing the last visit of a round opens the next round (and
// at the end of a sweep converges the item or clears its dirty flag). CTAs
// never wait on each other -- when nothing is claimable they back off and
// re-probe -- so there is no deadlock, no host polling and no per-round
// launch, and stragglers' rounds overlap other items' work.
template <int W2>
__global__ void __launch_bounds__(256, (W2 <= 32) ? BMPS_JAC_MINB : 1) jacobi_dynamic_kernel(JacArgs args) {
  using C = JacCfg<W2>;
  extern __shared__ __align__(16) double2 jsm[];
  double2* sQ = jsm;
  double2* sP = sQ + W2 * C::LDG;
  double2* sG = C::G_IN_BUF ? sP + C::BUF : sP + C::NBUF * C::BUF;
  __shared__ RotShared rs;
  __shared__ int s_item, s_v;
  __shared__ unsigned s_round;
  __shared__ unsigned long long jbar[2];
  JacStage st{jbar, 0u};
  stage_init(jbar);
  constexpr int w = W2 / 2;
  const int nitems = args.nitems;
  int cursor = blockIdx.x % nitems;
  volatile int* active = args.active;
  while (*active > 0) {
    if (threadIdx.x == 0) {
      s_item = -1;
      for (int probe = 0; probe < nitems; ++probe) {
        const int i = (cursor + probe) % nitems;
        JacSched* sc = args.sched + i;
        if (args.meta[i].conv) continue;
        const int c = args.meta[i].c;
        int nb = (c + w - 1) / w;
        nb += nb & 1;
        const unsigned nbv = (unsigned)(nb / 2);
        const unsigned long long peek = *((volatile unsigned long long*)&sc->ticket);
        if ((unsigned)(peek & 0xffffffffull) >= nbv) continue;
        const unsigned long long old = atomicAdd(&sc->ticket, 1ull);
        const unsigned v = (unsigned)(old & 0xffffffffull);
        if (v >= nbv) continue;
        s_item = i;
        s_v = (int)v;
        s_round = (unsigned)(old >> 32);
        cursor = i;
        break;
      }
      __threadfence();
    }
    __syncthreads();
    const int i = s_item;
    if (i < 0) {
      if (threadIdx.x == 0) __nanosleep(2000);
      __syncthreads();
      cursor = (cursor + 1) % nitems;
      continue;
    }
    const int v = s_v;
    const unsigned rnd = s_round;
    ItemMeta* m = args.meta + i;
    const int r = m->jrows, c = m->c;
    double2* X = (m->dq ? args.Z : m->precond ? args.Y : args.X) + (size_t)i * args.mat_stride;
    int nb = (c + w - 1) / w;
    nb += nb & 1;
    const double tol = args.tol_factor * sqrt((double)r) * kEps;
    const double noise2 = kNoiseRel * kNoiseRel * m->fro2;
    const double fro = sqrt(m->fro2);
    JacSched* sc = args.sched + i;
    if (nb == 2) {
      // single panel: the one claimer iterates the whole item to convergence
      const bool resident = r <= C::RC;
      if (resident) jac_load_resident<W2>(sP, X, r, c);
      int sweep = 0;
      bool clean = false;
      for (; sweep < args.max_sweeps; ++sweep) {
        if (!jac_visit<W2>(X, r, c, 0, 1, tol, noise2, fro, true, 64, resident, sG, sQ, sP, rs, st, args.tma)) {
          clean = true;
          break;
        }
      }
      if (resident) {
        __syncthreads();
        jac_store_chunk<W2>(sP, X, r, c, 0, 0, 1);
      }
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) {
        m->sweeps = sweep;
        if (!clean) m->status = BMPS_S_SVD_FAILED;
        __threadfence();
        m->conv = 1;
        atomicSub(args.active, 1);
      }
      __syncthreads();
      continue;
    }
    const int rounds = nb - 1;
    const int sweep = (int)(rnd / (unsigned)rounds), rho = (int)(rnd % (unsigned)rounds);
    int I, J;
    tourney_pair(nb, rho, v, I, J);
    double2* gc = args.gcache ? args.gcache + (size_t)i * args.gcache_stride : nullptr;
    // Exact skip of a cross visit whose outcome is known: the pair was checked clean
    // at round lc and neither block has been rotated since, so its columns -- hence
    // its Gram and the rotation test -- are bit-for-bit what they were (most visits
    // of the last sweeps of an item)
    int* last_rot = args.pairlog ? args.pairlog + (size_t)i * (args.nbcap + args.nbcap * args.nbcap)
                                 : nullptr;
    int* last_chk = last_rot ? last_rot + args.nbcap + I * args.nbcap + J : nullptr;
    bool skip = false;
    if (last_rot && rho > 0) {
      const int lc = *((volatile int*)last_chk);
      skip = lc >= 0 && *((volatile int*)(last_rot + I)) < lc && *((volatile int*)(last_rot + J)) < lc;
    }
    const bool dirty = skip ? false
                            : jac_visit<W2>(X, r, c, I, J, tol, noise2, fro, rho == 0,
                                            args.max_inner, false, sG, sQ, sP, rs, st, args.tma, gc);
    if (last_rot && !skip && threadIdx.x == 0) {
      if (dirty) {
        last_rot[I] = (int)rnd;
        last_rot[J] = (int)rnd;
        *last_chk = -1;
      } else {
        *last_chk = (int)rnd;
      }
    }
    // release: the CTA barrier orders every thread's panel / Gram-cache stores before
    // thread 0's GPU-scope fence, which is cumulative (the CUTLASS semaphore pattern);
    // one fence per visit instead of a MEMBAR.GPU stall in all 256 threads
    __syncthreads();
    if (threadIdx.x == 0) {
      if (dirty) atomicOr(&sc->dirty, 1);
      __threadfence();
      const int d = atomicAdd(&sc->done, 1);
      if (d == nb / 2 - 1) {
        // last visit of the round: open the next round (or finish the item)
        sc->done = 0;
        bool finished = false;
        if (rho == rounds - 1) {
          const int dsw = atomicAdd(&sc->dirty, 0);
          if (!dsw) {
            m->sweeps = sweep;
            finished = true;
          } else if (sweep + 1 >= args.max_sweeps) {
            m->sweeps = sweep + 1;
            m->status = BMPS_S_SVD_FAILED;
            finished = true;
          } else {
            sc->dirty = 0;
          }
        }
        __threadfence();
        if (finished) {
          m->conv = 1;
          atomicSub(args.active, 1);
        } else {
          atomicExch(&sc->ticket, (unsigned long long)(rnd + 1) << 32);
        }
      }
    }
    __syncthreads();
  }
}

}  // namespace bmps
