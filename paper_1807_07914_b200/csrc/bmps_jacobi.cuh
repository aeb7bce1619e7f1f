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

#ifndef BMPS_CLAIM_SLEEP_NS
#define BMPS_CLAIM_SLEEP_NS 2000   // dynamic Jacobi: back-off of a CTA that found no open visit
#endif

#ifdef BMPS_EXPERIMENTAL
constexpr bool kTmaStaging = true;    // TMA bulk panel staging compiled in (measured slower)
#else
constexpr bool kTmaStaging = false;
#endif

#ifndef BMPS_INNER_DEFER
#define BMPS_INNER_DEFER 1   // inner sweep: Q update of a batch under the next batch's rounds
#endif

#ifndef BMPS_JAC_MINB
#define BMPS_JAC_MINB 4   // resident Jacobi CTAs per SM the register budget is sized for
#endif

#ifdef BMPS_PHASE_TIMERS
// cycles spent in [0] Gram pass, [1] inner sweep (incl. check), [2] apply pass, [3] visits
__device__ unsigned long long g_phase_cycles[24];   // [16..20]: per-round segments of phase S
// per-warp arrival trace of the inner sweep's phase B (CTA 0, first 64 rounds): start of
// the phase, end of the warp's own work, release from the counting barrier
__device__ unsigned long long g_inner_trace[64 * 8 * 4];
__device__ int g_inner_trace_n;
#define BMPS_TICK(var) const long long var = clock64()
#define BMPS_ACC(slot, t0, t1) \
  if (threadIdx.x == 0) atomicAdd(&g_phase_cycles[slot], (unsigned long long)((t1) - (t0)))
#define WS_ACC(lead, slot, t0, t1) \
  if (threadIdx.x == (lead)) atomicAdd(&g_phase_cycles[slot], (unsigned long long)((t1) - (t0)))
#else
#define WS_ACC(lead, slot, t0, t1)
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
  int pad[4];                 // -DBMPS_DEBUG_CHECKS: [0..1] visit mask of the round, [2] round
};

// Invariant checks of the lock-free visit scheduling (-DBMPS_DEBUG_CHECKS; the
// pool's compute-sanitizer is closed, so the claim / completion protocol checks
// itself): every visit of a round completes exactly once, in the round its ticket
// was claimed for, and a round is closed only when all its visits completed.
BMPS_DEV void jac_debug_mark(JacSched* sc, int v, unsigned rnd, int nvis) {
#ifdef BMPS_DEBUG_CHECKS
  BMPS_CHECK(v >= 0 && v < nvis && nvis <= 64);
  BMPS_CHECK((unsigned)atomicAdd(&sc->pad[2], 0) == rnd);
  const unsigned long long old = atomicOr((unsigned long long*)sc->pad, 1ull << v);
  BMPS_CHECK(!(old & (1ull << v)));
#else
  (void)sc; (void)v; (void)rnd; (void)nvis;
#endif
}
// Called by the CTA that completed the last visit of round rnd, before it opens
// round rnd + 1 (or retires the item).
BMPS_DEV void jac_debug_close(JacSched* sc, unsigned rnd, int nvis) {
#ifdef BMPS_DEBUG_CHECKS
  unsigned long long* mask = (unsigned long long*)sc->pad;
  const unsigned long long full = nvis >= 64 ? ~0ull : ((1ull << nvis) - 1);
  BMPS_CHECK(atomicAdd(mask, 0ull) == full);
  atomicExch(mask, 0ull);
  atomicExch(&sc->pad[2], (int)(rnd + 1));
#else
  (void)sc; (void)rnd; (void)nvis;
#endif
}

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
  double thr_a, thr_b;        // dynamic mode: relative-coupling thresholds of the first
  int thr_a_sweeps, thr_b_sweeps;   // sweeps (< a_sweeps: thr_a, < b_sweeps: thr_b, then 0)
};

// Shared state of the inner (Gram-space) sweep, see jac_inner: per column group the
// four rotations (c, sigma) of the current round and the group's rotation count of the
// batch (double-buffered by batch parity).
template <int W2>
struct InnerShared {
  static constexpr int NG = W2 / 8;
  double2 sg[NG][4];
  double c[NG][4];
  int cnt[2][NG];
};

// Thread groups a Jacobi phase runs on. CtaGrp: the whole CTA (classic kernels,
// barrier 0). NamedGrp: a warp-aligned subset synchronised on its own named
// barrier (warp-specialised kernel: math warps and rotation warps).
struct CtaGrp {
  static constexpr int kN = 256;   // block size of every classic Jacobi launch
  BMPS_DEV static int tid() { return (int)threadIdx.x; }
  BMPS_DEV static int n() { return (int)blockDim.x; }
  BMPS_DEV static void sync() { __syncthreads(); }
  // BAR counts arrivals in units of warps: a warp must arrive converged (the compiler
  // does not always reconverge ahead of BAR.RED as it does ahead of BAR.SYNC)
  BMPS_DEV static int count(int p) {
    __syncwarp();
    return __syncthreads_count(p);
  }
};
template <int BASE, int N, int ID>
struct NamedGrp {
  static constexpr int kN = N;
  BMPS_DEV static int tid() { return (int)threadIdx.x - BASE; }
  BMPS_DEV static constexpr int n() { return N; }
  // __barrier_sync_count is a convergent intrinsic: the compiler reconverges the warp
  // before it (an inline-asm bar.sync after a divergent loop exit can be reached by a
  // split warp, which deadlocks or faults)
  BMPS_DEV static void sync() { __barrier_sync_count(ID, N); }
  // number of group threads with p != 0 (ballot per warp, one word per warp)
  BMPS_DEV static int count(int p) {
    __shared__ int s_w[N / 32];
    const unsigned bal = __ballot_sync(0xffffffffu, p != 0);
    if ((threadIdx.x & 31) == 0) s_w[tid() >> 5] = __popc(bal);
    sync();
    int r = 0;
#pragma unroll
    for (int k = 0; k < N / 32; ++k) r += s_w[k];
    sync();
    return r;
  }
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
template <int W2, class G = CtaGrp>
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
    G::sync();
    for (int idx = G::tid(); idx < C::GREM * 64; idx += G::n()) {
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
template <int W2, class G = CtaGrp>
BMPS_DEV void jac_gram_store_cross(const double (&acc)[JacCfg<W2>::GT + 1][kZ3], double2* sG,
                                   double2* scratch, const double2* cI, const double2* cJ) {
  using C = JacCfg<W2>;
  constexpr int w = W2 / 2, NTc = W2 / 16, CT = NTc * NTc;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rr = lane >> 2, cc = (lane & 3) * 2;
  for (int idx = G::tid(); idx < w * w; idx += G::n()) {
    const int i = idx % w, j = idx / w;
    sG[i + j * C::LDGG] = cI[i + j * w];
    sG[(w + i) + (w + j) * C::LDGG] = cJ[i + j * w];
  }
  if constexpr (CT >= 8) {
    constexpr int TPW = CT / 8;
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
  } else {
#pragma unroll
    for (int h = 0; h < 2; ++h)
      scratch[warp * 64 + rr * 8 + cc + h] = z3_get(acc[0], h);
    G::sync();
    constexpr int KS = 8 / CT;
    for (int idx = G::tid(); idx < CT * 64; idx += G::n()) {
      const int t = idx / 64, e = idx % 64;
      double2 v = scratch[(KS * t) * 64 + e];
      for (int k = 1; k < KS; ++k) v = cadd(v, scratch[(KS * t + k) * 64 + e]);
      const int i = (t / NTc) * 8 + e / 8, j = w + (t % NTc) * 8 + e % 8;
      sG[i + j * C::LDGG] = v;
      sG[j + i * C::LDGG] = cconj(v);
    }
  }
}

template <int W2, class G = CtaGrp>
BMPS_DEV void jac_cache_store(const double2* sG, double2* cI, double2* cJ) {
  using C = JacCfg<W2>;
  constexpr int w = W2 / 2;
  for (int idx = G::tid(); idx < w * w; idx += G::n()) {
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

// One (or more) cyclic Jacobi sweeps on the W2 x W2 Gram G, accumulating Q.
// Returns the number of rotations of the first sweep (block-uniform).
//
// Pair ordering: round R pairs column i with i ^ R -- R = 1 .. W2-1 for a full sweep,
// R = W2/2 .. W2-1 for the cross sweep between the two blocks of the panel (each pair
// exactly once either way). Rounds are taken in batches of four, R = 4 mm + r: within a
// batch every rotation stays inside a group of 8 columns (two aligned quads qa and
// qb = qa ^ mm; for mm = 0 the pairs stay inside each quad), so the W2/8 groups evolve
// independently for four rounds:
//   S. one warp per group runs the batch's rounds on the group's 8 x 8 diagonal block of
//      G (4 rotations per round on 4 lanes; the off-diagonal 2x2 pair blocks as lane
//      pairs, the rotated diagonal blocks in closed form) and accumulates the group's
//      8 x 8 unitary K_g = J_r0 .. J_r3 -- warp-synchronous, no CTA barrier inside;
//   M. after one barrier all warps apply the batch on FP64 tensor cores: the
//      off-diagonal group blocks G_pq <- K_p^H G_pq K_q (8 x 8 x 8 complex products,
//      3-product DMMA, the mirror block written from the same accumulators) and
//      Q[:, g] <- Q[:, g] K_g; second barrier.
// Two CTA barriers per four rounds, and the 2 (W2/8 - 1) / (W2/8) of the Gram-space
// work that lies outside the diagonal group blocks runs as dense 8 x 8 tiles on the
// tensor pipe instead of scalar FP64 with shared-memory round trips per round (the
// round-by-round sweep was bound by those and by two barriers per round). `work` holds
// the K_g (W2/8 x 64 complex; the idle staging buffer 0).
template <int W2>
BMPS_DEV int batch_col(int qa, int qb, int a) { return 4 * (a < 4 ? qa : qb) + (a & 3); }

BMPS_DEV double2 shfl_xor_z(double2 v, int mask) {
  return make_double2(__shfl_xor_sync(0xffffffffu, v.x, mask), __shfl_xor_sync(0xffffffffu, v.y, mask));
}

// Phase S of jac_inner for TWO column groups per warp (lanes 0..15: group ga, lanes
// 16..31: group gb): a run of rounds in which pair P of round ri joins local columns A_P
// and B_{P ^ ri}, register-resident.
//   MODE 0: A_P = P, B_P = 4 + P, rounds ri = 0..3 (quad qa against quad qb);
//   MODE 1: A_P = 2P, B_P = 2P + 1, one round (pairs (0,1)(2,3) inside each quad);
//   MODE 2: A_P = {0,1,4,5}, B_P = A_P + 2, rounds ri = 0, 1 ({0,1} x {2,3} per quad).
// Each half warp = lanes (t, u) holds the 2x2 pair blocks (rows of pair t, columns of pair
// u) of its group's 8 x 8 diagonal Gram block -- both triangles, each lane rotating its own
// copy -- and all 32 lanes = (row k, pair tk) hold the two columns of pair tk of both
// groups' K. From one round to the next only the B partners change (P ^ ri), i.e. the
// B-side entries move between lanes by XOR shuffles (inside a half warp); the rotations of a
// round are computed by the diagonal lanes (t, t) from their own registers and reach the
// other lanes through 96 bytes of shared memory per group -- the only memory round trip
// of a round. Two groups per warp because the scalar FP64 instructions cost the shared
// FP64 pipe two cycles per warp instruction however many lanes are active: with one
// group per warp, four CTAs' phase-S warps kept the pipe of their sub-partition ~85% busy
// in the cfg4 regime and every round waited for it. Returns the rotation counts
// (group ga | group gb << 16). `k_identity`: K starts as the identity (not loaded).
template <int W2, int MODE>
BMPS_DEV int jac_group_rounds(double2* sG, double2* Kga, double2* Kgb, InnerShared<W2>& is, int ga,
                              int qaa, int qba, int qab, int qbb, bool k_identity, double thr2,
                              double noise2) {
  using C = JacCfg<W2>;
  constexpr int NR = MODE == 0 ? 4 : MODE == 1 ? 1 : 2;
  const int lane = threadIdx.x & 31;
  const int hf = lane >> 4;                       // which of the warp's two groups (D role)
  const int t = (lane >> 2) & 3, u = lane & 3;
  const int k = lane & 7, tk = lane >> 3;
  const int g = ga + hf;
  const int qa = hf ? qab : qaa, qb = hf ? qbb : qba;
  auto la = [](int P) { return MODE == 0 ? P : MODE == 1 ? 2 * P : (P & 1) + 4 * (P >> 1); };
  auto lb = [](int P) { return MODE == 0 ? 4 + P : MODE == 1 ? 2 * P + 1 : (P & 1) + 4 * (P >> 1) + 2; };
  const int cAt = batch_col<W2>(qa, qb, la(t)), cAu = batch_col<W2>(qa, qb, la(u));
  double2 g00, g01, g10, g11;
  {
    const int cBt = batch_col<W2>(qa, qb, lb(t)), cBu = batch_col<W2>(qa, qb, lb(u));
    g00 = sG[cAt + cAu * C::LDGG];
    g01 = sG[cAt + cBu * C::LDGG];
    g10 = sG[cBt + cAu * C::LDGG];
    g11 = sG[cBt + cBu * C::LDGG];
  }
  double2 ka[2], kb[2];
  if (k_identity) {
#pragma unroll
    for (int z = 0; z < 2; ++z) {
      ka[z] = make_double2(k == la(tk) ? 1.0 : 0.0, 0.0);
      kb[z] = make_double2(k == lb(tk) ? 1.0 : 0.0, 0.0);
    }
  } else {
    ka[0] = Kga[k + 8 * la(tk)];
    kb[0] = Kga[k + 8 * lb(tk)];
    ka[1] = Kgb[k + 8 * la(tk)];
    kb[1] = Kgb[k + 8 * lb(tk)];
  }
  int cnt = 0;
#pragma unroll
  for (int ri = 0; ri < NR; ++ri) {
    if (ri > 0) {
      const int x = ri ^ (ri - 1);
      g01 = shfl_xor_z(g01, x);
      g10 = shfl_xor_z(g10, x << 2);
      g11 = shfl_xor_z(g11, x | (x << 2));
      kb[0] = shfl_xor_z(kb[0], x << 3);
      kb[1] = shfl_xor_z(kb[1], x << 3);
    }
    int act = 0;
    if (t == u) {
      double c;
      double2 sg;
      act = jacobi_rotation(g00.x, g11.x, g01, thr2, noise2, c, sg);
      is.c[g][t] = c;
      is.sg[g][t] = sg;
    }
    const unsigned am = __ballot_sync(0xffffffffu, act);
    __syncwarp();
    if (am) {
      cnt += __popc(am & 0xffffu) | (__popc(am >> 16) << 16);
      {
        // columns by pair u (right: J_u), then rows by pair t (left: J_t^H)
        const double cu = is.c[g][u], ct = is.c[g][t];
        const double2 su = is.sg[g][u], st = is.sg[g][t];
        const double2 r00 = cmsc(g00, cu, su, g01), r01 = cma(g01, cu, su, g00);
        const double2 r10 = cmsc(g10, cu, su, g11), r11 = cma(g11, cu, su, g10);
        g00 = cms(r00, ct, st, r10);
        g01 = cms(r01, ct, st, r11);
        g10 = cmac(r10, ct, st, r00);
        g11 = cmac(r11, ct, st, r01);
        if (act) {   // the rotated pair itself: diagonal by construction
          g00.y = 0.0;
          g11.y = 0.0;
          g01 = make_double2(0.0, 0.0);
          g10 = make_double2(0.0, 0.0);
        }
      }
#pragma unroll
      for (int z = 0; z < 2; ++z) {
        const double ck = is.c[ga + z][tk];
        const double2 sk = is.sg[ga + z][tk];
        const double2 na = cmsc(ka[z], ck, sk, kb[z]);
        kb[z] = cma(kb[z], ck, sk, ka[z]);
        ka[z] = na;
      }
    }
    __syncwarp();   // the parameters are consumed before the next round rewrites them
  }
  constexpr int xl = NR - 1;   // B partners of the last round
  {
    const int cBt = batch_col<W2>(qa, qb, lb(t ^ xl)), cBu = batch_col<W2>(qa, qb, lb(u ^ xl));
    sG[cAt + cAu * C::LDGG] = g00;
    sG[cAt + cBu * C::LDGG] = g01;
    sG[cBt + cAu * C::LDGG] = g10;
    sG[cBt + cBu * C::LDGG] = g11;
  }
  Kga[k + 8 * la(tk)] = ka[0];
  Kga[k + 8 * lb(tk ^ xl)] = kb[0];
  Kgb[k + 8 * la(tk)] = ka[1];
  Kgb[k + 8 * lb(tk ^ xl)] = kb[1];
  return cnt;
}

template <int W2, class G = CtaGrp>
BMPS_DEV int jac_inner(double2* sG, double2* sQ, double2* work, InnerShared<W2>& is, double tol,
                       double noise2, double fro, bool full, int max_inner) {
  using C = JacCfg<W2>;
  constexpr int NQ = W2 / 4, NG = W2 / 8, NW = G::kN / 32;
  constexpr int NBo = NG * (NG - 1) / 2;   // off-diagonal group blocks (p < q)
  constexpr int NT = NBo + NG * NG;        // + Q tiles (8 rows x one group)
  static_assert(2 * NW >= W2 / 8, "one warp per two column groups");
  const int tid = G::tid(), lane = tid & 31, wrp = tid >> 5;
  const int kr = lane & 3, rc = lane >> 2;
  for (int idx = tid; idx < W2 * W2; idx += G::n()) {
    const int i = idx % W2, j = idx / W2;
    sQ[i + j * C::LDG] = make_double2(i == j ? 1.0 : 0.0, 0.0);
  }
  int first = 0;
  const int nbatch = full ? NQ : NQ / 2;
  const double thr2 = (tol * fro) * (tol * fro);
  // Spare warps (W2 <= 32: half of the CTA) apply batch b's K_g to Q while the group
  // warps already run batch b + 1's rounds: Q is not read by the sweep itself, so only the
  // off-diagonal Gram blocks stay between the two barriers. K_g and the rotation counts
  // are double-buffered by batch parity.
  static_assert(NG % 2 == 0 || NG == 1, "two groups per phase-S warp");
  constexpr int NGW = (NG + 1) / 2;            // phase-S warps (two groups each)
  constexpr bool kDefer = BMPS_INNER_DEFER && NW >= 2 * NGW;
  constexpr int NSP = NW - NGW;                // warps of a deferred Q pass
  // quads of group g in batch mm: the g-th qa with qa < qa ^ mm (bit hb clear); mm = 0
  // pairs inside the quads 2g and 2g + 1
  auto group_quads = [](int mm, int g, int& qa, int& qb) {
    if (mm == 0) {
      qa = 2 * g;
      qb = 2 * g + 1;
    } else {
      const int hb = 31 - __clz(mm);
      qa = ((g >> hb) << (hb + 1)) | (g & ((1 << hb) - 1));
      qb = qa ^ mm;
    }
  };
  // Q[8 t .. 8 t + 7, group g] <- (same) K_g for tile = g + NG t (one warp)
  auto q_tile = [&](int tile, int mm, const double2* K, const int* cnt) {
    const int g = tile % NG, t8 = (tile / NG) * 8;
    if (!cnt[g]) return;
    int qa, qb;
    group_quads(mm, g, qa, qb);
    const double2* Kg = K + g * 64;
    double acc[kZ3];
#pragma unroll
    for (int z = 0; z < kZ3; ++z) acc[z] = 0.0;
#pragma unroll
    for (int sx = 0; sx < 2; ++sx)
      zmma3(acc, sQ[(t8 + rc) + batch_col<W2>(qa, qb, 4 * sx + kr) * C::LDG], Kg[(4 * sx + kr) + rc * 8]);
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h)
      sQ[(t8 + rc) + batch_col<W2>(qa, qb, 2 * kr + h) * C::LDG] = z3_get(acc, h);
  };
  for (int it = 0; it < max_inner; ++it) {
    int any = 0, nrot = 0, prev_nact = 0, prev_mm = 0;
    for (int bi = 0; bi < nbatch; ++bi) {
      BMPS_TICK(tr0);
      const int mm = full ? bi : NQ / 2 + bi;
      int* cnt = is.cnt[bi & 1];
      double2* K = work + (kDefer ? (bi & 1) * NG * 64 : 0);
      // the phase-S warps alternate between the CTA's last NGW warps and the NGW before
      // them from batch to batch, so every SM sub-partition gets its share of the scalar
      // work whatever the co-resident CTAs are doing
      const int gbase = (kDefer && (bi & 1)) ? NW - 2 * NGW : NW - NGW;
      const bool gwarp = wrp >= gbase && wrp < gbase + NGW;
      int my_act = 0;   // this warp's groups rotated in this batch (warp-uniform)
      if (gwarp) {
        // ---- S: the batch's rounds, two groups per warp ----
        const int ga = 2 * (wrp - gbase), gb = NG > 1 ? ga + 1 : ga;
        int qaa, qba, qab, qbb;
        group_quads(mm, ga, qaa, qba);
        group_quads(mm, gb, qab, qbb);
        double2* Kga = K + ga * 64;
        double2* Kgb = K + gb * 64;
        int gcnt;
        if (mm == 0) {
          // pairs inside each quad: (0,1)(2,3), then the 2 x 2 cross rounds of {0,1} x {2,3}
          gcnt = jac_group_rounds<W2, 1>(sG, Kga, Kgb, is, ga, qaa, qba, qab, qbb, true, thr2, noise2);
          __syncwarp();
          gcnt += jac_group_rounds<W2, 2>(sG, Kga, Kgb, is, ga, qaa, qba, qab, qbb, false, thr2, noise2);
        } else {
          gcnt = jac_group_rounds<W2, 0>(sG, Kga, Kgb, is, ga, qaa, qba, qab, qbb, true, thr2, noise2);
        }
        if (lane == 0) {
          cnt[ga] = gcnt & 0xffff;
          if (NG > 1) cnt[gb] = gcnt >> 16;
        }
        my_act = gcnt != 0;
      } else if (kDefer && prev_nact) {
        // the previous batch's Q update, under this batch's rounds
        const int sidx = wrp < gbase ? wrp : wrp - NGW;
        for (int tile = sidx; tile < NG * NG; tile += NSP)
          q_tile(tile, prev_mm, work + ((bi - 1) & 1) * NG * 64, is.cnt[(bi - 1) & 1]);
      }
      // one counting barrier closes phase S and tells every thread -- from the barrier
      // itself, not from shared memory -- whether any group rotated: the number of CTA
      // barriers a thread executes must never depend on a value it reads after one
      const int nact = G::count(my_act);
      BMPS_TICK(tr1);
      BMPS_ACC(4, tr0, tr1);
      any |= nact;
      if (nact) {
#pragma unroll
        for (int g = 0; g < NG; ++g) nrot += cnt[g];   // reported only, never branched on
      }
      if (nact) {
        // ---- M: the off-diagonal group blocks on the tensor cores ----
        for (int task = wrp; task < (kDefer ? NBo : NT); task += NW) {
          if (task < NBo) {
            int q = 1;
            while (q * (q + 1) / 2 <= task) ++q;
            const int p = task - q * (q - 1) / 2;
            if (!(cnt[p] | cnt[q])) continue;   // both K are the identity
            int pa, pb, qa, qb;
            group_quads(mm, p, pa, pb);
            group_quads(mm, q, qa, qb);
            const double2* Kp = K + p * 64;
            const double2* Kq = K + q * 64;
            const int row = batch_col<W2>(pa, pb, rc);
            double acc[kZ3];
#pragma unroll
            for (int z = 0; z < kZ3; ++z) acc[z] = 0.0;
            // T = G_pq K_q
#pragma unroll
            for (int sx = 0; sx < 2; ++sx)
              zmma3(acc, sG[row + batch_col<W2>(qa, qb, 4 * sx + kr) * C::LDGG], Kq[(4 * sx + kr) + rc * 8]);
            __syncwarp();
#pragma unroll
            for (int h = 0; h < 2; ++h)
              sG[row + batch_col<W2>(qa, qb, 2 * kr + h) * C::LDGG] = z3_get(acc, h);
            __syncwarp();
            // G_pq <- K_p^H T (and the mirror block)
#pragma unroll
            for (int z = 0; z < kZ3; ++z) acc[z] = 0.0;
            const int cq = batch_col<W2>(qa, qb, rc);
#pragma unroll
            for (int sx = 0; sx < 2; ++sx)
              zmma3(acc, cconj(Kp[(4 * sx + kr) + rc * 8]),
                    sG[batch_col<W2>(pa, pb, 4 * sx + kr) + cq * C::LDGG]);
            __syncwarp();
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int cc = batch_col<W2>(qa, qb, 2 * kr + h);
              const double2 v = z3_get(acc, h);
              sG[row + cc * C::LDGG] = v;
              sG[cc + row * C::LDGG] = cconj(v);
            }
          } else {
            q_tile(task - NBo, mm, K, cnt);
          }
        }
        G::sync();
      }
      prev_nact = nact;
      prev_mm = mm;
      BMPS_TICK(tr2);
      BMPS_ACC(5, tr1, tr2);
      BMPS_ACC(6, 0, 1);
    }
    if (kDefer) {
      if (prev_nact)
        for (int tile = wrp; tile < NG * NG; tile += NW)
          q_tile(tile, prev_mm, work + ((nbatch - 1) & 1) * NG * 64, is.cnt[(nbatch - 1) & 1]);
      G::sync();
    }
    if (it == 0) first = any ? max(nrot, 1) : 0;
    if (!any) break;
  }
  return first;
}

#ifndef BMPS_GRAM_RING3
#define BMPS_GRAM_RING3 1
#endif
// Slot k % 3 of the Gram pass's staging ring: buffers 0, 1, then the Q buffer.
template <int W2>
BMPS_DEV double2* jac_ring3(double2* sP, double2* sQ, int k) {
  const int m = k % 3;
  return m == 2 ? sQ : sP + m * JacCfg<W2>::BUF;
}

// One block-pair visit; returns true if any rotation was applied. If
// `resident`, the whole panel (r <= RC) already sits in buffer 0 and is
// neither loaded nor stored here. W2 = 32 streams the panel with TMA bulk
// copies (double buffered, mbarrier completion); W2 = 64 with cp.async.
// Returns 0: the pair is clean (no pair of columns fails the rotation test), 1: rotated,
// 2: deferred -- `thr2` > 0 and no pair's relative coupling |g|^2 / (a b) reaches it: the
// visit costs its Gram pass only and the caller keeps the sweep open (threshold Jacobi:
// early sweeps spend their inner sweeps and applies on the large couplings; the last
// sweeps run with thr2 = 0, so the final state is the same fixed point).
template <int W2, class G = CtaGrp>
BMPS_DEV int jac_visit(double2* X, int r, int c, int I, int J, double tol, double noise2,
                       double fro, bool full, int max_inner, bool resident, double2* sG,
                       double2* sQ, double2* sP, InnerShared<W2>& rs, JacStage& st, bool tma,
                       double2* gcache = nullptr, double thr2 = 0.0) {
  using C = JacCfg<W2>;
  BMPS_TICK(tv0);
  const int nch = (r + C::RC - 1) / C::RC;
  const bool bulk = kTmaStaging && !resident && tma;
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
    G::sync();
    jac_issue_bulk<W2>(sP, st, 0, X, r, c, 0, I, J);
    for (int k = 0; k < nch; ++k) {
      const int b = k & 1;
      if (k + 1 < nch) jac_issue_bulk<W2>(sP + (b ^ 1) * C::BUF, st, b ^ 1, X, r, c, (k + 1) * C::RC, I, J);
      jac_wait_bulk(st, b);
      G::sync();
      if (cross_gram) jac_gram_chunk_cross<W2>(gacc, sP + b * C::BUF, min(C::RC, r - k * C::RC));
      else jac_gram_chunk<W2>(gacc, sP + b * C::BUF, min(C::RC, r - k * C::RC));
      G::sync();
    }
  } else if (BMPS_GRAM_RING3 && C::NBUF == 2 && W2 * C::LDG >= C::BUF) {
    // three-slot ring (staging buffers 0, 1 and sQ, idle until the inner sweep):
    // two chunks in flight, one barrier per chunk -- the Gram pass reads the panel
    // from HBM and is latency-bound with a single chunk in flight
    G::sync();   // earlier users of the buffers are done
    jac_issue_chunk<W2>(jac_ring3<W2>(sP, sQ, 0), X, r, c, 0, I, J);
    if (nch > 1) jac_issue_chunk<W2>(jac_ring3<W2>(sP, sQ, 1), X, r, c, C::RC, I, J);
    for (int k = 0; k < nch; ++k) {
      if (k + 1 < nch) cp_async_wait<1>();
      else cp_async_wait<0>();
      G::sync();   // chunk k visible to all; every warp is done with chunk k - 1's slot
      if (k + 2 < nch) jac_issue_chunk<W2>(jac_ring3<W2>(sP, sQ, k + 2), X, r, c, (k + 2) * C::RC, I, J);
      const double2* cur = jac_ring3<W2>(sP, sQ, k);
      if (cross_gram) jac_gram_chunk_cross<W2>(gacc, cur, min(C::RC, r - k * C::RC));
      else jac_gram_chunk<W2>(gacc, cur, min(C::RC, r - k * C::RC));
    }
    G::sync();   // the Gram store reuses buffer 1 / sQ
  } else {
    G::sync();
    jac_issue_chunk<W2>(sP, X, r, c, 0, I, J);
    for (int k = 0; k < nch; ++k) {
      double2* cur = sP + (k % C::NBUF) * C::BUF;
      if (C::NBUF == 2 && k + 1 < nch) {
        jac_issue_chunk<W2>(sP + ((k + 1) % 2) * C::BUF, X, r, c, (k + 1) * C::RC, I, J);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      G::sync();
      if (cross_gram) jac_gram_chunk_cross<W2>(gacc, cur, min(C::RC, r - k * C::RC));
      else jac_gram_chunk<W2>(gacc, cur, min(C::RC, r - k * C::RC));
      G::sync();
      if (C::NBUF == 1 && k + 1 < nch) jac_issue_chunk<W2>(sP, X, r, c, (k + 1) * C::RC, I, J);
    }
  }
  BMPS_TICK(tv1);
  BMPS_ACC(0, tv0, tv1);
  // k-split partials need 8 warps x 64 complex: Q's space, or (W2 = 16) staging buffer 1,
  // whose last chunk every warp has consumed by now
  double2* scratch = W2 * C::LDG >= 512 ? sQ : sP + C::BUF;
  if (cross_gram) jac_gram_store_cross<W2, G>(gacc, sG, scratch, cI, cJ);
  else jac_gram_store<W2, G>(gacc, sG, scratch);
  G::sync();
  // staging buffer 0 is the inner sweep's workspace (the K_g), so the panel is
  // re-streamed for the apply even when it is a single chunk
  constexpr bool staged = false;
  // fast path: one parallel test of every pair the inner sweep would visit
  int need = 0;
  {
    constexpr int w = W2 / 2;
    const int npairs = full ? W2 * W2 : w * w;
    // no early exit: a warp must reach the counting barrier converged -- BAR counts
    // arrivals in units of warps, so a warp arriving in two fragments releases it early
    // (seen on the 64-column kernel: "Warp Illegal Instruction", cuda-gdb found one lane of
    // a warp a whole phase ahead of the other 31)
    for (int idx = G::tid(); idx < npairs; idx += G::n()) {
      int i, j;
      if (full) {
        i = idx % W2;
        j = idx / W2;
      } else {
        i = idx % w;
        j = w + idx / w;
      }
      if (i < j) {
        const double a = sG[i + i * C::LDGG].x, b = sG[j + j * C::LDGG].x;
        const double2 g = sG[i + j * C::LDGG];
        if (jacobi_needs(a, b, g, tol, noise2, fro)) need |= 1 | (cabs2(g) > thr2 * a * b ? 2 : 0);
      }
    }
    __syncwarp();
  }
  int needed = G::count(need & 1);
  bool deferred = false;
  if (needed && thr2 > 0.0) {          // block-uniform
    deferred = G::count(need & 2) == 0;
    if (deferred) needed = 0;
  }

  const int nrot = needed ? jac_inner<W2, G>(sG, sQ, sP, rs, tol, noise2, fro, full, max_inner) : 0;
  BMPS_TICK(tv2);
  BMPS_ACC(1, tv1, tv2);
  BMPS_ACC(3, 0, 1);
  if (gcache != nullptr && !resident && (full || nrot > 0)) jac_cache_store<W2, G>(sG, cI, cJ);
  if (C::G_IN_BUF) G::sync();  // sG (buffer 1) is read before the apply refills it
  if (nrot == 0) return deferred ? 2 : 0;
  double aacc[C::AT][kZ3];
  if (!resident) {
    if (bulk) jac_issue_bulk<W2>(sP, st, 0, X, r, c, 0, I, J);
    else jac_issue_chunk<W2>(sP, X, r, c, 0, I, J);
  }
  if (resident) {
    jac_apply_mma<W2>(aacc, sP, sQ);
    G::sync();
    jac_apply_writeback<W2>(aacc, sP);
    G::sync();
    return 1;
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
          G::sync();
        }
        jac_issue_bulk<W2>(sP + (b ^ 1) * C::BUF, st, b ^ 1, X, r, c, row1, I, J);
      }
      if (!staged) jac_wait_bulk(st, b);
      G::sync();
      jac_apply_mma<W2>(aacc, cur, sQ);
      G::sync();
      jac_apply_writeback<W2>(aacc, cur);
      G::sync();
      jac_store_bulk<W2>(cur, X, r, c, k * C::RC, I, J);
    }
    jac_flush_bulk();
    return 1;
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
    G::sync();
    jac_apply_mma<W2>(aacc, cur, sQ);
    jac_apply_store_global<W2>(aacc, X, r, c, k * C::RC, I, J);
    G::sync();  // every warp is done reading `cur` before it is refilled
    if (C::NBUF == 1 && !staged && k + 1 < nch) jac_issue_chunk<W2>(sP, X, r, c, (k + 1) * C::RC, I, J);
  }
  BMPS_TICK(tv3);
  BMPS_ACC(2, tv2, tv3);
  return 1;
}

template <int W2, class G = CtaGrp>
BMPS_DEV void jac_load_resident(double2* sP, const double2* X, int r, int c) {
  jac_issue_chunk<W2>(sP, X, r, c, 0, 0, 1);
  cp_async_wait<0>();
  G::sync();
}

template <int W2>
__global__ void __launch_bounds__(256, (W2 <= 32) ? BMPS_JAC_MINB : 1) jacobi_kernel(JacArgs args) {
  using C = JacCfg<W2>;
  extern __shared__ __align__(16) double2 jsm[];
  double2* sQ = jsm;
  double2* sP = sQ + W2 * C::LDG;
  double2* sG = C::G_IN_BUF ? sP + C::BUF : sP + C::NBUF * C::BUF;
  __shared__ InnerShared<W2> rs;
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
    const bool resident = false;   // (the inner sweep needs staging buffer 0)
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
  __shared__ InnerShared<W2> rs;
  __shared__ int s_item, s_v;
  __shared__ unsigned s_round;
  __shared__ unsigned long long jbar[2];
  JacStage st{jbar, 0u};
  stage_init(jbar);
  constexpr int w = W2 / 2;
  const int nitems = args.nitems;
  int cursor = blockIdx.x % nitems;
  volatile int* active = args.active;
  // The exit test is taken by one thread and broadcast with the claim (s_item = -2): a
  // per-thread `while (*active > 0)` let the warps of a CTA disagree when the last item
  // retired between their reads -- the warps that stayed re-ran the previous claim from
  // the stale shared words while warp 0 had left (found by the -DBMPS_DEBUG_CHECKS build:
  // "claimed item already retired", tools/debug_stress.py).
  for (;;) {
    BMPS_TICK(dc0);
    // warp 0 probes 32 items per round trip (lane l: item cursor + base + l), ballots
    // the ones with unclaimed visits and tries them in probe order; a claim used to
    // scan ~10 exhausted items one dependent load at a time (~7k cycles per visit)
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      int got = -1, gv = 0;
      unsigned grnd = 0;
      for (int base = 0; base < nitems && got < 0; base += 32) {
        const int probe = base + lane;
        const int i = (cursor + probe) % nitems;
        WS_ACC(0, 14, 0, min(32, nitems - base));   // probes (timer builds)
        bool cand = false;
        unsigned nbv = 0;
        if (probe < nitems && !((volatile ItemMeta*)args.meta)[i].conv) {
          int nb = (args.meta[i].c + w - 1) / w;
          nb += nb & 1;
          nbv = (unsigned)(nb / 2);
          const unsigned long long peek = *((volatile unsigned long long*)&args.sched[i].ticket);
          cand = (unsigned)(peek & 0xffffffffull) < nbv;
        }
        unsigned mask = __ballot_sync(0xffffffffu, cand);
        while (mask) {
          const int l = __ffs(mask) - 1;
          int ok = 0;
          unsigned long long old = 0;
          if (lane == l) {
            old = atomicAdd(&args.sched[i].ticket, 1ull);
            ok = (unsigned)(old & 0xffffffffull) < nbv;
          }
          if (__shfl_sync(0xffffffffu, ok, l)) {
            got = __shfl_sync(0xffffffffu, i, l);
            old = __shfl_sync(0xffffffffu, old, l);
            gv = (int)(old & 0xffffffffull);
            grnd = (unsigned)(old >> 32);
            break;
          }
          mask &= mask - 1;
        }
      }
      if (got >= 0) cursor = got;
      if (lane == 0) {
        s_item = (got < 0 && *active <= 0) ? -2 : got;
        s_v = gv;
        s_round = grnd;
        __threadfence();
      }
    }
    __syncthreads();
    const int i = s_item;
    if (i == -2) break;   // every item has converged (block-uniform)
    BMPS_TICK(dc1);
    if (i >= 0) { WS_ACC(0, 10, dc0, dc1); WS_ACC(0, 11, 0, 1); } else { WS_ACC(0, 12, dc0, dc1); }
    if (i < 0) {
      if (threadIdx.x == 0) __nanosleep(BMPS_CLAIM_SLEEP_NS);
      __syncthreads();
      cursor = (cursor + 1) % nitems;
      continue;
    }
    const int v = s_v;
    const unsigned rnd = s_round;
    ItemMeta* m = args.meta + i;
#ifdef BMPS_DEBUG_CHECKS
    if (!(i < nitems && !m->conv) && (threadIdx.x & 31) == 0)
      printf("claim check: block %d warp %d i %d nitems %d conv %d v %d rnd %u ticket %llx done %d c %d\n",
             (int)blockIdx.x, (int)(threadIdx.x >> 5), i, nitems, i < nitems ? m->conv : -1, v, rnd,
             i < nitems ? args.sched[i].ticket : 0ull, i < nitems ? args.sched[i].done : -1,
             i < nitems ? m->c : -1);
#endif
    BMPS_CHECK(i < nitems && !m->conv);
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
      const bool resident = false;   // (the inner sweep needs staging buffer 0)
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
    if (skip) { WS_ACC(0, 13, 0, 1); }
    const double thr = sweep < args.thr_a_sweeps ? args.thr_a : sweep < args.thr_b_sweeps ? args.thr_b : 0.0;
    const int ret = skip ? 0
                         : jac_visit<W2>(X, r, c, I, J, tol, noise2, fro, rho == 0, args.max_inner,
                                         false, sG, sQ, sP, rs, st, args.tma, gc, thr * thr);
    const bool dirty = ret != 0;   // rotated, or deferred by the sweep's threshold: not converged
    if (last_rot && !skip && threadIdx.x == 0) {
      if (ret == 1) {
        last_rot[I] = (int)rnd;
        last_rot[J] = (int)rnd;
        *last_chk = -1;
      } else if (ret == 2) {
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
      jac_debug_mark(sc, v, rnd, nb / 2);
      __threadfence();
      const int d = atomicAdd(&sc->done, 1);
      if (d == nb / 2 - 1) {
        // last visit of the round: open the next round (or finish the item)
        jac_debug_close(sc, rnd, nb / 2);
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

// ---------------------------------------------------------------------------
// Visit claiming and round bookkeeping shared by the cluster kernel.

// Round bookkeeping of a finished visit (one thread): the pair log for exact
// skipping, the item's dirty flag, and -- for the last visit of a round -- the
// opening of the next round or the end of the item (as in jacobi_dynamic_kernel).
template <int W2>
BMPS_DEV void jac_complete(const JacArgs& args, int i, unsigned rnd, int I, int J, bool dirty,
                           bool skipped, int v) {
  constexpr int w = W2 / 2;
  ItemMeta* m = args.meta + i;
  int nb = (m->c + w - 1) / w;
  nb += nb & 1;
  const int rounds = nb - 1;
  const int sweep = (int)(rnd / (unsigned)rounds), rho = (int)(rnd % (unsigned)rounds);
  JacSched* sc = args.sched + i;
  if (args.pairlog && !skipped) {
    int* last_rot = args.pairlog + (size_t)i * (args.nbcap + args.nbcap * args.nbcap);
    int* last_chk = last_rot + args.nbcap + I * args.nbcap + J;
    if (dirty) {
      last_rot[I] = (int)rnd;
      last_rot[J] = (int)rnd;
      *last_chk = -1;
    } else {
      *last_chk = (int)rnd;
    }
  }
  if (dirty) atomicOr(&sc->dirty, 1);
  if (v >= 0) jac_debug_mark(sc, v, rnd, nb / 2);
  __threadfence();
  const int d = atomicAdd(&sc->done, 1);
  if (d == nb / 2 - 1) {
    if (v >= 0) jac_debug_close(sc, rnd, nb / 2);
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

// Claim the next visit (one thread). Visits whose outcome is known (pair checked
// clean, neither block rotated since) are completed on the spot and the claim
// goes on. Returns the item (v, rnd set), -1 if nothing is claimable right now,
// -2 once every item has converged.
template <int W2>
BMPS_DEV int ws_claim(const JacArgs& args, int& cursor, int& v_out, unsigned& rnd_out) {
  constexpr int w = W2 / 2;
  const int nitems = args.nitems;
  for (;;) {
    if (*((volatile int*)args.active) <= 0) return -2;
    int got = -1;
    for (int probe = 0; probe < nitems; ++probe) {
      const int i = (cursor + probe) % nitems;
      JacSched* sc = args.sched + i;
      if (((volatile ItemMeta*)args.meta)[i].conv) continue;
      const int c = args.meta[i].c;
      int nb = (c + w - 1) / w;
      nb += nb & 1;
      const unsigned nbv = (unsigned)(nb / 2);
      const unsigned long long peek = *((volatile unsigned long long*)&sc->ticket);
      if ((unsigned)(peek & 0xffffffffull) >= nbv) continue;
      const unsigned long long old = atomicAdd(&sc->ticket, 1ull);
      const unsigned v = (unsigned)(old & 0xffffffffull);
      if (v >= nbv) continue;
      got = i;
      v_out = (int)v;
      rnd_out = (unsigned)(old >> 32);
      cursor = i;
      break;
    }
    __threadfence();
    if (got < 0) return -1;
    if (args.pairlog) {
      const int c = args.meta[got].c;
      int nb = (c + w - 1) / w;
      nb += nb & 1;
      const int rounds = nb - 1, rho = (int)(rnd_out % (unsigned)rounds);
      if (nb > 2 && rho > 0) {
        int I, J;
        tourney_pair(nb, rho, v_out, I, J);
        const int* last_rot = args.pairlog + (size_t)got * (args.nbcap + args.nbcap * args.nbcap);
        const int lc = *((volatile const int*)(last_rot + args.nbcap + I * args.nbcap + J));
        if (lc >= 0 && *((volatile const int*)(last_rot + I)) < lc &&
            *((volatile const int*)(last_rot + J)) < lc) {
          jac_complete<W2>(args, got, rnd_out, I, J, false, true, (int)v_out);
          continue;
        }
      }
    }
    return got;
  }
}

// ---------------------------------------------------------------------------
// Row-split cluster kernel (small batches: one circuit's brick layer).
//
// With few items the dynamic kernel cannot fill the GPU, and an item's ~9 x 31
// rounds run back to back at the latency of one visit (16 chunks of Gram pass,
// 16 inner rounds, 16 chunks of apply on one CTA). Here a thread-block cluster
// of CS CTAs works one visit: CTA k streams rows [k*rs, (k+1)*rs) of the panel,
// forms its partial Gram, the partials are summed through distributed shared
// memory in rank order (every CTA gets the bit-identical G), every CTA runs the
// same inner sweep (same G, same code -> the same Q, no broadcast), and applies
// Q to its own rows. Claiming, exact skipping and round bookkeeping are those of
// the dynamic kernel (rank 0 of the cluster).
template <int W2>
struct ClCfg {
  using C = JacCfg<W2>;
  static constexpr int PSZ = W2 * C::LDGG;   // partial Gram buffer
  static constexpr size_t kSmem = (size_t)(W2 * C::LDG + C::NBUF * C::BUF + PSZ) * sizeof(double2);
};

// Partial Gram over rows [row0, row1) (chunk-aligned), three-slot ring as in jac_visit.
template <int W2>
BMPS_DEV void cl_gram_rows(double (&gacc)[JacCfg<W2>::GT + 1][kZ3], const double2* X, int r, int c,
                           int I, int J, bool cross, double2* sP, double2* sQ, int row0, int row1) {
  using C = JacCfg<W2>;
  const int nch = (row1 - row0 + C::RC - 1) / C::RC;
#pragma unroll
  for (int u = 0; u < C::GT + 1; ++u)
#pragma unroll
    for (int q = 0; q < kZ3; ++q) gacc[u][q] = 0.0;
  __syncthreads();
  if (nch > 0) jac_issue_chunk<W2>(jac_ring3<W2>(sP, sQ, 0), X, r, c, row0, I, J);
  if (nch > 1) jac_issue_chunk<W2>(jac_ring3<W2>(sP, sQ, 1), X, r, c, row0 + C::RC, I, J);
  for (int k = 0; k < nch; ++k) {
    if (k + 1 < nch) cp_async_wait<1>();
    else cp_async_wait<0>();
    __syncthreads();
    if (k + 2 < nch)
      jac_issue_chunk<W2>(jac_ring3<W2>(sP, sQ, k + 2), X, r, c, row0 + (k + 2) * C::RC, I, J);
    const double2* cur = jac_ring3<W2>(sP, sQ, k);
    const int nrows = min(C::RC, row1 - (row0 + k * C::RC));
    if (cross) jac_gram_chunk_cross<W2>(gacc, cur, nrows);
    else jac_gram_chunk<W2>(gacc, cur, nrows);
  }
  __syncthreads();
}

// P <- P Q over rows [row0, row1) (chunk-aligned), cp.async double buffering.
template <int W2>
BMPS_DEV void cl_apply_rows(double2* X, int r, int c, int I, int J, const double2* sQ, double2* sP,
                            int row0, int row1) {
  using C = JacCfg<W2>;
  const int nch = (row1 - row0 + C::RC - 1) / C::RC;
  if (nch <= 0) return;
  double aacc[C::AT][kZ3];
  jac_issue_chunk<W2>(sP, X, r, c, row0, I, J);
  for (int k = 0; k < nch; ++k) {
    double2* cur = sP + (k & 1) * C::BUF;
    if (k + 1 < nch) {
      jac_issue_chunk<W2>(sP + ((k + 1) & 1) * C::BUF, X, r, c, row0 + (k + 1) * C::RC, I, J);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    jac_apply_mma<W2>(aacc, cur, sQ);
    jac_apply_store_global<W2>(aacc, X, r, c, row0 + k * C::RC, I, J);
    __syncthreads();
  }
}

template <int W2, int CS>
__global__ void __launch_bounds__(256, 3) jacobi_cluster_kernel(JacArgs args) {
  namespace cg = cooperative_groups;
  using C = JacCfg<W2>;
  using CC = ClCfg<W2>;
  constexpr int w = W2 / 2;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  extern __shared__ __align__(16) double2 jsm[];
  double2* sQ = jsm;
  double2* sP = sQ + W2 * C::LDG;
  double2* sG = C::G_IN_BUF ? sP + C::BUF : nullptr;   // W2 = 32 only
  double2* sPart = sP + C::NBUF * C::BUF;
  __shared__ InnerShared<W2> rs;
  __shared__ int c_item, c_v;
  __shared__ unsigned c_round;
  __shared__ unsigned long long jbar[2];
  JacStage st{jbar, 0u};
  const double2* rPart[CS];
#pragma unroll
  for (int k = 0; k < CS; ++k) rPart[k] = cl.map_shared_rank(sPart, k);
  const int* r_item = cl.map_shared_rank(&c_item, 0);
  const int* r_v = cl.map_shared_rank(&c_v, 0);
  const unsigned* r_round = cl.map_shared_rank(&c_round, 0);
  const int tid = threadIdx.x;
  int cursor = (int)(blockIdx.x / CS) % args.nitems;
  for (;;) {
    if (rank == 0 && tid == 0) {
      int v = 0;
      unsigned rnd = 0;
      int it;
      while ((it = ws_claim<W2>(args, cursor, v, rnd)) == -1) {
        __nanosleep(1000);
        cursor = (cursor + 1) % args.nitems;
      }
      c_item = it;
      c_v = v;
      c_round = rnd;
    }
    cl.sync();
    const int i = *r_item, v = *r_v;
    const unsigned rnd = *r_round;
    cl.sync();   // rank 0 may overwrite the claim only after every CTA has read it
    if (i < 0) break;
    ItemMeta* m = args.meta + i;
    const int r = m->jrows, c = m->c;
    double2* X = (m->dq ? args.Z : m->precond ? args.Y : args.X) + (size_t)i * args.mat_stride;
    int nb = (c + w - 1) / w;
    nb += nb & 1;
    const double tol = args.tol_factor * sqrt((double)r) * kEps;
    const double noise2 = kNoiseRel * kNoiseRel * m->fro2;
    const double fro = sqrt(m->fro2);
    if (nb == 2) {
      // single panel: rank 0 iterates the item alone (small; the others move on)
      if (rank == 0) {
        const bool resident = false;   // (the inner sweep needs staging buffer 0)
        if (resident) jac_load_resident<W2>(sP, X, r, c);
        int sweep = 0;
        bool clean = false;
        for (; sweep < args.max_sweeps; ++sweep) {
          if (!jac_visit<W2>(X, r, c, 0, 1, tol, noise2, fro, true, 64, resident, sG, sQ, sP, rs, st, false)) {
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
        if (tid == 0) {
          m->sweeps = sweep;
          if (!clean) m->status = BMPS_S_SVD_FAILED;
          __threadfence();
          m->conv = 1;
          atomicSub(args.active, 1);
        }
        __syncthreads();
      }
      continue;
    }
    const int rounds = nb - 1;
    const int rho = (int)(rnd % (unsigned)rounds);
    int I, J;
    tourney_pair(nb, rho, v, I, J);
    const bool full = rho == 0;
    double2* gc = args.gcache ? args.gcache + (size_t)i * args.gcache_stride : nullptr;
    double2* cI = gc ? gc + (size_t)I * w * w : nullptr;
    double2* cJ = gc ? gc + (size_t)J * w * w : nullptr;
    const bool cross = gc != nullptr && !full;
    // chunk-aligned row range of this rank
    const int rs_rows = ((r + C::RC - 1) / C::RC + CS - 1) / CS * C::RC;
    const int row0 = min(r, rank * rs_rows), row1 = min(r, row0 + rs_rows);
    double gacc[C::GT + 1][kZ3];
    cl_gram_rows<W2>(gacc, X, r, c, I, J, cross, sP, sQ, row0, row1);
    if (cross) jac_gram_store_cross<W2>(gacc, sPart, sQ, cI, cJ);
    else jac_gram_store<W2>(gacc, sPart, sQ);
    cl.sync();   // every rank's partial Gram is in place
    for (int idx = tid; idx < W2 * W2; idx += blockDim.x) {
      const int a = idx % W2, b2 = idx / W2;
      const int e = a + b2 * C::LDGG;
      if (cross && ((a < w) == (b2 < w))) {
        sG[e] = sPart[e];        // rotated intra-block Gram from the cache (same in every rank)
      } else {
        double2 acc = rPart[0][e];
#pragma unroll
        for (int k = 1; k < CS; ++k) acc = cadd(acc, rPart[k][e]);
        sG[e] = acc;
      }
    }
    cl.sync();   // partials consumed (the next visit rewrites them); sG complete in every rank
    int need = 0;
    {
      const int npairs = full ? W2 * W2 : w * w;
      for (int idx = tid; idx < npairs; idx += blockDim.x) {   // no early exit, see jac_visit
        int a, b2;
        if (full) {
          a = idx % W2;
          b2 = idx / W2;
        } else {
          a = idx % w;
          b2 = w + idx / w;
        }
        need |= (a < b2) && jacobi_needs(sG[a + a * C::LDGG].x, sG[b2 + b2 * C::LDGG].x,
                                         sG[a + b2 * C::LDGG], tol, noise2, fro);
      }
      __syncwarp();
    }
    const int nrot = __syncthreads_or(need) ? jac_inner<W2>(sG, sQ, sP, rs, tol, noise2, fro, full, args.max_inner)
                                            : 0;
    if (rank == 0 && gc != nullptr && (full || nrot > 0)) jac_cache_store<W2>(sG, cI, cJ);
    __syncthreads();   // sG (staging buffer 1) is read before the apply refills it
    if (nrot > 0) cl_apply_rows<W2>(X, r, c, I, J, sQ, sP, row0, row1);
    __threadfence();
    cl.sync();         // every rank's panel rows (and rank 0's cache) are written
    if (rank == 0 && tid == 0) jac_complete<W2>(args, i, rnd, I, J, nrot > 0, false, v);
  }
}

}  // namespace bmps
