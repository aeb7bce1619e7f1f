// Two-site update kernels: theta contraction (K2), block one-sided Jacobi SVD
// (K3), truncation + split (K4) and in-order stats (mps.py:94-136, 82-84).
#pragma once
#include <cooperative_groups.h>

#include "bmps_gemm.cuh"
#include "bmps_qr.cuh"

namespace bmps {

// ---------------------------------------------------------------------------
// K2 theta: M[(l,a),(b,r)] = sum_{s,t} G[2a+b][2s+t] * C[(l,s),(t,r)] with
// C = (lam_l * Gamma_q * lam_m) (2dl x dm) @ (Gamma_{q+1} * lam_r) (dm x 2dr)
// (mps.py:101-114). The GEMM runs on DMMA with GEMM columns interleaved as
// j = 2r + t so each 64x64 tile holds all four (s,t) entries of its 32x32
// (l,r) block; the 4x4 gate is applied in the epilogue. The result is written
// column-major as X0 = M (orient 0, dl >= dr) or X0 = M^H (orient 1) so the
// SVD always sees rows >= cols, into both the preserved copy M0 and the
// Jacobi working copy X.
// ---------------------------------------------------------------------------
struct ThetaOp {
  static constexpr bool kAKMajor = true;
  static constexpr bool kBKMajor = false;
  StateView sv;
  const int* items;
  const double2* ga;
  const double2* gb;
  const double* ll;
  const double* lm;
  const double* lr;
  int cap, dl, dm, dr;
  BMPS_DEV bool begin(int item, int& M, int& N, int& K) {
    const int s = items[2 * item], q = items[2 * item + 1];
    const int* d = sv.dimv(s);
    dl = d[q];
    dm = d[q + 1];
    dr = d[q + 2];
    cap = sv.cap;
    ga = sv.site(s, q);
    gb = sv.site(s, q + 1);
    ll = sv.bond(s, q);
    lm = sv.bond(s, q + 1);
    lr = sv.bond(s, q + 2);
    M = 2 * dl;
    N = 2 * dr;
    K = dm;
    return true;
  }
  BMPS_DEV double2 a(int i, int k) const {
    return cscale(ga[(size_t)i * cap + k], ll[i >> 1] * lm[k]);
  }
  BMPS_DEV double2 b(int k, int j) const {
    const int r = j >> 1, t = j & 1;
    return cscale(gb[(size_t)(2 * k + t) * cap + r], lr[r]);
  }
};

constexpr int kThetaLdc = 65;
constexpr size_t kThetaSmem = (size_t)kTile * kThetaLdc * sizeof(double2);

__global__ void __launch_bounds__(256, BMPS_GEMM_MINB) theta_kernel(StateView sv, const int* items,
                                                    const double2* gates, ItemMeta* meta,
                                                    double2* M0, double2* X, size_t mat_stride,
                                                    int tiles_per_dim, int qr_min_cols,
                                                    int double_qr, int col_sort,
                                                    double* fro_part, int fro_stride) {
  __shared__ __align__(16) double2 sA[kKC][kLds];
  __shared__ __align__(16) double2 sB[kKC][kLds];
  __shared__ double2 sG[16];
  extern __shared__ __align__(16) double2 sC[];  // 64 x kThetaLdc
  const int item = blockIdx.y;
  ThetaOp op;
  op.sv = sv;
  op.items = items;
  int M, N, K;
  op.begin(item, M, N, K);
  const int dl = op.dl, dm = op.dm, dr = op.dr;
  BMPS_CHECK(items[2 * item + 1] >= 0 && items[2 * item + 1] + 2 <= sv.n && dl >= 1 && dm >= 1 &&
             dr >= 1 && dl <= sv.cap && dm <= sv.cap && dr <= sv.cap);
  const int orient = dl >= dr ? 0 : 1;
  const int R = orient == 0 ? 2 * dl : 2 * dr;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ItemMeta* m = meta + item;
    m->r = R;
    m->c = orient == 0 ? 2 * dr : 2 * dl;
    m->orient = orient;
    m->dl = dl;
    m->dm = dm;
    m->dr = dr;
    const int c = orient == 0 ? 2 * dr : 2 * dl;
    m->precond = c >= qr_min_cols ? 1 : 0;
    m->dq = m->precond && double_qr ? 1 : 0;
    m->jrows = m->precond ? c : R;
  }
  const int tm = blockIdx.x / tiles_per_dim, tn = blockIdx.x % tiles_per_dim;
  const int m0 = tm * kTile, n0 = tn * kTile;
  if (m0 >= M || n0 >= N) {
    if (threadIdx.x == 0) fro_part[(size_t)item * fro_stride + blockIdx.x] = 0.0;
    return;
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;
  if (tid < 16) sG[tid] = gates[(size_t)item * 16 + tid];
  double acc[4][2][4];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[mi][ni][q] = 0.0;
  gemm_mainloop(op, acc, sA, sB, M, N, K, m0, n0, tid);
  {
    const int rr = lane >> 2, cc = (lane & 3) * 2;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int i = wm * 32 + mi * 8 + rr, j = wn * 16 + ni * 8 + cc + h;
          sC[i * kThetaLdc + j] = make_double2(acc[mi][ni][h], acc[mi][ni][2 + h]);
        }
  }
  __syncthreads();
  double2* m0p = M0 + (size_t)item * mat_stride;
  double2* xp = X + (size_t)item * mat_stride;
  // double-QR items get their working copy from dq_colsort_kernel (columns in
  // descending-norm order), the others straight from here
  const int ccols = orient == 0 ? 2 * dr : 2 * dl;
  const bool write_x = !(col_sort && double_qr && ccols >= qr_min_cols);
  double fro = 0.0;
  for (int idx = tid; idx < 32 * 32; idx += 256) {
    // orient 0 writes (2l+a) contiguous -> l fastest; orient 1 writes (b*dr+r) -> r fastest
    const int lloc = orient == 0 ? (idx & 31) : (idx >> 5);
    const int rloc = orient == 0 ? (idx >> 5) : (idx & 31);
    const int l = (m0 >> 1) + lloc, r = (n0 >> 1) + rloc;
    if (l >= dl || r >= dr) continue;
    double2 c4[4];
#pragma unroll
    for (int st = 0; st < 4; ++st) c4[st] = sC[(2 * lloc + (st >> 1)) * kThetaLdc + 2 * rloc + (st & 1)];
#pragma unroll
    for (int ab = 0; ab < 4; ++ab) {
      double2 v = make_double2(0.0, 0.0);
#pragma unroll
      for (int st = 0; st < 4; ++st) v = cfma(sG[ab * 4 + st], c4[st], v);
      const int a = ab >> 1, b = ab & 1;
      size_t off;
      if (orient == 0) {
        off = (size_t)(2 * l + a) + (size_t)(b * dr + r) * R;
      } else {
        off = (size_t)(b * dr + r) + (size_t)(2 * l + a) * R;
        v = cconj(v);
      }
      m0p[off] = v;
      if (write_x) xp[off] = v;
      fro += cabs2(v);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) fro += __shfl_xor_sync(0xffffffffu, fro, o);
  __shared__ double sfro[8];
  if (lane == 0) sfro[warp] = fro;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w8 = 0; w8 < 8; ++w8) t += sfro[w8];
    fro_part[(size_t)item * fro_stride + blockIdx.x] = t;
  }
}

// ||M||_F^2 = sum of theta's per-CTA partials in a fixed order (lane-strided
// sums, then a fixed shuffle tree), so every later decision that reads it (the
// Jacobi noise floor, the zero-sigma threshold of the split) is run-to-run
// bit-identical -- an atomicAdd over CTAs would depend on their completion order.
__global__ void fro_reduce_kernel(ItemMeta* meta, const double* fro_part, int fro_stride, int ntiles) {
  const int item = blockIdx.x, lane = threadIdx.x;
  const double* p = fro_part + (size_t)item * fro_stride;
  double t = 0.0;
  for (int k = lane; k < ntiles; k += 32) t += p[k];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (lane == 0) meta[item].fro2 = t;
}

}  // namespace bmps

#include "bmps_jacobi.cuh"

namespace bmps {

// End of a round-mode sweep: converge clean items, count the rest.
__global__ void sweep_end_kernel(ItemMeta* meta, int nitems, int max_sweeps, int* unconverged) {
  const int item = blockIdx.x * blockDim.x + threadIdx.x;
  if (item >= nitems) return;
  ItemMeta* m = meta + item;
  if (m->conv) return;
  if (!m->flag) {
    m->conv = 1;
    return;
  }
  m->flag = 0;
  m->sweeps += 1;
  if (m->sweeps >= max_sweeps) {
    m->conv = 1;
    m->status = BMPS_S_SVD_FAILED;
    return;
  }
  atomicAdd(unconverged, 1);
}

// ---------------------------------------------------------------------------
// K4a finalize: sigma_j = ||x_j||, sort descending, keep count (mps.py:43-49),
// discarded weight (mps.py:121-122), renormalised lambda (mps.py:123-127), new
// bond dim, and the side of the split read straight from X (U or V^H rows).
// ---------------------------------------------------------------------------
constexpr int kMaxCols = 2048;

__global__ void __launch_bounds__(512) finalize_kernel(StateView sv, const int* items,
                                                       ItemMeta* meta, const double2* X,
                                                       const double2* Yq,
                                                       size_t mat_stride, double* sig_ws,
                                                       int* perm_ws, int sig_stride,
                                                       double cutoff, int max_bond, int relative,
                                                       bmps_update_record* log,
                                                       const int* log_index) {
  __shared__ double ssig[kMaxCols];
  __shared__ int sidx[kMaxCols];
  __shared__ int s_keep;
  __shared__ double s_norm;
  const int item = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  ItemMeta* m = meta + item;
  const int r = m->jrows, c = m->c, dl = m->dl, dr = m->dr;
  const int side = m->orient ^ m->precond;   // 0: primary vectors -> Gamma_q, 1: -> Gamma_{q+1}
  const int s = items[2 * item], q = items[2 * item + 1];
  const double2* x = (m->precond || m->msel ? Yq : X) + (size_t)item * mat_stride;
  const bool presorted = m->msel != 0;  // double-QR: sigma already sorted by dq_sort_kernel
  int P2 = 1;
  while (P2 < c) P2 <<= 1;
  if (presorted) {
    const double* sg = sig_ws + (size_t)item * sig_stride;
    for (int j = tid; j < P2; j += blockDim.x) {
      ssig[j] = j < c ? sg[j] : -1.0;
      sidx[j] = j;
    }
  }
  for (int j = presorted ? P2 : warp; j < P2; j += 16) {
    double acc = 0.0;
    if (j < c)
      for (int i = lane; i < r; i += 32) acc += cabs2(x[(size_t)i + (size_t)j * r]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      ssig[j] = j < c ? sqrt(acc) : -1.0;
      sidx[j] = j;
    }
  }
  __syncthreads();
  // bitonic sort: descending sigma, ties by ascending column index
  for (int k = 2; k <= (presorted ? 1 : P2); k <<= 1) {
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      for (int t = tid; t < P2; t += blockDim.x) {
        const int u = t ^ jj;
        if (u > t) {
          const double st = ssig[t], su = ssig[u];
          const int it = sidx[t], iu = sidx[u];
          const bool u_first = su > st || (su == st && iu < it);
          const bool t_first = st > su || (st == su && it < iu);
          const bool swap = ((t & k) == 0) ? u_first : t_first;
          if (swap) {
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
    int status = m->status;
    if (!isfinite(ssig[0])) status = BMPS_S_SVD_FAILED;
    if (keep > sv.cap) {
      keep = sv.cap;
      if (!status) status = BMPS_S_CAPACITY;
    }
    // robustness of the keep decision: distance of the nearest singular value that
    // could move keep from the threshold, and the gap at the truncation boundary
    double margin = CUDART_INF, gap = CUDART_INF;
    const double s0 = ssig[0];
    if (cutoff > 0.0 && s0 > 0.0) {
      const double thr = cutoff * (relative ? s0 : 1.0);
      const int K = max_bond > 0 ? min(c, max_bond) : c;
      double mn = CUDART_INF;
      for (int k = 0; k < K; ++k) mn = fmin(mn, fabs(ssig[k] - thr));
      margin = mn / s0;
    }
    if (keep < c && s0 > 0.0) gap = (ssig[keep - 1] - ssig[keep]) / s0;
    double err = 0.0, nrm2 = 0.0;
    for (int k = keep; k < c; ++k) err += ssig[k] * ssig[k];
    for (int k = 0; k < keep; ++k) nrm2 += ssig[k] * ssig[k];
    const double nrm = sqrt(nrm2);
    if (nrm == 0.0 && !status) status = BMPS_S_ALL_TRUNCATED;
    BMPS_CHECK(keep >= 1 && keep <= sv.cap && keep <= c);
    m->keep = keep;
    m->err = err;
    m->norm = nrm;
    m->status = status;
    s_keep = status ? 0 : keep;
    s_norm = nrm;
    if (!status) sv.dimv(s)[q + 1] = keep;
    bmps_update_record rec;
    rec.err = err;
    rec.dl = dl;
    rec.dm = m->dm;
    rec.dr = dr;
    rec.keep = keep;
    rec.status = status;
    rec.site = q;
    rec.margin = margin;
    rec.gap = gap;
    log[log_index[item]] = rec;
  }
  __syncthreads();
  const int keep = s_keep;
  if (keep == 0) return;  // failure: leave the state untouched (host raises)
  const double nrm = s_norm;
  const double zero_sig = kNoiseRel * sqrt(m->fro2);
  double* sig_out = sig_ws + (size_t)item * sig_stride;
  int* perm_out = perm_ws + (size_t)item * sig_stride;
  double* lam_new = sv.bond(s, q + 1);
  for (int k = tid; k < keep; k += blockDim.x) {
    sig_out[k] = ssig[k];
    perm_out[k] = sidx[k];
    lam_new[k] = ssig[k] / nrm;
  }
  const int cap = sv.cap;
  if (side == 0) {
    // Gamma_q[l,a,k] = pinv(lam_l[l]) * x[2l+a, perm k] / sigma_k   (mps.py:131,133)
    double2* gq = sv.site(s, q);
    const double* ll = sv.bond(s, q);
    const int rows = 2 * dl;
    for (int idx = tid; idx < rows * keep; idx += blockDim.x) {
      const int k = idx % keep, i = idx / keep;
      const double sk = ssig[k];
      const double f = sk > zero_sig ? pinv(ll[i >> 1]) / sk : 0.0;
      gq[(size_t)i * cap + k] = cscale(x[(size_t)i + (size_t)sidx[k] * r], f);
    }
  } else {
    // Gamma_{q+1}[k,b,r] = conj(x[b*dr+r, perm k]) / sigma_k * pinv(lam_r[r])  (mps.py:132,134)
    double2* gb = sv.site(s, q + 1);
    const double* lr = sv.bond(s, q + 2);
    const int cols = 2 * dr;
    for (int idx = tid; idx < keep * cols; idx += blockDim.x) {
      const int jcol = idx % cols, k = idx / cols;
      const int b = jcol / dr, rr = jcol % dr;
      const double sk = ssig[k];
      const double f = sk > zero_sig ? pinv(lr[rr]) / sk : 0.0;
      gb[(size_t)(2 * k + b) * cap + rr] = cscale(cconj(x[(size_t)jcol + (size_t)sidx[k] * r]), f);
    }
  }
}

// ---------------------------------------------------------------------------
// K4b split GEMM: the other singular vectors W = M0^H Y Sigma^-1 with
// Y = X[:, perm] / sigma (i.e. W[:,k] = M0^H X[:,perm k] / sigma_k^2), written
// into Gamma_{q+1} (orient 0, as V^H rows) or Gamma_q (orient 1, as U columns)
// with the pseudo-inverse bond scaling of mps.py:129-134.
// ---------------------------------------------------------------------------
// PRE = false: W = X0^H X[:, perm] / sigma^2 (right vectors of X0, c x keep)
// PRE = true : W = X0 Y[:, perm] / sigma^2   (left vectors of X0, r x keep)
// side = orient ^ precond: 0 -> W goes to Gamma_{q+1} as V^H rows, 1 -> to Gamma_q.
template <bool PRE>
struct SplitOp {
  static constexpr bool kAKMajor = !PRE;
  static constexpr bool kBKMajor = true;
  StateView sv;
  const int* items;
  const ItemMeta* meta;
  const double2* M0;
  const double2* X;
  const double2* Yq;
  size_t mat_stride;
  const double* sig_ws;
  const int* perm_ws;
  int sig_stride;
  // per-CTA
  const double2* m0;
  const double2* x;
  const double* sig;
  const int* perm;
  double2* dst;
  const double* lb;
  int r, jr, side, dl, dr, cap;
  double zero_sig;
  BMPS_DEV bool begin(int item, int& M, int& N, int& K) {
    const ItemMeta* m = meta + item;
    if (m->status || m->keep <= 0 || (m->precond != 0) != PRE) return false;
    zero_sig = kNoiseRel * sqrt(m->fro2);
    const int s = items[2 * item], q = items[2 * item + 1];
    r = m->r;
    jr = m->jrows;
    side = m->orient ^ m->precond;
    dl = m->dl;
    dr = m->dr;
    cap = sv.cap;
    m0 = M0 + (size_t)item * mat_stride;
    x = (PRE || m->msel ? Yq : X) + (size_t)item * mat_stride;
    sig = sig_ws + (size_t)item * sig_stride;
    perm = perm_ws + (size_t)item * sig_stride;
    if (side == 0) {
      dst = sv.site(s, q + 1);
      lb = sv.bond(s, q + 2);
    } else {
      dst = sv.site(s, q);
      lb = sv.bond(s, q);
    }
    M = PRE ? r : m->c;
    N = m->keep;
    K = PRE ? m->c : r;
    return true;
  }
  BMPS_DEV double2 a(int i, int k) const {
    return PRE ? m0[(size_t)i + (size_t)k * r] : cconj(m0[(size_t)k + (size_t)i * r]);
  }
  BMPS_DEV double2 b(int k, int j) const { return x[(size_t)k + (size_t)perm[j] * jr]; }
  BMPS_DEV void store(int i, int j, double2 v) const {
    const double sj = sig[j];
    const double f = sj > zero_sig ? 1.0 / (sj * sj) : 0.0;
    if (side == 0) {
      const int b = i / dr, rr = i % dr;
      dst[(size_t)(2 * j + b) * cap + rr] = cscale(cconj(v), f * pinv(lb[rr]));
    } else {
      dst[(size_t)i * cap + j] = cscale(v, f * pinv(lb[i >> 1]));
    }
  }
};

// ---------------------------------------------------------------------------
// Stats replayed in program order per state (mps.py:82-84, 122):
// trunc_error_sq, total entries, peak entries, max_bond_seen, first failure.
// ---------------------------------------------------------------------------
__global__ void stats_replay_kernel(const bmps_update_record* log, const int* ranges, int nranges,
                                    double* trunc_err, long long* entries, long long* peak,
                                    int* max_bond_seen, int* status, int* status_bond,
                                    double* bond_err, int n, double* min_margin, double* min_gap) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nranges) return;
  const int s = ranges[3 * g], first = ranges[3 * g + 1], count = ranges[3 * g + 2];
  double te = trunc_err[s];
  long long ent = entries[s], pk = peak[s];
  int mb = max_bond_seen[s], st = status[s], sb = status_bond[s];
  double mm = min_margin ? min_margin[s] : 0.0, mg = min_gap ? min_gap[s] : 0.0;
  double* be = bond_err ? bond_err + (size_t)s * (n - 1) : nullptr;
  for (int it = first; it < first + count; ++it) {
    const bmps_update_record m = log[it];
    if (st) break;  // the reference raises at the first failure
    if (m.status == BMPS_S_SVD_FAILED) {
      st = m.status;
      sb = m.site;
      break;
    }
    te += m.err;  // added before the all-truncated check, as mps.py:122-126
    if (be) be[m.site] += m.err;   // per-bond discarded weight, same program order
    if (m.status) {
      st = m.status;
      sb = m.site;
      break;
    }
    const long long dl = m.dl, dm = m.dm, dr = m.dr, k = m.keep;
    ent += 2 * dl * k + 2 * k * dr - 2 * dl * dm - 2 * dm * dr;
    pk = ent > pk ? ent : pk;
    mb = m.keep > mb ? m.keep : mb;
    mm = fmin(mm, m.margin);
    mg = fmin(mg, m.gap);
  }
  trunc_err[s] = te;
  entries[s] = ent;
  peak[s] = pk;
  max_bond_seen[s] = mb;
  status[s] = st;
  status_bond[s] = sb;
  if (min_margin) min_margin[s] = mm;
  if (min_gap) min_gap[s] = mg;
}

}  // namespace bmps
