/*
 * bmps.h -- C ABI of the B200-native MPS hot path (libbmps.so, sm_100a).
 *
 * The reference (mpsqvm, /root/reference/pkg) has no FFI: its "operator API"
 * is the Python class MpsState + TruncationPolicy (src/mpsqvm/mps.py:24-237),
 * driven per gate by backends.mps_run (src/mpsqvm/backends.py:47-60). This
 * header is the boundary a drop-in binds to: every entry
 * point names the reference method it replaces.
 *
 * Conventions
 *   - Plain pointers and sizes only. All pointers are DEVICE pointers unless
 *     the name ends in _host. complex128 is two consecutive doubles (re, im).
 *   - A "state batch" holds S independent n-qubit states at bond capacity cap:
 *       gamma : complex128 [S][n][cap*2*cap]; site (s,k) element (l,p,r) at
 *               ((l*2 + p)*cap + r)  -- the reference's C-order (chi_l, 2, chi_r)
 *               tensor (mps.py:60-62) with row stride cap.
 *       lam   : float64 [S][n+1][cap]; bond b is the left bond of site b.
 *               Bonds 0 and n are the boundary vector [1.0]; internal bond b
 *               is the reference's bond_vectors[b-1] (mps.py:63).
 *       dims  : int32 [S][n+1]; dims[0] = dims[n] = 1.
 *       stats : float64 trunc_err[S], int64 entries[S], int64 peak[S],
 *               int32 max_bond_seen[S], int32 status[S], int32 status_bond[S]
 *               (RunRecord / MpsState bookkeeping, mps.py:64-84).
 *   - Every call is asynchronous on the given cudaStream_t (passed as void*),
 *     never allocates, never synchronises, and returns 0 or a negative
 *     BMPS_E_* launch/argument error. Numerical failures are reported through
 *     the per-state status words (BMPS_S_*) and read at the next host sync.
 *   - The library holds no mutable numerical state: every tunable of a call
 *     travels in its arguments (bmps_params). The only process-wide data are a
 *     per-device cache of kernel attributes / occupancy (set once under a
 *     mutex) and a read-only statistic (bmps_launch_count).
 *   - Work lists ("items") are int32 pairs (state index, site q), in program
 *     order per state; gates are complex128 row-major 2x2 / 4x4 matrices, one
 *     per item, 4x4 indexed [2a+b][2s+t] with a,s on site q (gates.py:3-4).
 */
#ifndef BMPS_H
#define BMPS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* launch / argument errors (return values) */
#define BMPS_OK 0
#define BMPS_E_ARG -1
#define BMPS_E_LAUNCH -2
#define BMPS_E_WORKSPACE -3
#define BMPS_PLAN_E_SITE -10       /* planner: site out of range (mps.py:161-163) */
#define BMPS_PLAN_E_SAME_SITE -11  /* planner: two-qubit gate on one site (mps.py:146-147) */
/* per-state numerical status (status[] words) */
#define BMPS_S_OK 0
#define BMPS_S_SVD_FAILED 1        /* mps.py:117-118 "SVD failed on bond q" */
#define BMPS_S_ALL_TRUNCATED 2     /* mps.py:125-126 "all singular values truncated" */
#define BMPS_S_CAPACITY 3          /* kept bond would exceed the allocated capacity */

typedef struct bmps_policy {
  double cutoff;     /* TruncationPolicy.cutoff   (mps.py:33) */
  int32_t max_bond;  /* TruncationPolicy.max_bond, <= 0 means None (mps.py:34) */
  int32_t relative;  /* TruncationPolicy.relative (mps.py:35) */
} bmps_policy;

/* ABI version and a human-readable message for a return/status code. */
int32_t bmps_version(void);
const char* bmps_status_string(int32_t code);

/* Number of kernels this library has launched so far (process-wide statistic). */
uint64_t bmps_launch_count(void);

/* Build flags: bit 0 = measured-slower development variants compiled in
 * (-DBMPS_EXPERIMENTAL: warp-specialised Jacobi, TMA bulk panel staging,
 * Jacobi modes 2 and 3). */
int32_t bmps_build_flags(void);

/* Development aid: cumulative cycles of the Jacobi phases (Gram pass, inner
 * sweep, apply pass, visit counts, warp-specialised waits) in a
 * -DBMPS_PHASE_TIMERS build; returns BMPS_E_ARG in normal builds. out4 is a host
 * array of 24 uint64. */
int32_t bmps_phase_cycles(uint64_t* out4);
/* Development aid (-DBMPS_PHASE_TIMERS builds; BMPS_E_ARG otherwise): per-warp clock
 * trace of the Jacobi inner sweep's rotation / Q-update phase, 64 x 8 x 4 uint64. */
int32_t bmps_inner_trace(uint64_t* out, int32_t n);

/* Test hook (no reference counterpart; tests/test_gpu_inner_sweep.py): one inner
 * Gram-space Jacobi sweep of a 32-column block-pair visit (jac_inner, the scalar part of
 * mps.py:116's SVD replacement) on a caller-supplied 32 x 32 Hermitian Gram (complex128,
 * column-major, device). full = 1: all 496 pairs, 0: the 256 pairs between columns 0..15
 * and 16..31. tol, noise2, fro as in the rotation test |g| > tol * min(|x_i|, |x_j|) * fro.
 * Writes the rotated Gram, the accumulated unitary Q (G_out = Q^H G_in Q) and the number
 * of rotations of the first sweep. */
int32_t bmps_debug_inner_sweep(const double* gram_in, double* gram_out, double* q_out,
                               int32_t full, double tol, double noise2, double fro,
                               int32_t max_inner, int32_t* nrot, void* stream);

/* MpsState.__init__ (mps.py:55-66): |0...0>, unit boundary bonds, stats reset. */
int32_t bmps_init_product(double* gamma, double* lam, int32_t* dims, double* trunc_err,
                          int64_t* entries, int64_t* peak, int32_t* max_bond_seen,
                          int32_t* status, int32_t* status_bond, int32_t S, int32_t n,
                          int32_t cap, void* stream);

/* MpsState.apply_one_qubit (mps.py:88-92) over a batch of (state, site) items. */
int32_t bmps_apply_1q(double* gamma, const int32_t* dims, int32_t S, int32_t n, int32_t cap,
                      const int32_t* items, const double* gates, int32_t nitems, void* stream);

/* Per-update record written by bmps_apply_2q (48 bytes): discarded weight
 * sum(sigma[keep:]^2) (mps.py:121-122), bond dims before the update, kept
 * dimension, status (BMPS_S_*), the site q, and two robustness figures of the
 * keep decision (mps.py:43-49) on the sorted spectrum sigma:
 *   margin = min_{k < min(p, max_bond)} |sigma_k - thr| / sigma_0, the distance of
 *            the nearest singular value that could change keep from the cutoff
 *            threshold (+inf when cutoff == 0);
 *   gap    = (sigma_{keep-1} - sigma_keep) / sigma_0, the spectral gap at the
 *            truncation boundary (+inf when nothing is discarded).
 * A margin below ~1e-12 is a cutoff tie: the reference's own zgesdd could
 * decide it either way. */
typedef struct bmps_update_record {
  double err;
  int32_t dl, dm, dr, keep, status, site;
  double margin, gap;
} bmps_update_record;

/* Tunables of bmps_apply_2q (per call; bmps_default_params fills defaults). */
typedef struct bmps_params {
  double tol_factor;     /* rotate while |g_ij| > tol_factor*sqrt(rows)*eps*sqrt(g_ii g_jj) (4) */
  int32_t max_sweeps;    /* Jacobi sweep cap; exceeding it is BMPS_S_SVD_FAILED (60) */
  int32_t max_inner;     /* Gram-space sweeps per block visit (1) */
  int32_t qr_min_cols;   /* Householder-QR preconditioning from this many columns (65) */
  int32_t jacobi_mode;   /* block Jacobi (> 64 columns): 1 one persistent CTA per item,
                            4 dynamic visit claiming (default); 2 round launches and
                            3 cluster per item need BMPS_EXPERIMENTAL */
  int32_t block_w2;      /* visit panel width 16 / 32 / 64 columns, 0 auto (32) */
  int32_t double_qr;     /* second QR of R^H before the Jacobi (1) */
  int32_t col_sort;      /* descending-norm column order ahead of the first QR (1) */
  int32_t gram_cache;    /* cross visits reuse rotated intra-block Grams (1) */
  int32_t pair_skip;     /* skip cross visits of provably clean block pairs (1) */
  int32_t jac_cluster;   /* row-split cluster visits: 2 / 4 CTAs per visit when forced; -1 (auto)
                            and 0 use single-CTA visits (-1) */
  int32_t jac_per_sm;    /* dynamic Jacobi CTAs per SM, 0 = occupancy maximum (0) */
  int32_t jac_ws;        /* reserved (the warp-specialised Jacobi was removed); must be 0 */
  int32_t tma_staging;   /* TMA bulk panel staging (BMPS_EXPERIMENTAL only) (0) */
  int32_t cluster_size;  /* CTAs per item in mode 3 (8) */
  int32_t qr_cluster;    /* QR panels taller than 384 rows on a row-split cluster when
                            the batch is small (2 x items <= SMs) (1) */
  int32_t n_svd_events;  /* capacity of svd_events in event pairs (0: no timing) */
  void** svd_events;     /* host array of 2*n_svd_events cudaEvent_t: the call records
                            a pair bracketing its SVD stage (column sort, QR
                            preconditioner, Jacobi, double-QR epilogue) at index
                            *svd_events_used, then increments it */
  int32_t* svd_events_used;
  /* threshold schedule of the dynamic Jacobi (jacobi_mode 4): in sweeps < thr_a_sweeps a
   * block-pair visit whose largest relative coupling |x_i^H x_j| / (|x_i| |x_j|) is below
   * thr_a only forms its Gram (no rotations, no panel update) and keeps the item's sweep
   * open; thr_b until thr_b_sweeps; afterwards every visit rotates down to tol_factor, so
   * the converged state is the same. 0 sweeps = off. */
  double thr_a;          /* (3e-2) */
  double thr_b;          /* (3e-3) */
  int32_t thr_a_sweeps;  /* (2) */
  int32_t thr_b_sweeps;  /* (5) */
  int32_t thr_auto;      /* 1: no thresholds when a round's visits do not fill the resident
                            CTAs (latency-bound launch: the sweep count is what matters) (1) */
  int32_t qr_small;      /* QR panels of <= 128 rows on the 128-thread short-panel kernel: -1 when
                            the batch exceeds the SM count, 0 never, 1 always (-1) */
  int32_t visits_hint;   /* the caller's estimate of the block-pair visits one Jacobi round of this
                            call has (sum over items of ceil(columns / 16) / 2, from its own bond
                            bounds); 0 = unknown: items x the widest item's count. Picks the CTAs
                            per SM of latency-bound launches. (0) */
} bmps_params;

void bmps_default_params(bmps_params* p);

/* Workspace bytes for bmps_apply_2q with nitems items at capacity cap. */
size_t bmps_apply_2q_workspace_bytes(int32_t cap, int32_t nitems);

/* MpsState.apply_two_qubit_adjacent (mps.py:94-136) over a batch of
 * independent items (no two items may share a site): contract (theta) ->
 * one-sided Jacobi SVD -> truncate (policy) -> split. Item i's record is
 * written to log[log_index[i]]; bookkeeping is applied by bmps_stats_replay in
 * program order. dim_bound (<= cap, 0 = cap) is an upper bound on the left /
 * right bond dims of every item, used only to size grids. params may be NULL
 * (defaults). Results are bit-deterministic: no reduction depends on the
 * order in which CTAs run. */
int32_t bmps_apply_2q(double* gamma, double* lam, int32_t* dims, int32_t S, int32_t n,
                      int32_t cap, const int32_t* items, const double* gates, int32_t nitems,
                      bmps_policy policy, bmps_update_record* log, const int32_t* log_index,
                      void* workspace, size_t workspace_bytes, int32_t dim_bound,
                      const bmps_params* params, void* stream);

/* Bookkeeping of MpsState._note_sizes / trunc_error_sq (mps.py:82-84, 122)
 * replayed over update records in PROGRAM order: ranges holds nranges int32
 * triples (state, first record, count; at most one range per state per call).
 * Sets the first failing record's status and site into status / status_bond.
 * Optional (NULL = skip): bond_err float64 [S][n-1] += each record's discarded
 * weight at its bond (the per-bond truncation error, summed in program order),
 * min_margin / min_gap float64 [S] = running minimum of the records' margin /
 * gap (cutoff-tie and truncation-gap detectors). */
int32_t bmps_stats_replay(const bmps_update_record* log, const int32_t* ranges, int32_t nranges,
                          double* trunc_err, int64_t* entries, int64_t* peak,
                          int32_t* max_bond_seen, int32_t* status, int32_t* status_bond,
                          double* bond_err, int32_t n, double* min_margin, double* min_gap,
                          void* stream);

/* Diagnostics of the last bmps_apply_2q on this workspace: per-item Jacobi
 * sweeps (int32), copied into a device buffer of length nitems. */
int32_t bmps_apply_2q_sweeps(const void* workspace, int32_t nitems, int32_t* sweeps,
                             void* stream);

/* MpsState.amplitude (mps.py:172-179) for a batch of (state, bitstring):
 * bits is uint8 [count][n] (0/1), out is complex128 [count]. */
int32_t bmps_amplitudes(const double* gamma, const double* lam, const int32_t* dims, int32_t S,
                        int32_t n, int32_t cap, const int32_t* state_idx, const uint8_t* bits,
                        int32_t count, double* out, void* stream);

/* MpsState.conditional_prob_zero (mps.py:206-214) for state `state`, qubit
 * `site`: prefix complex128 [dims[site]] (device), w0 / w1 complex128
 * [dims[site+1]] = prefix @ T_site[:, b, :], p01 float64 [2] = <w0,w0>, <w1,w1>
 * (the caller forms p0 / (p0 + p1), 0.5 when both vanish). */
int32_t bmps_conditional(const double* gamma, const double* lam, const int32_t* dims, int32_t S,
                         int32_t n, int32_t cap, int32_t state, int32_t site, const double* prefix,
                         double* w0, double* w1, double* p01, void* stream);

/* MpsState.sample / conditional_prob_zero (mps.py:206-237) for a batch of
 * shots: uniforms is float64 [shots][n] (the reference's rng.random() draws,
 * one per qubit per shot in qubit order), bits out uint8 [shots][n]. */
int32_t bmps_sample(const double* gamma, const double* lam, const int32_t* dims, int32_t S,
                    int32_t n, int32_t cap, const int32_t* state_idx, const double* uniforms,
                    int32_t shots, uint8_t* bits, void* stream);

/* One environment transfer step for a batch of (state, site, pauli) items,
 * the building block of MpsState.expectation_pauli / norm_sq
 * (mps.py:181-204): direction 0 (left, E_{k+1} from E_k, mps.py:200) or
 * 1 (right, R_k from R_{k+1}). Environments are cap x cap complex128
 * matrices (row stride cap); item i's input starts at env_in + j*in_stride
 * and its output at env_out + k*out_stride (strides in complex elements), with
 * j = in_idx[i] and k = out_idx[i] when those device index arrays are given,
 * else j = k = i (gather / scatter without copies).
 * pauli codes I=0 X=1 Y=2 Z=3. scratch: complex128 [2][count][2*cap*cap]. */
int32_t bmps_env_transfer(const double* gamma, const double* lam, const int32_t* dims, int32_t S,
                          int32_t n, int32_t cap, const int32_t* state_idx, const int32_t* site,
                          const uint8_t* pauli, int32_t direction, const double* env_in,
                          int64_t in_stride, const int32_t* in_idx, double* env_out,
                          int64_t out_stride, const int32_t* out_idx, double* scratch,
                          int32_t count, void* stream);

/* MpsState.expectation_pauli (mps.py:188-204) for a batch of (state, string)
 * items at small bonds (cap <= 32), fused: item i sweeps sites lo[i]..hi[i] (its
 * first / last non-identity site; hi < lo for an all-identity string) from the
 * cached left environment L_lo and closes with R_{hi+1} (R_lo if hi < lo).
 * Environments are complex128 [U][n+1][cap][cap] with env_stride = (n+1)*cap*cap
 * complex elements per environment set; env_idx[i] selects the set of item i;
 * codes uint8 [count][n] (I=0 X=1 Y=2 Z=3); out complex128 [count]. */
int32_t bmps_pauli_sweep(const double* gamma, const double* lam, const int32_t* dims, int32_t S,
                         int32_t n, int32_t cap, const int32_t* state_idx, const int32_t* env_idx,
                         const uint8_t* codes, const int32_t* lo, const int32_t* hi,
                         const double* env_l, const double* env_r, int64_t env_stride,
                         int32_t count, double* out, void* stream);

/* All identity environments of `count` states in one launch (small bonds,
 * cap <= 32): direction 0 fills L_1..L_n, direction 1 R_{n-1}..R_0, of env
 * complex128 [count][n+1][cap][cap] (env_stride = (n+1)*cap*cap complex
 * elements; the caller sets L_0 / R_n = [[1]] and zero padding). The
 * identity-Pauli case of the transfers above, kept in shared memory. */
int32_t bmps_env_sweep(const double* gamma, const double* lam, const int32_t* dims, int32_t S,
                       int32_t n, int32_t cap, const int32_t* states, int32_t count,
                       int32_t direction, double* env, int64_t env_stride, void* stream);

/* <E_left, R_right> contraction: out[i] = sum_{r,q} L_i[r,q] * R_i[r,q] over
 * the dims[s][b_i] x dims[s][b_i] leading block (complex128 out); L_i at
 * env_l + l*l_stride, R_i at env_r + r*r_stride (complex elements) with
 * l = l_idx[i], r = r_idx[i] when given (device int32), else l = r = i. */
int32_t bmps_env_close(const int32_t* dims, int32_t n, int32_t cap, const int32_t* state_idx,
                       const int32_t* bond, const double* env_l, int64_t l_stride,
                       const int32_t* l_idx, const double* env_r, int64_t r_stride,
                       const int32_t* r_idx, int32_t count, double* out, void* stream);

/* ---- dense statevector backend (R:src/mpsqvm/dense.py) --------------------
 * amps: complex128 [S][2^n], flat index with qubit 0 as the HIGH bit
 * (dense.py:23); n <= 33. Gates passed by host pointer are read during the
 * call (kernel parameters); no device allocation. */

/* DenseState.__init__ (dense.py:26-32): |0...0> for each of S states. */
int32_t bmps_dense_init(double* amps, int32_t S, int32_t n, void* stream);

/* DenseState.apply_one_qubit (dense.py:39-44): gate_host complex128 2x2. */
int32_t bmps_dense_apply_1q(double* amps, int32_t n, int32_t q, const double* gate_host,
                            void* stream);

/* DenseState.apply_two_qubit (dense.py:46-54): gate_host complex128 4x4
 * indexed [2a+b][2s+t], a/s on q1 (the first listed qubit), any q1 != q2. */
int32_t bmps_dense_apply_2q(double* amps, int32_t n, int32_t q1, int32_t q2,
                            const double* gate_host, void* stream);

/* dense_run (dense.py:112-123) of S states of n <= 12 qubits in one launch
 * (state resident in shared memory): ops int32 [S][nops][3] = (arity, q1,
 * q2), mats complex128 [S][nops][16] (a 2x2 gate in the first 4), device. */
int32_t bmps_dense_run_smem(double* amps, int32_t S, int32_t n, const int32_t* ops,
                            const double* mats, int32_t nops, void* stream);

/* DenseState.expectation_pauli / norm_sq (dense.py:61-81) for a batch of
 * (state, Pauli string): masks uint64 [count][2] = (X|Y bit mask, Z|Y bit
 * mask), ny int32 [count] = number of Y; out complex128 [count] (the caller
 * applies the 1e-10 imaginary-residue check). */
size_t bmps_dense_expect_workspace_bytes(int32_t count);
int32_t bmps_dense_expect(const double* amps, int32_t S, int32_t n, const int32_t* state_idx,
                          const uint64_t* masks, const int32_t* ny, int32_t count,
                          void* workspace, size_t workspace_bytes, double* out, void* stream);

/* Marginal-probability heap for DenseState.conditional_prob_zero / sample
 * (dense.py:88-110): tree float64 [2^(n+1)], node (level k, prefix v) at
 * tree[2^k + v], leaves |amp_i|^2 at tree[2^n + i]. */
int32_t bmps_dense_prob_tree(const double* amps, int32_t n, double* tree, void* stream);

/* DenseState.sample: uniforms float64 [shots][n] (rng.random() draws, one per
 * qubit per shot in qubit order), out uint64 [shots] basis indices. */
int32_t bmps_dense_sample(const double* tree, int32_t n, const double* uniforms, int32_t shots,
                          uint64_t* out, void* stream);

/* ---- host-side program planner (engine.compile_batch; no device work) ------
 * Input: the ops of nprogs programs concatenated (MEASUREs already dropped),
 * program p = ops [prog_off[p], prog_off[p+1]) for state prog_state[p];
 * arity 1/2, sites q1 (and q2 for arity 2, any order, any distance).
 * Output per EXPANDED op (SWAP routing of mps.py:138-157 applied, in program
 * order): state, arity, site (the left site of a two-site op), x_src = source
 * op index (>= 0), -i-2 for source op i applied as SWAP.G.SWAP (q1 > q2), -1
 * for a routing SWAP; x_layer = ASAP layer within the program; x_rec = the
 * op's record index (two-site ops numbered in program order across the batch)
 * or -1. On BMPS_PLAN_E_* *err_op is the offending source op. */
int64_t bmps_plan_expanded_count(const int8_t* arity, const int32_t* q1, const int32_t* q2,
                                 int64_t nops);
int32_t bmps_plan_build(int32_t nprogs, const int64_t* prog_off, const int32_t* prog_state,
                        const int8_t* arity, const int32_t* q1, const int32_t* q2, int32_t n,
                        int32_t* x_state, int8_t* x_arity, int32_t* x_site, int64_t* x_src,
                        int32_t* x_layer, int64_t* x_rec, int64_t* err_op);

#ifdef __cplusplus
}
#endif
#endif /* BMPS_H */
