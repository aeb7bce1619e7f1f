// Shared device helpers for libbmps: complex128 arithmetic, FP64 tensor-core
// (DMMA, mma.sync m8n8k4 f64) complex tile products, state indexing.
#pragma once
#include <cuda_runtime.h>
#include <cstdio>
#include <math_constants.h>
#include <stdint.h>

#include "bmps.h"

#define BMPS_DEV __device__ __forceinline__
#define BMPS_HOSTDEV __host__ __device__

namespace bmps {

// Device-side invariant checks of a -DBMPS_DEBUG_CHECKS build (bounds of the items
// a launch touches, the Jacobi scheduling protocol); compiled out otherwise.
#ifdef BMPS_DEBUG_CHECKS
#define BMPS_CHECK(cond)                                                                   \
  do {                                                                                     \
    if (!(cond)) {                                                                         \
      printf("BMPS_CHECK failed %s:%d block %d: %s\n", __FILE__, __LINE__, (int)blockIdx.x, #cond); \
      __trap();                                                                            \
    }                                                                                      \
  } while (0)
#else
#define BMPS_CHECK(cond) do { } while (0)
#endif

constexpr double kEps = 1.1102230246251565e-16;   // unit roundoff of float64
constexpr double kPinvFloor = 1e-12;              // mps.py:21 _PINV_FLOOR

BMPS_DEV double2 cmake(double x, double y) { return make_double2(x, y); }
BMPS_DEV double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
BMPS_DEV double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
BMPS_DEV double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
BMPS_DEV double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
BMPS_DEV double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// x*c -/+ y*z and x*c -/+ conj(y)*z with real c: 3 dependent FP64 ops per component.
BMPS_DEV double2 cms(double2 x, double c, double2 y, double2 z) {
  return make_double2(fma(y.y, z.y, fma(-y.x, z.x, x.x * c)), fma(-y.y, z.x, fma(-y.x, z.y, x.y * c)));
}
BMPS_DEV double2 cma(double2 x, double c, double2 y, double2 z) {
  return make_double2(fma(-y.y, z.y, fma(y.x, z.x, x.x * c)), fma(y.y, z.x, fma(y.x, z.y, x.y * c)));
}
BMPS_DEV double2 cmsc(double2 x, double c, double2 y, double2 z) {
  return make_double2(fma(-y.y, z.y, fma(-y.x, z.x, x.x * c)), fma(y.y, z.x, fma(-y.x, z.y, x.y * c)));
}
BMPS_DEV double2 cmac(double2 x, double c, double2 y, double2 z) {
  return make_double2(fma(y.y, z.y, fma(y.x, z.x, x.x * c)), fma(-y.y, z.x, fma(y.x, z.y, x.y * c)));
}
// a*b + c
BMPS_DEV double2 cfma(double2 a, double2 b, double2 c) {
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
BMPS_DEV double cabs2(double2 a) { return fma(a.x, a.x, a.y * a.y); }

// Reference pseudo-inverse of a bond entry: 1/x if x > 1e-12 else 0 (mps.py:129-130).
BMPS_DEV double pinv(double x) { return x > kPinvFloor ? 1.0 / x : 0.0; }

// d += a * b for one 8x8x4 FP64 tensor-core step (DMMA.8x8x4 on sm_100a).
// Fragment layout: A(8x4) row = lane>>2, col = lane&3; B(4x8) row = lane&3,
// col = lane>>2; D(8x8) row = lane>>2, cols 2*(lane&3) + {0,1}.
BMPS_DEV void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
// complex accumulate: c[0..1] real part, c[2..3] imaginary part.
BMPS_DEV void zmma(double (&c)[4], double2 a, double2 b) {
  dmma(c[0], c[1], a.x, b.x);
  dmma(c[0], c[1], -a.y, b.y);
  dmma(c[2], c[3], a.x, b.y);
  dmma(c[2], c[3], a.y, b.x);
}

// 3-product (Gauss) complex accumulate, 3 DMMA instead of 4 on the shared FP64
// pipe: c[0..1] += a.x b.x, c[2..3] += a.y b.y, c[4..5] += (a.x + a.y)(b.x + b.y);
// z3_get(c, h) = (c0 - c2, c4 - c0 - c2). Normwise error <= ~2 eps sum |a||b|, the
// same order as the 4-product form (ZGEMM3M).
#ifndef BMPS_Z3
#define BMPS_Z3 1
#endif
constexpr int kZ3 = BMPS_Z3 ? 6 : 4;   // accumulator doubles per complex tile
BMPS_DEV void zmma3(double (&c)[kZ3], double2 a, double2 b) {
#if BMPS_Z3
  dmma(c[0], c[1], a.x, b.x);
  dmma(c[2], c[3], a.y, b.y);
  dmma(c[4], c[5], a.x + a.y, b.x + b.y);
#else
  zmma(c, a, b);
#endif
}
BMPS_DEV double2 z3_get(const double (&c)[kZ3], int h) {
#if BMPS_Z3
  const double re = c[h], ri = c[2 + h];
  return make_double2(re - ri, c[4 + h] - re - ri);
#else
  return make_double2(c[h], c[2 + h]);
#endif
}

// Circle-method round robin over N (even) players: pair p of round rho.
BMPS_DEV void tourney_pair(int N, int rho, int p, int& i, int& j) {
  int a, b;
  if (p == 0) {
    a = rho;
    b = N - 1;
  } else {
    a = (rho + p) % (N - 1);
    b = (rho - p + N - 1) % (N - 1);
  }
  i = a < b ? a : b;
  j = a < b ? b : a;
}

// Complex Jacobi rotation zeroing the (i,j) entry of the 2x2 Hermitian Gram
// [[a, g], [conj(g), b]]. Column transform [x_i, x_j] <- [x_i, x_j] J with
// J = [[c, s], [-s*conj(e), c*conj(e)]], e = g/|g| (Rutishauser's tangent).
// A pair whose smaller squared norm is below kNegligible times the larger one
// (relative column norm < 1e-125) carries nothing that can reach a float64
// result; it is never rotated (this also keeps underflowed columns from
// looking non-orthogonal forever).
constexpr double kNegligible = 1e-250;
// Rounding-noise floor of a column relative to ||M||_F. With cutoff 0 the
// reference keeps numerically-zero singular values (rank-deficient theta);
// pairs of two such columns carry no information and relative orthogonality
// between them cannot converge, so they are not rotated, and singular vectors
// of sigma_k <= kNoiseRel * ||M||_F are written as zero in the split (their
// lambda entry is kept, so bond dims and spectra still match the reference;
// the state changes by <= kNoiseRel * ||M||_F).
constexpr double kNoiseRel = 1e-14;

// Rotation test for the pair (x_i, x_j) with squared norms a, b and g = x_i^H x_j:
//   |g| > tol * min(|x_i|, |x_j|) * ||M||_F
// i.e. relative orthogonality tol for columns near the top of the spectrum and
// absolute accuracy tol * ||M||_F for small ones (their contribution to any
// gauge-invariant output is |g| / min(|x_i|, |x_j|)). A purely relative test
// cannot converge for wide spectra: rounding of the dominant columns keeps
// re-injecting eps * ||M|| into small columns. fro = ||M||_F; noise2 =
// (kNoiseRel * fro)^2.
BMPS_DEV bool pair_needs_rotation(double a, double b, double2 g, double tol, double noise2,
                                  double fro) {
  const double lo = fmin(a, b), hi = fmax(a, b);
  if (!(hi > noise2)) return false;
  if (!(lo > kNegligible * hi)) return false;
  return hypot(g.x, g.y) > tol * sqrt(lo) * fro;
}

// 1/sqrt(x) for normal positive x: hardware approximation (MUFU, ~2^-23) plus two
// Newton steps -> full float64 accuracy without the library's special-case paths.
BMPS_DEV double fast_rsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return y;
}

// Same test as jacobi_rotation's early exits (no rotation math).
BMPS_DEV bool jacobi_needs(double a, double b, double2 g, double tol, double noise2, double fro) {
  const double lo = fmin(a, b), hi = fmax(a, b);
  if (!(hi > noise2) || !(lo > kNegligible * hi)) return false;
  const double thr = tol * fro;
  const double g2 = cabs2(g);
  return g2 > thr * thr * lo && g2 > 1e-290;
}

// Branch-free rotation of one pair: a, b = squared column norms, g = x_i^H x_j,
// thr2 = (tol ||M||_F)^2. Returns 1 and (c, sigma) if the pair rotates (the test of
// jacobi_needs, which includes |g|^2 > 1e-290 so every reciprocal square root below sees
// a normal number), else 0 and the identity. The column transform is
//   [x_i, x_j] <- [x_i, x_j] [[c, sigma], [-conj(sigma), c]],   c^2 + |sigma|^2 = 1:
// with delta = b - a and rho = sqrt(delta^2 + 4|g|^2),
//   c = sqrt((1 + |delta| / rho) / 2),   sigma = sign(delta) g / (rho c),
// the same small-angle rotation as Rutishauser's tangent formula (the phase of g rides
// on sigma, so no 1/|g| is needed). No branches: the call sits on the inner sweep's
// critical path.
BMPS_DEV int jacobi_rotation(double a, double b, double2 g, double thr2, double noise2, double& c,
                             double2& sigma) {
  const double lo = fmin(a, b), hi = fmax(a, b);
  const double g2 = cabs2(g);
  const bool act = (hi > noise2) && (lo > kNegligible * hi) && (g2 > thr2 * lo) && (g2 > 1e-290);
  const double g2s = act ? g2 : 1.0;                      // keeps the arithmetic finite
  const double delta = act ? b - a : 0.0;
  const double rr = fast_rsqrt(fma(delta, delta, 4.0 * g2s));
  const double c2 = fma(0.5 * fabs(delta), rr, 0.5);      // in [1/2, 1]
  const double rc = fast_rsqrt(c2);                       // 1 / c
  const double kap = delta < 0 ? -(rr * rc) : rr * rc;    // sign(delta) / (rho c)
  c = act ? c2 * rc : 1.0;
  sigma = act ? make_double2(g.x * kap, g.y * kap) : make_double2(0.0, 0.0);
  return act ? 1 : 0;
}

// cp.async 16-byte global -> shared copy, zero-filled when !valid.
BMPS_DEV void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem),
               "r"(valid ? 16 : 0));
}
BMPS_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
BMPS_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

struct StateView {
  double2* gamma;
  double* lam;
  int* dims;
  int n;
  int cap;
  BMPS_DEV double2* site(int s, int k) const {
    return gamma + ((size_t)s * n + k) * (size_t)(2 * (size_t)cap * cap);
  }
  BMPS_DEV double* bond(int s, int b) const { return lam + ((size_t)s * (n + 1) + b) * cap; }
  BMPS_DEV int* dimv(int s) const { return dims + (size_t)s * (n + 1); }
};

// Per-item bookkeeping of one two-site update (lives in the caller's workspace).
struct ItemMeta {
  int r, c, orient, dl, dm, dr;   // X0 rows/cols, orientation, bond dims before update
  int keep, status, sweeps, conv, flag;
  int precond;                    // 1: Jacobi runs on Y = R^H from X0 = QR
  int jrows;                      // rows of the Jacobi matrix (r, or c if precond)
  int dq;                         // 1: second QR (R1^H = Q2 R2), Jacobi on Z = R2^H
  int msel;                       // finalize/split read the result matrix from Y (not X)
  int keep_pre;                   // keep count known before finalize (double-QR path)
  double err, norm;
  double fro2;                    // ||M||_F^2 (accumulated by theta)
  double padd;
};

}  // namespace bmps
