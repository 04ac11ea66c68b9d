// Dense-matrix drop-ins of the reference's feasibility / semidual helpers
// for callers that hold a LINEAR-scale matrix (not a log plan) on the
// device: round_to_feasible (feasibility.py:44-69), bregman_div (72-85),
// c_transform + kkt_residual (88-122), gap (125-127) and
// hessian_matvec_exact (semidual.py:103-114).  The solver itself never
// calls these (its plans live in the log domain and go through the fused
// three-pass rounding of dense.cuh); they exist so that the reference's
// kernel-level functions keep their signatures and their arithmetic:
// every elementwise expression is numpy's, in numpy's order (the library is
// built with --fmad=false), and sums are fixed-order trees (deterministic,
// not numpy's pairwise order: agreement to a few ulp, not bitwise).
//
// Shapes: x (and C, log y, P) are m x n row-major with a leading dimension;
// row kernels use one 256-thread CTA per row (grid-stride over rows);
// column kernels a (ceil(n/256), RB) grid writing RB partial rows, summed in
// order by k_dapi_colfinish.
#pragma once

#include "common.cuh"

namespace otb {

constexpr int kDapiThreads = 256;
constexpr int kDapiRB = 64;   // row blocks of the column kernels

// Element of the rounding pipeline: (x_ij * z_i) * y_j with absent factors 1
// (feasibility.py:59, 63).
OTB_DEV double dapi_elem(const double* x, int64_t ld, int i, int j, const double* zr, const double* yc) {
  double v = x[(int64_t)i * ld + j];
  if (zr) v = v * zr[i];
  if (yc) v = v * yc[j];
  return v;
}

// Row sums of the rounding element, then per mode:
//   0: out_i = rowsum                 (plain)
//   1: out_i = r > 0 ? min(a_i / r, 1) : 1     (z, feasibility.py:56-58)
//   2: out_i = a_i - r                          (e_r, :64)
__global__ void __launch_bounds__(kDapiThreads) k_dapi_rows(const double* x, int64_t ld, int m, int n,
                                                           const double* zr, const double* yc, const double* a,
                                                           int mode, double* out) {
  __shared__ double slots[2 * kMaxWarps * 4];
  int phase = 0;
  for (int i = blockIdx.x; i < m; i += gridDim.x) {
    double s[1] = {0.0};
    for (int j = threadIdx.x; j < n; j += blockDim.x) s[0] += dapi_elem(x, ld, i, j, zr, yc);
    block_reduce<1, kSum>(s, slots, phase, blockDim.x);
    if (threadIdx.x == 0) {
      const double r = s[0];
      if (mode == 1) out[i] = (r > 0.0) ? fmin(div_rn(a[i], r), 1.0) : 1.0;
      else if (mode == 2) out[i] = a[i] - r;
      else out[i] = r;
    }
  }
}

// Column partial sums: part[blockIdx.y][j] over the rows of row block y.
__global__ void __launch_bounds__(kDapiThreads) k_dapi_cols(const double* x, int64_t ld, int m, int n,
                                                           const double* zr, const double* yc, double* part) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int RB = gridDim.y;
  const int i0 = (int)(((int64_t)blockIdx.y * m) / RB), i1 = (int)(((int64_t)(blockIdx.y + 1) * m) / RB);
  double s = 0.0;
  for (int i = i0; i < i1; ++i) s += dapi_elem(x, ld, i, j, zr, yc);
  part[(int64_t)blockIdx.y * n + j] = s;
}

// Fixed-order sum of the RB partial rows, then per mode:
//   0: out_j = colsum;  1: out_j = c > 0 ? min(b_j / c, 1) : 1 (y, :61-63);
//   2: out_j = b_j - c  (e_c, :65)
__global__ void __launch_bounds__(kDapiThreads) k_dapi_colfinish(const double* part, int RB, int n, const double* b,
                                                                int mode, double* out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double c = 0.0;
  for (int q = 0; q < RB; ++q) c += part[(int64_t)q * n + j];
  if (mode == 1) out[j] = (c > 0.0) ? fmin(div_rn(b[j], c), 1.0) : 1.0;
  else if (mode == 2) out[j] = b[j] - c;
  else out[j] = c;
}

// Single-CTA fixed-order reductions of a vector: out[0] = sum |v| (mode 0,
// the deficit, :66) or sum v (mode 1).
__global__ void __launch_bounds__(kDapiThreads) k_dapi_vsum(const double* v, int len, int mode, double* out) {
  __shared__ double slots[2 * kMaxWarps * 4];
  int phase = 0;
  double s[1] = {0.0};
  for (int i = threadIdx.x; i < len; i += blockDim.x) s[0] += (mode == 0) ? fabs(v[i]) : v[i];
  block_reduce<1, kSum>(s, slots, phase, blockDim.x);
  if (threadIdx.x == 0) out[0] = s[0];
}

// F^ = F + outer(e_r, e_c) / deficit when deficit > 0 (feasibility.py:67-68),
// F = (x z) y.
__global__ void k_dapi_round_out(const double* x, int64_t ld, int m, int n, const double* zr, const double* yc,
                                 const double* er, const double* ec, const double* deficit, double* out,
                                 int64_t ldo) {
  const double def = *deficit;
  const int64_t total = (int64_t)m * n;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(k / n), j = (int)(k - (int64_t)i * n);
    double f = dapi_elem(x, ld, i, j, zr, yc);
    if (def > 0.0) f = f + div_rn(er[i] * ec[j], def);
    out[(int64_t)i * ldo + j] = f;
  }
}

// bregman_div (feasibility.py:72-85): per row [sum terms, sum x, sum exp(log y)]
// with terms = x > 0 ? x (log x - log y) : 0.
__global__ void __launch_bounds__(kDapiThreads) k_dapi_bregman(const double* x, int64_t ldx, const double* ly,
                                                              int64_t ldy, int m, int n, double* rows3) {
  __shared__ double slots[2 * kMaxWarps * 4];
  int phase = 0;
  for (int i = blockIdx.x; i < m; i += gridDim.x) {
    double s[3] = {0.0, 0.0, 0.0};
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      const double xv = x[(int64_t)i * ldx + j], lv = ly[(int64_t)i * ldy + j];
      if (xv > 0.0) s[0] += xv * (log(xv) - lv);
      s[1] += xv;
      s[2] += exp(lv);
    }
    block_reduce<3, kSum>(s, slots, phase, blockDim.x);
    if (threadIdx.x == 0) {
      rows3[3 * (int64_t)i] = s[0];
      rows3[3 * (int64_t)i + 1] = s[1];
      rows3[3 * (int64_t)i + 2] = s[2];
    }
  }
}

// kkt_residual (feasibility.py:93-122) on x AS GIVEN, plus <C, x> for gap
// (:125-127).  Per row i: zeta_i = min_j (C_ij - gamma_j) (c_transform,
// :88-90), slack = (C - gamma) - zeta, and the row sums
//   [row sum of x, sum min(x,0)^2, sum x^2, sum min(slack,0)^2, sum x slack, sum C x]
// into rows6[6 i ..]; column sums of x come from k_dapi_cols.
__global__ void __launch_bounds__(kDapiThreads) k_dapi_kkt(const double* x, int64_t ldx, const double* C,
                                                          int64_t ldc, const double* gamma, int m, int n,
                                                          double* zeta, double* rows6) {
  __shared__ double slots[2 * kMaxWarps * 4];
  int phase = 0;
  for (int i = blockIdx.x; i < m; i += gridDim.x) {
    const double* cr = C + (int64_t)i * ldc;
    const double* xr = x + (int64_t)i * ldx;
    double mn[1] = {INFINITY};
    for (int j = threadIdx.x; j < n; j += blockDim.x) mn[0] = fmin(mn[0], cr[j] - gamma[j]);
    block_reduce<1, kMin>(mn, slots, phase, blockDim.x);
    const double z = mn[0];
    double s[3] = {0.0, 0.0, 0.0}, t[3] = {0.0, 0.0, 0.0};
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      const double xv = xr[j], cv = cr[j];
      const double sl = (cv - gamma[j]) - z;
      const double xn = fmin(xv, 0.0), sn = fmin(sl, 0.0);
      s[0] += xv;
      s[1] += xn * xn;
      s[2] += xv * xv;
      t[0] += sn * sn;
      t[1] += xv * sl;
      t[2] += cv * xv;
    }
    block_reduce<3, kSum>(s, slots, phase, blockDim.x);
    block_reduce<3, kSum>(t, slots, phase, blockDim.x);
    if (threadIdx.x == 0) {
      zeta[i] = z;
      double* o = rows6 + 6 * (int64_t)i;
      o[0] = s[0];
      o[1] = s[1];
      o[2] = s[2];
      o[3] = t[0];
      o[4] = t[1];
      o[5] = t[2];
    }
  }
}

// Fixed-order column sums of a [m][K] row-stats array: out[k] = sum_i rows[i K + k]
// (out[k] for k < K; one warp per k, lanes strided, then the warp tree).
// With `res` (length m) also out[K] = sum_i (rows[i K] - res_i)^2.
__global__ void k_dapi_rowstats(const double* rows, int m, int K, const double* res, double* out) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nk = K + (res ? 1 : 0);
  for (int k = w; k < nk; k += blockDim.x >> 5) {
    double s = 0.0;
    for (int i = lane; i < m; i += 32) {
      if (k < K) {
        s += rows[(int64_t)i * K + k];
      } else {
        const double e = rows[(int64_t)i * K] - res[i];
        s += e * e;
      }
    }
    s = warp_sum(s);
    if (lane == 0) out[k] = s;
  }
}

// sum_j (v_j - b_j)^2 (column residual), single CTA.
__global__ void __launch_bounds__(kDapiThreads) k_dapi_sqdiff(const double* v, const double* b, int n, double* out) {
  __shared__ double slots[2 * kMaxWarps * 4];
  int phase = 0;
  double s[1] = {0.0};
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const double e = v[j] - b[j];
    s[0] += e * e;
  }
  block_reduce<1, kSum>(s, slots, phase, blockDim.x);
  if (threadIdx.x == 0) out[0] = s[0];
}

// hessian_matvec_exact (semidual.py:103-114), dense P: pv_i = P_i . v (row
// kernel writes w_i = a_i * pv_i), then col sums of P a and of P w.
__global__ void __launch_bounds__(kDapiThreads) k_dapi_rowdot(const double* P, int64_t ld, int m, int n,
                                                             const double* v, const double* a, double* w) {
  __shared__ double slots[2 * kMaxWarps * 4];
  int phase = 0;
  for (int i = blockIdx.x; i < m; i += gridDim.x) {
    double s[1] = {0.0};
    for (int j = threadIdx.x; j < n; j += blockDim.x) s[0] += P[(int64_t)i * ld + j] * v[j];
    block_reduce<1, kSum>(s, slots, phase, blockDim.x);
    if (threadIdx.x == 0) w[i] = a[i] * s[0];   // semidual.py:113: a * pv
  }
}

// Column partials of P^T u for two row weights at once (u0 = a, u1 = a pv).
__global__ void __launch_bounds__(kDapiThreads) k_dapi_cols2(const double* P, int64_t ld, int m, int n,
                                                            const double* u0, const double* u1, double* part0,
                                                            double* part1) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int RB = gridDim.y;
  const int i0 = (int)(((int64_t)blockIdx.y * m) / RB), i1 = (int)(((int64_t)(blockIdx.y + 1) * m) / RB);
  double s0 = 0.0, s1 = 0.0;
  for (int i = i0; i < i1; ++i) {
    const double p = P[(int64_t)i * ld + j];
    s0 += p * u0[i];
    s1 += p * u1[i];
  }
  part0[(int64_t)blockIdx.y * n + j] = s0;
  part1[(int64_t)blockIdx.y * n + j] = s1;
}

// out_j = (cw_j * v_j - y_j) / eta, cw = P^T a, y = P^T (a pv) (semidual.py:114).
__global__ void k_dapi_hv_out(const double* part0, const double* part1, int RB, int n, const double* v, double eta,
                              double* out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double cw = 0.0, y = 0.0;
  for (int q = 0; q < RB; ++q) {
    cw += part0[(int64_t)q * n + j];
    y += part1[(int64_t)q * n + j];
  }
  out[j] = div_rn(cw * v[j] - y, eta);
}

}  // namespace otb
