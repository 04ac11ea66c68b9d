// Column-parallel "finish" kernels: reduce the per-cluster partial rows of a
// dense pass in fixed order, apply the per-column post-operation, and fold
// scalar partials with the last-block pattern (deterministic).  When the
// rows are sharded over ranks, phase 1 (k_colreduce) fills a send buffer,
// the host all-reduces it with NCCL, and phase 2 (the *_post kernels) runs
// on the globally reduced vector.
#pragma once

#include "common.cuh"

namespace otb {

struct DevScalars {
  double value, gnorm, alse, bgam;     // eval
  double slope;                        // g . direction
  double sumx, deficit;                // test pass A / B
  double s8[8];                        // test pass C scalar totals
  double row_sq, col_sq;               // KKT marginal residual sums of squares
  double warm_err;
  double drift;
  double cnorm_sq;                     // ||C||_F^2 when the caller gave it as a device scalar
  double ev0[3];                       // value, ||g||, non-finite count of an eval not yet read by the host
  double scratch[4];
  double sp_glob[2];                   // multi-rank sparsify: overflow on any rank, total kept entries
  unsigned long long alloc;            // CSR bump allocator
  unsigned long long nnzc;             // kept entries of the last sparsify
  int flags;
  int pad;
  unsigned int cnt[16];                // last-block counters
};

enum CounterIdx {
  CNT_COLRED = 0, CNT_EVALPOST = 1, CNT_DOT = 2, CNT_ROWS = 3, CNT_VECPOST = 4, CNT_SUM = 5, CNT_WARM = 6,
  CNT_SCALED = 7
};

// out[j] = sum_c part[c*n + j]; out[n + k] = sum_c spart[c*sstride + k].
// One block = 32 columns; the 8 warps split the partial rows (fixed order).
// Single rank (nothing to all-reduce in between), the elementwise finish of
// k_vec_post can be applied here (post = POST_COPY / POST_Y / POST_EC into
// post_out) and scalar k also stored at sdst[k] — one launch instead of two
// plus the scalar copies.  post < 0: plain column sums into out.
struct ColPost {
  int post;                // < 0: none
  const double* b;
  double* out;
  double* sdst[2];         // optional destinations of scalars 0, 1
};
__global__ void __launch_bounds__(256) k_colreduce(const double* part, int nparts, int n, double* out,
                                                   const double* spart, int nspart, int sstride, int nscal,
                                                   unsigned int* counter, ColPost cp) {
  __shared__ double red[8 * 32];
  const double s = reduce_partials32(part, nparts, n, blockIdx.x * 32, red);
  const int j = blockIdx.x * 32 + threadIdx.x;
  if (threadIdx.x < 32 && j < n) {
    if (cp.post < 0) out[j] = s;
    else if (cp.post == 0) cp.out[j] = s;                                            // POST_COPY
    else if (cp.post == 1) cp.out[j] = (s > 0.0) ? fmin(div_rn(cp.b[j], s), 1.0) : 1.0;   // POST_Y
    else cp.out[j] = cp.b[j] - s;                                                     // POST_EC
  }
  if (nscal > 0) {
    if (last_block(counter)) {
      if (threadIdx.x < 32) {
        for (int k = 0; k < nscal; ++k) {
          const double v = warp_fixed_sum(spart + k, nspart, sstride);
          if (threadIdx.x == 0) {
            out[n + k] = v;
            if (k < 2 && cp.sdst[k] != nullptr) *cp.sdst[k] = v;
          }
        }
      }
    }
  }
}

// semidual.py:90-100 finish: g = (P^T a) - b, ||g||, L = -b.gamma + eta a.lse.
// buf[0..n) = column sums of a_i P_ij, buf[n] = a.lse.
__global__ void __launch_bounds__(256) k_eval_post(int n, const double* buf, const double* b, const double* gamma,
                                                   double eta, double* g, DevScalars* ds, double* bpart) {
  __shared__ double red[2][kMaxWarps * 4];
  double sq = 0.0, bg = 0.0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const double gj = buf[j] - b[j];
    g[j] = gj;
    sq = fma(gj, gj, sq);
    bg += (-b[j]) * gamma[j];
  }
  int ph = 0;
  double t[2] = {sq, bg};
  block_reduce<2, kSum>(t, &red[0][0], ph, blockDim.x);
  if (threadIdx.x == 0) {
    bpart[2 * blockIdx.x] = t[0];
    bpart[2 * blockIdx.x + 1] = t[1];
  }
  if (last_block(&ds->cnt[CNT_EVALPOST])) {
    if (threadIdx.x < 32) {
      const double s = warp_fixed_sum(bpart, gridDim.x, 2);
      const double bgs = warp_fixed_sum(bpart + 1, gridDim.x, 2);
      if (threadIdx.x == 0) {
        const double alse = buf[n];
        ds->scratch[0] = buf[n + 1];   // count of non-finite rows
        ds->gnorm = sqrt(s);
        ds->alse = alse;
        ds->bgam = bgs;
        ds->value = bgs + eta * alse;
      }
    }
  }
}

// Single rank: k_colreduce and k_eval_post in one kernel (one launch less per
// eval) with k_eval_post's summation tree reproduced exactly, so the bits of
// ||g|| and L are those of the two-kernel path: level 1 = xor tree over the
// 32 columns of a block (a k_eval_post warp), level 2 = xor tree over 8
// consecutive blocks (a k_eval_post block of 256 columns), level 3 =
// warp_fixed_sum over those groups (k_eval_post's grid, colgrid groups).
// Valid while colgrid * 256 >= n (one column per k_eval_post thread).
__global__ void __launch_bounds__(256) k_colreduce_eval(const double* part, int nparts, int n, const double* spart,
                                                        int nspart, const double* b, const double* gamma, double eta,
                                                        double* g, DevScalars* ds, double* bpart, int colgrid,
                                                        bool save_ev0 = false) {
  __shared__ double red[8 * 32];
  __shared__ double l2[2][512];
  const double s = reduce_partials32(part, nparts, n, blockIdx.x * 32, red);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < 32) {
    const int j = blockIdx.x * 32 + lane;
    double sq = 0.0, bg = 0.0;
    if (j < n) {
      const double gj = s - b[j];
      g[j] = gj;
      sq = fma(gj, gj, sq);
      bg += (-b[j]) * gamma[j];
    }
    sq = warp_sum(sq);
    bg = warp_sum(bg);
    if (lane == 0) {
      bpart[2 * blockIdx.x] = sq;
      bpart[2 * blockIdx.x + 1] = bg;
    }
  }
  if (last_block(&ds->cnt[CNT_EVALPOST])) {
    const int nb = gridDim.x;
    for (int B = warp; B < colgrid; B += 8) {   // level 2: groups of 8 blocks, xor tree as in block_reduce
      const int k = 8 * B + lane;
      double x0 = (lane < 8 && k < nb) ? bpart[2 * k] : 0.0;
      double x1 = (lane < 8 && k < nb) ? bpart[2 * k + 1] : 0.0;
      x0 = warp_sum(x0);
      x1 = warp_sum(x1);
      if (lane == 0) {
        l2[0][B] = x0;
        l2[1][B] = x1;
      }
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const double sqs = warp_fixed_sum(&l2[0][0], colgrid, 1);
      const double bgs = warp_fixed_sum(&l2[1][0], colgrid, 1);
      const double alse = warp_fixed_sum(spart, nspart, 2);       // as k_colreduce's scalars (stride 2)
      const double nbad = warp_fixed_sum(spart + 1, nspart, 2);
      if (threadIdx.x == 0) {
        ds->scratch[0] = nbad;   // count of non-finite rows
        ds->gnorm = sqrt(sqs);
        ds->alse = alse;
        ds->bgam = bgs;
        ds->value = bgs + eta * alse;
        if (save_ev0) {          // kept for a host read after later evals (otb_inner_iteration)
          ds->ev0[0] = ds->value;
          ds->ev0[1] = ds->gnorm;
          ds->ev0[2] = nbad;
        }
      }
    }
  }
}

// Single rank: the finish of test pass B (mode 0) or C (mode 1) in one
// kernel — blocks [0, col32) reduce the column partials (k_colreduce),
// blocks [col32, col32 + colgrid) do k_rows_post's work with its own thread
// mapping, and the last block combines — reproducing the summation trees of
// k_rows_post, k_colreduce and k_vec_post(POST_COLRES) exactly (same bits).
//   mode 0: er_i = a_i - rowsum_i; deficit = sum |er|; ec_j = b_j - colsum_j
//   mode 1: s8[0..6] = CTA scalar totals, s8[7] = sum (rowsum_i - a_i)^2,
//           col_sq = sum_j (colsum_j - b_j)^2
struct TestFinishIO {
  int mode;
  const double* colpart;   // [nparts][n]
  int nparts;
  int n;
  const double* b;
  double* ec;              // mode 0
  const double* rowpart;   // [m_loc][cl]
  int m_loc, cl;
  const double* a;
  int64_t row0;
  double* er;              // mode 0
  const double* spart;     // mode 1: [nspart][8] CTA scalars
  int nspart;
  int col32, colgrid;
  DevScalars* ds;
  double* bpart;           // col32 + colgrid doubles
};
__global__ void __launch_bounds__(256) k_test_finish(TestFinishIO io) {
  __shared__ double red[8 * 32];
  __shared__ double red2[2][kMaxWarps * 4];
  __shared__ double l2[512];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* bcol = io.bpart;
  double* brow = io.bpart + io.col32;
  if ((int)blockIdx.x < io.col32) {
    const double s = reduce_partials32(io.colpart, io.nparts, io.n, blockIdx.x * 32, red);
    if (threadIdx.x < 32) {
      const int j = blockIdx.x * 32 + lane;
      if (io.mode == 0) {
        if (j < io.n) io.ec[j] = io.b[j] - s;   // feasibility.py:65
      } else {
        double sq = 0.0;
        if (j < io.n) {
          const double e = s - io.b[j];
          sq = fma(e, e, sq);
        }
        sq = warp_sum(sq);
        if (lane == 0) bcol[blockIdx.x] = sq;
      }
    }
  } else {
    const int rb = blockIdx.x - io.col32;
    double s = 0.0;
    for (int i = rb * blockDim.x + threadIdx.x; i < io.m_loc; i += io.colgrid * blockDim.x) {
      double rs = 0.0;
      for (int q = 0; q < io.cl; ++q) rs += io.rowpart[(size_t)i * io.cl + q];
      const double ai = io.a[io.row0 + i];
      if (io.mode == 0) {
        const double e = ai - rs;
        io.er[i] = e;
        s += fabs(e);
      } else {
        const double e = rs - ai;
        s = fma(e, e, s);
      }
    }
    int ph = 0;
    double t[1] = {s};
    block_reduce<1, kSum>(t, &red2[0][0], ph, blockDim.x);
    if (threadIdx.x == 0) brow[rb] = t[0];
  }
  if (last_block(&io.ds->cnt[CNT_ROWS])) {
    if (io.mode == 1) {
      for (int B = warp; B < io.colgrid; B += 8) {   // the column residual's level 2 (k_vec_post blocks)
        const int k = 8 * B + lane;
        double x = (lane < 8 && k < io.col32) ? bcol[k] : 0.0;
        x = warp_sum(x);
        if (lane == 0) l2[B] = x;
      }
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const double rows = warp_fixed_sum(brow, io.colgrid, 1);
      if (io.mode == 0) {
        if (threadIdx.x == 0) {
          io.ds->scratch[2] = rows;
          io.ds->deficit = rows;   // feasibility.py:66
        }
      } else {
        const double colsq = warp_fixed_sum(l2, io.colgrid, 1);
        double v[7];
#pragma unroll
        for (int k = 0; k < 7; ++k) v[k] = warp_fixed_sum(io.spart + k, io.nspart, 8);
        if (threadIdx.x == 0) {
#pragma unroll
          for (int k = 0; k < 7; ++k) io.ds->s8[k] = v[k];
          io.ds->s8[7] = rows;
          io.ds->col_sq = colsq;
        }
      }
    }
  }
}

// Dot product x.y into *out (fixed-order), e.g. slope = g.dir.
__global__ void __launch_bounds__(256) k_dot(int n, const double* x, const double* y, DevScalars* ds,
                                             double* bpart, double* out) {
  __shared__ double red[2][kMaxWarps * 4];
  double s = 0.0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) s = fma(x[j], y[j], s);
  int ph = 0;
  double t[1] = {s};
  block_reduce<1, kSum>(t, &red[0][0], ph, blockDim.x);
  if (threadIdx.x == 0) bpart[blockIdx.x] = t[0];
  if (last_block(&ds->cnt[CNT_DOT])) {
    if (threadIdx.x < 32) {
      const double v = warp_fixed_sum(bpart, gridDim.x, 1);
      if (threadIdx.x == 0) *out = v;
    }
  }
}

// Sum of v into *out.
__global__ void __launch_bounds__(256) k_sum(int n, const double* v, DevScalars* ds, double* bpart, double* out) {
  __shared__ double red[2][kMaxWarps * 4];
  double s = 0.0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) s += v[j];
  int ph = 0;
  double t[1] = {s};
  block_reduce<1, kSum>(t, &red[0][0], ph, blockDim.x);
  if (threadIdx.x == 0) bpart[blockIdx.x] = t[0];
  if (last_block(&ds->cnt[CNT_SUM])) {
    if (threadIdx.x < 32) {
      const double v2 = warp_fixed_sum(bpart, gridDim.x, 1);
      if (threadIdx.x == 0) *out = v2;
    }
  }
}

// inner_newton.py:88: trial = gamma + t * direction.
__global__ void k_trial(int n, const double* gamma, const double* dir, double t, double* out) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    out[j] = gamma[j] + t * dir[j];
}

// Slope g.dir (as k_dot) fused with the first Armijo trial gamma + t dir
// (as k_trial): one pass over the three vectors, one launch less.
__global__ void __launch_bounds__(256) k_dot_trial(int n, const double* x, const double* y, DevScalars* ds,
                                                   double* bpart, double* out, const double* gamma, double t,
                                                   double* trial) {
  __shared__ double red[2][kMaxWarps * 4];
  double s = 0.0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const double yj = y[j];
    s = fma(x[j], yj, s);
    trial[j] = gamma[j] + t * yj;
  }
  int ph = 0;
  double tt[1] = {s};
  block_reduce<1, kSum>(tt, &red[0][0], ph, blockDim.x);
  if (threadIdx.x == 0) bpart[blockIdx.x] = tt[0];
  if (last_block(&ds->cnt[CNT_DOT])) {
    if (threadIdx.x < 32) {
      const double v = warp_fixed_sum(bpart, gridDim.x, 1);
      if (threadIdx.x == 0) *out = v;
    }
  }
}

// out = -v
__global__ void k_neg(int n, const double* v, double* out) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) out[j] = -v[j];
}

// v +/- (*total) / divisor   (sinkhorn.py:102-103 recentring)
__global__ void k_shift(int len, double* v, const double* total, double divisor, double sign) {
  const double drift = *total / divisor;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < len; j += gridDim.x * blockDim.x)
    v[j] = (sign > 0) ? v[j] + drift : v[j] - drift;
}

// Per-column post operations on a reduced vector buf (length n).
enum VecPost { POST_COPY = 0, POST_Y = 1, POST_EC = 2, POST_COLRES = 3, POST_WARMERR = 4 };

// POST_COPY:     out = buf
// POST_Y:        out = buf > 0 ? min(b / buf, 1) : 1        (feasibility.py:62)
// POST_EC:       out = b - buf                              (feasibility.py:65)
// POST_COLRES:   *out_s = sum (buf - b)^2                   (feasibility.py:111)
// POST_WARMERR:  *out_s = sum (buf - b)^2                   (sinkhorn.py:65)
__global__ void __launch_bounds__(256) k_vec_post(int mode, int n, const double* buf, const double* b,
                                                  double* out, DevScalars* ds, double* bpart, double* out_s) {
  __shared__ double red[2][kMaxWarps * 4];
  double s = 0.0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const double v = buf[j];
    if (mode == POST_COPY) out[j] = v;
    else if (mode == POST_Y) out[j] = (v > 0.0) ? fmin(div_rn(b[j], v), 1.0) : 1.0;
    else if (mode == POST_EC) out[j] = b[j] - v;
    else {
      const double e = v - b[j];
      s = fma(e, e, s);
    }
  }
  if (mode >= POST_COLRES) {
    int ph = 0;
    double t[1] = {s};
    block_reduce<1, kSum>(t, &red[0][0], ph, blockDim.x);
    if (threadIdx.x == 0) bpart[blockIdx.x] = t[0];
    if (last_block(&ds->cnt[CNT_VECPOST])) {
      if (threadIdx.x < 32) {
        const double v2 = warp_fixed_sum(bpart, gridDim.x, 1);
        if (threadIdx.x == 0) *out_s = v2;
      }
    }
  }
}

// Local-group all-reduce (otb_attach_group): out = op over ranks 0..N-1, in
// rank order, of the ranks' buffers (same device).  Every rank runs this on
// its own stream after waiting for the others' events, so every rank gets
// the same bits.
constexpr int kMaxGroup = 16;
struct LocalRed {
  const double* src[kMaxGroup];
  int nranks;
  int op;            // 0 sum, 2 max (NCCL op codes)
  int64_t count;
  double* out;
};
__global__ void __launch_bounds__(256) k_local_reduce(LocalRed r) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < r.count; j += (int64_t)gridDim.x * blockDim.x) {
    double t = r.src[0][j];
    for (int q = 1; q < r.nranks; ++q) {
      const double v = r.src[q][j];
      t = (r.op == 2) ? fmax(t, v) : t + v;
    }
    r.out[j] = t;
  }
}

// Multi-rank sparsify: [capacity-overflow flag, kept entries] as doubles
// after the n column sums, so that the all-reduce of d also tells every rank
// whether ANY rank must redo the pass (the collectives stay matched).
__global__ void k_sparsify_scalars(const DevScalars* ds, double* dst) {
  if (threadIdx.x == 0) {
    dst[0] = (ds->flags & 2) ? 1.0 : 0.0;
    dst[1] = (double)ds->nnzc;
  }
}

// Row-side finishes over local rows (rowpart [m_loc][cl]):
//   mode 0 (test pass B): er_i = a_i - rowsum_i, *out_s = sum |er_i|  (feasibility.py:64-66)
//   mode 1 (test pass C): *out_s = sum (rowsum_i - a_i)^2            (feasibility.py:110)
__global__ void __launch_bounds__(256) k_rows_post(int mode, int m_loc, int cl, const double* rowpart,
                                                   const double* a, int64_t row0, double* er, DevScalars* ds,
                                                   double* bpart, double* out_s) {
  __shared__ double red[2][kMaxWarps * 4];
  double s = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m_loc; i += gridDim.x * blockDim.x) {
    double rs = 0.0;
    for (int q = 0; q < cl; ++q) rs += rowpart[(size_t)i * cl + q];
    const double ai = a[row0 + i];
    if (mode == 0) {
      const double e = ai - rs;
      er[i] = e;
      s += fabs(e);
    } else {
      const double e = rs - ai;
      s = fma(e, e, s);
    }
  }
  int ph = 0;
  double t[1] = {s};
  block_reduce<1, kSum>(t, &red[0][0], ph, blockDim.x);
  if (threadIdx.x == 0) bpart[blockIdx.x] = t[0];
  if (last_block(&ds->cnt[CNT_ROWS])) {
    if (threadIdx.x < 32) {
      const double v = warp_fixed_sum(bpart, gridDim.x, 1);
      if (threadIdx.x == 0) *out_s = v;
    }
  }
}

// Warm-start gamma finish (sinkhorn.py:36-39, 54-58): combine the per-cluster
// (max, sum) pairs of each column.  mode 0: write M and S (multi-rank phase
// 1); mode 1: write gamma_j = eta (log b_j - (M + log S)) directly.
// One block = 32 columns; warp w folds partials w, w+8, ... with the online
// (max, sum) rule, then warp 0 folds the 8 warp results in order.
__global__ void __launch_bounds__(256) k_warm_gamma_combine(int mode, int n, const double* part, int nparts,
                                                            double* outM, double* outS, const double* log_b,
                                                            double eta, double* gamma) {
  __shared__ double rm[8 * 32], rs[8 * 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int j = blockIdx.x * 32 + lane;
  double M = -INFINITY, S = 0.0;
  if (j < n) {
    for (int c = warp; c < nparts; c += nw) {
      const double mc = part[((size_t)c * 2) * n + j];
      if (mc == -INFINITY) continue;
      const double sc = part[((size_t)c * 2 + 1) * n + j];
      if (mc > M) {
        S = S * exp(M - mc) + sc;
        M = mc;
      } else {
        S += sc * exp(mc - M);
      }
    }
  }
  rm[warp * 32 + lane] = M;
  rs[warp * 32 + lane] = S;
  __syncthreads();
  if (warp == 0 && j < n) {
    double Mg = -INFINITY;
    for (int w = 0; w < nw; ++w) Mg = fmax(Mg, rm[w * 32 + lane]);
    double Sg = 0.0;
    for (int w = 0; w < nw; ++w) {
      const double mw = rm[w * 32 + lane];
      if (mw != -INFINITY) Sg += rs[w * 32 + lane] * exp(mw - Mg);
    }
    if (mode == 0) {
      outM[j] = Mg;
      outS[j] = Sg;
    } else {
      gamma[j] = eta * (log_b[j] - (Mg + log(Sg)));
    }
  }
}

// Multi-rank: rescale the local S to the global max, before the sum reduce.
__global__ void k_warm_rescale(int n, const double* Mloc, const double* Mglob, double* S) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const double ml = Mloc[j];
    S[j] = (ml == -INFINITY) ? 0.0 : S[j] * exp(ml - Mglob[j]);
  }
}

__global__ void k_warm_gamma_post(int n, const double* M, const double* S, const double* log_b, double eta,
                                  double* gamma) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    gamma[j] = eta * (log_b[j] - (M[j] + log(S[j])));
}

// zeta_i = eta (log a_i - lse_i): the row potential of the accepted dual
// (bregman_outer.py:123-126 -> sinkhorn.py:47-51 on the cached lse).
// Kept-density estimate before a context's first sparsify (no history to
// choose dense P_rho or the bitmap runs from): the fraction of P >= rho
// (P > 0) over every `stride`-th local row of the stored P.  One count in
// *out (relaxed atomic: only compared against a threshold).
__global__ void k_density_sample(const double* __restrict__ P, int64_t ld, int m_loc, int n, int stride,
                                 const double* gnorm, double eta, double mn, double rho_host,
                                 unsigned long long* out) {
  const double rho = gnorm != nullptr ? (eta * *gnorm) / mn : rho_host;   // inner_newton.py:112-114
  unsigned long long cnt = 0;
  const int rows = (m_loc + stride - 1) / stride;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)rows * n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx / n) * stride, j = (int)(idx % n);
    const double p = P[(size_t)r * ld + j];
    cnt += (p >= rho && p > 0.0) ? 1ull : 0ull;
  }
  cnt = (unsigned long long)warp_sum_i((int)cnt);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(out, cnt);
}

__global__ void k_zeta_from_lse(int m_loc, const double* log_a, int64_t row0, const double* lse, double eta,
                                double* zeta) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m_loc; i += gridDim.x * blockDim.x)
    zeta[i] = eta * (log_a[row0 + i] - lse[i]);
}

// Test hook: CSR rows gathered into local-row order (int32 columns).
__global__ void k_csr_compact(int m_loc, const int64_t* row_start, const int* row_len, const int64_t* rowpre,
                              const uint16_t* cols, const double* vals, int32_t* out_cols, double* out_vals) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int r = gw; r < m_loc; r += nw) {
    const int64_t s = row_start[r], o = rowpre[r];
    for (int k = lane; k < row_len[r]; k += 32) {
      out_cols[o + k] = cols[s + k];
      out_vals[o + k] = vals[s + k];
    }
  }
}

}  // namespace otb

namespace otb {
// X^0 = a b^T in the log domain, clamped (bregman_outer.py:91-93, core.py:141-145).
__global__ void k_init_plan(double* X, int64_t ld, int m_loc, int n, const double* log_a, int64_t row0,
                            const double* log_b) {
  const int64_t total = (int64_t)m_loc * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx / n), j = (int)(idx % n);
    X[(size_t)r * ld + j] = fmax(log_a[row0 + r] + log_b[j], kLogFloor);
  }
}
// sinkhorn.py:41-43 scaled_plan_log, then core.py:141-145: log X + (zeta_i +
// gamma_j - C_ij)/eta, NaN / +inf counted in *bad, clamped at LOG_FLOOR.
__global__ void k_scaled_plan(const double* __restrict__ C, const double* __restrict__ X, int64_t ld, int m_loc, int n,
                              const double* __restrict__ zeta, const double* __restrict__ gamma, double eta,
                              double* __restrict__ out, unsigned int* bad) {
  const Divider DIV(eta);
  const int64_t total = (int64_t)m_loc * n;
  unsigned int nb = 0;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx / n), j = (int)(idx % n);
    const size_t o = (size_t)r * ld + j;
    const double v = X[o] + DIV((zeta[r] + gamma[j]) - C[o]);
    nb += (isnan(v) || v == INFINITY) ? 1u : 0u;
    out[o] = fmax(v, kLogFloor);
  }
  if (nb) atomicAdd(bad, nb);
}

// On-device instance construction: C_rj = sum_k (x_rk -
// y_jk)^2 over the coordinates in order (numpy's axis-sum of d*d), rows
// [row0, row0 + m_loc) of x; the local maximum goes to *peak (as ordered
// bits: C >= 0).  --fmad=false keeps every product and sum one rounding,
// so the matrix equals numpy's bit for bit.
__global__ void k_sq_dist(const double* __restrict__ x, const double* __restrict__ y, int m_loc, int n, int dim,
                          int64_t row0, double* __restrict__ C, int64_t ld, unsigned long long* peak) {
  const int64_t total = (int64_t)m_loc * n;
  double mx = 0.0;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx / n), j = (int)(idx % n);
    const double* xr = x + (row0 + r) * dim;
    const double* yj = y + (int64_t)j * dim;
    double acc = 0.0;
    for (int k = 0; k < dim; ++k) {
      const double d = xr[k] - yj[k];
      acc = (k == 0) ? d * d : acc + d * d;
    }
    C[(size_t)r * ld + j] = acc;
    mx = fmax(mx, acc);
  }
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) atomicMax(peak, (unsigned long long)__double_as_longlong(mx));
}

// C /= peak (core.py:174: cost / peak), skipped when peak == 0.
__global__ void k_scale_cost(double* C, int64_t ld, int m_loc, int n, double peak) {
  if (peak == 0.0) return;
  const Divider D(peak);
  const int64_t total = (int64_t)m_loc * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx / n), j = (int)(idx % n);
    C[(size_t)r * ld + j] = D(C[(size_t)r * ld + j]);
  }
}

// CSR export with the bitmap index (pair-layout runs, dense.cuh): kept
// entries per row, then, one warp per row walking its words in order, the
// kept entries of each lane's pair at their element position.
__global__ void k_bm_rownnz(const uint4* __restrict__ bm, int nq, int m_loc, int* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < m_loc; r += (gridDim.x * blockDim.x) >> 5) {
    int k = 0;
    for (int q = lane; q < nq; q += 32) {
      const uint4 w = bm[(size_t)r * nq + q];
      k += __popc(w.x) + __popc(w.y);
    }
    for (int o = 16; o > 0; o >>= 1) k += __shfl_xor_sync(0xffffffffu, k, o);
    if (lane == 0) cnt[r] = k;
  }
}

__global__ void k_bm_export(const uint4* __restrict__ bm, int nq, int m_loc, const int64_t* __restrict__ row_start,
                            const double* __restrict__ vals, const int64_t* __restrict__ rowpre,
                            int32_t* __restrict__ out_cols, double* __restrict__ out_vals) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < m_loc; r += (gridDim.x * blockDim.x) >> 5) {
    const double* vr = vals + row_start[r];
    int64_t o = rowpre[r];
    for (int q = 0; q < nq; ++q) {
      const uint4 w = bm[(size_t)r * nq + q];
      const unsigned k0 = (w.x >> lane) & 1u, k1 = (w.y >> lane) & 1u;
      const int64_t pos = o + __popc(w.x & lt) + __popc(w.y & lt);
      const double* e = vr + 2 * ((int)w.z + __popc((w.x | w.y) & lt));
      if (k0) {
        out_cols[pos] = 64 * q + 2 * lane;
        out_vals[pos] = e[0];
      }
      if (k1) {
        out_cols[pos + k0] = 64 * q + 2 * lane + 1;
        out_vals[pos + k0] = e[1];
      }
      o += __popc(w.x) + __popc(w.y);
    }
  }
}

// CSR export of a dense P_rho (window-cluster dense mode): a row's kept
// entries are its nonzeros (kept values are > 0), except the anchor row,
// stored whole like the reference's anchor_row (zeros included).
__global__ void k_dense_rownnz(const double* __restrict__ Pr, int64_t ld, int m_loc, int n, int64_t anchor_local,
                               int* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < m_loc; r += (gridDim.x * blockDim.x) >> 5) {
    int k = 0;
    if (r == anchor_local) {
      k = n;
    } else {
      for (int j = lane; j < n; j += 32) k += Pr[(size_t)r * ld + j] != 0.0;
      for (int o = 16; o > 0; o >>= 1) k += __shfl_xor_sync(0xffffffffu, k, o);
    }
    if (lane == 0) cnt[r] = k;
  }
}

__global__ void k_dense_export(const double* __restrict__ Pr, int64_t ld, int m_loc, int n, int64_t anchor_local,
                               const int64_t* __restrict__ rowpre, int32_t* __restrict__ out_cols,
                               double* __restrict__ out_vals) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < m_loc; r += (gridDim.x * blockDim.x) >> 5) {
    int64_t o = rowpre[r];
    for (int j0 = 0; j0 < n; j0 += 32) {
      const int j = j0 + lane;
      const double v = j < n ? Pr[(size_t)r * ld + j] : 0.0;
      const bool k = j < n && (r == anchor_local || v != 0.0);
      const unsigned b = __ballot_sync(0xffffffffu, k);
      if (k) {
        out_cols[o + __popc(b & lt)] = j;
        out_vals[o + __popc(b & lt)] = v;
      }
      o += __popc(b);
    }
  }
}

// Test hook for log_fast (common.cuh).
__global__ void k_selftest_log(const double* __restrict__ x, int64_t n, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = log_fast(x[i]);
}

// core.py:141-145 on an uploaded log plan in one pass: count NaN / +inf
// entries (InvalidCost) and clamp below at LOG_FLOOR (NaN stays NaN).
__global__ void k_check_clamp(double* __restrict__ X, int64_t ld, int m, int n, double floor_v,
                              unsigned long long* __restrict__ bad) {
  unsigned long long nb = 0;
  for (int r = blockIdx.x; r < m; r += gridDim.x) {   // one row per block step, columns by pairs
    double* row = X + (int64_t)r * ld;
    for (int j = 2 * threadIdx.x; j < n; j += 2 * blockDim.x) {
      if (j + 1 < n) {
        double2 v = *reinterpret_cast<double2*>(row + j);   // rows are 256-byte aligned, j even
        nb += (v.x != v.x || v.x == INFINITY) + (v.y != v.y || v.y == INFINITY);
        const bool c0 = v.x < floor_v, c1 = v.y < floor_v;
        if (c0 || c1) {
          v.x = c0 ? floor_v : v.x;
          v.y = c1 ? floor_v : v.y;
          *reinterpret_cast<double2*>(row + j) = v;
        }
      } else {
        const double v = row[j];
        nb += (v != v || v == INFINITY);
        if (v < floor_v) row[j] = floor_v;
      }
    }
  }
  nb = (unsigned long long)warp_sum_i((int)nb);
  if ((threadIdx.x & 31) == 0 && nb) atomicAdd(bad, nb);
}

// Test hook for exp_fast (common.cuh): out[i] = exp_fast(x_i) (exp() where
// the fast path does not apply), out[n + i] = exp(x_i).
__global__ void k_selftest_exp(const double* __restrict__ x, int64_t n, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    bool ok = true;
    const double f = exp_fast(x[i], ok);
    out[i] = ok ? f : exp(x[i]);
    out[n + i] = exp(x[i]);
  }
}

// Test hook for the table-driven exp_tab / log_tab of the dense passes
// (common.cuh), with the kernels' fallbacks: out[i] = exp, out[n + i] = log.
__global__ void k_selftest_tab(const double* __restrict__ x, int64_t n, double* __restrict__ out) {
  __shared__ double2 etab[128];
  __shared__ double4 ltab[128];
  if (threadIdx.x < 128) {
    etab[threadIdx.x] = kExp2Tab[threadIdx.x];
    ltab[threadIdx.x] = kLogTab[threadIdx.x];
  }
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    bool ok = true;
    const double e = exp_tab(x[i], ok, etab);
    out[i] = ok ? e : exp(x[i]);
    bool lok = true;
    const double l = log_tab(x[i], lok, ltab);
    out[n + i] = lok ? l : log_fast(x[i]);
  }
}

// Test hook for Divider (common.cuh): out_i = x_i / y.
__global__ void k_selftest_div(const double* __restrict__ x, int64_t n, double y, double* __restrict__ out) {
  const Divider D(y);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = D(x[i]);
}

}  // namespace otb
