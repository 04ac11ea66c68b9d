// Sparse Hessian-vector product (K4) and the device-resident CG loop (K5).
//
// CSR layout: every local row r owns one
// contiguous run [row_start[r], row_start[r] + row_len[r]) of 16-bit column
// indices and float64 values, ascending columns; the anchor row is stored
// dense and unnormalised (sparsify.py:125).  Runs of different rows are not
// in row order (chunked allocation), so a row prefix `rowpre` of lengths is
// built once per Newton step for nnz-balanced scheduling.
#pragma once

#include "common.cuh"

namespace otb {

struct Csr {
  const int64_t* row_start;
  const int* row_len;
  const int64_t* rowpre;   // m_loc + 1 prefix of row_len
  const uint16_t* cols;
  const double* vals;
  int m_loc;
  int64_t row0;
};

enum CgStatus { CG_RUN = 0, CG_DONE = 1, CG_NOTPD = 2, CG_MAXIT = 3, CG_INCONSISTENT = 4 };

struct CgState {
  double rs, curv, alpha, beta, target, bnorm, shift, res;
  long long iters, max_iters;
  int status, pad;
  unsigned int cnt[4];
};

// rowpre[r] = sum_{q<r} row_len[q]; single CTA (m_loc <= a few 1e5).
__global__ void k_row_prefix(const int* row_len, int m_loc, int64_t* rowpre) {
  __shared__ long long wsum[32];
  __shared__ long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int base = 0; base < m_loc; base += blockDim.x) {
    const int i = base + threadIdx.x;
    long long v = (i < m_loc) ? row_len[i] : 0;
    long long inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      long long w = (lane < nw) ? wsum[lane] : 0;
      long long wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long t = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += t;
      }
      if (lane < nw) wsum[lane] = wi - w;
    }
    __syncthreads();
    const long long excl = carry + wsum[warp] + inc - v;
    if (i < m_loc) rowpre[i] = excl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) rowpre[m_loc] = carry;
}

OTB_DEV int lower_bound_i64(const int64_t* a, int n, int64_t key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// ---------------------------------------------------------------- hess_apply
// sparsify.py:151-153 with SparseRowStochastic.matvec/rmatvec (64-78):
// y = P_rho^T (a * (P_rho v)).  One pass over each row: s_r = P_r . v from a
// shared-memory copy of v, then a_r s_r P_rj scattered into a shared-memory
// column accumulator.  All threads of the CTA work on the same row between
// two barriers, and a row has distinct columns, so the scatter needs no
// atomics.  Each CTA writes its accumulator as one partial row.
// With `update`, the CTA first forms v = r + beta p_prev (krylov.py:83) and
// stores its slice of v into p_cur.
struct HvArgs {
  Csr A;
  const double* a;
  int n;
  const double* v_src;     // used when !update
  const double* r;
  const double* p_prev;
  double* p_cur;
  int update;
  const CgState* st;       // nullptr: standalone product
  double* colpart;         // [gridDim][n]
};

__global__ void __launch_bounds__(512, 1) k_hv_smem(HvArgs h) {
  extern __shared__ __align__(16) double hsm[];
  if (h.st != nullptr && h.st->status != CG_RUN) return;
  const int n = h.n;
  const int npad = (n + 1) & ~1;
  double* vsm = hsm;
  double* acc = hsm + npad;
  double* slots = acc + npad;
  const int tid = threadIdx.x, nt = blockDim.x;
  const double beta = h.update ? h.st->beta : 0.0;
  const int sl0 = (int)(((int64_t)blockIdx.x * n) / gridDim.x);
  const int sl1 = (int)(((int64_t)(blockIdx.x + 1) * n) / gridDim.x);
  for (int j = tid; j < n; j += nt) {
    double v;
    if (h.update) {
      v = h.r[j] + beta * h.p_prev[j];
      if (j >= sl0 && j < sl1) h.p_cur[j] = v;
    } else {
      v = h.v_src[j];
    }
    vsm[j] = v;
    acc[j] = 0.0;
  }
  __syncthreads();
  const int64_t total = h.A.rowpre[h.A.m_loc];
  const int64_t lo = (total * blockIdx.x) / gridDim.x;
  const int64_t hi = (total * (blockIdx.x + 1)) / gridDim.x;
  const int rb = (blockIdx.x == 0) ? 0 : lower_bound_i64(h.A.rowpre, h.A.m_loc, lo);
  const int re = (blockIdx.x + 1 == gridDim.x) ? h.A.m_loc : lower_bound_i64(h.A.rowpre, h.A.m_loc, hi);
  int rphase = 0;
  for (int r = rb; r < re; ++r) {
    const int len = h.A.row_len[r];
    const int64_t st0 = h.A.row_start[r];
    const double* vals = h.A.vals + st0;
    const uint16_t* cols = h.A.cols + st0;
    double dot = 0.0;
#pragma unroll 4
    for (int k = tid; k < len; k += nt) dot = fma(vals[k], vsm[cols[k]], dot);
    double t[1] = {dot};
    block_reduce<1, kSum>(t, slots, rphase, nt);
    const double w = __ldg(h.a + h.A.row0 + r) * t[0];
#pragma unroll 4
    for (int k = tid; k < len; k += nt) {
      const int j = cols[k];
      acc[j] = acc[j] + vals[k] * w;
    }
  }
  __syncthreads();
  double* dst = h.colpart + (size_t)blockIdx.x * n;
  for (int j = tid; j < n; j += nt) dst[j] = acc[j];
}

// Warp-per-row variant for n too large for a shared accumulator: the
// scatter goes to global memory with fp64 RED (non-deterministic order).
struct HvAtomicArgs {
  Csr A;
  const double* a;
  const double* v;
  double* y;               // accumulated, zeroed by the consumer
  const CgState* st;
};

__global__ void __launch_bounds__(256) k_hv_atomic(HvAtomicArgs h) {
  if (h.st != nullptr && h.st->status != CG_RUN) return;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int r = gw; r < h.A.m_loc; r += nw) {
    const int len = h.A.row_len[r];
    const int64_t st0 = h.A.row_start[r];
    const double* vals = h.A.vals + st0;
    const uint16_t* cols = h.A.cols + st0;
    double dot = 0.0;
    for (int k = lane; k < len; k += 32) dot = fma(vals[k], __ldg(h.v + cols[k]), dot);
    dot = warp_sum(dot);
    const double w = __ldg(h.a + h.A.row0 + r) * dot;
    for (int k = lane; k < len; k += 32) atomicAdd(h.y + cols[k], vals[k] * w);
  }
}

// p_cur = r + beta p_prev (krylov.py:83), for the atomic variant.
__global__ void k_cg_p(int n, const double* r, const double* p_prev, double* p_cur, const CgState* st) {
  if (st->status != CG_RUN) return;
  const double beta = st->beta;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    p_cur[j] = r[j] + beta * p_prev[j];
}

// Column sums of the hv partials (or the RED accumulator) into `out`.
OTB_DEV double hv_column(int j, int n, const double* colpart, int nparts, double* yatomic) {
  if (yatomic != nullptr) {
    const double v = yatomic[j];
    yatomic[j] = 0.0;
    return v;
  }
  double s = 0.0;
  for (int c = 0; c < nparts; ++c) s += colpart[(size_t)c * n + j];
  return s;
}

// krylov.py:63-66 (ap = Hp + shift p; curvature = p.ap) and 70-75.
// `ysum` != nullptr: column sums already reduced (multi-rank, after the
// all-reduce); else reduce colpart / yatomic here.
struct CgApArgs {
  int n;
  const double* colpart;
  int nparts;
  double* yatomic;
  const double* ysum;
  const double* d;
  const double* p;
  double eta;
  double* ap;
  CgState* st;
  double* bpart;
};

__global__ void __launch_bounds__(256) k_cg_ap(CgApArgs c) {
  if (c.st->status != CG_RUN) return;
  __shared__ double red[2][32 * 4];
  const double shift = c.st->shift;
  double part = 0.0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < c.n; j += gridDim.x * blockDim.x) {
    const double y = c.ysum ? c.ysum[j] : hv_column(j, c.n, c.colpart, c.nparts, c.yatomic);
    const double pj = c.p[j];
    const double apj = div_rn(c.d[j] * pj - y, c.eta) + shift * pj;
    c.ap[j] = apj;
    part = fma(pj, apj, part);
  }
  int ph = 0;
  double t[1] = {part};
  block_reduce<1, kSum>(t, &red[0][0], ph, blockDim.x);
  if (threadIdx.x == 0) c.bpart[blockIdx.x] = t[0];
  if (last_block(&c.st->cnt[0])) {
    if (threadIdx.x < 32) {
      const double curv = warp_fixed_sum(c.bpart, gridDim.x, 1);
      if (threadIdx.x == 0) {
        CgState* s = c.st;
        s->curv = curv;
        if (curv <= 0.0) {
          s->status = (sqrt(s->rs) <= s->target) ? CG_DONE : CG_NOTPD;
          s->res = sqrt(s->rs);
        } else {
          s->alpha = s->rs / curv;
        }
      }
    }
  }
}

// krylov.py:76-84: x += alpha p, r -= alpha ap, convergence test, beta.
__global__ void __launch_bounds__(256) k_cg_update(int n, double* x, double* r, const double* p, const double* ap,
                                                   CgState* st, double* bpart) {
  if (st->status != CG_RUN) return;
  __shared__ double red[2][32 * 4];
  const double alpha = st->alpha;
  double part = 0.0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    x[j] = x[j] + alpha * p[j];
    const double rj = r[j] - alpha * ap[j];
    r[j] = rj;
    part = fma(rj, rj, part);
  }
  int ph = 0;
  double t[1] = {part};
  block_reduce<1, kSum>(t, &red[0][0], ph, blockDim.x);
  if (threadIdx.x == 0) bpart[blockIdx.x] = t[0];
  if (last_block(&st->cnt[1])) {
    if (threadIdx.x < 32) {
      const double rsn = warp_fixed_sum(bpart, gridDim.x, 1);
      if (threadIdx.x == 0) {
        st->iters += 1;
        if (sqrt(rsn) <= st->target) {
          st->rs = rsn;
          st->status = CG_DONE;
        } else {
          st->beta = rsn / st->rs;
          st->rs = rsn;
          if (st->iters >= st->max_iters) st->status = CG_MAXIT;
        }
        st->res = sqrt(st->rs);
      }
    }
  }
}

// krylov.py:51-67 set-up: x = 0, r = p = rhs, rs = r.r, stop target.
__global__ void __launch_bounds__(256) k_cg_init(int n, const double* rhs, double* x, double* r, double* p0,
                                                 CgState* st, double* bpart, double shift, double rel_tol,
                                                 long long max_iters) {
  __shared__ double red[2][32 * 4];
  double sq = 0.0, sm = 0.0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const double v = rhs[j];
    x[j] = 0.0;
    r[j] = v;
    p0[j] = v;
    sq = fma(v, v, sq);
    sm += v;
  }
  int ph = 0;
  double t[2] = {sq, sm};
  block_reduce<2, kSum>(t, &red[0][0], ph, blockDim.x);
  if (threadIdx.x == 0) {
    bpart[2 * blockIdx.x] = t[0];
    bpart[2 * blockIdx.x + 1] = t[1];
  }
  if (last_block(&st->cnt[2])) {
    if (threadIdx.x < 32) {
      const double rs = warp_fixed_sum(bpart, gridDim.x, 2);
      const double sum = warp_fixed_sum(bpart + 1, gridDim.x, 2);
      if (threadIdx.x == 0) {
        const double bnorm = sqrt(rs);
        st->rs = rs;
        st->bnorm = bnorm;
        st->shift = shift;
        st->target = rel_tol * bnorm;
        st->iters = 0;
        st->max_iters = max_iters;
        st->beta = 0.0;
        st->res = bnorm;
        if (shift == 0.0 && fabs(sum) > 1e-12 * fmax(1.0, bnorm)) st->status = CG_INCONSISTENT;
        else if (bnorm == 0.0) {
          st->status = CG_DONE;
          st->res = 0.0;
        } else if (max_iters <= 0) st->status = CG_MAXIT;
        else st->status = CG_RUN;
      }
    }
  }
}

// Standalone H v (+ shift v) for parity tests: out_j = (d v - y)/eta + shift v.
__global__ void k_hv_out(int n, const double* colpart, int nparts, double* yatomic, const double* d,
                         const double* v, double eta, double shift, double* out) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const double y = hv_column(j, n, colpart, nparts, yatomic);
    out[j] = div_rn(d[j] * v[j] - y, eta) + shift * v[j];
  }
}

}  // namespace otb
