// Sparse Hessian-vector product (K4) and the device-resident CG loop (K5).
//
// CSR layout: every local row r owns one
// contiguous run [row_start[r], row_start[r] + row_len[r]) of 16-bit column
// indices and float64 values, ascending columns, starting on an 8-entry
// boundary (so a thread can load 8 entries as one 16-byte vector of columns
// and four 16-byte vectors of values); the anchor row is stored dense and
// unnormalised (sparsify.py:125).  Runs are not in row order (chunked
// allocation); `rowpre` (prefix of row lengths) drives nnz-balanced
// scheduling.
//
// H v = (d * v - P^T (a * (P v))) / eta is applied in ONE pass over the
// CSR: the CTA's warps are split into NG groups, each group walks its own
// rows (s_r = P_r . v from a shared-memory copy of v, then a_r s_r P_rj
// scattered into the group's private shared-memory column accumulator —
// no atomics: within a group one row at a time, rows have distinct
// columns).  The next row's first chunk is prefetched into registers while
// the current row is reduced and scattered.  The group accumulators are
// summed and written as one partial row per CTA; partial rows are reduced
// in fixed order (deterministic).
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

namespace otb {

struct Csr {
  const int64_t* row_start;
  const int* row_len;
  const int64_t* rowpre;   // m_loc + 1 prefix of row_len
  const int* cta_rb;       // [nb + 1] nnz-balanced row bounds of the hv CTAs (or nullptr)
  const uint16_t* cols;
  const double* vals;
  int m_loc;
  int64_t row0;
};

enum CgStatus { CG_RUN = 0, CG_DONE = 1, CG_NOTPD = 2, CG_MAXIT = 3, CG_INCONSISTENT = 4 };

struct CgState {
  double rs, curv, alpha, beta, target, bnorm, shift, res;
  long long iters, max_iters;
  int status, precond;     // precond: Jacobi PCG (z = r / diag(H_rho + shift I)), else plain CG
  unsigned int cnt[4];
  double rz;               // PCG: r . z
};

constexpr int kCsrAlign = 8;   // row runs start on 8-entry boundaries

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

// Rows of CTA `b` out of `nb`: [rb, re), balanced by nonzeros.
OTB_DEV void cta_rows_search(const Csr& A, int b, int nb, int& rb, int& re) {
  const int64_t total = A.rowpre[A.m_loc];
  const int64_t lo = (total * b) / nb;
  const int64_t hi = (total * (b + 1)) / nb;
  rb = (b == 0) ? 0 : lower_bound_i64(A.rowpre, A.m_loc, lo);
  re = (b + 1 == nb) ? A.m_loc : lower_bound_i64(A.rowpre, A.m_loc, hi);
}

// The bounds are computed once per sparsify (k_cta_bounds): a binary search
// of dependent global loads at every kernel start costs several us.
OTB_DEV void cta_rows(const Csr& A, int b, int nb, int& rb, int& re) {
  if (A.cta_rb != nullptr) {
    rb = A.cta_rb[b];
    re = A.cta_rb[b + 1];
  } else {
    cta_rows_search(A, b, nb, rb, re);
  }
}

// by_rows: equal row counts — the bitmap kernels visit every column slot of
// a row whatever its nnz, so their cost is per row, not per entry.
__global__ void k_cta_bounds(Csr A, int nb, int* bounds, int by_rows) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b > nb) return;
  if (b == nb) {
    bounds[b] = A.m_loc;
    return;
  }
  if (by_rows) {
    bounds[b] = (int)(((int64_t)b * A.m_loc) / nb);
    return;
  }
  int rb, re;
  cta_rows_search(A, b, nb, rb, re);
  bounds[b] = rb;
}

// Sum over the threads of one warp group (TG threads, named barrier `bar`).
OTB_DEV double group_sum(double v, double* slots, int& phase, int tg, int TG, int bar) {
  v = warp_sum(v);
  double* s = slots + phase * 32;
  if ((tg & 31) == 0) s[tg >> 5] = v;
  bar_sync(bar, TG);
  double acc = s[0];
  for (int w = 1; w < (TG >> 5); ++w) acc += s[w];
  phase ^= 1;
  return acc;
}

// A thread's share of one chunk of a row: entries base + i*stride, i < 8.
// Consecutive threads hold consecutive entries, so for the dense-ish rows
// of P_rho the 32 lanes of a warp touch ~consecutive columns: the
// shared-memory gathers of v and the accumulator updates are (nearly)
// bank-conflict free, and the global loads are fully coalesced.
constexpr int kEA = 8;
struct Chunk {
  double v[kEA];
  int c[kEA];
};

OTB_DEV void load_chunk(const Csr& A, int64_t st0, int base, int stride, int len, Chunk& ch) {
#pragma unroll
  for (int i = 0; i < kEA; ++i) {
    const int k = base + i * stride;
    if (k < len) {
      ch.v[i] = A.vals[st0 + k];
      ch.c[i] = A.cols[st0 + k];
    } else {
      ch.v[i] = 0.0;     // contributes 0 * v[0] to the dot product
      ch.c[i] = 0;
    }
  }
}

OTB_DEV double chunk_dot(const Chunk& ch, const double* v) {
  double d = 0.0;
#pragma unroll
  for (int i = 0; i < kEA; ++i) d = fma(ch.v[i], v[ch.c[i]], d);
  return d;
}

// sparsify.py:78 product then sum: acc_j += val * (a_i s_i)
OTB_DEV void chunk_scatter(const Chunk& ch, int base, int stride, int len, double* acc, double w) {
#pragma unroll
  for (int i = 0; i < kEA; ++i) {
    if (base + i * stride < len) {
      const int j = ch.c[i];
      acc[j] = acc[j] + ch.v[i] * w;
    }
  }
}

// One CTA's share of y = P^T (a * (P v)): rows [rb, re) split round-robin
// over NG warp groups; `acc` holds NG accumulators of `npad` doubles.
OTB_DEV void hv_rows(const Csr& A, const double* a, const double* vsm, double* acc, int npad, int rb, int re,
                     int NG, double* gslots) {
  const int TG = blockDim.x / NG;
  const int g = threadIdx.x / TG, tg = threadIdx.x % TG;
  double* myacc = acc + (size_t)g * npad;
  double* slots = gslots + g * 64;
  const int bar = 1 + g;
  const int span = kEA * TG;     // entries covered by one chunk of the group
  int phase = 0;
  Chunk nx;
  int64_t nst = 0;
  int nlen = 0;
  int r = rb + g;
  if (r < re) {
    nst = A.row_start[r];
    nlen = A.row_len[r];
    load_chunk(A, nst, tg, TG, nlen, nx);
  }
  for (; r < re; r += NG) {
    const int64_t st0 = nst;
    const int len = nlen;
    const Chunk c0 = nx;
    Chunk c1;
    const int b1 = tg + span;
    load_chunk(A, st0, b1, TG, len, c1);
    const int rn = r + NG;
    if (rn < re) {                                   // prefetch the next row
      nst = A.row_start[rn];
      nlen = A.row_len[rn];
      load_chunk(A, nst, tg, TG, nlen, nx);
    }
    double dot = chunk_dot(c0, vsm) + chunk_dot(c1, vsm);
    for (int base = b1 + span; base < len + tg; base += span) {
      Chunk ct;
      load_chunk(A, st0, base, TG, len, ct);
      dot += chunk_dot(ct, vsm);
    }
    const double s_r = group_sum(dot, slots, phase, tg, TG, bar);
    const double w = __ldg(a + A.row0 + r) * s_r;    // sparsify.py:153: weights * pv
    chunk_scatter(c0, tg, TG, len, myacc, w);
    chunk_scatter(c1, b1, TG, len, myacc, w);
    for (int base = b1 + span; base < len + tg; base += span) {
      Chunk ct;
      load_chunk(A, st0, base, TG, len, ct);
      chunk_scatter(ct, base, TG, len, myacc, w);
    }
  }
}

// ------------------------------------------------------------ bitmap rows
// Second index over the same CSR values, written by k_sparsify: per local
// row, 16*NQ words of 64 columns (zero past n), each a uint4 {b0, b1, off,
// 0}.  Bit l of b0 (b1) marks column 64q+2l (64q+2l+1) as kept and `off`
// is the position, relative to the row start, of the word's first kept
// entry.  Values are in column order, so the entry of column 64q+2l+e sits
// at off + popc(b0 & lt) + popc(b1 & lt) + (e ? bit l of b0 : 0).
//
// hess_apply over it: thread (warp w, lane l) owns the columns
// 64(w + 16t) + 2l + e (t < NQ, e < 2), so its slices of v and of the
// accumulator live in registers.  Rows go R at a time: the words, row
// starts and a_r of the next R rows are staged in shared memory by
// cp.async while the current ones are processed; every thread issues the
// loads of all its kept values of the R rows at once (a warp's entries of
// one word are contiguous, so they coalesce), forms its partial dots, ONE
// block reduction yields the R row dots, and every thread adds
// val * a_r * dot_r to its own columns.  No shared-memory scatter, no
// atomics, rows summed in order (deterministic).  n <= 8192 (NQ <= 8).
constexpr int kMaxNQ = 8;

// Column ownership: thread (warp w, lane l) of a CTA with W = 16 warps owns
// the columns 64(w + W t) + 2l + e, t < NQ, e < 2; bitmap rows hold
// 16 NQ words.
template <int W>
OTB_DEV int bm_col(int t, int e) { return 64 * ((threadIdx.x >> 5) + W * t) + 2 * (threadIdx.x & 31) + e; }

OTB_DEV void cp_async(void* dst, const void* src, int bytes, bool ok) {
  // src-size 0 zero-fills the destination (rows past the CTA's range)
  if (bytes == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(ok ? 16 : 0)
                 : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(ok ? 8 : 0)
                 : "memory");
}
OTB_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
OTB_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Pair layout (dense.cuh, SparsifyIO): the lane's pair (columns 2l, 2l+1)
// of word w sits at 2 (w.z + popc(pairs below l)) of the row run, 16-byte
// aligned, with 0.0 for an unkept half.  The position is always inside the
// run or its padding (the value buffer has 16 entries of slack), so the load
// is issued unconditionally.
OTB_DEV unsigned bm_pairs(const uint4& w) { return w.x | w.y; }
OTB_DEV const double* bm_entry(const double* vr, const uint4& w, unsigned lt) {
  return vr + 2 * ((int)w.z + __popc(bm_pairs(w) & lt));
}
// Zero the loaded pair when the lane's pair is not in the run (it then read
// a later pair; no FP op on that data).
OTB_DEV void bm_select(const uint4& w, unsigned lb, double& e0, double& e1) {
  const bool kp = (bm_pairs(w) & lb) != 0u;
  e0 = kp ? e0 : 0.0;
  e1 = kp ? e1 : 0.0;
}

// ---- one pass, 16 warps: R rows per block reduction
template <int NQ>
struct BmCfg {
  static constexpr int R = NQ <= 4 ? 4 : 2;   // rows per block reduction
  static constexpr int NQP = 16 * NQ;         // words per row
};
constexpr int kBmStageBytes = 256 * 16 + 4 * 16;   // words of R rows, R row starts, R a_r
constexpr int kBmSmemBytes = 2 * kBmStageBytes;

// Words [woff, woff + NQP) of rows r0..r0+R-1 (row stride `stride` words).
template <int NQ>
OTB_DEV void bm_stage(const Csr& A, const uint4* bm, const double* a, int r0, int re, unsigned char* stage,
                      int stride, int woff) {
  constexpr int R = BmCfg<NQ>::R, NQP = BmCfg<NQ>::NQP;
  const int t = threadIdx.x;
  if (t < R * NQP) {
    const int k = t / NQP;
    const bool ok = r0 + k < re;
    cp_async(reinterpret_cast<uint4*>(stage) + t, ok ? bm + (size_t)(r0 + k) * stride + woff + (t - k * NQP) : bm,
             16, ok);
  } else if (t >= 256 && t < 256 + R) {
    const int k = t - 256;
    const bool ok = r0 + k < re;
    cp_async(stage + 256 * 16 + 8 * k, ok ? A.row_start + r0 + k : A.row_start, 8, ok);
  } else if (t >= 288 && t < 288 + R) {
    const int k = t - 288;
    const bool ok = r0 + k < re;
    cp_async(stage + 256 * 16 + 32 + 8 * k, ok ? a + A.row0 + r0 + k : a, 8, ok);
  }
  cp_async_commit();
}

// Row dots split over the column windows of a thread-block cluster: each
// CTA's partial dots of a batch go to every CTA of the cluster through DSMEM
// (remote stores + a release arrive on the peer's mbarrier), and every CTA
// adds the W partials in window order, so all windows apply the same dots.
// send(b) and recv(b) are split so that the exchange of batch b overlaps the
// loads and dots of batch b+1; four buffers / barriers rotate (a CTA can be
// at most three sends ahead of a peer's reads).
constexpr int kXBufs = 4;
struct ClusterDots {
  double* xbuf;     // [kXBufs][16][4]
  uint64_t* xbar;   // [kXBufs], initialised with W arrivals
  int W, cr, nsend, nrecv;
  int nthreads;     // threads taking part (the consumer warps)

  template <int R>
  OTB_DEV void send(const double (&v)[R]) {
    const int q = nsend % kXBufs;
    double* base = xbuf + q * 16 * 4;
    if (threadIdx.x < W) {            // thread rk serves cluster rank rk, in parallel
      const uint32_t rk = threadIdx.x;
      const uint32_t dst = mapa(smem_u32(base + cr * 4), rk);
#pragma unroll
      for (int k = 0; k < R; ++k) st_cluster_f64(dst + 8u * k, v[k]);
      mbar_arrive_remote(mapa(smem_u32(&xbar[q]), rk));
    }
    ++nsend;
  }
  template <int R>
  OTB_DEV void recv(double (&v)[R]) {
    const int q = nrecv % kXBufs;
    const uint32_t par = (uint32_t)((nrecv / kXBufs) & 1);
    const double* base = xbuf + q * 16 * 4;
    if (threadIdx.x == 0) {
      while (!mbar_try_wait_cluster(&xbar[q], par)) {
      }
    }
    bar_sync(1, nthreads);
#pragma unroll
    for (int k = 0; k < R; ++k) {
      double t = 0.0;
      for (int rk = 0; rk < W; ++rk) t += base[rk * 4 + k];
      v[k] = t;
    }
    ++nrecv;
  }
};

template <int NQ>
OTB_DEV void hv_bitmap_rows(const Csr& A, const uint4* __restrict__ bm, const double* __restrict__ a,
                            const double (&v)[2 * NQ], double (&acc)[2 * NQ], int rb, int re, double* slots,
                            unsigned char* ring, int stride = BmCfg<NQ>::NQP, int woff = 0) {
  constexpr int R = BmCfg<NQ>::R, NQP = BmCfg<NQ>::NQP;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lb = 1u << lane, lt = lb - 1u;
  int phase = 0, buf = 0;
  if (rb < re) bm_stage<NQ>(A, bm, a, rb, re, ring, stride, woff);
  cp_async_wait_all();
  __syncthreads();
  for (int r0 = rb; r0 < re; r0 += R, buf ^= 1) {
    if (r0 + R < re) bm_stage<NQ>(A, bm, a, r0 + R, re, ring + (buf ^ 1) * kBmStageBytes, stride, woff);
    const unsigned char* cur = ring + buf * kBmStageBytes;
    const uint4* wsm = reinterpret_cast<const uint4*>(cur);
    const int64_t* rsm = reinterpret_cast<const int64_t*>(cur + 256 * 16);
    const double* asm_ = reinterpret_cast<const double*>(cur + 256 * 16 + 32);
    double val[R][2 * NQ];
    double dot[R], ar[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const double* vr = A.vals + rsm[k];
      ar[k] = asm_[k];
#pragma unroll
      for (int t = 0; t < NQ; ++t) {
        const double2 e = __ldg(reinterpret_cast<const double2*>(bm_entry(vr, wsm[k * NQP + warp + 16 * t], lt)));
        val[k][2 * t] = e.x;
        val[k][2 * t + 1] = e.y;
      }
    }
#pragma unroll
    for (int k = 0; k < R; ++k) {
      dot[k] = 0.0;
#pragma unroll
      for (int t = 0; t < NQ; ++t) {
        bm_select(wsm[k * NQP + warp + 16 * t], lb, val[k][2 * t], val[k][2 * t + 1]);
        dot[k] = fma(val[k][2 * t], v[2 * t], dot[k]);
        dot[k] = fma(val[k][2 * t + 1], v[2 * t + 1], dot[k]);
      }
    }
    cp_async_wait_all();   // next stage lands before the barrier below publishes it
    block_sum_split<R>(dot, slots, phase, blockDim.x);
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const double w = ar[k] * dot[k];   // sparsify.py:153: weights * pv
#pragma unroll
      for (int i = 0; i < 2 * NQ; ++i) acc[i] = fma(val[k][i], w, acc[i]);
    }
  }
}

// ---- staged variant: values and words brought in by TMA
// One producer lane streams, for each batch of kStR rows, the row's run of
// values (or, in a cluster, the segment of this CTA's 4096-column window)
// and its bitmap words into a ring of shared-memory stages with 1-D bulk
// copies (cp.async.bulk, completion on the stage's mbarrier).  The 512
// consumer threads never touch global memory inside the row loop: offsets
// from the staged words, values from the staged run, select, dot, one
// split-shuffle block reduction (+ the cluster exchange), update of the
// owned columns.  The next stages are in flight meanwhile.
constexpr int kStR = 2;                      // rows per batch
constexpr int kStWords = 64;                 // staged words per row (one 4096-column window)
constexpr int kStRowVals = 4096 + 8;         // staged values per row (window + alignment slack)
constexpr int kStZero = 4096;                // zero pair in each row slot (never a copy target)
constexpr int kStHdrBytes = 128;
constexpr int kStBytes = kStR * kStWords * 16 + kStHdrBytes + kStR * kStRowVals * 8;
constexpr int kStConsumers = 512;
constexpr int kStThreads = kStConsumers + 32;   // + one producer warp

struct StHdr {
  int base[kStR];     // stage index of the row's entry 0 (row-relative offsets add to it)
  int count;          // valid rows in the batch
  int pad;
  double ar[kStR];    // a_r
};

struct StRing {
  unsigned char* mem;
  uint64_t* full;
  uint64_t* empty;
  int S;
  int stage;
  uint32_t phase;
  OTB_DEV unsigned char* at(int s) const { return mem + (size_t)s * kStBytes; }
  OTB_DEV void advance() {
    if (++stage == S) {
      stage = 0;
      phase ^= 1u;
    }
  }
};

OTB_DEV size_t st_smem_bytes(int S) { return (size_t)S * kStBytes + 2 * (size_t)S * 8; }

// Carve a ring of S stages at `p` (16-byte aligned); thread 0 initialises
// the barriers (the caller synchronises before use).
OTB_DEV StRing st_ring(unsigned char* p, int S, int consumers = kStConsumers) {
  StRing rg;
  rg.mem = p;
  rg.full = reinterpret_cast<uint64_t*>(p + (size_t)S * kStBytes);
  rg.empty = rg.full + S;
  rg.S = S;
  rg.stage = 0;
  rg.phase = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&rg.full[s], 1);
      mbar_init(&rg.empty[s], consumers);
    }
    fence_mbar_init();
  }
  if (threadIdx.x < S * kStR * 2) {   // the zero pairs read by lanes without a pair
    const int s = threadIdx.x / (kStR * 2), k = (threadIdx.x / 2) % kStR, h = threadIdx.x & 1;
    reinterpret_cast<double*>(rg.at(s) + kStR * kStWords * 16 + kStHdrBytes)[k * kStRowVals + kStZero + h] = 0.0;
  }
  return rg;
}

// Producer (the whole producer warp): batches of rows [rb, re).  NQP words
// per row are staged from word `woff` of each row (row stride `stride`
// words); the value segment is the row's whole run (last_window with
// woff == 0), or the entries of this window: from word woff's `off` to the
// next window's first word's `off` (the row length for the last window).
// The row metadata of 32 rows is fetched at once, one row per lane, so the
// per-batch work of lane 0 is a barrier wait and the bulk-copy issue.
OTB_DEV void st_produce(const Csr& A, const uint4* bm, const double* a, int rb, int re, int stride, int woff, int nqp,
                        bool last_window, StRing& rg) {
  const int lane = threadIdx.x & 31;
  for (int g0 = rb; g0 < re; g0 += 32) {
    const int r = g0 + lane;
    int64_t a0 = 0;
    int cnt = 0, off = 0;
    double ar = 0.0;
    if (r < re) {
      const int64_t st = A.row_start[r];
      // pair offsets -> doubles (row_len counts stored doubles)
      const int fo = (woff > 0) ? 2 * (int)bm[(size_t)r * stride + woff].z : 0;
      const int lo = last_window ? A.row_len[r] : 2 * (int)bm[(size_t)r * stride + woff + nqp].z;
      a0 = (st + fo) & ~(int64_t)1;                        // 16-byte aligned source
      cnt = (int)(((st + lo + 1) & ~(int64_t)1) - a0);
      off = (int)(st - a0);
      ar = a[A.row0 + r];
    }
    const int rows = min(32, re - g0);
    for (int k0 = 0; k0 < rows; k0 += kStR) {
      int64_t ka0[kStR];
      int kcnt[kStR], koff[kStR];
      double kar[kStR];
#pragma unroll
      for (int k = 0; k < kStR; ++k) {
        ka0[k] = __shfl_sync(0xffffffffu, a0, k0 + k);
        kcnt[k] = __shfl_sync(0xffffffffu, cnt, k0 + k);
        koff[k] = __shfl_sync(0xffffffffu, off, k0 + k);
        kar[k] = __shfl_sync(0xffffffffu, ar, k0 + k);
      }
      if (lane == 0) {
        mbar_wait(&rg.empty[rg.stage], rg.phase ^ 1u);
        unsigned char* sp = rg.at(rg.stage);
        StHdr* h = reinterpret_cast<StHdr*>(sp + kStR * kStWords * 16);
        double* vdst = reinterpret_cast<double*>(sp + kStR * kStWords * 16 + kStHdrBytes);
        uint32_t bytes = 0;
        int count = 0;
#pragma unroll
        for (int k = 0; k < kStR; ++k) {
          const bool ok = k0 + k < rows;
          h->base[k] = koff[k] + k * kStRowVals;
          h->ar[k] = kar[k];
          if (ok) {
            bytes += (uint32_t)kcnt[k] * 8u + (uint32_t)nqp * 16u;
            ++count;
          }
        }
        h->count = count;
        mbar_arrive_expect_tx(&rg.full[rg.stage], bytes);
#pragma unroll
        for (int k = 0; k < kStR; ++k) {
          if (k0 + k < rows) {
            if (kcnt[k] > 0)
              bulk_g2s(vdst + k * kStRowVals, A.vals + ka0[k], (uint32_t)kcnt[k] * 8u, &rg.full[rg.stage]);
            bulk_g2s(sp + k * kStWords * 16, bm + (size_t)(g0 + k0 + k) * stride + woff, (uint32_t)nqp * 16u,
                     &rg.full[rg.stage]);
          }
        }
      }
      rg.advance();
    }
  }
}

// Consumers (512 threads): the same batches.  Column 2l keeps e0, column
// 2l+1 keeps e1 (e0 when 2l is not kept); columns that are not kept carry
// 0, and fma(0, x, s) == s for finite x.
// One staged row against the thread's columns: select the pair of every
// word; accumulate the dot (DOT) or add val * w to the columns (!DOT).
template <int NQ, bool DOT, int CW = 16, bool CLAMP = true>
OTB_DEV void st_row(const uint4* words, const double* vals, int k, int base, unsigned lb, unsigned lt,
                    const double (&v)[2 * NQ], double (&acc)[2 * NQ], double& dot, double w,
                    double (*val)[2 * NQ] = nullptr) {
  const int warp = threadIdx.x >> 5;
  double d0 = 0.0, d1 = 0.0;   // two independent fma chains for the dot
#pragma unroll
  for (int t = 0; t < NQ; ++t) {
    const uint4 wd = words[k * kStWords + warp + CW * t];
    const unsigned pm = bm_pairs(wd);
    // window kernels: words past n are zero (off 0 lies before a later
    // window's segment); keep the address inside the row's stage slot —
    // their masks are 0.  Single CTA: off 0 is the row start, no clamp.
    int idx = base + 2 * ((int)wd.z + __popc(pm & lt));
    if constexpr (CLAMP) idx = min(max(idx, k * kStRowVals), (k + 1) * kStRowVals - 2);
    // a lane whose pair is not in the run reads the slot's zero pair
    idx = (pm & lb) ? idx : k * kStRowVals + kStZero;
    const double2 e = *reinterpret_cast<const double2*>(vals + idx);
    const double e0 = e.x, e1 = e.y;
    if constexpr (DOT) {
      d0 = fma(e0, v[2 * t], d0);
      d1 = fma(e1, v[2 * t + 1], d1);
      if (val != nullptr) {
        (*val)[2 * t] = e0;
        (*val)[2 * t + 1] = e1;
      }
    } else {
      acc[2 * t] = fma(e0, w, acc[2 * t]);
      acc[2 * t + 1] = fma(e1, w, acc[2 * t + 1]);
    }
  }
  if constexpr (DOT) dot += d0 + d1;
}

// Consumers (512 threads): the same batches.  Single CTA: the values of a
// batch stay in registers from the dot to the update and the stage is
// released right after the dots.  Cluster (CL): the exchange of batch b's
// window partials overlaps batch b+1 (send b, dots of b+1, receive b), and
// batch b is applied by re-reading its stage, released only then — no
// second register copy of the values.
template <int NQ, bool CL, int CW = 16>
OTB_DEV void st_consume(int rb, int re, const double (&v)[2 * NQ], double (&acc)[2 * NQ], double* slots, StRing& rg,
                        ClusterDots* cx) {
  constexpr int kCons = CW * 32;
  const int lane = threadIdx.x & 31;
  const unsigned lb = 1u << lane, lt = lb - 1u;
  int rphase = 0;
  int pstage = 0;          // CL: stage of the batch still to be applied
  bool have_prev = false;
  double pdot[kStR];
  for (int r0 = rb; r0 < re; r0 += kStR) {
    mbar_wait(&rg.full[rg.stage], rg.phase);
    const unsigned char* sp = rg.at(rg.stage);
    const uint4* words = reinterpret_cast<const uint4*>(sp);
    const StHdr* h = reinterpret_cast<const StHdr*>(sp + kStR * kStWords * 16);
    const double* vals = reinterpret_cast<const double*>(sp + kStR * kStWords * 16 + kStHdrBytes);
    const int count = h->count;
    double dot[kStR];
    if constexpr (CL) {
#pragma unroll
      for (int k = 0; k < kStR; ++k) {
        dot[k] = 0.0;
        if (k < count) st_row<NQ, true>(words, vals, k, h->base[k], lb, lt, v, acc, dot[k], 0.0);
      }
      block_sum_split<kStR>(dot, slots, rphase, kCons);
      cx->send<kStR>(dot);                 // this batch's window partials go out ...
      if (have_prev) {                     // ... while the previous batch's come in
        cx->recv<kStR>(pdot);
        const unsigned char* pp = rg.at(pstage);
        const uint4* pw = reinterpret_cast<const uint4*>(pp);
        const StHdr* ph = reinterpret_cast<const StHdr*>(pp + kStR * kStWords * 16);
        const double* pv = reinterpret_cast<const double*>(pp + kStR * kStWords * 16 + kStHdrBytes);
        double unused = 0.0;
#pragma unroll
        for (int k = 0; k < kStR; ++k)
          if (k < ph->count)
            st_row<NQ, false>(pw, pv, k, ph->base[k], lb, lt, v, acc, unused, ph->ar[k] * pdot[k]);
        mbar_arrive(&rg.empty[pstage]);
      }
#pragma unroll
      for (int k = 0; k < kStR; ++k) pdot[k] = dot[k];
      pstage = rg.stage;
      have_prev = true;
      rg.advance();
    } else {
      double val[kStR][2 * NQ], ar[kStR];
#pragma unroll
      for (int k = 0; k < kStR; ++k) {
        dot[k] = 0.0;
        ar[k] = 0.0;
#pragma unroll
        for (int i = 0; i < 2 * NQ; ++i) val[k][i] = 0.0;
        if (k < count) {
          ar[k] = h->ar[k];
          st_row<NQ, true, CW, false>(words, vals, k, h->base[k], lb, lt, v, acc, dot[k], 0.0, &val[k]);
        }
      }
      mbar_arrive(&rg.empty[rg.stage]);   // stage consumed; values live on in registers
      rg.advance();
      block_sum_split<kStR>(dot, slots, rphase, kCons);
#pragma unroll
      for (int k = 0; k < kStR; ++k) {
        const double w = ar[k] * dot[k];   // sparsify.py:153: weights * pv
#pragma unroll
        for (int i = 0; i < 2 * NQ; ++i) acc[i] = fma(val[k][i], w, acc[i]);
      }
    }
  }
  if constexpr (CL) {
    if (have_prev) {
      cx->recv<kStR>(pdot);
      const unsigned char* pp = rg.at(pstage);
      const uint4* pw = reinterpret_cast<const uint4*>(pp);
      const StHdr* ph = reinterpret_cast<const StHdr*>(pp + kStR * kStWords * 16);
      const double* pv = reinterpret_cast<const double*>(pp + kStR * kStWords * 16 + kStHdrBytes);
      double unused = 0.0;
#pragma unroll
      for (int k = 0; k < kStR; ++k)
        if (k < ph->count) st_row<NQ, false>(pw, pv, k, ph->base[k], lb, lt, v, acc, unused, ph->ar[k] * pdot[k]);
      mbar_arrive(&rg.empty[pstage]);
    }
  }
}

// Variant code of the hess_apply kernels: 0 group smem accumulators,
// 1..8 bitmap with NQ = V words per warp (cp.async-staged words, loads from
// global), 9..12 TMA-staged bitmap (n <= 4096) with NQ = V - 8.  (32
// consumer warps + the producer would exceed 1024 threads per CTA.)
constexpr int kHvVariants = kMaxNQ + 5;
template <int V>
struct HvVar {
  static constexpr bool kBitmap = V > 0;
  static constexpr bool kStaged = V > 8;
  static constexpr int CW = 16;                               // consumer warps
  static constexpr int NQ = V > 8 ? V - 8 : (V > 0 ? V : 1);
  static constexpr int W = CW;
  static constexpr int kThreads = V > 8 ? CW * 32 + 32 : 512;
};

// Partial row of y = P^T (a * (P v)) over this CTA's rows, bitmap variants:
// v read from shared memory (vsm), result to dst (its own columns).
template <int V>
OTB_DEV void hv_bitmap_partial(const Csr& A, const uint4* bm, const double* a, const double* vsm, int n, int rb,
                               int re, double* slots, unsigned char* scratch, double* dst) {
  constexpr int NQ = HvVar<V>::NQ, W = HvVar<V>::W;
  double vr[2 * NQ], ar[2 * NQ];
#pragma unroll
  for (int i = 0; i < 2 * NQ; ++i) {
    const int j = bm_col<W>(i >> 1, i & 1);
    vr[i] = (j < n) ? vsm[j] : 0.0;
    ar[i] = 0.0;
  }
  hv_bitmap_rows<NQ>(A, bm, a, vr, ar, rb, re, slots, scratch);
#pragma unroll
  for (int i = 0; i < 2 * NQ; ++i) {
    const int j = bm_col<W>(i >> 1, i & 1);
    if (j < n) dst[j] = ar[i];
  }
}

// Staged variant of hv_bitmap_partial: the producer warp streams, the 512
// consumer threads compute; `rg` persists across calls (ring position).
template <int V>
// upd (persistent CG): vsm holds the previous direction and the CG update
// p = r + beta p (krylov.py:83) is done here, by the thread that owns the
// column, instead of in a separate pass over all n.
OTB_DEV void hv_staged_partial(const Csr& A, const uint4* bm, const double* a, double* vsm, int n, int nq, int rb,
                               int re, double* slots, StRing& rg, double* dst, const double* rsm = nullptr,
                               double beta = 0.0, bool upd = false) {
  constexpr int NQ = HvVar<V>::NQ, CW = HvVar<V>::CW;
  if (threadIdx.x >= CW * 32) {
    st_produce(A, bm, a, rb, re, nq, 0, CW * NQ, true, rg);
    return;
  }
  double vr[2 * NQ], ar[2 * NQ];
#pragma unroll
  for (int i = 0; i < 2 * NQ; ++i) {
    const int j = bm_col<CW>(i >> 1, i & 1);
    double v = 0.0;
    if (j < n) {
      v = vsm[j];
      if (upd) {
        v = rsm[j] + beta * v;   // krylov.py:83
        vsm[j] = v;
      }
    }
    vr[i] = v;
    ar[i] = 0.0;
  }
  st_consume<NQ, false, CW>(rb, re, vr, ar, slots, rg, nullptr);
#pragma unroll
  for (int i = 0; i < 2 * NQ; ++i) {
    const int j = bm_col<CW>(i >> 1, i & 1);
    if (j < n) dst[j] = ar[i];
  }
}

// Shared-memory layout of the group hv: v[npad] | acc[NG][npad] | slots.
OTB_DEV size_t hv_smem_doubles(int npad, int NG) { return (size_t)npad * (1 + NG) + 16 * 64; }

struct HvArgs {
  Csr A;
  const double* a;
  int n;
  int ng;
  const double* v_src;     // used when !update
  const double* r;
  const double* p_prev;
  double* p_cur;
  int update;
  const CgState* st;       // nullptr: standalone product
  double* colpart;         // [gridDim][n]
  const uint4* bm;         // bitmap index (NQ > 0)
  int nq;
  int nwin;                // window-cluster variant: CTAs per cluster
  int64_t ld;              // window-cluster dense mode: row stride of the dense P_rho (A.vals)
};

// Standalone hess_apply partials (multi-rank CG iterations, otb_hess_apply).
template <int V>
__global__ void __launch_bounds__(HvVar<V>::kThreads, 1) k_hv_grp(HvArgs h) {
  extern __shared__ __align__(16) double hsm[];
  if (h.st != nullptr && h.st->status != CG_RUN) return;
  const int n = h.n, npad = (n + 1) & ~1, NG = h.ng;
  double* vsm = hsm;
  double* acc = hsm + npad;
  double* gslots = acc + (size_t)npad * NG;
  const double beta = h.update ? h.st->beta : 0.0;
  const int sl0 = (int)(((int64_t)blockIdx.x * n) / gridDim.x);
  const int sl1 = (int)(((int64_t)(blockIdx.x + 1) * n) / gridDim.x);
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double v;
    if (h.update) {
      v = h.r[j] + beta * h.p_prev[j];       // krylov.py:83
      if (j >= sl0 && j < sl1) h.p_cur[j] = v;
    } else {
      v = h.v_src[j];
    }
    vsm[j] = v;
  }
  int rb, re;
  cta_rows(h.A, blockIdx.x, gridDim.x, rb, re);
  double* dst = h.colpart + (size_t)blockIdx.x * n;
  if constexpr (HvVar<V>::kStaged) {
    StRing rg = st_ring(reinterpret_cast<unsigned char*>(gslots + 16 * 64), 2, HvVar<V>::CW * 32);
    __syncthreads();
    hv_staged_partial<V>(h.A, h.bm, h.a, vsm, n, h.nq, rb, re, gslots, rg, dst);
  } else if constexpr (HvVar<V>::kBitmap) {
    __syncthreads();
    hv_bitmap_partial<V>(h.A, h.bm, h.a, vsm, n, rb, re, gslots, reinterpret_cast<unsigned char*>(gslots + 16 * 64),
                        dst);
  } else {
    for (int j = threadIdx.x; j < npad * NG; j += blockDim.x) acc[j] = 0.0;
    __syncthreads();
    hv_rows(h.A, h.a, vsm, acc, npad, rb, re, NG, gslots);
    __syncthreads();
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      double t = acc[j];
      for (int g = 1; g < NG; ++g) t += acc[(size_t)g * npad + j];
      dst[j] = t;
    }
  }
}

// Window-cluster hess_apply for n > 8192 (configs 4-5): a cluster of W
// CTAs shares one row block; CTA rank q owns window q = bitmap words
// [WW q, WW (q + 1)) of every row, WW = 16 NQ words = 1024 NQ columns (NQ
// words per consumer warp, v and the accumulator in registers).  W and NQ are
// chosen at context creation so the clusters that are co-resident cover the
// most SMs per window column (otb.cu, hv geometry).
//
// The row dot of row k needs all W windows' partials, so a plain schedule
// (dots, exchange, update) stalls every row on the slowest CTA of the
// cluster.  Here the exchange is decoupled by D rows:
//   step k: (a) issue the global (L2) loads of row k-D's values at the pair
//               positions saved when its dots were formed,
//           (b) row k from the TMA ring: partial dots from shared memory,
//               pair positions saved (uint16, registers), stage released,
//               CTA sum, partial sent to every peer (DSMEM + remote arrive),
//           (c) receive row k-D's W partials (window order), apply
//               a_r * dot_r * P_rj to the owned columns.
// Row k-D's values were brought to the SM by TMA D rows earlier, so the
// re-read is an L2 hit; HBM sees each value once.  The ring holds only the
// rows in flight (loads + dots); the exchange waits hold no stage.  Rows are
// applied in order, partials summed in window order: deterministic.
// kept density from which sparsify writes P_rho dense (OTB_HV_DENSE forces either).  0: always.
// The bitmap kernel visits every column slot of a row whatever is kept, so its time does not fall
// with the density (tools/hv_density_sweep.py: config 4, 37% -> 18% kept: 2.37 ms flat, config 5
// 76% -> 46%: 5.6 -> 5.5 ms) and the dense kernel's 1.37 ms / 3.13 ms wins at every density
// (sparsify too: 5.1 against 7.2 ms at config 4).  The bitmap runs remain the format when the
// eval's P is not stored (OTB_STORE_P=0) and the comparison format of the tests.
constexpr double kDenseRhoMin = 0.0;
constexpr int kWcD = 4;                  // exchange lookahead (rows)
constexpr int kWcX = 2 * kWcD + 2;       // exchange buffers (>= 2 D + 1: see the note in wc_consume)
constexpr int kWcMaxW = 16;
constexpr int kWcMaxStages = 16;   // ring stages of the window-cluster kernels
constexpr int kWcHdr = 32;

template <int NQ>
struct WcGeo {
  static constexpr int WW = 16 * NQ;                  // words per window
  static constexpr int kVals = 1024 * NQ + 8;         // staged values per row (window + zero pair + slack)
  static constexpr int kZero = 1024 * NQ;             // zero pair (never a copy target)
  static constexpr int kStage = WW * 16 + kWcHdr + kVals * 8;
  static constexpr int kVsm = 1024 * NQ * 8;          // the window of v
};

struct WcHdr {
  long long st;      // row_start of the row (doubles)
  double ar;         // a_r
  int base;          // stage value index of the row's pair 0 (= -2 off(first word))
  int pad[3];
};

__host__ __device__ inline size_t wc_smem_bytes(int nqw, int stage_bytes, int S) {
  return (size_t)1024 * nqw * 8 + (size_t)S * stage_bytes + 2 * (size_t)S * 8;
}

// DENSE: the rows are the dense P_rho of sparsify's dense mode (vals = its
// base, row stride ld): the window is copied as is (no words), and a value's
// position is its column.
template <int NQ, bool DENSE>
OTB_DEV void wc_produce(const Csr& A, const uint4* bm, const double* a, int rb, int re, int stride, int woff,
                        bool last_window, unsigned char* ring, uint64_t* full, uint64_t* empty, int S,
                        int64_t ld, int wcols) {
  using G = WcGeo<NQ>;
  const int lane = threadIdx.x & 31;
  int stage = 0;
  uint32_t phase = 0;
  for (int g0 = rb; g0 < re; g0 += 32) {
    const int r = g0 + lane;
    long long st = 0, src = 0;
    int cnt = 0, base = 0;
    double ar = 0.0;
    if (r < re) {
      if constexpr (DENSE) {
        st = (long long)r * ld + 64LL * woff;   // window start (column 64 woff)
        src = st;
        cnt = wcols;
        base = 0;
      } else {
        st = A.row_start[r];
        const int fo = (woff > 0) ? 2 * (int)bm[(size_t)r * stride + woff].z : 0;
        const int lo = last_window ? A.row_len[r] : 2 * (int)bm[(size_t)r * stride + woff + G::WW].z;
        src = st + fo;                     // even: runs start on 8-entry boundaries, offsets count pairs
        cnt = max(lo - fo, 0);
        base = -fo;
      }
      ar = a[A.row0 + r];
    }
    const int rows = min(32, re - g0);
    for (int k = 0; k < rows; ++k) {
      const long long kst = __shfl_sync(0xffffffffu, st, k);
      const long long ksrc = __shfl_sync(0xffffffffu, src, k);
      const int kcnt = __shfl_sync(0xffffffffu, cnt, k);
      const int kbase = __shfl_sync(0xffffffffu, base, k);
      const double kar = __shfl_sync(0xffffffffu, ar, k);
      if (lane == 0) {
        mbar_wait(&empty[stage], phase ^ 1u);
        unsigned char* sp = ring + (size_t)stage * G::kStage;
        WcHdr* h = reinterpret_cast<WcHdr*>(sp + G::WW * 16);
        double* vdst = reinterpret_cast<double*>(sp + G::WW * 16 + kWcHdr);
        h->st = kst;
        h->ar = kar;
        h->base = kbase;
        mbar_arrive_expect_tx(&full[stage], (uint32_t)kcnt * 8u + (DENSE ? 0u : (uint32_t)G::WW * 16u));
        if (kcnt > 0) bulk_g2s(vdst, A.vals + ksrc, (uint32_t)kcnt * 8u, &full[stage]);
        if (!DENSE) bulk_g2s(sp, bm + (size_t)(g0 + k) * stride + woff, (uint32_t)G::WW * 16u, &full[stage]);
      }
      if (++stage == S) {
        stage = 0;
        phase ^= 1u;
      }
    }
  }
}

// The CTA's partial of row k's dot, sent to the W peers.  Every warp sums
// its lanes, writes the warp partial to slot buffer k mod 8 and ARRIVES on
// named barrier 2 + (k mod 8); only the row's reducer warp (k mod 16) waits
// there and forms the CTA partial with the same tree as block_reduce (the
// same bits), its lanes q < W sending it to peer q.  The other 15 warps go
// straight on to the next row.  Reuse of buffer / barrier k mod 8 at row
// k + 8: a warp at the dots of row k + 8 has done the update of row
// k + 8 - D (D <= 4), which needed row k's full dot, i.e. row k's reducer
// has read its slots and passed its barrier.
constexpr int kWcNB = 8;
OTB_DEV void wc_send_partial(double v, int k, double* slots, double* xbuf, uint64_t* xbar, int W, int cr) {
  static_assert(kStConsumers == 512 && kWcD < kWcNB, "reducer rotation assumes 16 consumer warps");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double ws = warp_sum(v);
  double* sl = slots + (k & (kWcNB - 1)) * 16;
  if (lane == 0) sl[warp] = ws;
  const int bid = 2 + (k & (kWcNB - 1));
  if (warp == (k & 15)) {
    bar_sync(bid, kStConsumers);
    const double t = warp_sum(lane < 16 ? sl[lane] : 0.0);
    if (lane < W) {   // lane q serves peer q, in parallel
      const int q = k % kWcX;
      st_async_f64(mapa(smem_u32(xbuf + q * kWcMaxW + cr), (uint32_t)lane), t, mapa(smem_u32(&xbar[q]), (uint32_t)lane));
    }
  } else {
    bar_arrive(bid, kStConsumers);
  }
}

// Dense P_rho consumers, values KEPT in registers: row k's window values
// are read from the stage once (dots), kept in a register slot, and applied
// to the accumulator when row k's full dot arrives D rows later — no second
// read of the values at all (HBM and L2 see each value once).  D = 1: the
// exchange of row k overlaps the dots of row k+1; two register slots of
// 2 NQ doubles.  Same per-thread sums and row order as wc_consume: the same
// bits.
template <int NQ>
OTB_DEV void wc_consume_keep(int cnt, const double* vsm, double (&acc)[2 * NQ], unsigned char* ring, uint64_t* full,
                             uint64_t* empty, int S, double* xbuf, uint64_t* xbar, int W, int cr, double* slots,
                             WcHdr* hring) {
  using G = WcGeo<NQ>;
  constexpr int D = 1;
  const int lane = threadIdx.x & 31;
  int stage = 0;
  uint32_t phase = 0;
  double kv[D + 1][2 * NQ];
  double kar[D + 1];
  for (int k0 = 0; k0 < cnt + D; k0 += D + 1) {
#pragma unroll
    for (int j = 0; j <= D; ++j) {
      const int k = k0 + j, ku = k - D;
      if (k < cnt) {   // dots of row k; its values stay in slot j
        mbar_wait(&full[stage], phase);
        const unsigned char* sp = ring + (size_t)stage * G::kStage;
        const WcHdr* h = reinterpret_cast<const WcHdr*>(sp + G::WW * 16);
        const double* sv = reinterpret_cast<const double*>(sp + G::WW * 16 + kWcHdr);
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int t = 0; t < NQ; ++t) {
          const double2 x = *reinterpret_cast<const double2*>(sv + bm_col<16>(t, 0));
          const double2 vv = *reinterpret_cast<const double2*>(vsm + bm_col<16>(t, 0));
          kv[j][2 * t] = x.x;
          kv[j][2 * t + 1] = x.y;
          d0 = fma(x.x, vv.x, d0);
          d1 = fma(x.y, vv.y, d1);
        }
        kar[j] = h->ar;
        mbar_arrive(&empty[stage]);
        if (++stage == S) {
          stage = 0;
          phase ^= 1u;
        }
        wc_send_partial(d0 + d1, k, slots, xbuf, xbar, W, cr);
      }
      if (ku >= 0 && ku < cnt) {   // row ku (slot (j + 1) mod (D + 1)): full dot, then the update
        const int ju = (j + 1) % (D + 1);   // static after unrolling
        const int q = ku % kWcX;
        mbar_wait(&xbar[q], (uint32_t)((ku / kWcX) & 1));
        double dot = (lane < W) ? xbuf[q * kWcMaxW + lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        if (threadIdx.x == 0) mbar_arrive_expect_tx(&xbar[q], 8u * (uint32_t)W);
        const double w = kar[ju] * dot;   // sparsify.py:153: weights * pv
#pragma unroll
        for (int i = 0; i < 2 * NQ; ++i) acc[i] = fma(kv[ju][i], w, acc[i]);
      }
    }
  }
}

// Consumers (512 threads).  Exchange buffer safety: a CTA at dot row k has
// received row k-D, so every peer has sent row >= k-D and (being at dot row
// >= k-D) has received rows <= k-2D-1... a sender of row k reuses buffer
// k % X, last used for row k-X; with X >= 2D+1 every CTA has consumed row k-X
// before any peer can send row k.
template <int NQ, bool DENSE>
OTB_DEV void wc_consume(int cnt, const double* __restrict__ vals, const double* vsm, double (&acc)[2 * NQ],
                        unsigned char* ring, uint64_t* full, uint64_t* empty, int S, double* xbuf, uint64_t* xbar,
                        int W, int cr, double* slots, WcHdr* hring, int lim) {
  // lim (DENSE): columns of this window inside the matrix (the last window's
  // tail is neither staged nor loaded)
  const bool wfull = lim >= 1024 * NQ;
  using G = WcGeo<NQ>;
  constexpr int D = kWcD;
  constexpr int NI = (NQ + 1) / 2;   // uint32 words of packed uint16 pair positions per row
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lb = 1u << lane, lt = lb - 1u;
  int stage = 0;
  uint32_t phase = 0;
  uint32_t pidx[D][NI];
#pragma unroll
  for (int j = 0; j < D; ++j)
#pragma unroll
    for (int i = 0; i < NI; ++i) pidx[j][i] = 0xffffffffu;
  for (int k0 = 0; k0 < cnt + D; k0 += D) {
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const int k = k0 + j, ku = k - D;
      // (a) row ku: loads of its values from L2 (positions saved in slot j)
      double e[2 * NQ];
      double ar_u = 0.0;
      const bool upd = ku >= 0 && ku < cnt;
      if (upd) {
        const WcHdr hu = hring[warp * (D + 1) + ku % (D + 1)];   // this warp's copy (no CTA barrier per row)
        ar_u = hu.ar;
        const double* vr = vals + hu.st;
        if constexpr (DENSE) {
          if (wfull) {   // fixed positions: no per-value test outside the last window
#pragma unroll
            for (int t = 0; t < NQ; ++t) {
#ifdef OTB_HV_NO_REREAD   // experiment: timing without the L2 re-read (wrong results)
              const double2 x = make_double2(0.0, 0.0);
#else
              const double2 x = __ldg(reinterpret_cast<const double2*>(vr + bm_col<16>(t, 0)));
#endif
              e[2 * t] = x.x;
              e[2 * t + 1] = x.y;
            }
          } else {
#pragma unroll
            for (int t = 0; t < NQ; ++t) {
              double2 x = make_double2(0.0, 0.0);
              if (bm_col<16>(t, 0) < lim) x = __ldg(reinterpret_cast<const double2*>(vr + bm_col<16>(t, 0)));
              e[2 * t] = x.x;
              e[2 * t + 1] = x.y;
            }
          }
        } else {
#pragma unroll
          for (int t = 0; t < NQ; ++t) {
            double2 x = make_double2(0.0, 0.0);
            const uint32_t p = (pidx[j][t >> 1] >> (16 * (t & 1))) & 0xffffu;
            if (p != 0xffffu) x = __ldg(reinterpret_cast<const double2*>(vr + 2 * (int)p));
            e[2 * t] = x.x;
            e[2 * t + 1] = x.y;
          }
        }
      }
      // (b) row k: partial dots from the staged window, positions saved
      if (k < cnt) {
        mbar_wait(&full[stage], phase);
        const unsigned char* sp = ring + (size_t)stage * G::kStage;
        const uint4* words = reinterpret_cast<const uint4*>(sp);
        const WcHdr* h = reinterpret_cast<const WcHdr*>(sp + G::WW * 16);
        const double* sv = reinterpret_cast<const double*>(sp + G::WW * 16 + kWcHdr);
        const int base = h->base;
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int i = 0; i < NI; ++i) pidx[j][i] = 0xffffffffu;
        if constexpr (DENSE) {   // (the stage tail past the matrix was zeroed at start)
#pragma unroll
          for (int t = 0; t < NQ; ++t) {
            const double2 x = *reinterpret_cast<const double2*>(sv + bm_col<16>(t, 0));
            const double2 vv = *reinterpret_cast<const double2*>(vsm + bm_col<16>(t, 0));
            d0 = fma(x.x, vv.x, d0);
            d1 = fma(x.y, vv.y, d1);
          }
        }
#pragma unroll
        for (int t = 0; t < (DENSE ? 0 : NQ); ++t) {
          const uint4 wd = words[warp + 16 * t];
          const unsigned pm = bm_pairs(wd);
          const int P = (int)wd.z + __popc(pm & lt);   // pair index in the row run
          const bool kp = (pm & lb) != 0u;
          const int idx = kp ? base + 2 * P : G::kZero;
          const double2 x = *reinterpret_cast<const double2*>(sv + idx);
          const double2 vv = *reinterpret_cast<const double2*>(vsm + bm_col<16>(t, 0));
          d0 = fma(x.x, vv.x, d0);
          d1 = fma(x.y, vv.y, d1);
          if (kp) pidx[j][t >> 1] = (pidx[j][t >> 1] & ~(0xffffu << (16 * (t & 1)))) | ((uint32_t)P << (16 * (t & 1)));
        }
        if (lane == 0) hring[warp * (D + 1) + k % (D + 1)] = *h;
        __syncwarp();
        mbar_arrive(&empty[stage]);
        if (++stage == S) {
          stage = 0;
          phase ^= 1u;
        }
        wc_send_partial(d0 + d1, k, slots, xbuf, xbar, W, cr);
      }
      // (c) row ku: the W partials in window order, then the update
      if (upd) {
        const int q = ku % kWcX;
        const uint32_t par = (uint32_t)((ku / kWcX) & 1);
        mbar_wait(&xbar[q], par);
        // the W partials: lane rk loads partial rk, then a xor butterfly —
        // every lane of every warp and every CTA of the cluster forms the
        // same tree (each step pairs the same two values), so the same bits
        double dot = (lane < W) ? xbuf[q * kWcMaxW + lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        // re-arm buffer q for row ku + X once every consumer has read it (the
        // next block reduction is that barrier; peers cannot send row ku + X
        // before this CTA has sent row ku + X - D, i.e. after this point)
        if (threadIdx.x == 0) mbar_arrive_expect_tx(&xbar[q], 8u * (uint32_t)W);
        const double w = ar_u * dot;   // sparsify.py:153: weights * pv
#pragma unroll
        for (int i = 0; i < 2 * NQ; ++i) acc[i] = fma(e[i], w, acc[i]);
      }
    }
  }
}

// Dense-P_rho window-cluster hess_apply without a producer warp: 16
// consumer warps (128 registers), the window of v in REGISTERS (no second
// shared-memory read per value: the stage values are the only LDS traffic),
// the ring refilled by the warp whose arrival completes a stage's round (as
// in rowpipe.cuh Dense<.., true>).  Same per-thread sums, row order, row
// reduction tree and exchange as wc_consume_keep: the same bits.
template <int NQ>
__global__ void __launch_bounds__(kStConsumers, 1) k_hv_wcd(HvArgs h) {
  using G = WcGeo<NQ>;
  extern __shared__ __align__(16) unsigned char wsm[];
  __shared__ double xbuf[kWcX * kWcMaxW];
  __shared__ uint64_t xbar[kWcX];
  __shared__ double slots[2 * kMaxWarps * 4];
  __shared__ uint32_t arrivals[kWcMaxStages];
  const int W = h.nwin;
  const int S = h.ng;   // ring stages
  const int cr = (int)cluster_ctarank(), cid = blockIdx.x / W, ncl = gridDim.x / W;
  const int lane = threadIdx.x & 31;
  unsigned char* ring = wsm;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)S * G::kStage);
  const int cb = 1024 * NQ * cr;                              // first column of this window
  const int wcols = min(1024 * NQ, (int)(h.ld - cb));         // columns of the window inside the matrix
  int rb, re;
  cta_rows(h.A, cid, ncl, rb, re);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    for (int q = 0; q < kWcX; ++q) mbar_init(&xbar[q], 1);
    fence_mbar_init();
    for (int q = 0; q < kWcX; ++q) mbar_arrive_expect_tx(&xbar[q], 8u * (uint32_t)W);
  }
  if (threadIdx.x < kWcMaxStages) arrivals[threadIdx.x] = 0u;
  if (wcols < 1024 * NQ)   // the last window's stage tail (past the matrix) reads as 0.0
    for (int i = threadIdx.x; i < S * (1024 * NQ - wcols); i += blockDim.x) {
      const int st = i / (1024 * NQ - wcols), col = wcols + i % (1024 * NQ - wcols);
      reinterpret_cast<double*>(ring + (size_t)st * G::kStage + G::WW * 16 + kWcHdr)[col] = 0.0;
    }
  fence_proxy_async();
  __syncwarp();
  cluster_sync_all();
  // bulk copy of local row r's window into stage st
  auto issue = [&](int st, int r) {
    unsigned char* sp = ring + (size_t)st * G::kStage;
    mbar_arrive_expect_tx(&full[st], (uint32_t)wcols * 8u);
    bulk_g2s(sp + G::WW * 16 + kWcHdr, h.A.vals + (size_t)r * h.ld + cb, (uint32_t)wcols * 8u, &full[st]);
  };
  if (h.st == nullptr || h.st->status == CG_RUN) {   // same decision in every CTA
    if (threadIdx.x == 0)
      for (int s = 0; s < S && rb + s < re; ++s) issue(s, rb + s);
    // the window of v in registers; p = r + beta p by the column's owner (krylov.py:83)
    const double beta = h.update ? h.st->beta : 0.0;
    double vr[2 * NQ], acc[2 * NQ];
#pragma unroll
    for (int i = 0; i < 2 * NQ; ++i) {
      const int j = cb + bm_col<16>(i >> 1, i & 1);
      double v = 0.0;
      if (j < h.n) {
        if (h.update) {
          v = h.r[j] + beta * h.p_prev[j];
          if (cid == 0) h.p_cur[j] = v;
        } else {
          v = h.v_src[j];
        }
      }
      vr[i] = v;
      acc[i] = 0.0;
    }
    const int cnt = re - rb;
    const uint32_t nwarps = kStConsumers / 32;
    int stage = 0, fill = S;   // fill: local index of the row the next refill of `stage` loads
    uint32_t phase = 0, rounds = 1;
    constexpr int D = 1;
    double kv[D + 1][2 * NQ];
    double kar[D + 1];
    for (int k0 = 0; k0 < cnt + D; k0 += D + 1) {
#pragma unroll
      for (int j = 0; j <= D; ++j) {
        const int k = k0 + j, ku = k - D;
        if (k < cnt) {   // dots of row k; its values stay in slot j
          mbar_wait(&full[stage], phase);
          kar[j] = __ldg(h.a + h.A.row0 + rb + k);   // a_r, used by the update one row later
          const unsigned char* sp = ring + (size_t)stage * G::kStage;
          const double* sv = reinterpret_cast<const double*>(sp + G::WW * 16 + kWcHdr);
          double d0 = 0.0, d1 = 0.0;
#pragma unroll
          for (int t = 0; t < NQ; ++t) {
            const double2 x = *reinterpret_cast<const double2*>(sv + bm_col<16>(t, 0));
            kv[j][2 * t] = x.x;
            kv[j][2 * t + 1] = x.y;
            d0 = fma(x.x, vr[2 * t], d0);
            d1 = fma(x.y, vr[2 * t + 1], d1);
          }
          __syncwarp();
          // the arrival that completes the stage's round refills it; its
          // count is checked after the row's partial went out (the atomic's
          // round trip overlaps the reduction)
          uint32_t old = 0u;
          if (lane == 0)
            asm volatile("atom.relaxed.cta.shared::cta.add.u32 %0, [%1], 1;"
                         : "=r"(old)
                         : "r"(smem_u32(&arrivals[stage]))
                         : "memory");
          const int rst = stage, rfill = fill;
          const uint32_t tgt = rounds * nwarps - 1u;
          ++fill;
          if (++stage == S) {
            stage = 0;
            phase ^= 1u;
            ++rounds;
          }
          wc_send_partial(d0 + d1, k, slots, xbuf, xbar, W, cr);
          if (lane == 0 && old == tgt && rfill < cnt) {
            fence_proxy_async();
            issue(rst, rb + rfill);
          }
        }
        if (ku >= 0 && ku < cnt) {   // row ku: full dot, then the update
          const int ju = (j + 1) % (D + 1);
          const int q = ku % kWcX;
          mbar_wait(&xbar[q], (uint32_t)((ku / kWcX) & 1));
          double dot = (lane < W) ? xbuf[q * kWcMaxW + lane] : 0.0;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
          if (threadIdx.x == 0) mbar_arrive_expect_tx(&xbar[q], 8u * (uint32_t)W);
          const double w = kar[ju] * dot;   // sparsify.py:153: weights * pv
#pragma unroll
          for (int i = 0; i < 2 * NQ; ++i) acc[i] = fma(kv[ju][i], w, acc[i]);
        }
      }
    }
    double* dst = h.colpart + (size_t)cid * h.n;
#pragma unroll
    for (int i = 0; i < 2 * NQ; ++i) {
      const int jj = cb + bm_col<16>(i >> 1, i & 1);
      if (jj < h.n) dst[jj] = acc[i];
    }
  }
  __syncwarp();
  cluster_sync_all();   // no CTA leaves while a peer may still address its shared memory
}

template <int NQ, bool DENSE>
__global__ void __launch_bounds__(kStThreads, 1) k_hv_wc(HvArgs h) {
  using G = WcGeo<NQ>;
  extern __shared__ __align__(16) unsigned char wsm[];
  __shared__ double xbuf[kWcX * kWcMaxW];
  __shared__ uint64_t xbar[kWcX];
  __shared__ double slots[2 * kMaxWarps * 4];
  __shared__ WcHdr hring[(kStConsumers / 32) * (kWcD + 1)];   // per consumer warp
  const int W = h.nwin;
  const int S = h.ng;   // ring stages (HvArgs.ng reused)
  const int cr = (int)cluster_ctarank(), cid = blockIdx.x / W, ncl = gridDim.x / W;
  double* vsm = reinterpret_cast<double*>(wsm);            // [1024 NQ] the window of v
  unsigned char* ring = wsm + (size_t)G::kVsm;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)S * G::kStage);
  uint64_t* empty = full + S;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kStConsumers);
    }
    for (int q = 0; q < kWcX; ++q) mbar_init(&xbar[q], 1);
    fence_mbar_init();
    // exchange buffer q expects W partials (st.async, 8 bytes each) per use;
    // armed here for rows 0..X-1, re-armed by the receiver after each use
    for (int q = 0; q < kWcX; ++q) mbar_arrive_expect_tx(&xbar[q], 8u * (uint32_t)W);
  }
  if (threadIdx.x < S * 2) {   // the zero pair of every stage
    double* sv = reinterpret_cast<double*>(ring + (size_t)(threadIdx.x >> 1) * G::kStage + G::WW * 16 + kWcHdr);
    sv[G::kZero + (threadIdx.x & 1)] = 0.0;
  }
  if (DENSE) {   // the last window's stage tail (past the matrix) reads as 0.0
    const int lim = min(1024 * NQ, (int)(h.ld - 64LL * G::WW * cr));
    if (lim < 1024 * NQ)
      for (int i = threadIdx.x; i < S * (1024 * NQ - lim); i += blockDim.x) {
        const int st = i / (1024 * NQ - lim), col = lim + i % (1024 * NQ - lim);
        reinterpret_cast<double*>(ring + (size_t)st * G::kStage + G::WW * 16 + kWcHdr)[col] = 0.0;
      }
  }
  __syncwarp();
  cluster_sync_all();
  if (h.st == nullptr || h.st->status == CG_RUN) {   // same decision in every CTA
    const int n = h.n, cb = 64 * G::WW * cr;
    int rb, re;
    cta_rows(h.A, cid, ncl, rb, re);
    if (threadIdx.x >= kStConsumers) {
      wc_produce<NQ, DENSE>(h.A, h.bm, h.a, rb, re, h.nq, G::WW * cr, cr + 1 == W, ring, full, empty, S, h.ld,
                            min(1024 * NQ, (int)(h.ld - 64LL * G::WW * cr)));
    } else {
      // the window of v in shared memory (registers hold the accumulator and
      // the values in flight); p = r + beta p by the column's owner (krylov.py:83)
      const double beta = h.update ? h.st->beta : 0.0;
      double ar[2 * NQ];
#pragma unroll
      for (int i = 0; i < 2 * NQ; ++i) {
        const int jl = bm_col<16>(i >> 1, i & 1), j = cb + jl;
        double v = 0.0;
        if (j < n) {
          if (h.update) {
            v = h.r[j] + beta * h.p_prev[j];
            if (cid == 0) h.p_cur[j] = v;
          } else {
            v = h.v_src[j];
          }
        }
        vsm[jl] = v;
        ar[i] = 0.0;
      }
      bar_sync(1, kStConsumers);
      if constexpr (DENSE)
        wc_consume_keep<NQ>(re - rb, vsm, ar, ring, full, empty, S, xbuf, xbar, W, cr, slots, hring);
      else
        wc_consume<NQ, DENSE>(re - rb, h.A.vals, vsm, ar, ring, full, empty, S, xbuf, xbar, W, cr, slots, hring,
                              min(1024 * NQ, (int)(h.ld - 64LL * G::WW * cr)));
      double* dst = h.colpart + (size_t)cid * n;
#pragma unroll
      for (int i = 0; i < 2 * NQ; ++i) {
        const int j = cb + bm_col<16>(i >> 1, i & 1);
        if (j < n) dst[j] = ar[i];
      }
    }
  }
  __syncwarp();
  cluster_sync_all();   // no CTA leaves while a peer may still address its shared memory
}

// Warp-per-row variant for n too large for shared accumulators: the
// scatter goes to global memory with fp64 RED (order not deterministic).
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
    double dot = 0.0;
    for (int base = lane; base < len; base += 32 * kEA) {
      Chunk ch;
      load_chunk(h.A, st0, base, 32, len, ch);
#pragma unroll
      for (int i = 0; i < kEA; ++i) dot = fma(ch.v[i], __ldg(h.v + ch.c[i]), dot);
    }
    dot = warp_sum(dot);
    const double w = __ldg(h.a + h.A.row0 + r) * dot;
    for (int base = lane; base < len; base += 32 * kEA) {
      Chunk ch;
      load_chunk(h.A, st0, base, 32, len, ch);
#pragma unroll
      for (int i = 0; i < kEA; ++i)
        if (base + i * 32 < len) atomicAdd(h.y + ch.c[i], ch.v[i] * w);
    }
  }
}

// p_cur = r + beta p_prev (krylov.py:83), for the atomic variant.
__global__ void k_cg_p(int n, const double* r, const double* p_prev, double* p_cur, const CgState* st) {
  if (st->status != CG_RUN) return;
  const double beta = st->beta;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    p_cur[j] = r[j] + beta * p_prev[j];
}

// krylov.py:63-75 for the multi-kernel path: ap = Hp + shift p, curvature.
// Column sums come from colpart (reduced here), yatomic, or ysum
// (multi-rank, after the all-reduce).  One block = 32 columns.
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
  __shared__ double red[8 * 32];
  __shared__ double red2[2][kMaxWarps * 4];
  const double shift = c.st->shift;
  const int j = blockIdx.x * 32 + (threadIdx.x & 31);
  double y = 0.0;
  if (c.colpart != nullptr) {
    y = reduce_partials32(c.colpart, c.nparts, c.n, blockIdx.x * 32, red);
  } else if (threadIdx.x < 32 && j < c.n) {
    if (c.ysum) {
      y = c.ysum[j];
    } else {
      y = c.yatomic[j];
      c.yatomic[j] = 0.0;
    }
  }
  double part = 0.0;
  if (threadIdx.x < 32 && j < c.n) {
    const double pj = c.p[j];
    const double apj = Divider(c.eta)(c.d[j] * pj - y) + shift * pj;   // sparsify.py:153 + krylov.py:65
    c.ap[j] = apj;
    part = pj * apj;
  }
  int ph = 0;
  double t[1] = {part};
  block_reduce<1, kSum>(t, &red2[0][0], ph, blockDim.x);
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
          s->alpha = (s->precond ? s->rz : s->rs) / curv;
        }
      }
    }
  }
}

// krylov.py:76-84: x += alpha p, r -= alpha ap, convergence test, beta.
// PCG (minv != nullptr): z = minv r, beta = (r.z)_new / (r.z); the stopping
// test stays on ||r|| (krylov.py:79-82), so plain and preconditioned CG
// stop at the same residual.
__global__ void __launch_bounds__(256) k_cg_update(int n, double* x, double* r, const double* p, const double* ap,
                                                   CgState* st, double* bpart, const double* minv = nullptr,
                                                   double* z = nullptr) {
  if (st->status != CG_RUN) return;
  __shared__ double red[2][kMaxWarps * 4];
  const double alpha = st->alpha;
  double part = 0.0, pz = 0.0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    x[j] = x[j] + alpha * p[j];
    const double rj = r[j] - alpha * ap[j];
    r[j] = rj;
    part = fma(rj, rj, part);
    if (minv != nullptr) {
      const double zj = rj * minv[j];
      z[j] = zj;
      pz = fma(rj, zj, pz);
    }
  }
  int ph = 0;
  double t[2] = {part, pz};
  block_reduce<2, kSum>(t, &red[0][0], ph, blockDim.x);
  if (threadIdx.x == 0) {
    bpart[2 * blockIdx.x] = t[0];
    bpart[2 * blockIdx.x + 1] = t[1];
  }
  if (last_block(&st->cnt[1])) {
    if (threadIdx.x < 32) {
      const double rsn = warp_fixed_sum(bpart, gridDim.x, 2);
      const double rzn = warp_fixed_sum(bpart + 1, gridDim.x, 2);
      if (threadIdx.x == 0) {
        st->iters += 1;
        if (sqrt(rsn) <= st->target) {
          st->rs = rsn;
          st->status = CG_DONE;
        } else {
          st->beta = st->precond ? rzn / st->rz : rsn / st->rs;
          st->rs = rsn;
          st->rz = rzn;
          if (st->iters >= st->max_iters) st->status = CG_MAXIT;
        }
        st->res = sqrt(st->rs);
      }
    }
  }
}

// krylov.py:51-67 set-up: x = 0, r = p = rhs, rs = r.r, stop target.
// neg_of != nullptr: the right-hand side is -neg_of, written to rhs_out
// (inner_newton.py:117's -g without a separate pass).
// PCG (pc.q != nullptr): the Jacobi preconditioner of H_rho + shift I,
// minv_j = 1 / ((d_j - q_j) / eta + shift) with q = (P_rho o P_rho)^T a
// (diag of P_rho^T diag(a) P_rho), z = minv r, p0 = z, rz = r.z.
struct PcgInit {
  const double* d;
  const double* q;     // nullptr: plain CG (the reference's krylov.py)
  double eta;
  double* minv;
  double* z;
};
__global__ void __launch_bounds__(256) k_cg_init(int n, const double* rhs, double* x, double* r, double* p0,
                                                 CgState* st, double* bpart, double shift, double rel_tol,
                                                 long long max_iters, const double* neg_of = nullptr,
                                                 double* rhs_out = nullptr, const double* shift_dev = nullptr,
                                                 PcgInit pc = PcgInit{nullptr, nullptr, 1.0, nullptr, nullptr}) {
  __shared__ double red[2][kMaxWarps * 4];
  double sq = 0.0, sm = 0.0, rzp = 0.0;
  const double sh0 = shift_dev != nullptr ? *shift_dev : shift;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const double v = (neg_of != nullptr) ? -neg_of[j] : rhs[j];
    if (rhs_out != nullptr) rhs_out[j] = v;
    x[j] = 0.0;
    r[j] = v;
    if (pc.q != nullptr) {
      const double dj = div_rn(pc.d[j] - pc.q[j], pc.eta) + sh0;
      const double mi = dj > 0.0 ? div_rn(1.0, dj) : 1.0;
      pc.minv[j] = mi;
      const double zj = v * mi;
      pc.z[j] = zj;
      p0[j] = zj;
      rzp = fma(v, zj, rzp);
    } else {
      p0[j] = v;
    }
    sq = fma(v, v, sq);
    sm += v;
  }
  int ph = 0;
  double t[4] = {sq, sm, rzp, 0.0};
  block_reduce<4, kSum>(t, &red[0][0], ph, blockDim.x);
  if (threadIdx.x == 0) {
    bpart[4 * blockIdx.x] = t[0];
    bpart[4 * blockIdx.x + 1] = t[1];
    bpart[4 * blockIdx.x + 2] = t[2];
  }
  if (last_block(&st->cnt[2])) {
    if (threadIdx.x < 32) {
      const double rs = warp_fixed_sum(bpart, gridDim.x, 4);
      const double sum = warp_fixed_sum(bpart + 1, gridDim.x, 4);
      const double rz = warp_fixed_sum(bpart + 2, gridDim.x, 4);
      if (threadIdx.x == 0) {
        st->precond = pc.q != nullptr;
        st->rz = rz;
        const double bnorm = sqrt(rs);
        const double sh = shift_dev != nullptr ? *shift_dev : shift;   // ||g|| of an eval the host has not read
        st->rs = rs;
        st->bnorm = bnorm;
        st->shift = sh;
        st->target = rel_tol * bnorm;
        st->iters = 0;
        st->max_iters = max_iters;
        st->beta = 0.0;
        st->res = bnorm;
        if (sh == 0.0 && fabs(sum) > 1e-12 * fmax(1.0, bnorm)) st->status = CG_INCONSISTENT;
        else if (bnorm == 0.0) {
          st->status = CG_DONE;
          st->res = 0.0;
        } else if (max_iters <= 0) st->status = CG_MAXIT;
        else st->status = CG_RUN;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Persistent single-GPU CG: the whole krylov.py:68-84 loop in ONE
// cooperative launch (one CTA per SM), TWO grid barriers per iteration.
// Every CTA keeps full copies of p and r in shared memory and updates them
// redundantly, so only the H p product has to be exchanged:
//   phase 1  group hess_apply of the CTA's rows -> one partial row (HBM)
//   --sync-- phase 2  the CTA's column slice: y = fixed-order sum of the
//            partial rows, ap = (d p - y)/eta + shift p (to HBM), p.ap partial
//   --sync-- every CTA: curvature = fixed-order sum of the partials ->
//            alpha; x += alpha p on its slice; r -= alpha ap and r.r over ALL
//            columns (same order in every CTA -> bitwise-identical r.r, so
//            every CTA takes the same stop / beta decision); p = r + beta p.
// No host round trip; status, iteration count and residual end in *st.
struct CgFusedArgs {
  Csr A;
  const double* a;
  const double* d;
  int n;
  int ng;
  double eta;
  double* x;
  const double* r0;  // initial residual (= rhs)
  double* ap;
  double* colpart;   // [gridDim][n]
  double* scal;      // [gridDim]
  CgState* st;
  const uint4* bm;   // bitmap index (NQ > 0)
  int nq;
  unsigned long long* trace;   // optional: [gridDim][kCgTraceIters][6] globaltimer stamps
  const int* flags;            // sparsify flags: bit 1 = CSR overflow (nothing to solve with)
};

constexpr int kCgTraceIters = 16;
OTB_DEV unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// phase stamps of the first kCgTraceIters iterations, thread 0 of each CTA:
// 0 start, 1 hv done, 2 after barrier 1, 3 column slice done, 4 after barrier 2, 5 end
#define CG_STAMP(k)                                                                         \
  do {                                                                                      \
    if (c.trace != nullptr && tid == 0 && it < kCgTraceIters)                               \
      c.trace[((size_t)b * kCgTraceIters + (size_t)it) * 6 + (k)] = globaltimer();           \
  } while (0)

// Shared memory of k_cg_fused: p[npad] | r[npad] | acc[NG][npad] | slots.
OTB_DEV size_t cg_fused_smem_doubles(int npad, int NG) { return (size_t)npad * (2 + NG) + 16 * 64; }

template <int V>
__global__ void __launch_bounds__(HvVar<V>::kThreads, 1) k_cg_fused(CgFusedArgs c) {
  namespace cgrp = cooperative_groups;
  extern __shared__ __align__(16) double hsm[];
  __shared__ double red[40 * 32];   // reduce_partials32: one row of 32 per warp (<= 40 warps)
  __shared__ double red2[2][kMaxWarps * 4];
  __shared__ double bcast;
  cgrp::grid_group grid = cgrp::this_grid();
  if (c.st->status != CG_RUN || (*c.flags & 2)) return;
  const int n = c.n, npad = (n + 1) & ~1, NG = c.ng;
  const int B = gridDim.x, b = blockIdx.x, tid = threadIdx.x, nth = blockDim.x;
  double* psm = hsm;
  double* rsm = hsm + npad;
  double* acc = rsm + npad;
  double* gslots = acc + (size_t)npad * NG;
  const double eta = c.eta, shift = c.st->shift, target = c.st->target;
  const Divider DIV(eta);
  const long long max_iters = c.st->max_iters;
  double rs = c.st->rs, beta = 0.0, alpha = 0.0, curv = 0.0;
  long long it = 0;
  int status = CG_RUN;
  const int j0 = (int)(((int64_t)b * n) / B), j1 = (int)(((int64_t)(b + 1) * n) / B);
  int rb, re;
  cta_rows(c.A, b, B, rb, re);
  for (int j = tid; j < n; j += nth) {                 // x0 = 0, r = p = rhs (krylov.py:60-62)
    const double v = c.r0[j];
    psm[j] = v;
    rsm[j] = v;
  }
  StRing rg;
  if constexpr (HvVar<V>::kStaged) rg = st_ring(reinterpret_cast<unsigned char*>(gslots + 16 * 64), 2, HvVar<V>::CW * 32);
  __syncthreads();
  for (;;) {
    CG_STAMP(0);
    // ---- phase 1: the hess_apply partial row of this CTA
    double* dst = c.colpart + (size_t)b * n;
    if constexpr (HvVar<V>::kStaged) {
      hv_staged_partial<V>(c.A, c.bm, c.a, psm, n, c.nq, rb, re, gslots, rg, dst, rsm, beta, it > 0);
    } else if constexpr (HvVar<V>::kBitmap) {
      hv_bitmap_partial<V>(c.A, c.bm, c.a, psm, n, rb, re, gslots,
                          reinterpret_cast<unsigned char*>(gslots + 16 * 64), dst);
    } else {
      for (int j = tid; j < npad * NG; j += nth) acc[j] = 0.0;
      __syncthreads();
      hv_rows(c.A, c.a, psm, acc, npad, rb, re, NG, gslots);
      __syncthreads();
      for (int j = tid; j < n; j += nth) {
        double t = acc[j];
        for (int g = 1; g < NG; ++g) t += acc[(size_t)g * npad + j];
        dst[j] = t;
      }
    }
    CG_STAMP(1);
    grid.sync();
    CG_STAMP(2);
    // ---- phase 2: column slice of ap, curvature partial
    double part = 0.0;
    for (int jc = j0; jc < j1; jc += 32) {
      const double y = reduce_partials32(c.colpart, B, n, jc, red);
      const int j = jc + (tid & 31);
      if (tid < 32 && j < j1) {
        const double pj = psm[j];
        const double apj = DIV(c.d[j] * pj - y) + shift * pj;   // sparsify.py:153 + krylov.py:65
        c.ap[j] = apj;
        part += pj * apj;
      }
    }
    {
      int ph = 0;
      double t[1] = {part};
      block_reduce<1, kSum>(t, &red2[0][0], ph, nth);
      if (tid == 0) c.scal[b] = t[0];
    }
    CG_STAMP(3);
    grid.sync();
    CG_STAMP(4);
    // ap (written by every CTA in phase 2) and this CTA's slice of x are
    // loaded now, so their latency overlaps the curvature reduction
    constexpr int kApRegs = HvVar<V>::kThreads > 600 ? 4 : 16;   // covers n <= 4096 / 8192 (loop beyond)
    double apr[kApRegs];
#pragma unroll
    for (int i = 0; i < kApRegs; ++i) {
      const int j = tid + i * nth;
      apr[i] = (j < n) ? c.ap[j] : 0.0;
    }
    const int jx = j0 + tid;
    const double xj = (jx < j1) ? c.x[jx] : 0.0;
    if (tid < 32) {
      const double v = warp_fixed_sum(c.scal, B, 1);
      if (tid == 0) bcast = v;
    }
    __syncthreads();
    curv = bcast;
    if (curv <= 0.0) {                                   // krylov.py:70-74
      status = (sqrt(rs) <= target) ? CG_DONE : CG_NOTPD;
      break;
    }
    alpha = rs / curv;
    // ---- phase 3 (redundant in every CTA): x on the slice, r and r.r everywhere
    if (jx < j1) c.x[jx] = xj + alpha * psm[jx];
    for (int j = jx + nth; j < j1; j += nth) c.x[j] = c.x[j] + alpha * psm[j];
    double rr = 0.0;
#pragma unroll
    for (int i = 0; i < kApRegs; ++i) {
      const int j = tid + i * nth;
      if (j < n) {
        const double rj = rsm[j] - alpha * apr[i];
        rsm[j] = rj;
        rr = fma(rj, rj, rr);
      }
    }
    for (int j = tid + kApRegs * nth; j < n; j += nth) {
      const double rj = rsm[j] - alpha * c.ap[j];
      rsm[j] = rj;
      rr = fma(rj, rj, rr);
    }
    {
      int ph = 1;
      double t[1] = {rr};
      block_reduce<1, kSum>(t, &red2[0][0], ph, nth);
      rr = t[0];
    }
    ++it;
    if (sqrt(rr) <= target) {                            // krylov.py:79-82
      rs = rr;
      status = CG_DONE;
      break;
    }
    beta = rr / rs;
    rs = rr;
    if (it >= max_iters) {
      status = CG_MAXIT;
      break;
    }
    if constexpr (!HvVar<V>::kStaged) {   // staged variants update p in the next hess_apply (owned columns)
      for (int j = tid; j < n; j += nth) psm[j] = rsm[j] + beta * psm[j];   // krylov.py:83
    }
    if (c.trace != nullptr && tid == 0 && it - 1 < kCgTraceIters)          // (it already counts this one)
      c.trace[((size_t)b * kCgTraceIters + (size_t)(it - 1)) * 6 + 5] = globaltimer();
    if constexpr (!HvVar<V>::kStaged) __syncthreads();
  }
  if (b == 0 && tid == 0) {
    CgState* s = c.st;
    s->rs = rs;
    s->curv = curv;
    s->alpha = alpha;
    s->beta = beta;
    s->iters = it;
    s->status = status;
    s->res = sqrt(rs);
  }
}

// Standalone H v (+ shift v) for parity tests: out_j = (d v - y)/eta + shift v.
// One block = 32 columns.
__global__ void __launch_bounds__(256) k_hv_out(int n, const double* colpart, int nparts, double* yatomic,
                                                const double* d, const double* v, double eta, double shift,
                                                double* out) {
  __shared__ double red[8 * 32];
  const int j = blockIdx.x * 32 + (threadIdx.x & 31);
  double y = 0.0;
  if (colpart != nullptr) {
    y = reduce_partials32(colpart, nparts, n, blockIdx.x * 32, red);
  } else if (threadIdx.x < 32 && j < n) {
    y = yatomic[j];
  }
  if (threadIdx.x < 32 && j < n) out[j] = Divider(eta)(d[j] * v[j] - y) + shift * v[j];
}

}  // namespace otb
