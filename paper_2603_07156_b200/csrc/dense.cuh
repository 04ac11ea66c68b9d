// Dense passes over (C, log X): each kernel streams every local row once
// through the TMA ring of rowpipe.cuh.  Reference sites are cited per kernel.
#pragma once

#include "rowpipe.cuh"

namespace otb {

#ifndef OTB_DENSE_MAXT
#define OTB_DENSE_MAXT 544
#endif
constexpr int kMaxThreads = OTB_DENSE_MAXT;   // 512 consumers + 1 producer warp (register budget: 96)
#ifndef OTB_DENSE_MINB
#define OTB_DENSE_MINB 1           // CTAs per SM the register allocation is sized for
#endif
constexpr int kTabInts = 2 * kMaxNS * 32;
// test_c with two slices per fetch (as eval, test_a, test_b): measured SLOWER at config 5 (29.8 ->
// 32.5 ms: the pass sits at the 128-register cap and the paired form spills), so off.
#ifndef OTB_TESTC_PAIRS
#define OTB_TESTC_PAIRS 0
#endif
#ifndef OTB_ZETA_A_NS
#define OTB_ZETA_A_NS 6   // rows of more than this many slices take the KKT c-transform from pass A
#endif

// ---------------------------------------------------------------- eval (K1)
// semidual.py:51-100: logits = logX + (gamma - C)/eta, row max, shifted
// exponentials, row sums, lse = max + log(sum); column sums of a_i P_ij
// (gradient before -b) and a.lse (objective) are reduced without
// materialising P.  Per-row max / sum are kept for the sparsify pass.
struct EvalIO {
  const double* gamma;
  const double* a;      // global-row indexed
  double eta;
  double* rowM;
  double* rowS;
  double* lse;
  double* colpart;      // [ncl][n]
  double* vpart;        // [ncl][2]: a.lse, count of non-finite rows
  double* P;            // optional: P = shifted / row_sum (local rows x ld), read by sparsify
};

// Streams (C, log X, gamma) with no producer warp (Dense<3, true, 1>: 16
// consumer warps, 128 registers): gamma's window slice comes through the
// TMA ring with the two matrices, so no consumer waits on a global load.
// gamma is padded with -1e300 past n, so the masked columns of a partial
// last slice (stale but finite C, log X) give z = -1e302 and exp() = 0: no
// per-element masks in the row max, and only the P store of that slice is
// masked.  Exps: CUDA's
// fast path, branch-free per pair; a pair with an argument outside
// (-708.4, 708.4) (subnormal or zero result, -inf, NaN) is redone with exp().
constexpr int kSelfThreads = 512;
template <int NS>
__global__ void __launch_bounds__(kSelfThreads, 1) k_eval(Geom geo, EvalIO io) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ double2 etab[128];
  for (int i = threadIdx.x; i < 128; i += blockDim.x) etab[i] = kExp2Tab[i];   // visible after setup's barrier
  Dense<3, true, 1> D;
  D.setup(geo, smem);
  const Divider DIV(io.eta);
  const int nsl = D.nsl;
  const bool tail = D.tail;
  // valid columns of the thread's pair in the last slice (tail only)
  const int lastv = D.c1 - (D.c0 + (nsl - 1) * D.slice) - 2 * D.tid;
  double alse = 0.0, nbad = 0.0;
  for (int r = D.r0; r < D.r1; ++r) {
    double z[2 * NS];
    double mx = -INFINITY;
#pragma unroll
    for (int s = 0; s < NS; s += 2) {
      if (s + 1 < NS && s + 1 < nsl) {   // two slices at once: four interleaved chains
        double2 v[2][3];                 // [slice][C, log X, gamma]
        D.fetchn2(v);
        const double dq[4] = {v[0][2].x - v[0][0].x, v[0][2].y - v[0][0].y, v[1][2].x - v[1][0].x,
                              v[1][2].y - v[1][0].y};
        double q[4];
        DIV.quad(dq, q);   // semidual.py:52
        z[2 * s] = v[0][1].x + q[0];
        z[2 * s + 1] = v[0][1].y + q[1];
        z[2 * s + 2] = v[1][1].x + q[2];
        z[2 * s + 3] = v[1][1].y + q[3];
        const double zm0 = z[2 * s] > z[2 * s + 1] ? z[2 * s] : z[2 * s + 1];
        const double zm1 = z[2 * s + 2] > z[2 * s + 3] ? z[2 * s + 2] : z[2 * s + 3];
        mx = zm0 > mx ? zm0 : mx;
        mx = zm1 > mx ? zm1 : mx;
        D.refill2_deferred();
      } else if (s < nsl) {
        double2 c, x, gm;
        D.fetch3(c, x, gm);
        double q0, q1;
        DIV.pair(gm.x - c.x, gm.y - c.y, q0, q1);   // semidual.py:52
        z[2 * s] = x.x + q0;
        z[2 * s + 1] = x.y + q1;
        const double zm = z[2 * s] > z[2 * s + 1] ? z[2 * s] : z[2 * s + 1];
        mx = zm > mx ? zm : mx;
      }   // z of slices >= nsl is never read
    }
    // row max over the whole row (cluster-wide when the row is split), so
    // that exp(z - M) is the reference's shifted value bit for bit
    double t[1] = {mx};
    D.reduce<1, kMax>(t);
    double M = t[0];
    if (D.g.cl > 1) {
      const double* all = D.exchange<1>(t);
      M = all[0];
      for (int q = 1; q < D.g.cl; ++q) M = fmax(M, all[q * 4]);
    }
    // semidual.py:81: exp(logits - row_max)
    double se = 0.0;
#pragma unroll
    for (int s = 0; s < NS; s += 2) {
      if (s + 1 < NS && s + 1 < nsl) {   // four exps, one range check (se in column order, as below)
        double x[4], e[4];
        bool ok = true;
#pragma unroll
        for (int i = 0; i < 4; ++i) x[i] = z[2 * s + i] - M;
#pragma unroll
        for (int i = 0; i < 4; ++i) e[i] = exp_tab(x[i], ok, etab);
        if (!ok) {
#pragma unroll
          for (int i = 0; i < 4; ++i) e[i] = exp_t(x[i], etab);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          z[2 * s + i] = e[i];
          se += e[i];
        }
      } else if (s < nsl) {
        const double x0 = z[2 * s] - M, x1 = z[2 * s + 1] - M;
        bool ok = true;
        double e0 = exp_tab(x0, ok, etab), e1 = exp_tab(x1, ok, etab);
        if (!ok) {   // per element, as everywhere P is formed (exp_t)
          e0 = exp_t(x0, etab);
          e1 = exp_t(x1, etab);
        }
        z[2 * s] = e0;
        z[2 * s + 1] = e1;
        se += e0;
        se += e1;
      }
    }
    const double S = D.row_sum(se);
    const double ai = __ldg(io.a + D.g.row0 + r);
    const double w = ai / S;
    const Divider DS(S);
    double* Prow = io.P != nullptr ? io.P + (size_t)r * D.g.ld + D.col(0, 0) : nullptr;
#pragma unroll
    for (int s = 0; s < NS; s += 2) {
      if (s + 1 < NS && s + 1 < nsl) {   // two slices at once
        double2* a0 = D.acc2(0, s);
        double2* a1 = D.acc2(0, s + 1);
        double2 v0 = *a0, v1 = *a1;
        v0.x = fma(w, z[2 * s], v0.x);
        v0.y = fma(w, z[2 * s + 1], v0.y);
        v1.x = fma(w, z[2 * s + 2], v1.x);
        v1.y = fma(w, z[2 * s + 3], v1.y);
        *a0 = v0;
        *a1 = v1;
        if (Prow != nullptr) {                    // semidual.py:82-83: shifted / row_sum
          const double e4[4] = {z[2 * s], z[2 * s + 1], z[2 * s + 2], z[2 * s + 3]};
          double p[4];
          DS.quad(e4, p);
          double* dst = Prow + s * D.slice;
          *reinterpret_cast<double2*>(dst) = make_double2(p[0], p[1]);   // slice s is not the last
          dst += D.slice;
          if (s + 1 < nsl - 1 || !tail || lastv > 1) {
            *reinterpret_cast<double2*>(dst) = make_double2(p[2], p[3]);
          } else if (lastv > 0) {
            dst[0] = p[2];
          }
        }
      } else if (s < nsl) {
        double2* a2 = D.acc2(0, s);
        double2 v = *a2;
        v.x = fma(w, z[2 * s], v.x);
        v.y = fma(w, z[2 * s + 1], v.y);
        *a2 = v;
        if (Prow != nullptr) {                    // semidual.py:82-83: shifted / row_sum
          double p0, p1;
          DS.pair(z[2 * s], z[2 * s + 1], p0, p1);
          double* dst = Prow + s * D.slice;
          if (s < nsl - 1 || !tail || lastv > 1) {
            *reinterpret_cast<double2*>(dst) = make_double2(p0, p1);
          } else if (lastv > 0) {
            dst[0] = p0;
          }
        }
      }
    }
    if (D.tid == 0 && D.cr == 0) {
      const double l = M + log(S);   // semidual.py:79
      io.rowM[r] = M;
      io.rowS[r] = S;
      io.lse[r] = l;
      alse = fma(ai, l, alse);
      if (!isfinite(l) || !isfinite(S)) nbad += 1.0;
    }
  }
  bar_sync(1, D.g.nt);
  D.store_acc(0, io.colpart + (size_t)D.cid * D.g.n);
  if (D.tid == 0 && D.cr == 0) {
    io.vpart[2 * D.cid] = alse;
    io.vpart[2 * D.cid + 1] = nbad;
  }
  D.finish();
}

// ------------------------------------------------------------ sparsify (K2/K3)
// sparsify.py:90-127 + 143-145: keep P >= rho and P > 0 off the anchor row,
// empty rows keep their first argmax with value 1, kept values divided by
// the kept sum, anchor row stored unnormalised and dense.  Rows are written
// as contiguous runs (ascending columns) into chunks obtained with one
// atomicAdd per chunk; d = P_rho^T a is accumulated on the fly.
struct SparsifyIO {
  const double* gamma;
  const double* a;
  double eta;
  double rho;
  int64_t anchor_local;   // local row of the anchor, -1 if not on this rank
  const double* rowM;
  const double* rowS;
  const double* rowL;     // lse of the same eval (M + log S)
  uint16_t* cols;
  double* vals;
  int64_t cap;
  int64_t* row_start;     // [m_loc]
  int* row_len;           // [m_loc]
  unsigned long long* alloc;
  unsigned long long* nnzc;   // += kept entries (one atomic per CTA)
  int64_t chunk;
  double* colpart;        // [ncl][n] partial of d
  int* flags;             // bit 1: capacity overflow
  uint4* bm;              // bitmap index [m_loc][nq] (sparse.cuh), or nullptr
  int nq;
  const double* gnorm;    // non-null: rho = (eta ||g||) / mn from this device scalar (no host round trip)
  double mn;
  double* colpart2;       // non-null (Jacobi PCG): [ncl][n] partial of q = (P_rho o P_rho)^T a, accumulator 1
  double* dense;          // non-null: P_rho written DENSE (local rows x ld, 0 where dropped) instead of
                          // the row runs; may alias the P being streamed (each element is read before
                          // its own thread overwrites it)
};
// With the bitmap index, a row's run holds column PAIRS (2l, 2l+1) with at
// least one kept entry, 16 bytes each (the unkept one stored as 0.0), and
// the word's offset counts pairs: lane l of hess_apply finds its pair at
// 2 (off + popc(pairs below l)) with no per-element select.  Kept entries
// come in long runs (cfg2: 40 columns on average), so pairs cost ~1.5% more
// bytes than single entries.  Without it, runs hold the kept entries.

// Dense P_rho row (window-cluster hess_apply at high density): the same
// values as the runs, 0.0 where dropped, d (and the PCG diagonal)
// accumulated in the same order.  A row with nothing kept keeps its first
// argmax with value 1 (sparsify.py:103-107), as in the run path.
template <int NS, class DT>
OTB_DEV void sparsify_dense_row(DT& D, const SparsifyIO& io, int r, bool anc, double (&P)[2 * NS], unsigned skip,
                                unsigned keep, double ksum, int kcnt, const Divider& DS, unsigned long long& kept,
                                const double2* etab) {
  int jbest = -1;
  const bool fallback = !anc && kcnt == 0;
  if (fallback) {
#pragma unroll
    for (int k = 0; k < 2 * NS; ++k)
      if ((skip >> k) & 1u) P[k] = DS(exp_t(P[k], etab));   // skipped entries take part in the argmax
    double pm = -1.0;
#pragma unroll
    for (int k = 0; k < 2 * NS; ++k) pm = fmax(pm, P[k]);
    double u[1] = {pm};
    D.template reduce<1, kMax>(u);
    const double pmax = u[0];
    double jm = 1e300;
#pragma unroll
    for (int k = 0; k < 2 * NS; ++k)
      if (P[k] >= 0.0 && P[k] == pmax) jm = fmin(jm, (double)D.col(k >> 1, k & 1));
    u[0] = jm;
    D.template reduce<1, kMin>(u);
    jm = u[0];
    if (D.g.cl > 1) {
      double v2[2] = {pmax, jm};
      const double* all = D.template exchange<2>(v2);
      double bp = all[0], bj = all[1];
      for (int q = 1; q < D.g.cl; ++q) {
        if (all[q * 4] > bp || (all[q * 4] == bp && all[q * 4 + 1] < bj)) {
          bp = all[q * 4];
          bj = all[q * 4 + 1];
        }
      }
      jm = bj;
    }
    jbest = (int)jm;
    kcnt = 1;
  }
  const double ai = __ldg(io.a + D.g.row0 + r);
  double* drow = io.dense + (size_t)r * D.g.ld;
  const Divider DK(ksum);
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    if (s < D.nsl) {
      const int j = D.col(s, 0);
      double v0, v1;
      bool k0, k1;
      if (fallback) {
        k0 = j == jbest && P[2 * s] >= 0.0;
        k1 = j + 1 == jbest && P[2 * s + 1] >= 0.0;
        v0 = k0 ? 1.0 : 0.0;
        v1 = k1 ? 1.0 : 0.0;
      } else {
        k0 = (keep >> (2 * s)) & 1u;
        k1 = (keep >> (2 * s + 1)) & 1u;
        double n0, n1;   // sparsify.py:109-110: kept / kept_sum (the anchor row unnormalised)
        DK.pair(P[2 * s], P[2 * s + 1], n0, n1);
        v0 = k0 ? (anc ? P[2 * s] : n0) : 0.0;
        v1 = k1 ? (anc ? P[2 * s + 1] : n1) : 0.0;
      }
      if (j + 1 < D.c1) {
        *reinterpret_cast<double2*>(drow + j) = make_double2(v0, v1);
      } else if (j < D.c1) {
        drow[j] = v0;
      }
      double2* a2 = D.acc2(0, s);
      if (k0) a2->x += ai * v0;
      if (k1) a2->y += ai * v1;
      if (io.colpart2 != nullptr) {   // Jacobi diagonal of P_rho^T diag(a) P_rho
        double2* q2 = D.acc2(1, s);
        if (k0) q2->x += ai * (v0 * v0);
        if (k1) q2->y += ai * (v1 * v1);
      }
    }
  }
  if (D.tid == 0 && D.cr == 0) kept += kcnt;
}

// FROMP: stream the P stored by the eval of the same gamma (one matrix, no
// exp / division) instead of recomputing it from C and log X.
// FROMP kernels have no producer warp (Dense<1, true>: the consumers refill
// the ring, 128 registers).
template <int NS, bool FROMP>
__global__ void __launch_bounds__(FROMP ? kSelfThreads : kMaxThreads, OTB_DENSE_MINB) k_sparsify(Geom geo, SparsifyIO io) {
  extern __shared__ __align__(128) unsigned char smem[];
  OTB_EXP_TABLE(etab);   // (the eval's exp, for P recomputed or for the empty-row fallback)
  Dense<FROMP ? 1 : 2, FROMP> D;
  D.setup(geo, smem);
  if (D.producer) {
    D.produce();
    D.finish();
    return;
  }
  __shared__ int tab[kTabInts];
  __shared__ unsigned long long chunk_base;
  const double eta = io.eta;
  const double rho = io.gnorm != nullptr ? (eta * *io.gnorm) / io.mn : io.rho;   // inner_newton.py:112-114
  const Divider DIV(eta);
  const double log_rho = log(rho);
  const int nw = D.g.nt >> 5;
  const unsigned lt = (1u << D.lane) - 1u;
  const bool pairs = io.bm != nullptr;
  const bool dmode = io.dense != nullptr;   // dense P_rho output (uniform over the grid)
  const int bq0 = (D.c0 >> 6) + D.warp, bqs = D.slice >> 6;   // word of slice 0, words per slice (64-col words)
  unsigned long long cur = 0, end = 0;
  unsigned long long kept = 0;
  int rowpar = 0;
  for (int r = D.r0; r < D.r1; ++r) {
    const bool anc = (r == io.anchor_local);
    const double M = io.rowM[r], S = io.rowS[r];
    const Divider DS(S);
    // P = exp(z - M) / S < rho whenever z - M < log(rho S): such entries are
    // dropped without the exp and the division (margin 1e-9 >> rounding).
    // log S = lse - M up to a few ulp of lse, far inside the margin.
    const double dmin = (anc || !(rho > 0.0)) ? -INFINITY : (log_rho + (io.rowL[r] - M)) - 1e-9;
    double P[2 * NS];       // P_ij, or z - M for skipped entries (bit set in `skip`)
    unsigned keep = 0, skip = 0;
    unsigned bb0[NS], bb1[NS];   // per-slice keep masks of the warp (ballots), reused by the write loop
    double ks = 0.0;
    int* tb = tab + rowpar * kMaxNS * 32;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      P[2 * s] = -1.0;
      P[2 * s + 1] = -1.0;
      if (s < D.nsl) {
        double2 c, x;
        D.fetch(c, x);
        const int j = D.col(s, 0);
        if constexpr (FROMP) {
          if (j < D.c1) P[2 * s] = c.x;
          if (j + 1 < D.c1) P[2 * s + 1] = c.y;
        } else {
          const double2 gm = load_pair(io.gamma, j, D.c1);
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            if (j + e < D.c1) {
              const double dz = ((e ? x.y : x.x) + DIV((e ? gm.y : gm.x) - (e ? c.y : c.x))) - M;
              if (dz < dmin) {
                P[2 * s + e] = dz;
                skip |= 1u << (2 * s + e);
              } else {
                P[2 * s + e] = DS(exp_t(dz, etab));   // semidual.py:82-83: shifted / row_sum
              }
            }
          }
        }
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double p = P[2 * s + e];
        const bool valid = D.col(s, e) < D.c1 && !((skip >> (2 * s + e)) & 1u);
        const bool k = valid && (anc || (p >= rho && p > 0.0));
        if (k) {
          keep |= 1u << (2 * s + e);
          ks += p;
        }
      }
      bb0[s] = bb1[s] = 0u;
      if (s < D.nsl && !dmode) {   // dense P_rho needs no run layout: no ballots, no scan
        bb0[s] = __ballot_sync(0xffffffffu, (keep >> (2 * s)) & 1u);
        bb1[s] = __ballot_sync(0xffffffffu, (keep >> (2 * s + 1)) & 1u);
        // packed count of the warp's chunk: stored units (pairs, or entries) | entries << 16
        // (a window has at most 10240 columns, so neither field carries)
        const int ents = __popc(bb0[s]) + __popc(bb1[s]);
        if (D.lane == 0) tb[s * 32 + D.warp] = (pairs ? __popc(bb0[s] | bb1[s]) : ents) | (ents << 16);
      }
    }
    if (dmode) {
      // kept sum and kept count of the row: one block reduction of both
      // (per-value trees as in the run path, so the same ksum bits), one
      // cluster exchange
      double t2[2] = {ks, (double)__popc(keep)};
      D.template reduce<2, kSum>(t2);
      double ksum = t2[0], kcnt = t2[1];
      if (D.g.cl > 1) {
        const double* all = D.template exchange<2>(t2);
        ksum = 0.0;
        kcnt = 0.0;
        for (int q = 0; q < D.g.cl; ++q) {
          ksum += all[q * 4];
          kcnt += all[q * 4 + 1];
        }
      }
      sparsify_dense_row<NS>(D, io, r, anc, P, skip, keep, ksum, (int)kcnt, DS, kept, etab);
      rowpar ^= 1;
      continue;
    }
    double t[1] = {ks};
    D.template reduce<1, kSum>(t);   // barrier also publishes tb
    double ksum = t[0];
    // Exclusive scan of the packed counts over (slice, warp) — the order of
    // the row run.  Two slices per round, one 16-lane segment each (lane =
    // warp index); pre[s] = start of this warp's chunk of slice s.
    int pre[NS];
    int run = 0;
    {
      const int seg = D.lane >> 4, wl = D.lane & 15;
#pragma unroll
      for (int q = 0; q < (NS + 1) / 2; ++q) {
        const int sl = 2 * q + seg;
        const int v = (sl < D.nsl && wl < nw) ? tb[sl * 32 + wl] : 0;
        int inc = v;
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) {
          const int u = __shfl_up_sync(0xffffffffu, inc, o, 16);
          if (wl >= o) inc += u;
        }
        const int tot0 = __shfl_sync(0xffffffffu, inc, 15), tot1 = __shfl_sync(0xffffffffu, inc, 31);
        const int ex0 = __shfl_sync(0xffffffffu, inc - v, D.warp);
        const int ex1 = __shfl_sync(0xffffffffu, inc - v, 16 + D.warp);
        pre[2 * q] = run + ex0;
        run += tot0;
        if (2 * q + 1 < NS) pre[2 * q + 1] = run + ex1;
        run += tot1;
      }
    }
    int ecnt = run >> 16;                              // kept entries of the row (this window)
    int need = run & 0xffff;                           // kept (entries or pairs) in this CTA's window
    int cnt = need;                                    // ... in the whole row
    int myoff = 0;                                     // offset of this window in the row
    if (D.g.cl > 1) {
      double v3[3] = {(double)need, ksum, (double)ecnt};
      const double* all = D.template exchange<3>(v3);
      double cs = 0.0, kss = 0.0, es = 0.0;
      for (int q = 0; q < D.g.cl; ++q) {
        if (q < D.cr) myoff += (int)all[q * 4];
        cs += all[q * 4];
        kss += all[q * 4 + 1];
        es += all[q * 4 + 2];
      }
      cnt = (int)cs;
      ksum = kss;
      ecnt = (int)es;
    }
    bool fallback = false;
    int jbest = -1;
    if (!anc && cnt == 0) {
      // sparsify.py:103-107: keep the first argmax of the row with value 1.
      fallback = true;
#pragma unroll
      for (int k = 0; k < 2 * NS; ++k)
        if ((skip >> k) & 1u) P[k] = DS(exp_t(P[k], etab));   // skipped entries take part in the argmax
      double pm = -1.0;
#pragma unroll
      for (int k = 0; k < 2 * NS; ++k) pm = fmax(pm, P[k]);
      double u[1] = {pm};
      D.template reduce<1, kMax>(u);
      double pmax = u[0];
      double jm = 1e300;
#pragma unroll
      for (int k = 0; k < 2 * NS; ++k)
        if (P[k] >= 0.0 && P[k] == pmax) jm = fmin(jm, (double)D.col(k >> 1, k & 1));
      u[0] = jm;
      D.template reduce<1, kMin>(u);
      jm = u[0];
      if (D.g.cl > 1) {
        double v2[2] = {pmax, jm};
        const double* all = D.template exchange<2>(v2);
        double bp = all[0], bj = all[1];
        for (int q = 1; q < D.g.cl; ++q) {
          if (all[q * 4] > bp || (all[q * 4] == bp && all[q * 4 + 1] < bj)) {
            bp = all[q * 4];
            bj = all[q * 4 + 1];
          }
        }
        jm = bj;
      }
      jbest = (int)jm;
      need = (jbest >= D.c0 && jbest < D.c1) ? 1 : 0;
      cnt = 1;
      ecnt = 1;
      myoff = 0;
    }
    // Contiguous row run: cluster rank 0 bump-allocates from its current
    // chunk (state replicated in all of its consumer threads) and shares
    // the start with the other ranks of the cluster.
    // The (cur, end) chunk state is the same in every rank of the cluster
    // (cnt is the cluster-wide count), so only a refill needs rank 0's new
    // chunk base sent to the others — about one row in ten at cfg5 instead
    // of every row.
    const int sto = pairs ? 2 * cnt : cnt;   // stored doubles of the row
    const int cnt_al = (sto + 7) & ~7;      // runs start on 8-entry boundaries (vector loads in hess_apply)
    if (cur + (unsigned long long)cnt_al > end) {
      const unsigned long long want = (unsigned long long)max((int64_t)cnt_al, io.chunk);
      if (D.cr == 0) {
        if (D.tid == 0) chunk_base = atomicAdd(io.alloc, want);
        bar_sync(1, D.g.nt);
        cur = chunk_base;
        bar_sync(1, D.g.nt);   // chunk_base may be rewritten next time
      }
      if (D.g.cl > 1) {
        double v1[1] = {(double)cur};
        const double* all = D.template exchange<1>(v1);
        cur = (unsigned long long)all[0];   // rank 0's base
      }
      end = cur + want;
    }
    const unsigned long long start = cur;
    cur += (unsigned long long)cnt_al;
    const bool ovf = (int64_t)(start + cnt_al) > io.cap;
    if (ovf && D.tid == 0 && D.cr == 0) atomicOr(io.flags, 2);
    const double ai = __ldg(io.a + D.g.row0 + r);
    const unsigned long long wbase = start + (pairs ? 2 * myoff : myoff);
    uint4* bmr = pairs ? io.bm + (size_t)r * io.nq : nullptr;   // the row's bitmap words
    const Divider DK(ksum);
    if (!ovf) {
      if (fallback) {
#pragma unroll
        for (int k = 0; k < 2 * NS; ++k) {
          if (D.col(k >> 1, k & 1) == jbest && P[k] >= 0.0) {
            if (io.cols != nullptr) io.cols[wbase] = (uint16_t)jbest;
            if (pairs) {
              io.vals[wbase + (k & 1)] = 1.0;
              io.vals[wbase + 1 - (k & 1)] = 0.0;
            } else {
              io.vals[wbase] = 1.0;
            }
            double2* a2 = D.acc2(0, k >> 1);
            if (k & 1) a2->y += ai * 1.0;
            else a2->x += ai * 1.0;
            if (io.colpart2 != nullptr) {
              double2* q2 = D.acc2(1, k >> 1);
              if (k & 1) q2->y += ai * (1.0 * 1.0);
              else q2->x += ai * (1.0 * 1.0);
            }
          }
        }
        if (io.bm != nullptr && D.lane == 0) {
          for (int s = 0; s < D.nsl; ++s) {
            const int cs = D.c0 + s * D.slice + 64 * D.warp;   // this warp's 64-column word
            if (cs < D.c1) {
              uint4 w = make_uint4(0u, 0u, 0u, 0u);
              const int o = jbest - cs;
              if (o >= 0 && o < 64) {
                if (o & 1) w.y = 1u << (o >> 1);
                else w.x = 1u << (o >> 1);
              }
              io.bm[(size_t)r * io.nq + cs / 64] = w;
            }
          }
        }
      } else {
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          if (s < D.nsl) {
            const unsigned k0 = (keep >> (2 * s)) & 1u, k1 = (keep >> (2 * s + 1)) & 1u;
            const unsigned b0 = bb0[s], b1 = bb1[s];
            const int base = pre[s] & 0xffff;
            const int j = D.col(s, 0);
            if (bmr != nullptr && D.lane == 0 && D.c0 + s * D.slice + 64 * D.warp < D.c1)   // this warp's word
              bmr[bq0 + s * bqs] = make_uint4(b0, b1, (unsigned)(myoff + base), 0u);
            double2* a2 = D.acc2(0, s);
            if (pairs) {
              if (k0 | k1) {
                const int off = base + __popc((b0 | b1) & lt);
                double n0, n1;   // sparsify.py:109-110: kept / kept_sum (the anchor row unnormalised)
                DK.pair(P[2 * s], P[2 * s + 1], n0, n1);
                const double v0 = k0 ? (anc ? P[2 * s] : n0) : 0.0;
                const double v1 = k1 ? (anc ? P[2 * s + 1] : n1) : 0.0;
                *reinterpret_cast<double2*>(io.vals + wbase + 2 * off) = make_double2(v0, v1);
                if (k0) a2->x += ai * v0;
                if (k1) a2->y += ai * v1;
                if (io.colpart2 != nullptr) {
                  double2* q2 = D.acc2(1, s);
                  if (k0) q2->x += ai * (v0 * v0);
                  if (k1) q2->y += ai * (v1 * v1);
                }
              }
              continue;
            }
            const int off = base + __popc(b0 & lt) + __popc(b1 & lt);
            if (k0) {
              const double v = anc ? P[2 * s] : DK(P[2 * s]);
              if (io.cols != nullptr) io.cols[wbase + off] = (uint16_t)j;
              io.vals[wbase + off] = v;
              a2->x += ai * v;
              if (io.colpart2 != nullptr) D.acc2(1, s)->x += ai * (v * v);
            }
            if (k1) {
              const double v = anc ? P[2 * s + 1] : DK(P[2 * s + 1]);
              if (io.cols != nullptr) io.cols[wbase + off + k0] = (uint16_t)(j + 1);
              io.vals[wbase + off + k0] = v;
              a2->y += ai * v;
              if (io.colpart2 != nullptr) D.acc2(1, s)->y += ai * (v * v);
            }
          }
        }
      }
    }
    if (D.tid == 0 && D.cr == 0) {
      io.row_start[r] = (int64_t)start;
      io.row_len[r] = ovf ? 0 : sto;
      kept += ovf ? 0 : ecnt;
    }
    rowpar ^= 1;
  }
  if (D.tid == 0 && D.cr == 0 && kept) atomicAdd(io.nnzc, kept);
  bar_sync(1, D.g.nt);
  D.store_acc(0, io.colpart + (size_t)D.cid * D.g.n);
  if (io.colpart2 != nullptr) D.store_acc(1, io.colpart2 + (size_t)D.cid * D.g.n);
  D.finish();
}

// Dense P_rho from the stored P, lean (sparsify's dense mode when P is
// valid): the same kept set, kept sum, values and d (and PCG diagonal)
// bits as k_sparsify<NS, true> with io.dense, with the keep decision
// recomputed from P in the write loop instead of per-row bit masks, no
// run/bitmap machinery, and the masked columns of a partial last slice
// handled by one uniform branch.
template <int NS>
__global__ void __launch_bounds__(kSelfThreads, 1) k_sparsify_dense(Geom geo, SparsifyIO io) {
  extern __shared__ __align__(128) unsigned char smem[];
  Dense<1, true> D;
  D.setup(geo, smem);
  const double rho = io.gnorm != nullptr ? (io.eta * *io.gnorm) / io.mn : io.rho;   // inner_newton.py:112-114
  const int nsl = D.nsl;
  const bool tail = D.tail;
  const int lastv = D.c1 - (D.c0 + (nsl - 1) * D.slice) - 2 * D.tid;   // valid columns of the last pair
  const bool pcg = io.colpart2 != nullptr;
  unsigned long long kept = 0;
  for (int r = D.r0; r < D.r1; ++r) {
    const bool anc = (r == io.anchor_local);
    double P[2 * NS];
    double ks = 0.0;
    int kc = 0;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      if (s < nsl) {
        double2 v[1];
        D.fetchn(v);
        P[2 * s] = v[0].x;
        P[2 * s + 1] = v[0].y;
        if (tail && s == nsl - 1) {   // masked columns: -1 (never kept, never the argmax)
          P[2 * s] = lastv > 0 ? P[2 * s] : -1.0;
          P[2 * s + 1] = lastv > 1 ? P[2 * s + 1] : -1.0;
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {   // sparsify.py:96-101
          const double p = P[2 * s + e];
          const bool k = anc ? p >= 0.0 : (p >= rho && p > 0.0);
          if (k) {
            ks += p;
            ++kc;
          }
        }
      }
    }
    // kept sum and kept count of the row: one block reduction of both, one
    // cluster exchange (the trees of k_sparsify's dense mode)
    double t2[2] = {ks, (double)kc};
    D.template reduce<2, kSum>(t2);
    double ksum = t2[0], kcnt = t2[1];
    if (D.g.cl > 1) {
      const double* all = D.template exchange<2>(t2);
      ksum = 0.0;
      kcnt = 0.0;
      for (int q = 0; q < D.g.cl; ++q) {
        ksum += all[q * 4];
        kcnt += all[q * 4 + 1];
      }
    }
    int jbest = -1;
    const bool fallback = !anc && kcnt == 0.0;
    if (fallback) {   // sparsify.py:103-107: keep the first argmax of the row with value 1
      double pm = -1.0;
#pragma unroll
      for (int k = 0; k < 2 * NS; ++k)
        if ((k >> 1) < nsl) pm = fmax(pm, P[k]);
      double u[1] = {pm};
      D.template reduce<1, kMax>(u);
      const double pmax = u[0];
      double jm = 1e300;
#pragma unroll
      for (int k = 0; k < 2 * NS; ++k)
        if ((k >> 1) < nsl && P[k] >= 0.0 && P[k] == pmax) jm = fmin(jm, (double)D.col(k >> 1, k & 1));
      u[0] = jm;
      D.template reduce<1, kMin>(u);
      jm = u[0];
      if (D.g.cl > 1) {
        double v2[2] = {pmax, jm};
        const double* all = D.template exchange<2>(v2);
        double bp = all[0], bj = all[1];
        for (int q = 1; q < D.g.cl; ++q) {
          if (all[q * 4] > bp || (all[q * 4] == bp && all[q * 4 + 1] < bj)) {
            bp = all[q * 4];
            bj = all[q * 4 + 1];
          }
        }
        jm = bj;
      }
      jbest = (int)jm;
    }
    const double ai = __ldg(io.a + D.g.row0 + r);
    double* drow = io.dense + (size_t)r * D.g.ld + D.col(0, 0);
    const Divider DK(ksum);
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      if (s < nsl) {
        const double p0 = P[2 * s], p1 = P[2 * s + 1];
        double v0, v1;
        if (fallback) {
          const int j = D.col(s, 0);
          v0 = (j == jbest && p0 >= 0.0) ? 1.0 : 0.0;
          v1 = (j + 1 == jbest && p1 >= 0.0) ? 1.0 : 0.0;
        } else {   // sparsify.py:109-110: kept / kept_sum (the anchor row unnormalised)
          const bool k0 = anc ? p0 >= 0.0 : (p0 >= rho && p0 > 0.0);
          const bool k1 = anc ? p1 >= 0.0 : (p1 >= rho && p1 > 0.0);
          double n0 = p0, n1 = p1;
          if (!anc) DK.pair(p0, p1, n0, n1);
          v0 = k0 ? n0 : 0.0;
          v1 = k1 ? n1 : 0.0;
        }
        double* dst = drow + s * D.slice;
        if (!(tail && s == nsl - 1) || lastv > 1) {
          *reinterpret_cast<double2*>(dst) = make_double2(v0, v1);
        } else if (lastv > 0) {
          dst[0] = v0;
        }
        double2* a2 = D.acc2(0, s);   // d += a_i v (0 where dropped: the same bits as adding only kept)
        a2->x += ai * v0;
        a2->y += ai * v1;
        if (pcg) {   // Jacobi diagonal of P_rho^T diag(a) P_rho
          double2* q2 = D.acc2(1, s);
          q2->x += ai * (v0 * v0);
          q2->y += ai * (v1 * v1);
        }
      }
    }
    if (D.tid == 0 && D.cr == 0) kept += fallback ? 1ull : (unsigned long long)kcnt;
  }
  if (D.tid == 0 && D.cr == 0 && kept) atomicAdd(io.nnzc, kept);
  bar_sync(1, D.g.nt);
  D.store_acc(0, io.colpart + (size_t)D.cid * D.g.n);
  if (pcg) D.store_acc(1, io.colpart2 + (size_t)D.cid * D.g.n);
  D.finish();
}

// ------------------------------------------------- inexact test, pass A (K7/K8)
// inner_newton.py:160-167 + core.py:141-145 (candidate log plan, NaN/+inf
// check, floor clamp) fused with feasibility.py:56-60 (row sums, z, column
// sums of F = X diag-scaled).  Writes the candidate into Xout.
struct TestAIO {
  const double* gamma;
  const double* a;
  const double* log_a;
  const double* lse;
  double eta;
  double* Xout;
  double* zrow;
  double* colpart;   // [ncl][n]
  double* spart;     // [gridDim][2]: sum of exp(candidate), count of NaN/+inf
  int recover;       // 0: round the given log plan as is (no candidate write)
  double* czeta;     // metrics: c-transform zeta_i = min_j (C_ij - gamma_j) per row (feasibility.py:103), or nullptr
};

// No producer warp (Dense<3, true, 1>: 128 registers); gamma streamed with
// (C, log X) through the ring (-1e300 padding past n).  Only the last slice
// of a partial window is masked (candidate store, exp of the plan as given).
template <int NS>
__global__ void __launch_bounds__(kSelfThreads, 1) k_test_a(Geom geo, TestAIO io) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ double2 etab[128];
  for (int i = threadIdx.x; i < 128; i += blockDim.x) etab[i] = kExp2Tab[i];   // visible after setup's barrier
  Dense<3, true, 1> D;
  D.setup(geo, smem);
  const int nsl = D.nsl;
  const bool tail = D.tail;
  const int lastv = D.c1 - (D.c0 + (nsl - 1) * D.slice) - 2 * D.tid;   // valid columns of the last pair
  const Divider DIV(io.eta);
  double sumx = 0.0;
  bool bad = false;
  // wide rows (NS > 6) also reduce the c-transform for pass C (see k_test_c)
  constexpr bool kCtr = NS > OTB_ZETA_A_NS;
  const bool ctr = kCtr && io.czeta != nullptr;
  for (int r = D.r0; r < D.r1; ++r) {
    const int64_t gi = D.g.row0 + r;
    const double la = io.recover ? __ldg(io.log_a + gi) : 0.0;
    const double l = io.recover ? io.lse[r] : 0.0;
    double* Xrow = io.Xout + (size_t)r * D.g.ld + D.col(0, 0);   // this thread's slice-0 pair of the row
    double xv[2 * NS];
    double rs = 0.0;
    double shmin = INFINITY;
#pragma unroll
    for (int s = 0; s < NS; s += 2) {
      if (s + 1 < NS && s + 1 < nsl) {   // two slices at once: four interleaved chains, one range check each
        double2 v[2][3];                 // [slice][C, log X, gamma]
        D.fetchn2(v);
        const bool part = tail && s + 1 == nsl - 1;   // only the second slice can be the partial one
        const double cc[4] = {v[0][0].x, v[0][0].y, v[1][0].x, v[1][0].y};
        const double xx[4] = {v[0][1].x, v[0][1].y, v[1][1].x, v[1][1].y};
        const double gg[4] = {v[0][2].x, v[0][2].y, v[1][2].x, v[1][2].y};
        if (kCtr && ctr) {   // the slack's c-transform for pass C's KKT metrics
#pragma unroll
          for (int i = 0; i < 4; ++i) shmin = fmin(shmin, cc[i] - gg[i]);
        }
        double l4[4] = {xx[0], xx[1], xx[2], xx[3]};   // log entries (candidate, or the plan as given)
        if (io.recover) {                               // inner_newton.py:160-167, core.py:141-145
          double dq[4], q[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) dq[i] = gg[i] - cc[i];
          DIV.quad(dq, q);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const double raw = ((la + xx[i]) + q[i]) - l;
            bad |= isnan(raw) || raw == INFINITY;
            l4[i] = fmax(raw, kLogFloor);
          }
          double* dst = Xrow + s * D.slice;
          *reinterpret_cast<double2*>(dst) = make_double2(l4[0], l4[1]);   // slice s is not the last
          dst += D.slice;
          if (!part || lastv > 1) {
            *reinterpret_cast<double2*>(dst) = make_double2(l4[2], l4[3]);
          } else if (lastv > 0) {
            dst[0] = l4[2];
          }
        }
        bool ok = true;   // four exps branch-free (exp() only when out of range)
        double e[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) e[i] = exp_tab(l4[i], ok, etab);
        if (!ok) {   // per element (exp_t), as k_materialize_rounded forms X
#pragma unroll
          for (int i = 0; i < 4; ++i) e[i] = exp_t(l4[i], etab);
        }
        if (part) {
          e[2] = lastv > 0 ? e[2] : 0.0;
          e[3] = lastv > 1 ? e[3] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) xv[2 * s + i] = e[i];
        rs += e[0] + e[1];
        rs += e[2] + e[3];
        D.refill2_deferred();
      } else if (s < nsl) {
        double2 c, x, gm;
        D.fetch3(c, x, gm);
        const bool part = tail && s == nsl - 1;
        if (kCtr && ctr) {   // the slack's c-transform for pass C's KKT metrics
          shmin = fmin(shmin, c.x - gm.x);
          shmin = fmin(shmin, c.y - gm.y);
        }
        double l0 = x.x, l1 = x.y;   // the slice's log entries (candidate, or the plan as given)
        if (io.recover) {            // inner_newton.py:160-167, core.py:141-145
          double q0, q1;
          DIV.pair(gm.x - c.x, gm.y - c.y, q0, q1);
          const double raw0 = ((la + x.x) + q0) - l, raw1 = ((la + x.y) + q1) - l;
          bad |= isnan(raw0) || raw0 == INFINITY || isnan(raw1) || raw1 == INFINITY;
          l0 = fmax(raw0, kLogFloor);
          l1 = fmax(raw1, kLogFloor);
          double* dst = Xrow + s * D.slice;
          if (!part || lastv > 1) {
            *reinterpret_cast<double2*>(dst) = make_double2(l0, l1);
          } else if (lastv > 0) {
            dst[0] = l0;
          }
        }
        bool ok = true;   // both exps branch-free (exp() only when out of range)
        double e0 = exp_tab(l0, ok, etab), e1 = exp_tab(l1, ok, etab);
        if (!ok) {   // per element (exp_t), as k_materialize_rounded forms X
          e0 = exp_t(l0, etab);
          e1 = exp_t(l1, etab);
        }
        if (part) {
          e0 = lastv > 0 ? e0 : 0.0;
          e1 = lastv > 1 ? e1 : 0.0;
        }
        xv[2 * s] = e0;
        xv[2 * s + 1] = e1;
        rs += e0 + e1;
      }
    }
    double rsum;
    if (kCtr && ctr) {
      double zeta;
      D.row_sum_min(rs, shmin, rsum, zeta);
      if (D.tid == 0 && D.cr == 0) io.czeta[r] = zeta;
    } else {
      rsum = D.row_sum(rs);
    }
    const double ai = __ldg(io.a + gi);
    const double z = (rsum > 0.0) ? fmin(div_rn(ai, rsum), 1.0) : 1.0;   // feasibility.py:56-58
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      if (s < nsl) {
        double2* a2 = D.acc2(0, s);
        double2 v = *a2;
        v.x = fma(xv[2 * s], z, v.x);   // column sums: a reduction, fused multiply-add
        v.y = fma(xv[2 * s + 1], z, v.y);
        *a2 = v;
      }
    }
    if (D.tid == 0 && D.cr == 0) {
      io.zrow[r] = z;
      sumx += rsum;
    }
  }
  double bv[1] = {bad ? 1.0 : 0.0};
  D.reduce<1, kSum>(bv);
  D.store_acc(0, io.colpart + (size_t)D.cid * D.g.n);
  if (D.tid == 0) {
    io.spart[2 * blockIdx.x] = (D.cr == 0) ? sumx : 0.0;
    io.spart[2 * blockIdx.x + 1] = bv[0];
  }
  D.finish();
}

// ------------------------------------------------------ inexact test, pass B
// feasibility.py:61-66: F = (X z) y; row sums -> e_r, column sums -> e_c.
struct TestBIO {
  const double* zrow;
  const double* y;
  double* rowpart;   // [m_loc * cl]
  double* colpart;   // [ncl][n]
};

// No producer warp (Dense<2, true, 1>: 128 registers), y streamed through
// the ring with the candidate rows (zero padding past n: a partial last
// slice's masked columns give f = 0), column sums in registers (no shared
// accumulator: the ring takes the whole shared memory).
template <int NS>
__global__ void __launch_bounds__(kSelfThreads, 1) k_test_b(Geom geo, TestBIO io) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ double rsl[2 * 8 * 16];
  __shared__ double2 etab[128];
  for (int i = threadIdx.x; i < 128; i += blockDim.x) etab[i] = kExp2Tab[i];   // visible after setup's barrier
  Dense<2, true, 1> D;
  D.setup(geo, smem);
  const int nsl = D.nsl;
  double acc[2 * NS];
#pragma unroll
  for (int k = 0; k < 2 * NS; ++k) acc[k] = 0.0;
  for (int r = D.r0; r < D.r1; ++r) {
    const double z = io.zrow[r];
    double rs = 0.0;
#pragma unroll
    for (int s = 0; s < NS; s += 2) {
      if (s + 1 < NS && s + 1 < nsl) {   // two slices at once: four interleaved chains, one range check
        double2 v[2][2];                 // [slice][candidate log entries, y]
        D.fetchn2(v);
        const double x[4] = {v[0][0].x, v[0][0].y, v[1][0].x, v[1][0].y};
        const double yv[4] = {v[0][1].x, v[0][1].y, v[1][1].x, v[1][1].y};
        double e[4], f[4];
        bool ok = true;
#pragma unroll
        for (int i = 0; i < 4; ++i) e[i] = exp_tab(x[i], ok, etab);
        if (!ok) {   // per element (exp_t), as k_materialize_rounded forms X
#pragma unroll
          for (int i = 0; i < 4; ++i) e[i] = exp_t(x[i], etab);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) f[i] = (e[i] * z) * yv[i];   // feasibility.py:65
        rs += f[0] + f[1];
        rs += f[2] + f[3];
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[2 * s + i] += f[i];
        D.refill2_deferred();
      } else if (s < nsl) {
        double2 v[2];   // candidate log entries, y
        D.fetchn(v);
        bool ok = true;
        double e0 = exp_tab(v[0].x, ok, etab), e1 = exp_tab(v[0].y, ok, etab);
        if (!ok) {   // per element (exp_t), as k_materialize_rounded forms X
          e0 = exp_t(v[0].x, etab);
          e1 = exp_t(v[0].y, etab);
        }
        const double f0 = (e0 * z) * v[1].x, f1 = (e1 * z) * v[1].y;   // feasibility.py:65
        rs += f0 + f1;
        acc[2 * s] += f0;
        acc[2 * s + 1] += f1;
      }
    }
    D.row_sum_deferred(rs, r, io.rowpart, rsl);
  }
  double* dst = io.colpart + (size_t)D.cid * D.g.n;
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    if (s < nsl) {
      const int j = D.col(s, 0);
      if (j < D.c1) dst[j] = acc[2 * s];
      if (j + 1 < D.c1) dst[j + 1] = acc[2 * s + 1];
    }
  }
  D.finish();
}

// ------------------------------------------------------ inexact test, pass C
// feasibility.py:67-68 (rank-one correction) + 80-85 (Bregman divergence)
// and, with METRICS, bregman_outer.py:53 (objective) + feasibility.py:103-122
// (c-transform, slack, KKT sums).  Scalar partials per CTA (8 slots):
//   0 sum f(log f - logY) [f>0]  1 sum f  2 sum C f  3 sum f^2
//   4 sum min(f,0)^2  5 sum min(slack,0)^2  6 sum f*slack
struct TestCIO {
  const double* zrow;
  const double* y;
  const double* er;
  const double* ec;
  const double* deficit;   // device scalar (feasibility.py:66)
  const double* gamma;
  double* rowpart;   // [m_loc * cl] row sums of the rounded plan
  double* colpart;   // [ncl][n] column sums of the rounded plan
  double* spart;     // [gridDim][8]
  const double* czeta;   // METRICS: row c-transform from pass A
};

// No producer warp (Dense<.., true, ..>: 128 registers); y, e_c and (with
// METRICS) gamma streamed through the ring with the rows (X [, C], y, e_c
// [, gamma]); their padding past n (0, 0, -1e300) makes a partial last
// slice's masked columns contribute nothing (f = 0, slack = +1e300 > 0), so
// there are no per-element masks; column sums in registers.
template <int NS, bool METRICS>
__global__ void __launch_bounds__(kSelfThreads, 1) k_test_c(Geom geo, TestCIO io) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int NM = METRICS ? 2 : 1, NA = NM + (METRICS ? 3 : 2);
  __shared__ double rsl[2 * 8 * 16];
  __shared__ double2 etab[128];
  __shared__ double4 ltab[128];
  for (int i = threadIdx.x; i < 128; i += blockDim.x) {   // visible after setup's barrier (blocks may be < 128)
    etab[i] = kExp2Tab[i];
    ltab[i] = kLogTab[i];
  }
  Dense<NA, true, NA - NM> D;
  D.setup(geo, smem);
  const int nsl = D.nsl;
  const double deficit = *io.deficit;
  const Divider DD(deficit);
  // The slack needs the row c-transform zeta (feasibility.py:103, row min of
  // C - gamma).  Up to 6 slices the row's f and C - gamma stay in registers
  // and zeta is reduced here; wider rows take zeta from pass A (k_test_a,
  // czeta) so that they do not spill.  Same values, same summation order.
  constexpr bool kZetaFromA = NS > OTB_ZETA_A_NS;
  constexpr int KR = (METRICS && !kZetaFromA) ? 2 * NS : 1;
  double acc[7] = {0, 0, 0, 0, 0, 0, 0};
  double cacc[2 * NS];
#pragma unroll
  for (int k = 0; k < 2 * NS; ++k) cacc[k] = 0.0;
  for (int r = D.r0; r < D.r1; ++r) {
    const double z = io.zrow[r];
    const double e_r = io.er[r];
    const double zeta_a = (METRICS && kZetaFromA) ? io.czeta[r] : 0.0;
    double fk[KR], shk[KR];
    double shmin = INFINITY;
    double rs = 0.0;
#pragma unroll
    for (int s = 0; s < NS; s += (OTB_TESTC_PAIRS ? 2 : 1)) {
      if (OTB_TESTC_PAIRS && s + 1 < NS && s + 1 < nsl) {   // two slices at once (off: see OTB_TESTC_PAIRS)
        double2 v[2][NA];
        D.fetchn2(v);
        const double xl[4] = {v[0][0].x, v[0][0].y, v[1][0].x, v[1][0].y};
        const double yv[4] = {v[0][NM].x, v[0][NM].y, v[1][NM].x, v[1][NM].y};
        double ex[4], f[4], lg[4];
        bool ok = true;
#pragma unroll
        for (int i = 0; i < 4; ++i) ex[i] = exp_tab(xl[i], ok, etab);
        if (!ok) {   // per element (exp_t), as k_materialize_rounded forms X
#pragma unroll
          for (int i = 0; i < 4; ++i) ex[i] = exp_t(xl[i], etab);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) f[i] = (ex[i] * z) * yv[i];   // feasibility.py:65
        if (deficit > 0.0) {                                         // feasibility.py:67-68
          const double ev[4] = {e_r * v[0][NM + 1].x, e_r * v[0][NM + 1].y, e_r * v[1][NM + 1].x,
                                e_r * v[1][NM + 1].y};
          double d[4];
          DD.quad(ev, d);
#pragma unroll
          for (int i = 0; i < 4; ++i) f[i] = f[i] + d[i];
        }
        // feasibility.py:84 terms: table logs, branch-free; log_fast per PAIR with an entry near 1,
        // zero, subnormal, negative or non-finite (the same pairs, the same bits as the single-slice path)
        bool lok0 = true, lok1 = true;
        lg[0] = log_tab(f[0], lok0, ltab);
        lg[1] = log_tab(f[1], lok0, ltab);
        lg[2] = log_tab(f[2], lok1, ltab);
        lg[3] = log_tab(f[3], lok1, ltab);
        if (!(lok0 && lok1)) {
          if (!lok0) {
            lg[0] = f[0] > 0.0 ? log_fast(f[0]) : 0.0;
            lg[1] = f[1] > 0.0 ? log_fast(f[1]) : 0.0;
          }
          if (!lok1) {
            lg[2] = f[2] > 0.0 ? log_fast(f[2]) : 0.0;
            lg[3] = f[3] > 0.0 ? log_fast(f[3]) : 0.0;
          }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double fv = f[i];
          acc[0] = fma(fv > 0.0 ? fv : 0.0, lg[i] - xl[i], acc[0]);
          acc[1] += fv;
          rs += fv;
          if constexpr (METRICS) {
            const double2 c2 = v[i >> 1][1], g2 = v[i >> 1][NM + 2];
            const double cv = (i & 1) ? c2.y : c2.x;
            const double gv = (i & 1) ? g2.y : g2.x;
            acc[2] = fma(cv, fv, acc[2]);
            acc[3] = fma(fv, fv, acc[3]);
            const double fm = fmin(fv, 0.0);
            acc[4] = fma(fm, fm, acc[4]);
            const double shv = cv - gv;
            if constexpr (kZetaFromA) {   // slack >= 0: acc[5] stays 0 (see the single-slice path)
              acc[6] = fma(fv, shv - zeta_a, acc[6]);
            } else {
              fk[2 * s + i] = fv;
              shk[2 * s + i] = shv;
              shmin = fmin(shmin, shv);
            }
          }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) cacc[2 * s + i] += f[i];
        D.refill2_deferred();
      } else if (s < nsl) {
        double2 v[NA];
        D.fetchn(v);
        const double2 x = v[0];
        const double2 yy = v[NM], ee = v[NM + 1];
        bool ok = true;   // both exps of the slice branch-free (exp() only when out of range)
        double ex2[2] = {exp_tab(x.x, ok, etab), exp_tab(x.y, ok, etab)};
        if (!ok) {   // per element (exp_t), as k_materialize_rounded forms X
          ex2[0] = exp_t(x.x, etab);
          ex2[1] = exp_t(x.y, etab);
        }
        double f2[2] = {(ex2[0] * z) * yy.x, (ex2[1] * z) * yy.y};   // feasibility.py:65
        if (deficit > 0.0) {                                          // feasibility.py:67-68
          double d0, d1;
          DD.pair(e_r * ee.x, e_r * ee.y, d0, d1);
          f2[0] = f2[0] + d0;
          f2[1] = f2[1] + d1;
        }
        // feasibility.py:84 terms f (log f - log y) for f > 0: table logs,
        // branch-free; log_fast only for a pair with an entry near 1, zero,
        // subnormal, negative or non-finite
        bool lok = true;
        double lg[2] = {log_tab(f2[0], lok, ltab), log_tab(f2[1], lok, ltab)};
        if (!lok) {
          lg[0] = f2[0] > 0.0 ? log_fast(f2[0]) : 0.0;
          lg[1] = f2[1] > 0.0 ? log_fast(f2[1]) : 0.0;
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double xl = e ? x.y : x.x;
          const double fv = f2[e];
          // the sums below are reductions (their order differs from numpy's
          // anyway): fused multiply-adds
          acc[0] = fma(fv > 0.0 ? fv : 0.0, lg[e] - xl, acc[0]);
          acc[1] += fv;
          rs += fv;
          if constexpr (METRICS) {
            const double cv = e ? v[1].y : v[1].x;
            const double gv = e ? v[NM + 2].y : v[NM + 2].x;
            acc[2] = fma(cv, fv, acc[2]);
            acc[3] = fma(fv, fv, acc[3]);
            const double fm = fmin(fv, 0.0);
            acc[4] = fma(fm, fm, acc[4]);
            const double shv = cv - gv;
            // slack = shv - zeta >= 0 exactly (zeta is the row minimum of the
            // same shv values, and fl(a - b) >= 0 for a >= b), so the
            // reference's sum min(slack, 0)^2 (feasibility.py:117) is 0:
            // acc[5] stays 0
            if constexpr (kZetaFromA) {
              acc[6] = fma(fv, shv - zeta_a, acc[6]);
            } else {
              fk[2 * s + e] = fv;
              shk[2 * s + e] = shv;
              shmin = fmin(shmin, shv);
            }
          }
        }
        cacc[2 * s] += f2[0];
        cacc[2 * s + 1] += f2[1];
      }
    }
    if constexpr (KR > 1) {
      const double zeta = D.row_min(shmin);
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        if (s < nsl) {
#pragma unroll
          for (int e = 0; e < 2; ++e) acc[6] = fma(fk[2 * s + e], shk[2 * s + e] - zeta, acc[6]);   // slack >= 0: acc[5] = 0
        }
      }
    }
    D.row_sum_deferred(rs, r, io.rowpart, rsl);
  }
  // CTA-level scalar partials
  double v4[4] = {acc[0], acc[1], acc[2], acc[3]};
  D.template reduce<4, kSum>(v4);
  double w3[3] = {acc[4], acc[5], acc[6]};
  D.template reduce<3, kSum>(w3);
  if (D.tid == 0) {
    double* sp = io.spart + (size_t)blockIdx.x * 8;
    sp[0] = v4[0];
    sp[1] = v4[1];
    sp[2] = v4[2];
    sp[3] = v4[3];
    sp[4] = w3[0];
    sp[5] = w3[1];
    sp[6] = w3[2];
    sp[7] = 0.0;
  }
  double* dst = io.colpart + (size_t)D.cid * D.g.n;
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    if (s < nsl) {
      const int j = D.col(s, 0);
      if (j < D.c1) dst[j] = cacc[2 * s];
      if (j + 1 < D.c1) dst[j + 1] = cacc[2 * s + 1];
    }
  }
  D.finish();
}

// -------------------------------------------------------- warm start, zeta
// sinkhorn.py:47-51 (zeta = eta (log a - LSE_row(logX + (gamma - C)/eta)))
// fused with sinkhorn.py:61-65 (column sums of exp(logX + (zeta + gamma -
// C)/eta), evaluated with the reference's own expression order).
struct WarmZIO {
  const double* gamma;
  const double* log_a;
  double eta;
  double* zeta;      // local rows
  double* colpart;   // [ncl][n]
};

template <int NS>
__global__ void __launch_bounds__(kMaxThreads, OTB_DENSE_MINB) k_warm_zeta(Geom geo, WarmZIO io) {
  extern __shared__ __align__(128) unsigned char smem[];
  Dense<2> D;
  D.setup(geo, smem);
  if (D.producer) {
    D.produce();
    D.finish();
    return;
  }
  const double eta = io.eta;
  const Divider DIV(eta);
  for (int r = D.r0; r < D.r1; ++r) {
    double xs[2 * NS], cs[2 * NS];
    double mx = -INFINITY;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      xs[2 * s] = xs[2 * s + 1] = 0.0;
      cs[2 * s] = cs[2 * s + 1] = 0.0;
      if (s < D.nsl) {
        double2 c, x;
        D.fetch(c, x);
        xs[2 * s] = x.x;
        xs[2 * s + 1] = x.y;
        cs[2 * s] = c.x;
        cs[2 * s + 1] = c.y;
        const int j = D.col(s, 0);
        const double2 gm = load_pair(io.gamma, j, D.c1);
        double q0, q1;
        DIV.pair(gm.x - c.x, gm.y - c.y, q0, q1);
        if (j < D.c1) mx = fmax(mx, x.x + q0);
        if (j + 1 < D.c1) mx = fmax(mx, x.y + q1);
      }
    }
    double t[1] = {mx};
    D.reduce<1, kMax>(t);
    double M = t[0];
    double se = 0.0;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      if (s < D.nsl) {
        const int j = D.col(s, 0);
        const double2 gm = load_pair(io.gamma, j, D.c1);
        double q0, q1;
        DIV.pair(gm.x - cs[2 * s], gm.y - cs[2 * s + 1], q0, q1);
        bool ok = true;
        double e0 = exp_fast((xs[2 * s] + q0) - M, ok), e1 = exp_fast((xs[2 * s + 1] + q1) - M, ok);
        if (!ok) {
          e0 = exp((xs[2 * s] + q0) - M);
          e1 = exp((xs[2 * s + 1] + q1) - M);
        }
        if (j < D.c1) se += e0;
        if (j + 1 < D.c1) se += e1;
      }
    }
    t[0] = se;
    D.reduce<1, kSum>(t);
    double S = t[0];
    if (D.g.cl > 1) {
      double v2[2] = {M, S};
      const double* all = D.exchange<2>(v2);
      double Mg = all[0];
      for (int q = 1; q < D.g.cl; ++q) Mg = fmax(Mg, all[q * 4]);
      double Sg = 0.0;
      for (int q = 0; q < D.g.cl; ++q) Sg += all[q * 4 + 1] * exp(all[q * 4] - Mg);
      M = Mg;
      S = Sg;
    }
    const int64_t gi = D.g.row0 + r;
    const double zeta = eta * (__ldg(io.log_a + gi) - (M + log(S)));
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      if (s < D.nsl) {
        const int j = D.col(s, 0);
        const double2 gm = load_pair(io.gamma, j, D.c1);
        double q0, q1;
        DIV.pair((zeta + gm.x) - cs[2 * s], (zeta + gm.y) - cs[2 * s + 1], q0, q1);
        bool ok = true;
        double e0 = exp_fast(xs[2 * s] + q0, ok), e1 = exp_fast(xs[2 * s + 1] + q1, ok);
        if (!ok) {
          e0 = exp(xs[2 * s] + q0);
          e1 = exp(xs[2 * s + 1] + q1);
        }
        if (j >= D.c1) e0 = 0.0;
        if (j + 1 >= D.c1) e1 = 0.0;
        double2* a2 = D.acc2(0, s);
        double2 v = *a2;
        v.x += e0;
        v.y += e1;
        *a2 = v;
      }
    }
    if (D.tid == 0 && D.cr == 0) io.zeta[r] = zeta;
  }
  bar_sync(1, D.g.nt);
  D.store_acc(0, io.colpart + (size_t)D.cid * D.g.n);
  D.finish();
}

// ------------------------------------------------------- warm start, gamma
// sinkhorn.py:54-58: column log-sum-exp of logX + (zeta - C)/eta, as an
// online (max, sum) pair per column; partial pairs per cluster.
struct WarmGIO {
  const double* zeta;
  double eta;
  double* colpart;   // [ncl][2][n]
};

template <int NS>
__global__ void __launch_bounds__(kMaxThreads, OTB_DENSE_MINB) k_warm_gamma(Geom geo, WarmGIO io) {
  extern __shared__ __align__(128) unsigned char smem[];
  Dense<2> D;
  D.setup(geo, smem);
  if (D.producer) {
    D.produce();
    D.finish();
    return;
  }
  const double eta = io.eta;
  const Divider DIV(eta);
#pragma unroll
  for (int s = 0; s < NS; ++s)
    if (s < D.nsl) *D.acc2(0, s) = make_double2(-INFINITY, -INFINITY);
  for (int r = D.r0; r < D.r1; ++r) {
    const double zi = io.zeta[r];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      if (s < D.nsl) {
        double2 c, x;
        D.fetch(c, x);
        const int j = D.col(s, 0);
        double2* m2 = D.acc2(0, s);
        double2* s2 = D.acc2(1, s);
        double2 m = *m2, sm = *s2;
        double q0, q1;
        DIV.pair(zi - c.x, zi - c.y, q0, q1);
        if (j < D.c1) {
          const double tv = x.x + q0;
          if (tv > m.x) {
            sm.x = sm.x * exp(m.x - tv) + 1.0;
            m.x = tv;
          } else {
            sm.x += exp(tv - m.x);
          }
        }
        if (j + 1 < D.c1) {
          const double tv = x.y + q1;
          if (tv > m.y) {
            sm.y = sm.y * exp(m.y - tv) + 1.0;
            m.y = tv;
          } else {
            sm.y += exp(tv - m.y);
          }
        }
        *m2 = m;
        *s2 = sm;
      }
    }
  }
  bar_sync(1, D.g.nt);
  D.store_acc(0, io.colpart + ((size_t)D.cid * 2 + 0) * D.g.n);
  D.store_acc(1, io.colpart + ((size_t)D.cid * 2 + 1) * D.g.n);
  D.finish();
}

// -------------------------------------------------------- test-only hook
// Dense P = exp(logit - M_i) / S_i using the row statistics of the last
// eval (semidual.py:82-83).  Used by RowSoftmaxCache.p in parity tests.
__global__ void k_materialize_p(const double* C, const double* X, int64_t ld, int m_loc, int n,
                                const double* gamma, double eta, const double* rowM, const double* rowS,
                                double* P, int64_t ldp) {
  OTB_EXP_TABLE(etab);
  __syncthreads();
  const int64_t total = (int64_t)m_loc * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx / n), j = (int)(idx % n);
    const double z = X[(size_t)r * ld + j] + Divider(eta)(gamma[j] - C[(size_t)r * ld + j]);
    P[(size_t)r * ldp + j] = div_rn(exp_t(z - rowM[r], etab), rowS[r]);
  }
}

// Dense rounded plan F^ of the last test (feasibility.py:63-68), test /
// result hook: ((exp(logX) z_i) y_j) + (e_r_i e_c_j) / deficit.
__global__ void k_materialize_rounded(const double* X, int64_t ld, int m_loc, int n, const double* zrow,
                                      const double* y, const double* er, const double* ec,
                                      const double* deficit_ptr, double* out, int64_t ldo) {
  OTB_EXP_TABLE(etab);
  __syncthreads();
  const double deficit = *deficit_ptr;
  const int64_t total = (int64_t)m_loc * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx / n), j = (int)(idx % n);
    double f = (exp_t(X[(size_t)r * ld + j], etab) * zrow[r]) * y[j];
    if (deficit > 0.0) f = f + div_rn(er[r] * ec[j], deficit);
    out[(size_t)r * ldo + j] = f;
  }
}

}  // namespace otb
