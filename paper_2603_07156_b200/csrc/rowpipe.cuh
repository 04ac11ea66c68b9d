// Row-streaming machinery shared by the dense passes over C and log X.
//
// Layout and mapping:
//   * a matrix is m_loc rows x ld doubles in HBM (ld = round_up(n, 32), so
//     every row starts 256-byte aligned);
//   * a cluster of `cl` CTAs owns a contiguous block of rows; CTA rank q of
//     the cluster owns the column window [q*colw, min((q+1)*colw, n));
//   * a CTA = `nt` consumer threads + one producer warp.  The producer's
//     elected lane streams the window of each row, one "slice" of 2*nt
//     columns at a time, into an `nstage`-deep shared-memory ring with 1-D
//     TMA bulk copies (cp.async.bulk ... complete_tx on an mbarrier);
//   * consumer thread t owns columns c0 + s*2*nt + 2t + {0,1} of every row
//     (slice s < NS), reads them from the ring as one 16-byte vector, and
//     keeps the row in registers until the per-row reductions are done;
//   * per-column accumulators live in shared memory at the thread's own
//     slots (conflict-free, no atomics), and are written once per CTA as a
//     partial row that a column-parallel "finish" kernel reduces in fixed
//     order (deterministic);
//   * per-row reductions (max / sum / min) are warp shuffles + one named
//     barrier; when cl > 1 the per-CTA results are exchanged through DSMEM
//     (remote st.shared::cluster + remote mbarrier arrive).
#pragma once

#include "common.cuh"

namespace otb {

constexpr int kMaxCluster = 16;   // > 8: non-portable cluster sizes
constexpr int kXb = 4;       // cluster exchange buffers (rotating; >= 3 needed, see exchange())
constexpr int kMaxNS = 10;   // 1024-column slices per CTA: one CTA per row up to n = 10240
#ifndef OTB_F2_DEFER
#define OTB_F2_DEFER 0   // fetchn2's refill decision after the slices' arithmetic (refill2_deferred)
#endif

struct Geom {
  const double* mat0;   // first streamed matrix (row-major, ld)
  const double* mat1;   // second streamed matrix or nullptr
  const double* vec[3]; // NV row-invariant length-n vectors (gamma, y, ...) streamed as the last NV
                        // arrays of every stage, a whole slice each: 16-byte aligned, with at least
                        // one slice of padding past n (its value chosen so masked columns drop out)
  int64_t ld;           // leading dimension (doubles)
  int m_loc;            // local rows
  int n;                // columns
  int64_t row0;         // global index of local row 0
  int nt;               // consumer threads per CTA
  int ns;               // slices per row per CTA (<= NS template)
  int cl;               // cluster size
  int colw;             // columns per CTA window (even)
  int nstage;           // ring depth
  int nacc;             // accumulator vectors in smem (0..2)
};

// Shared-memory carve-up; identical for every dense kernel.
struct SmemMap {
  double* ring;      // nstage * nmat * 2nt
  double* acc;       // nacc * ns * 2nt
  double* slots;     // 2 * kMaxWarps * 4
  double* xbuf;      // kXb * kMaxCluster * 4
  uint64_t* full;    // nstage
  uint64_t* empty;   // nstage
  uint64_t* xbar;    // kXb
  int* misc;         // 64 ints
};

OTB_DEV size_t smem_bytes_for(const Geom& g, int nmat) {
  size_t slice = 2 * (size_t)g.nt;
  size_t d = (size_t)g.nstage * nmat * slice + (size_t)g.nacc * g.ns * slice + 2 * kMaxWarps * 4 + kXb * kMaxCluster * 4;
  return d * 8 + (2 * (size_t)g.nstage + kXb) * 8 + 64 * 4;
}

OTB_DEV SmemMap carve(const Geom& g, int nmat, unsigned char* base) {
  SmemMap s;
  const size_t slice = 2 * (size_t)g.nt;
  double* p = reinterpret_cast<double*>(base);
  s.ring = p;
  p += (size_t)g.nstage * nmat * slice;
  s.acc = p;
  p += (size_t)g.nacc * g.ns * slice;
  s.slots = p;
  p += 2 * kMaxWarps * 4;
  s.xbuf = p;
  p += kXb * kMaxCluster * 4;
  uint64_t* b = reinterpret_cast<uint64_t*>(p);
  s.full = b;
  s.empty = b + g.nstage;
  s.xbar = b + 2 * g.nstage;
  s.misc = reinterpret_cast<int*>(b + 2 * g.nstage + kXb);
  return s;
}

// Per-CTA context of a dense pass.
//
// SELF = false: a producer warp (threads nt..nt+31) streams the ring; the
// consumers release a stage on its `empty` barrier.
// SELF = true: no producer warp (the CTA is the nt consumer threads, 16
// warps at 512: 128 registers instead of 96).  Thread 0 issues the first
// nstage slices; afterwards the LAST warp to finish reading a stage refills
// it with the slice nstage positions ahead: every warp's lane 0 adds to the
// stage's arrival counter (acq_rel), the one that completes the round
// (count = rounds * nwarps - 1 before it) fences the async proxy and issues
// the bulk copies.  Every thread advances the same refill cursor.
template <int NMAT, bool SELF = false, int NV = 0>
struct Dense {
  static_assert(NV >= 0 && NV <= 3 && NMAT - NV >= 1 && NMAT - NV <= 2, "1-2 matrices and 0-3 vectors");
  static constexpr int NM = NMAT - NV;   // streamed matrices
  Geom g;
  SmemMap sm;
  int tid, lane, warp;
  bool producer;
  int cr;        // rank in cluster
  int cid;       // cluster index
  int ncl;       // number of clusters
  int r0, r1;    // local rows of this cluster
  int c0, c1;    // column window of this CTA
  int nsl;       // slices actually used by this CTA
  int slice;     // 2*nt
  // pipeline state
  int stage;
  uint32_t phase;
  int rphase;    // block-reduce slot parity
  int xcount;    // DSMEM exchanges done
  bool tail;     // the window's last slice is partial (columns >= c1 masked)
  // SELF: refill cursor (row, slice) of the slice nstage positions ahead of
  // the one being consumed, and the ring rounds completed
  int fr, fs;
  uint32_t rounds;

  OTB_DEV void setup(const Geom& geo, unsigned char* smem) {
    g = geo;
    sm = carve(g, NMAT, smem);
    tid = threadIdx.x;
    lane = tid & 31;
    warp = tid >> 5;
    producer = SELF ? false : tid >= g.nt;
    cr = (g.cl > 1) ? (int)cluster_ctarank() : 0;
    cid = blockIdx.x / g.cl;
    ncl = gridDim.x / g.cl;
    r0 = (int)(((int64_t)cid * g.m_loc) / ncl);
    r1 = (int)(((int64_t)(cid + 1) * g.m_loc) / ncl);
    c0 = cr * g.colw;
    c1 = min(c0 + g.colw, g.n);
    slice = 2 * g.nt;
    nsl = (c1 > c0) ? (c1 - c0 + slice - 1) / slice : 0;
    tail = nsl > 0 && (c1 - c0) < nsl * slice;
    stage = 0;
    phase = 0;
    rphase = 0;
    xcount = 0;
    rounds = 1;
    fr = r0 + (nsl > 0 ? g.nstage / nsl : 0);
    fs = nsl > 0 ? g.nstage % nsl : 0;
    if (tid == 0) {
      for (int s = 0; s < g.nstage; ++s) {
        mbar_init(&sm.full[s], 1);
        if (!SELF) mbar_init(&sm.empty[s], g.nt / 32);
        if (SELF) sm.misc[s] = 0;
      }
      // exchange buffers: one local arrival + 32 bytes (4 doubles) from every
      // CTA of the cluster per use (st.async complete_tx), armed here for the
      // first kXb exchanges and re-armed by the receiver after each one
      for (int q = 0; q < kXb; ++q) mbar_init(&sm.xbar[q], 1);
      fence_mbar_init();
      if (g.cl > 1)
        for (int q = 0; q < kXb; ++q) mbar_arrive_expect_tx(&sm.xbar[q], 32u * (uint32_t)g.cl);
    }
    // zero accumulators (consumer-owned slots only, but any thread may do it)
    const int na = g.nacc * g.ns * slice;
    for (int i = tid; i < na; i += blockDim.x) sm.acc[i] = 0.0;
    if (SELF) {
      // the ring too: a partial last slice leaves stale columns in its stage,
      // which must be finite (the kernels mask them through the vectors'
      // padding)
      const int nr = g.nstage * NMAT * slice;
      for (int i = tid; i < nr; i += blockDim.x) sm.ring[i] = 0.0;
      fence_proxy_async();
      __syncthreads();
      if (tid == 0 && nsl > 0) {
        int rr = r0, ss = 0;
        for (int k = 0; k < g.nstage && rr < r1; ++k) {
          issue(k, rr, ss);
          if (++ss == nsl) {
            ss = 0;
            ++rr;
          }
        }
      }
    }
    if (g.cl > 1) {
      __syncwarp();
      cluster_sync_all();
    } else {
      __syncthreads();
    }
  }

  OTB_DEV double* stage_buf(int st, int mat) const { return sm.ring + ((size_t)st * NMAT + mat) * slice; }

  // Bulk copies of slice (r, s) of the window into stage st: the matrices'
  // columns inside the window, the vectors as a whole slice (their padding
  // past n covers a partial last slice).
  OTB_DEV void issue(int st, int r, int s) {
    int cols = min(slice, c1 - c0 - s * slice);
    cols = (cols + 1) & ~1;
    const uint32_t bytes = (uint32_t)cols * 8u;
    const uint32_t vbytes = (uint32_t)slice * 8u;
    mbar_arrive_expect_tx(&sm.full[st], bytes * NM + vbytes * NV);
    const size_t off = (size_t)r * g.ld + c0 + (size_t)s * slice;
    bulk_g2s(stage_buf(st, 0), g.mat0 + off, bytes, &sm.full[st]);
    if (NM > 1) bulk_g2s(stage_buf(st, 1), g.mat1 + off, bytes, &sm.full[st]);
    if constexpr (NV > 0) {
#pragma unroll
      for (int v = 0; v < NV; ++v)
        bulk_g2s(stage_buf(st, NM + v), g.vec[v] + c0 + (size_t)s * slice, vbytes, &sm.full[st]);
    }
  }

  // Producer: stream every (row, slice) of this CTA's window.
  OTB_DEV void produce() {
    if constexpr (SELF) return;
    if (lane != 0) return;
    for (int r = r0; r < r1; ++r) {
      for (int s = 0; s < nsl; ++s) {
        mbar_wait(&sm.empty[stage], phase ^ 1u);
        issue(stage, r, s);
        advance();
      }
    }
  }

  // Releases the stage just read (consumer side, all threads of the warp).
  OTB_DEV void release() {
    __syncwarp();
    if (!SELF) {
      if (lane == 0) mbar_arrive(&sm.empty[stage]);
    } else {
      // the warp whose arrival completes the stage's round refills it.  A
      // relaxed atomic (no fence: acq_rel compiles to a MEMBAR that waits
      // for the warp's outstanding global stores): every warp's reads of the
      // stage are issued before its arrival, in the same in-order shared
      // memory pipeline, and the refill's bulk copy lands a global round
      // trip after the last arrival.
      // The count is checked at once: deferring the check (and the refill)
      // by even one slice's arithmetic was measured slower (config 5: eval
      // 17.6 -> 20.0 ms, test_c 28.1 -> 35.2 ms) — the ring is shallow and
      // the refill latency matters more than the atomic's round trip.
      if (lane == 0) {
        uint32_t old;
        asm volatile("atom.relaxed.cta.shared::cta.add.u32 %0, [%1], 1;"
                     : "=r"(old)
                     : "r"(smem_u32(&sm.misc[stage]))
                     : "memory");
        if (old == rounds * (uint32_t)(g.nt >> 5) - 1u && fr < r1) {   // last reader of this round
          fence_proxy_async();
          issue(stage, fr, fs);
        }
      }
      if (++fs == nsl) {
        fs = 0;
        ++fr;
      }
    }
  }

  OTB_DEV void advance() {
    if (++stage == g.nstage) {
      stage = 0;
      phase ^= 1u;
      ++rounds;
    }
  }

  // Consumer: column index of element e (0/1) of slice s for this thread.
  OTB_DEV int col(int s, int e) const { return c0 + s * slice + 2 * tid + e; }
  OTB_DEV bool valid(int s, int e) const { return col(s, e) < c1; }

  // Wait for slice s of the current row; returns the thread's two values of
  // each matrix (garbage where !valid).
  OTB_DEV void fetch(double2& v0, double2& v1) {
    mbar_wait(&sm.full[stage], phase);
    const double2* b0 = reinterpret_cast<const double2*>(stage_buf(stage, 0));
    v0 = b0[tid];
    if (NMAT > 1) {
      const double2* b1 = reinterpret_cast<const double2*>(stage_buf(stage, 1));
      v1 = b1[tid];
    }
    release();
    advance();
  }

  // The same for every streamed array (matrices first, then vectors).
  OTB_DEV void fetchn(double2 (&v)[NMAT]) {
    mbar_wait(&sm.full[stage], phase);
#pragma unroll
    for (int k = 0; k < NMAT; ++k) v[k] = reinterpret_cast<const double2*>(stage_buf(stage, k))[tid];
    release();
    advance();
  }
  // TWO consecutive slices of the current row at once (SELF only): both
  // stages are waited for, read and released together, so the arithmetic of
  // the four elements forms one basic block and their dependent fp64 chains
  // interleave.  With one slice per fetch a warp has two elements in flight
  // and every slice costs the full latency of its chain (the wait loop and
  // the release are block boundaries the scheduler does not move code
  // across): the dense passes ran latency bound at ~45% issue-active.  The
  // two arrival atomics go out back to back (one round trip, not two).
  OTB_DEV void fetchn2(double2 (&v)[2][NMAT]) {
    static_assert(SELF, "fetchn2 is for the self-fed ring");
    const int st0 = stage;
    const uint32_t ph0 = phase, rd0 = rounds;
    advance();
    const int st1 = stage;
    const uint32_t ph1 = phase, rd1 = rounds;
    advance();
    mbar_wait(&sm.full[st0], ph0);
    mbar_wait(&sm.full[st1], ph1);
#pragma unroll
    for (int k = 0; k < NMAT; ++k) {
      v[0][k] = reinterpret_cast<const double2*>(stage_buf(st0, k))[tid];
      v[1][k] = reinterpret_cast<const double2*>(stage_buf(st1, k))[tid];
    }
    __syncwarp();
    if (lane == 0) {
      asm volatile("atom.relaxed.cta.shared::cta.add.u32 %0, [%1], 1;"
                   : "=r"(pend_old[0])
                   : "r"(smem_u32(&sm.misc[st0]))
                   : "memory");
      asm volatile("atom.relaxed.cta.shared::cta.add.u32 %0, [%1], 1;"
                   : "=r"(pend_old[1])
                   : "r"(smem_u32(&sm.misc[st1]))
                   : "memory");
    }
    pend_st[0] = st0;
    pend_st[1] = st1;
    pend_tgt[0] = rd0 * (uint32_t)(g.nt >> 5) - 1u;
    pend_tgt[1] = rd1 * (uint32_t)(g.nt >> 5) - 1u;
#if !OTB_F2_DEFER
    refill2();
#endif
  }
  // The refill decision of the last fetchn2 (lane 0: did this warp's arrival
  // complete a stage's round?).  With OTB_F2_DEFER the kernel calls it after
  // the slices' arithmetic, so the atomics' round trip is not waited for.
  uint32_t pend_old[2], pend_tgt[2];
  int pend_st[2];
  OTB_DEV void refill2() {
    int fr1 = fr, fs1 = fs + 1;
    if (fs1 == nsl) {
      fs1 = 0;
      ++fr1;
    }
    if (lane == 0) {
      const bool f0 = pend_old[0] == pend_tgt[0] && fr < r1, f1 = pend_old[1] == pend_tgt[1] && fr1 < r1;
      if (f0 || f1) {
        fence_proxy_async();
        if (f0) issue(pend_st[0], fr, fs);
        if (f1) issue(pend_st[1], fr1, fs1);
      }
    }
    fr = fr1;
    fs = fs1 + 1;
    if (fs == nsl) {
      fs = 0;
      ++fr;
    }
  }
  OTB_DEV void refill2_deferred() {
#if OTB_F2_DEFER
    refill2();
#endif
  }

  OTB_DEV void fetch3(double2& v0, double2& v1, double2& v2) {
    static_assert(NMAT == 3, "fetch3 needs three streamed arrays");
    double2 v[3];
    fetchn(v);
    v0 = v[0];
    v1 = v[1];
    v2 = v[2];
  }

  // Accumulator slots of this thread for slice s (double2 at acc[k]).
  OTB_DEV double2* acc2(int k, int s) const {
    return reinterpret_cast<double2*>(sm.acc + (size_t)k * g.ns * slice + (size_t)s * slice) + tid;
  }

  template <int K, int OP>
  OTB_DEV void reduce(double (&v)[K]) {
    block_reduce<K, OP>(v, sm.slots, rphase, g.nt);
  }

  // Exchange K (<=4) values among the cl (> 1) CTAs of the cluster.  Returns
  // the shared-memory table: entry [q*4 + k] is CTA q's value k.  Every
  // value goes out as st.async (async proxy) completing 32 bytes per CTA on
  // the peer's buffer barrier, so the wait is a cta-scope one (no L1
  // invalidation, unlike a cluster-scope acquire).  Buffers rotate over
  // kXb = 4: a peer can write buffer x mod 4 again only at exchange x + 4,
  // i.e. after this CTA sent exchange x + 3, which its warp 0 does only after
  // the block reduction that precedes it — by then every thread has finished
  // reading table x (read right after exchange x returns).  The table is
  // readable until the next block reduction.  Consumer threads only.
  template <int K>
  OTB_DEV const double* exchange(const double (&v)[K]) {
    static_assert(K >= 1 && K <= 4, "exchange of 1..4 values");
    const int q = xcount & (kXb - 1);
    const uint32_t par = (uint32_t)((xcount / kXb) & 1);
    double* mine = sm.xbuf + (q * kMaxCluster + cr) * 4;
    if (warp == 0 && lane < g.cl) {   // lane rk serves cluster rank rk: the remote ops go out in parallel
      const uint32_t dst = mapa(smem_u32(mine), (uint32_t)lane);
      const uint32_t bar = mapa(smem_u32(&sm.xbar[q]), (uint32_t)lane);
      st_async_v2f64(dst, v[0], K > 1 ? v[K > 1 ? 1 : 0] : 0.0, bar);
      st_async_v2f64(dst + 16u, K > 2 ? v[K > 2 ? 2 : 0] : 0.0, K > 3 ? v[K > 3 ? 3 : 0] : 0.0, bar);
    }
    mbar_wait(&sm.xbar[q], par);   // every consumer thread: the async-proxy data is then visible to it
    ++xcount;
    if (tid == 0) mbar_arrive_expect_tx(&sm.xbar[q], 32u * (uint32_t)g.cl);   // re-arm for exchange + kXb
    return sm.xbuf + q * kMaxCluster * 4;
  }

  // Row-wide (cluster-wide) sum of a per-thread value.
  OTB_DEV double row_sum(double v) {
    double t[1] = {v};
    reduce<1, kSum>(t);
    if (g.cl == 1) return t[0];
    const double* all = exchange<1>(t);
    double s = 0.0;
    for (int q = 0; q < g.cl; ++q) s += all[q * 4];
    return s;
  }
  // row_sum and row_min of two per-thread values with one barrier (and one
  // exchange when the row is split); same bits as the separate calls.
  OTB_DEV void row_sum_min(double s, double mn, double& S, double& MN) {
    block_reduce2<kSum, kMin>(s, mn, sm.slots, rphase, g.nt);
    if (g.cl == 1) {
      S = s;
      MN = mn;
      return;
    }
    const double t[2] = {s, mn};
    const double* all = exchange<2>(t);
    S = 0.0;
    MN = all[1];
    for (int q = 0; q < g.cl; ++q) S += all[q * 4];
    for (int q = 1; q < g.cl; ++q) MN = fmin(MN, all[q * 4 + 1]);
  }
  OTB_DEV double row_min(double v) {
    double t[1] = {v};
    reduce<1, kMin>(t);
    if (g.cl == 1) return t[0];
    const double* all = exchange<1>(t);
    double s = all[0];
    for (int q = 1; q < g.cl; ++q) s = fmin(s, all[q * 4]);
    return s;
  }

  // Row sum of a per-thread value written to out[r * cl + cr] WITHOUT a
  // barrier per row: each warp's lane sum goes to slot [row mod 8][warp]
  // (rsl: 2 x 8 x 16 doubles, double-buffered by batch); every 8th row (and
  // the last) one barrier, after which warp w reduces batch row w's 16 slots
  // with block_reduce's second-level tree (the same bits as reduce<1, kSum>).
  // Buffer b of batch k is written again by batch k + 2, after the barrier
  // of batch k + 1 that every warp reaches only after its reads of batch k.
  static constexpr int kRB = 8;
  OTB_DEV void row_sum_deferred(double v, int r, double* out, double* rsl) {
    const int i = r - r0, slot = i % kRB, buf = (i / kRB) & 1;
    const double ws = warp_sum(v);
    if (lane == 0) rsl[(buf * kRB + slot) * 16 + warp] = ws;
    if (slot == kRB - 1 || r == r1 - 1) {
      bar_sync(1, g.nt);
      if (warp <= slot) {
        const int nw = g.nt >> 5;
        const double t = warp_sum(lane < nw ? rsl[(buf * kRB + warp) * 16 + lane] : 0.0);
        if (lane == 0) out[(size_t)(r - slot + warp) * g.cl + cr] = t;
      }
    }
  }

  // Writes accumulator k to the partial row `dst` (global columns).
  OTB_DEV void store_acc(int k, double* dst) const {
    for (int s = 0; s < nsl; ++s) {
      const double2 a = *acc2(k, s);
      const int j = col(s, 0);
      if (j < c1) dst[j] = a.x;
      if (j + 1 < c1) dst[j + 1] = a.y;
    }
  }

  OTB_DEV void finish() {
    if (g.cl > 1) {
      __syncwarp();
      cluster_sync_all();
    }
  }
};

// Loads gamma-like column vectors as pairs (bounds-checked at n).
OTB_DEV double2 load_pair(const double* v, int j, int lim) {
  double2 r;
  r.x = (j < lim) ? __ldg(v + j) : 0.0;
  r.y = (j + 1 < lim) ? __ldg(v + j + 1) : 0.0;
  return r;
}

}  // namespace otb
