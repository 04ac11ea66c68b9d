// libotb host side: context, C ABI (include/otb.h) and the orchestration of
// one IBSN inner iteration on the device.  The host only reads scalars back
// (objective, gradient norm, CG status every kCgBatch iterations, slope,
// test results); every vector stays in HBM.
#include "otb.h"

#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "dense.cuh"
#include "dense_api.cuh"
#include "finish.cuh"
#include "sparse.cuh"

using namespace otb;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(expr)                                                                    \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess) return fail(OTB_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define TRY(expr)                  \
  do {                             \
    int s_ = (expr);               \
    if (s_ != OTB_OK) return s_;   \
  } while (0)

#define LAUNCH_CHECK()            \
  do {                            \
    ++c->launches;                \
    CUDA_TRY(cudaGetLastError()); \
  } while (0)

// ------------------------------------------------------------------ NCCL
struct NcclId {
  char internal[128];
};
typedef void* NcclComm;
struct Nccl {
  void* h = nullptr;
  int (*getUniqueId)(NcclId*) = nullptr;
  int (*commInitRank)(NcclComm*, int, NcclId, int) = nullptr;
  int (*allReduce)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
  int (*commDestroy)(NcclComm) = nullptr;
  const char* (*getErrorString)(int) = nullptr;
};
constexpr int kNcclFloat64 = 8;
constexpr int kNcclSum = 0;
constexpr int kNcclMax = 2;

int load_nccl(const char* path, Nccl& api) {
  if (api.h) return OTB_OK;
  void* h = dlopen(path && path[0] ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return fail(OTB_ERR_NCCL, std::string("dlopen nccl: ") + dlerror());
  api.getUniqueId = (int (*)(NcclId*))dlsym(h, "ncclGetUniqueId");
  api.commInitRank = (int (*)(NcclComm*, int, NcclId, int))dlsym(h, "ncclCommInitRank");
  api.allReduce = (int (*)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t))dlsym(h, "ncclAllReduce");
  api.commDestroy = (int (*)(NcclComm))dlsym(h, "ncclCommDestroy");
  api.getErrorString = (const char* (*)(int))dlsym(h, "ncclGetErrorString");
  if (!api.getUniqueId || !api.commInitRank || !api.allReduce || !api.commDestroy)
    return fail(OTB_ERR_NCCL, "nccl symbols missing");
  api.h = h;
  return OTB_OK;
}

// ------------------------------------------------------------- kernels
enum DenseKind {
  DK_EVAL = 0, DK_SPARSIFY, DK_TESTA, DK_TESTB, DK_TESTC0, DK_TESTC1, DK_WARMZ, DK_WARMG, DK_SPARSP, DK_SPDENSE,
  DK_COUNT
};
// streamed arrays: eval and test_a C, log X, gamma; test_b X, y; test_c X, y, e_c (+ C, gamma with
// the metrics)
const int kNmat[DK_COUNT] = {3, 2, 3, 2, 3, 5, 2, 2, 1, 1};
const int kNacc[DK_COUNT] = {1, 1, 1, 0, 0, 0, 1, 2, 1, 1};   // shared accumulators (test_b, test_c: registers)
// static shared memory (sparsify: scan table; test_b/test_c: deferred row-sum slots; exp/log tables)
const int kStaticSmem[DK_COUNT] = {2048, (int)(kTabInts * 4 + 16 + 2048), 2048, 4096, 8192, 8192, 0, 0,
                                   (int)(kTabInts * 4 + 16 + 2048), 0};
// kinds whose CTA has no producer warp (Dense<NMAT, true>: the consumers refill the ring)
const bool kSelfFeed[DK_COUNT] = {true, false, true, true, true, true, false, false, true, true};
int dense_block(int kind, int nt) { return nt + (kSelfFeed[kind] ? 0 : 32); }
constexpr int kMaxStageSelf = 16;   // ring depth cap of the self-fed kinds (misc holds their counters)

#define NS_ROW(K)                                                                                   \
  { nullptr, (const void*)K<1>, (const void*)K<2>, (const void*)K<3>, (const void*)K<4>,             \
    (const void*)K<5>, (const void*)K<6>, (const void*)K<7>, (const void*)K<8>, (const void*)K<9>,  \
    (const void*)K<10> }
#define NS_ROW2(K, B)                                                                                \
  { nullptr, (const void*)K<1, B>, (const void*)K<2, B>, (const void*)K<3, B>, (const void*)K<4, B>, \
    (const void*)K<5, B>, (const void*)K<6, B>, (const void*)K<7, B>, (const void*)K<8, B>,          \
    (const void*)K<9, B>, (const void*)K<10, B> }
static_assert(kMaxNS == 10, "kDenseFn rows list NS = 1..10");
const void* const kDenseFn[DK_COUNT][kMaxNS + 1] = {
    NS_ROW(k_eval),          NS_ROW2(k_sparsify, false), NS_ROW(k_test_a),    NS_ROW(k_test_b),
    NS_ROW2(k_test_c, false), NS_ROW2(k_test_c, true),   NS_ROW(k_warm_zeta), NS_ROW(k_warm_gamma),
    NS_ROW2(k_sparsify, true), NS_ROW(k_sparsify_dense)};

#define HV_ROW(K)                                                                                    \
  {                                                                                                  \
    (const void*)K<0>, (const void*)K<1>, (const void*)K<2>, (const void*)K<3>, (const void*)K<4>,   \
        (const void*)K<5>, (const void*)K<6>, (const void*)K<7>, (const void*)K<8>, (const void*)K<9>, \
        (const void*)K<10>, (const void*)K<11>, (const void*)K<12>                                   \
  }
const void* const kHvFn[kHvVariants] = HV_ROW(k_hv_grp);     // variant codes: sparse.cuh HvVar
const void* const kCgFn[kHvVariants] = HV_ROW(k_cg_fused);
#define WC_ROW(D)                                                                                     \
  {                                                                                                   \
    nullptr, (const void*)k_hv_wc<1, D>, (const void*)k_hv_wc<2, D>, (const void*)k_hv_wc<3, D>,     \
        (const void*)k_hv_wc<4, D>, (const void*)k_hv_wc<5, D>, (const void*)k_hv_wc<6, D>,           \
        (const void*)k_hv_wc<7, D>, (const void*)k_hv_wc<8, D>                                        \
  }
const void* const kWcFn[2][kMaxNQ + 1] = {WC_ROW(false), WC_ROW(true)};   // [dense P_rho][NQ]
// dense P_rho without a producer warp (the one used for dense mode)
const void* const kWcdFn[kMaxNQ + 1] = {nullptr,           (const void*)k_hv_wcd<1>, (const void*)k_hv_wcd<2>,
                                        (const void*)k_hv_wcd<3>, (const void*)k_hv_wcd<4>, (const void*)k_hv_wcd<5>,
                                        (const void*)k_hv_wcd<6>, (const void*)k_hv_wcd<7>, (const void*)k_hv_wcd<8>};
int wc_stage_bytes(int nqw) {
  switch (nqw) {
    case 1: return WcGeo<1>::kStage;
    case 2: return WcGeo<2>::kStage;
    case 3: return WcGeo<3>::kStage;
    case 4: return WcGeo<4>::kStage;
    case 5: return WcGeo<5>::kStage;
    case 6: return WcGeo<6>::kStage;
    case 7: return WcGeo<7>::kStage;
    default: return WcGeo<8>::kStage;
  }
}

enum ProfClass {
  PC_EVAL = 0, PC_SPARSIFY, PC_HV, PC_CGVEC, PC_TESTA, PC_TESTB, PC_TESTC, PC_WARMZ, PC_WARMG, PC_CGFUSED,
  PC_SKIP = 15,   // CG iterations launched past convergence (no-op kernels): not reported
  PC_N = 16
};

constexpr int kCgBatch = 16;
constexpr size_t kMaxDynSmem = 232448;  // 227 KB

}  // namespace

// Local group (otb_attach_group): the ranks of one process, one host thread
// each.  A generation barrier with a timeout; `broken` releases everyone.
struct otb_group {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool broken = false;
  double timeout_s = 300.0;
  const double* bufs[kMaxGroup] = {};
  int64_t counts[kMaxGroup] = {};
  int ops[kMaxGroup] = {};
  cudaEvent_t ready[kMaxGroup] = {}, done[kMaxGroup] = {};
  int devices[kMaxGroup] = {};

  int barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (broken) return fail(OTB_ERR_NCCL, "local group broken (a rank failed or timed out)");
    const uint64_t g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return OTB_OK;
    }
    const bool ok = cv.wait_for(lk, std::chrono::duration<double>(timeout_s), [&] { return gen != g || broken; });
    if (!ok) {
      broken = true;
      cv.notify_all();
      return fail(OTB_ERR_NCCL, "local group: barrier timed out (collective sequences of the ranks differ?)");
    }
    if (broken) return fail(OTB_ERR_NCCL, "local group broken (a rank failed or timed out)");
    return OTB_OK;
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    broken = true;
    cv.notify_all();
  }
};

struct otb_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int64_t m_glob = 0, n = 0, row0 = 0, row1 = 0, m_loc = 0, ld = 0;
  int num_sms = 148;
  // dense geometry
  int nt = 0, ns = 0, cl = 1, colw = 0, ncl = 0, grid = 0, per_sm = 1;
  int nstage[DK_COUNT] = {};
  size_t smem[DK_COUNT] = {};
  // hess_apply
  int hv_mode = 0, hv_grid = 0, hv_ng = 1;   // hv_mode 0 group smem, 1 global RED, 2 bitmap, 3 window clusters
  int hv_nb = 0, hv_win = 1;                   // row blocks (partial rows), CTAs per cluster (mode 3)
  int hv_var = 0, nq = 0, hv_threads = 512;   // kernel variant (sparse.cuh HvVar), bitmap words per row
  int hv_ng_d = 0;                             // ring stages of the dense-P_rho window-cluster kernel
  size_t hv_smem_d = 0;
  bool hv_wcd = true;                          // OTB_HV_WCD=0: the producer-warp dense kernel (comparison)
  // dense-P_rho overlay of a group-kernel context (hv_mode 0, n > 8192, e.g. config 3): while the
  // kept density is >= ov_min_density sparsify writes P_rho dense over the stored P and hess_apply
  // is k_hv_wcd<ov_nq> on ov_ncl clusters of ov_win CTAs; below it the CSR group kernel runs
  bool ov_ok = false;
  double ov_min_density = 0.25;                // kept density from which the overlay's dense product is the faster one
  int ov_nq = 0, ov_win = 0, ov_ncl = 0, ov_stages = 0;
  size_t ov_smem = 0;
  int* ov_rb = nullptr;                        // [ov_ncl + 1] equal row counts per cluster
  uint4* bm = nullptr;
  double* Pbuf = nullptr;    // P of the last eval (local rows x ld), streamed by sparsify
  unsigned long long* cg_trace = nullptr;   // OTB_CG_TRACE=1: phase stamps of the fused CG
  bool p_valid = false;
  bool rho_dense = false;    // the last sparsify wrote P_rho dense into Pbuf (window-cluster hess_apply)
  int dense_policy = -1;     // OTB_HV_DENSE: 0 never, 1 always, -1 by the last kept density
  double last_density = 0.0; // kept entries / (m_loc n) of the last sparsify
  bool have_density = false; // last_density is from a sparsify of this context (else sampled)
  int precond = 0;           // CG preconditioner: 0 none (the reference's plain CG), 1 Jacobi
  bool force_post = false;   // OTB_FORCE_EVAL_POST=1 (tests): the multi-rank eval finish on one rank
  // CUDA graphs of a 16-iteration CG batch (per-iteration path): [0] the
  // first batch of a solve (k = 0 has no direction update), [1] the others
  bool cg_graph = true;      // OTB_CG_GRAPH=0: eager launches
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t cg_exec[2] = {nullptr, nullptr};
  unsigned char cg_key[2][160] = {};
  int64_t cg_batch_launches[2] = {0, 0};
  double *jq = nullptr, *minv = nullptr, *zv = nullptr, *colpart2 = nullptr;   // PCG vectors
  bool rowpre_valid = false;
  size_t hv_smem = 0;
  bool cg_fused = false;     // persistent cooperative CG available (1 rank, smem hv)
  int fused_ng = 1;
  size_t fused_smem = 0;
  int* cta_rb = nullptr;     // [hv_grid + 1] row bounds of the hess_apply CTAs
  int colgrid = 0, col32 = 0;
  double* scal = nullptr;    // [hv_grid][2] per-CTA scalars of the fused CG
  // problem
  const double *C = nullptr, *a = nullptr, *b = nullptr, *log_a = nullptr, *log_b = nullptr;
  double eta = 0.0, norm_c = 0.0, norm_a = 0.0, norm_b = 0.0;
  bool norm_c_dev = false;   // ||C|| from ds->cnorm_sq (otb_set_cost_norm_sq)
  int64_t anchor = -1;
  bool bound = false;
  // buffers
  double *rowM = nullptr, *rowS = nullptr, *lse = nullptr, *zrow = nullptr, *er = nullptr, *rowpart = nullptr;
  double* czeta = nullptr;   // row c-transform of the KKT metrics (pass A -> pass C)
  double *colpart = nullptr, *vpart = nullptr, *sendbuf = nullptr, *bpart = nullptr;
  double *g = nullptr, *d = nullptr, *rhs = nullptr, *dir = nullptr, *cg_r = nullptr, *cg_p[2] = {nullptr, nullptr};
  double *cg_ap = nullptr, *cg_y = nullptr, *gtrial = nullptr, *yv = nullptr, *ec = nullptr;
  double* gev = nullptr;      // aligned copy of a caller's gamma for the eval's TMA stream
  double *Mloc = nullptr, *Mglob = nullptr, *Sloc = nullptr;
  int64_t *row_start = nullptr, *rowpre = nullptr;
  int* row_len = nullptr;        // stored doubles of each row run
  int* row_nnz = nullptr;        // kept entries per row (CSR export with the bitmap index)
  uint16_t* cols = nullptr;
  double* vals = nullptr;
  int64_t cap = 0, chunk = 0, nnz = 0;
  DevScalars* ds = nullptr;
  DevScalars* hs = nullptr;   // pinned
  CgState* cg = nullptr;
  CgState* hcg = nullptr;     // pinned
  double* hbuf = nullptr;     // pinned, 16 doubles
  // state
  double last_value = 0.0, last_gnorm = 0.0;
  bool have_eval = false;
  const double* round_src = nullptr;
  // NCCL
  Nccl nccl;
  NcclComm comm = nullptr;
  otb_group* group = nullptr;   // local group (instead of NCCL)
  double* lg_tmp = nullptr;     // its reduction target
  int nranks = 1, rank = 0;
  int64_t nnz_glob = 0;         // kept entries over all ranks
  int64_t launches = 0;       // kernels launched by this context
  // profiling
  bool prof = false;
  struct Rec {
    int cls;
    cudaEvent_t e0, e1;
    double bytes;
  };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  double prof_ms[PC_N] = {}, prof_bytes[PC_N] = {};
  int64_t prof_cnt[PC_N] = {};
};

namespace {

int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
int64_t rup(int64_t a, int64_t b) { return cdiv(a, b) * b; }

template <class T>
int dalloc(T** p, size_t count) {
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(OTB_ERR_NOMEM, std::string("cudaMalloc ") + std::to_string(count * sizeof(T)) + " bytes: " +
                                   cudaGetErrorString(e));
  }
  return OTB_OK;
}

// The dynamic shared-memory limit is a per-FUNCTION (process-wide)
// attribute: raise it once to the device maximum instead of to this
// context's need, so contexts of different shapes never lower it for each
// other.
cudaError_t allow_max_smem(const void* fn, int device) {
  int optin = 0;
  cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  if (e != cudaSuccess) return e;
  cudaFuncAttributes fa;
  e = cudaFuncGetAttributes(&fa, fn);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
}

// Jacobi PCG: sparsify also accumulates q = (P_rho o P_rho)^T a (accumulator 1)
int nacc_of(const otb_ctx* c, int kind) {
  return ((kind == DK_SPARSIFY || kind == DK_SPARSP || kind == DK_SPDENSE) && c->precond) ? 2 : kNacc[kind];
}

size_t dense_smem(const otb_ctx* c, int kind, int nstage) {
  const size_t slice = 2 * (size_t)c->nt;
  const size_t dbl = (size_t)nstage * kNmat[kind] * slice + (size_t)nacc_of(c, kind) * c->ns * slice + 2 * kMaxWarps * 4 +
                     kXb * kMaxCluster * 4;
  return dbl * 8 + (2 * (size_t)nstage + kXb) * 8 + 64 * 4;
}

Geom make_geom(const otb_ctx* c, int kind, const double* m0, const double* m1) {
  Geom g;
  g.mat0 = m0;
  g.mat1 = m1;
  g.vec[0] = g.vec[1] = g.vec[2] = nullptr;
  g.ld = c->ld;
  g.m_loc = (int)c->m_loc;
  g.n = (int)c->n;
  g.row0 = c->row0;
  g.nt = c->nt;
  g.ns = c->ns;
  g.cl = c->cl;
  g.colw = c->colw;
  g.nstage = c->nstage[kind];
  g.nacc = nacc_of(c, kind);
  return g;
}

// ---------------------------------------------------------- profiling
int prof_begin(otb_ctx* c, cudaEvent_t* e0) {
  if (!c->prof) return OTB_OK;
  if (c->pool.empty()) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreate(&e));
    c->pool.push_back(e);
  }
  *e0 = c->pool.back();
  c->pool.pop_back();
  CUDA_TRY(cudaEventRecord(*e0, c->stream));
  return OTB_OK;
}

int prof_end(otb_ctx* c, int cls, cudaEvent_t e0, double bytes) {
  if (!c->prof) return OTB_OK;
  if (c->pool.empty()) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreate(&e));
    c->pool.push_back(e);
  }
  cudaEvent_t e1 = c->pool.back();
  c->pool.pop_back();
  CUDA_TRY(cudaEventRecord(e1, c->stream));
  c->recs.push_back({cls, e0, e1, bytes});
  return OTB_OK;
}

int prof_collect(otb_ctx* c) {
  if (c->recs.empty()) return OTB_OK;
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  for (auto& r : c->recs) {
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, r.e0, r.e1));
    c->prof_ms[r.cls] += ms;
    c->prof_bytes[r.cls] += r.bytes;
    c->prof_cnt[r.cls] += 1;
    c->pool.push_back(r.e0);
    c->pool.push_back(r.e1);
  }
  c->recs.clear();
  return OTB_OK;
}

// ------------------------------------------------------------- helpers
int launch_dense(otb_ctx* c, int kind, Geom geo, void* io) {
  const void* fn = kDenseFn[kind][geo.ns];
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)c->grid);
  cfg.blockDim = dim3((unsigned)dense_block(kind, geo.nt));
  cfg.dynamicSmemBytes = c->smem[kind];
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)c->cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* args[2] = {&geo, io};
  CUDA_TRY(cudaLaunchKernelExC(&cfg, fn, args));
  ++c->launches;
  return OTB_OK;
}

// Local group all-reduce: publish, barrier, wait for every rank's event,
// fixed-order sum into lg_tmp, barrier (no rank overwrites its buffer while a
// peer still reads it), copy back.
int group_allreduce(otb_ctx* c, double* buf, size_t count, int op) {
  otb_group* G = c->group;
  const int r = c->rank, N = G->n;
  if (count > (size_t)(rup(c->n, 2) + 16)) return fail(OTB_ERR_ARG, "local group all-reduce larger than its buffer");
  G->bufs[r] = buf;
  G->counts[r] = (int64_t)count;
  G->ops[r] = op;
  CUDA_TRY(cudaEventRecord(G->ready[r], c->stream));
  TRY(G->barrier());
  LocalRed lr{};
  for (int q = 0; q < N; ++q) {
    if (G->counts[q] != (int64_t)count || G->ops[q] != op) {
      G->abort();
      return fail(OTB_ERR_NCCL, "local group: ranks issued different all-reduces");
    }
    if (q != r) CUDA_TRY(cudaStreamWaitEvent(c->stream, G->ready[q], 0));
    lr.src[q] = G->bufs[q];
  }
  lr.nranks = N;
  lr.op = op;
  lr.count = (int64_t)count;
  lr.out = c->lg_tmp;
  k_local_reduce<<<(int)std::min<int64_t>(cdiv((int64_t)count, 256), 2 * c->num_sms), 256, 0, c->stream>>>(lr);
  LAUNCH_CHECK();
  CUDA_TRY(cudaEventRecord(G->done[r], c->stream));
  TRY(G->barrier());
  for (int q = 0; q < N; ++q)
    if (q != r) CUDA_TRY(cudaStreamWaitEvent(c->stream, G->done[q], 0));
  CUDA_TRY(cudaMemcpyAsync(buf, c->lg_tmp, count * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  return OTB_OK;
}

int allreduce(otb_ctx* c, double* buf, size_t count, int op) {
  if (c->nranks <= 1) return OTB_OK;
  if (c->group) return group_allreduce(c, buf, count, op);
  const int r = c->nccl.allReduce(buf, buf, count, kNcclFloat64, op, c->comm, c->stream);
  if (r != 0)
    return fail(OTB_ERR_NCCL, std::string("ncclAllReduce: ") + (c->nccl.getErrorString ? c->nccl.getErrorString(r) : "?"));
  return OTB_OK;
}

int sync_scalars(otb_ctx* c) {
  CUDA_TRY(cudaMemcpyAsync(c->hs, c->ds, sizeof(DevScalars), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return OTB_OK;
}

int colreduce(otb_ctx* c, int nparts, const double* spart, int nspart, int sstride, int nscal,
              ColPost cp = ColPost{-1, nullptr, nullptr, {nullptr, nullptr}}) {
  k_colreduce<<<c->col32, 256, 0, c->stream>>>(c->colpart, nparts, (int)c->n, c->sendbuf, spart, nspart, sstride,
                                                 nscal, &c->ds->cnt[CNT_COLRED], cp);
  LAUNCH_CHECK();
  return OTB_OK;
}

int require_bound(const otb_ctx* c) {
  if (!c) return fail(OTB_ERR_ARG, "null context");
  if (!c->bound) return fail(OTB_ERR_ARG, "no problem bound (otb_bind)");
  return OTB_OK;
}

// ------------------------------------------------------------- eval
// Launch part of an eval (no host synchronisation).
int eval_launch(otb_ctx* c, const double* X, const double* gamma, bool save_ev0 = false) {
  const int n = (int)c->n;
  // gamma is streamed by TMA with the rows, a whole slice at a time: it is
  // copied into gev, whose padding past n holds -inf (set at creation)
  if (gamma != c->gev) {
    CUDA_TRY(cudaMemcpyAsync(c->gev, gamma, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
    gamma = c->gev;
  }
  Geom geo = make_geom(c, DK_EVAL, c->C, X);
  geo.vec[0] = gamma;
  EvalIO io{gamma, c->a, c->eta, c->rowM, c->rowS, c->lse, c->colpart, c->vpart, c->Pbuf};
  c->p_valid = false;
  cudaEvent_t e0 = nullptr;
  TRY(prof_begin(c, &e0));
  TRY(launch_dense(c, DK_EVAL, geo, &io));
  TRY(prof_end(c, PC_EVAL, e0, 16.0 * c->m_loc * n + 8.0 * c->m_loc + 24.0 * n));
  if (c->nranks == 1 && (int64_t)c->colgrid * 256 >= n && c->colgrid <= 512 && !c->force_post) {
    k_colreduce_eval<<<c->col32, 256, 0, c->stream>>>(c->colpart, c->ncl, n, c->vpart, c->ncl, c->b, gamma, c->eta,
                                                      c->g, c->ds, c->bpart, c->colgrid, save_ev0);
    LAUNCH_CHECK();
    return OTB_OK;
  }
  TRY(colreduce(c, c->ncl, c->vpart, c->ncl, 2, 2));
  TRY(allreduce(c, c->sendbuf, (size_t)n + 2, kNcclSum));
  k_eval_post<<<c->colgrid, 256, 0, c->stream>>>(n, c->sendbuf, c->b, gamma, c->eta, c->g, c->ds, c->bpart);
  LAUNCH_CHECK();
  if (save_ev0) {
    CUDA_TRY(cudaMemcpyAsync(&c->ds->ev0[0], &c->ds->value, 2 * sizeof(double), cudaMemcpyDeviceToDevice,
                             c->stream));
    CUDA_TRY(cudaMemcpyAsync(&c->ds->ev0[2], &c->ds->scratch[0], sizeof(double), cudaMemcpyDeviceToDevice,
                             c->stream));
  }
  return OTB_OK;
}

// Host side of an eval whose scalars are in c->hs (after sync_scalars).
int eval_finish(otb_ctx* c) {
  if (c->hs->scratch[0] != 0.0) {
    c->have_eval = false;
    return fail(OTB_ERR_NONFINITE, "row softmax produced non-finite values after stabilization");
  }
  c->last_value = c->hs->value;
  c->last_gnorm = c->hs->gnorm;
  c->have_eval = true;
  c->p_valid = c->Pbuf != nullptr;
  return OTB_OK;
}

int do_eval(otb_ctx* c, const double* X, const double* gamma) {
  TRY(eval_launch(c, X, gamma));
  TRY(sync_scalars(c));
  return eval_finish(c);
}

// --------------------------------------------------------- sparsify
Csr csr_view(const otb_ctx* c);

int grow_csr(otb_ctx* c, int64_t want) {
  if (want <= c->cap) return OTB_OK;
  int64_t ncap = std::max<int64_t>(want, (int64_t)(c->cap * 1.5));
  ncap = std::min<int64_t>(ncap, c->m_loc * rup(c->n, kCsrAlign) + (int64_t)c->ncl * c->chunk + c->n);
  if (c->cols) cudaFree(c->cols);
  if (c->vals) cudaFree(c->vals);
  c->cols = nullptr;
  c->vals = nullptr;
  c->cap = 0;
  TRY(dalloc(&c->cols, (size_t)ncap));
  TRY(dalloc(&c->vals, (size_t)ncap + 16));   // slack: hess_apply reads up to 2 entries past a run
  c->cap = ncap;
  return OTB_OK;
}

int row_prefix(otb_ctx* c) {
  k_row_prefix<<<1, 1024, 0, c->stream>>>(c->row_len, (int)c->m_loc, c->rowpre);
  LAUNCH_CHECK();
  return OTB_OK;
}

// Launch part of a sparsify pass (no host synchronisation): kernel, CTA
// bounds / row prefix where hess_apply needs them, Hessian diagonal.  The
// kept count and the capacity flag land in c->ds; *rec is the profiling
// record whose byte count needs nnz (or -1).
int sparsify_launch(otb_ctx* c, const double* X, const double* gamma, double rho, int64_t* rec,
                    const double* gnorm_dev = nullptr) {
  const int n = (int)c->n;
  const int64_t anchor_local = (c->anchor >= c->row0 && c->anchor < c->row1) ? c->anchor - c->row0 : -1;
  // alloc, nnzc, flags are adjacent in DevScalars
  CUDA_TRY(cudaMemsetAsync(&c->ds->alloc, 0, 2 * sizeof(unsigned long long) + sizeof(int), c->stream));
  const int kind = c->p_valid ? DK_SPARSP : DK_SPARSIFY;
  const bool bitmap = c->hv_mode == 2 || c->hv_mode == 3;   // hess_apply reads the bitmap, not the columns
  // window-cluster hess_apply: dense P_rho (written over the stored P) when
  // most pairs are kept — a fixed position per value instead of bitmap
  // offsets; the products are bitwise the same (dropped entries are 0.0 and
  // every thread sums the same columns in the same order)
  const char* env_hd = std::getenv("OTB_HV_DENSE");   // read per call: an experiment / test knob
  c->dense_policy = env_hd ? (std::atoi(env_hd) > 0 ? 1 : 0) : -1;
  double density = c->last_density;
  const bool dense_cap = c->hv_mode == 3 || c->ov_ok;
  const double dense_min = c->hv_mode == 3 ? kDenseRhoMin : c->ov_min_density;
  if (dense_cap && dense_min > 0.0 && c->Pbuf != nullptr && c->p_valid && c->dense_policy < 0 && !c->have_density) {
    // no kept density yet on this context: estimate it from every 64th row
    // of the stored P (one host synchronisation, first sparsify only)
    const int stride = 64;
    const int64_t rows = (c->m_loc + stride - 1) / stride;
    CUDA_TRY(cudaMemsetAsync(&c->ds->scratch[3], 0, sizeof(double), c->stream));
    k_density_sample<<<c->num_sms * 4, 256, 0, c->stream>>>(c->Pbuf, c->ld, (int)c->m_loc, n, stride, gnorm_dev,
                                                            c->eta, (double)c->m_glob * (double)c->n, rho,
                                                            reinterpret_cast<unsigned long long*>(&c->ds->scratch[3]));
    LAUNCH_CHECK();
    TRY(sync_scalars(c));
    unsigned long long cnt = 0;
    std::memcpy(&cnt, &c->hs->scratch[3], sizeof cnt);
    density = (double)cnt / std::max(1.0, (double)rows * (double)n);
  }
  // (a group-kernel context can write the dense P_rho only from the stored P: its recomputing
  // sparsify writes the CSR columns)
  const bool dense = dense_cap && c->Pbuf != nullptr && (c->hv_mode == 3 || c->p_valid) &&
                     (c->dense_policy == 1 || (c->dense_policy < 0 && density >= dense_min));
  // dense P_rho from the stored P: the lean kernel (same bits as k_sparsify's dense mode)
  const int launch_kind = (dense && c->p_valid) ? (int)DK_SPDENSE : kind;
  Geom geo = c->p_valid ? make_geom(c, launch_kind, c->Pbuf, nullptr) : make_geom(c, DK_SPARSIFY, c->C, X);
  SparsifyIO io{gamma, c->a, c->eta, rho, anchor_local, c->rowM, c->rowS, c->lse, bitmap ? nullptr : c->cols,
                c->vals, c->cap,
                c->row_start, c->row_len, &c->ds->alloc, &c->ds->nnzc, c->chunk, c->colpart, &c->ds->flags,
                bitmap ? c->bm : nullptr, c->nq, gnorm_dev, (double)c->m_glob * (double)c->n,
                c->precond ? c->colpart2 : nullptr, dense ? c->Pbuf : nullptr};
  c->rho_dense = dense;
  cudaEvent_t e0 = nullptr;
  TRY(prof_begin(c, &e0));
  TRY(launch_dense(c, launch_kind, geo, &io));
  if (dense) c->p_valid = false;   // Pbuf now holds P_rho
  *rec = c->prof ? (int64_t)c->recs.size() : -1;
  TRY(prof_end(c, PC_SPARSIFY, e0, 0.0));
  // the row prefix (CSR export, nnz-balanced bounds) only where it is used
  if (!bitmap && !dense) {
    TRY(row_prefix(c));
    // nnz-balanced row bounds of the hess_apply CTAs, once per sparsify
    // (the bitmap kernels use fixed equal row counts, set at creation)
    Csr A = csr_view(c);
    A.cta_rb = nullptr;
    k_cta_bounds<<<(int)cdiv(c->hv_nb + 1, 256), 256, 0, c->stream>>>(A, c->hv_nb, c->cta_rb, 0);
    LAUNCH_CHECK();
  }
  c->rowpre_valid = !bitmap && !dense;
  if (c->precond) {   // q = (P_rho o P_rho)^T a for the Jacobi diagonal, summed over ranks
    k_colreduce<<<c->col32, 256, 0, c->stream>>>(c->colpart2, c->ncl, n, c->jq, nullptr, 0, 0, 0,
                                                   &c->ds->cnt[CNT_COLRED], ColPost{-1, nullptr, nullptr, {nullptr, nullptr}});
    LAUNCH_CHECK();
    TRY(allreduce(c, c->jq, (size_t)n, kNcclSum));
  }
  if (c->nranks == 1) {   // d = column sums, written by the reduction itself
    TRY(colreduce(c, c->ncl, nullptr, 0, 0, 0, ColPost{POST_COPY, c->b, c->d, {nullptr, nullptr}}));
    return OTB_OK;
  }
  TRY(colreduce(c, c->ncl, nullptr, 0, 0, 0));
  // [overflow flag, kept entries] ride along with d: a redo after a CSR
  // overflow on ANY rank is then taken by every rank (matched collectives)
  k_sparsify_scalars<<<1, 32, 0, c->stream>>>(c->ds, c->sendbuf + n);
  LAUNCH_CHECK();
  TRY(allreduce(c, c->sendbuf, (size_t)n + 2, kNcclSum));
  k_vec_post<<<c->colgrid, 256, 0, c->stream>>>(POST_COPY, n, c->sendbuf, c->b, c->d, c->ds, c->bpart, nullptr);
  LAUNCH_CHECK();
  CUDA_TRY(cudaMemcpyAsync(c->ds->sp_glob, c->sendbuf + n, 2 * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  return OTB_OK;
}

// Host side of a sparsify pass whose scalars are in c->hs.  Returns 1 when
// the CSR overflowed its capacity (grown here; the pass must be redone).
int sparsify_finish(otb_ctx* c, int64_t rec, bool* redo) {
  const int64_t nnz = (int64_t)c->hs->nnzc;
  if (rec >= 0 && rec < (int64_t)c->recs.size())
    c->recs[(size_t)rec].bytes = 16.0 * c->m_loc * c->n + 12.0 * nnz + 8.0 * (c->m_loc + 1);
  const bool mine = (c->hs->flags & 2) != 0;
  *redo = c->nranks > 1 ? c->hs->sp_glob[0] != 0.0 : mine;
  if (*redo) {
    if (!mine) return OTB_OK;   // another rank overflowed: same redo, nothing to grow here
    const int64_t need = (int64_t)c->hs->alloc + (int64_t)c->ncl * c->chunk;
    return grow_csr(c, need + need / 8);
  }
  c->nnz = nnz;
  c->nnz_glob = c->nranks > 1 ? (int64_t)c->hs->sp_glob[1] : nnz;
  c->last_density = (double)nnz / std::max(1.0, (double)c->m_loc * (double)c->n);
  c->have_density = true;
  return OTB_OK;
}

int do_sparsify(otb_ctx* c, const double* X, const double* gamma, double rho) {
  for (int attempt = 0; attempt < 8; ++attempt) {
    int64_t rec = -1;
    TRY(sparsify_launch(c, X, gamma, rho, &rec));
    TRY(sync_scalars(c));
    bool redo = false;
    TRY(sparsify_finish(c, rec, &redo));
    if (!redo) return OTB_OK;
  }
  return fail(OTB_ERR_NOMEM, "CSR capacity could not be grown");
}

Csr csr_view(const otb_ctx* c) {
  Csr A;
  A.row_start = c->row_start;
  A.row_len = c->row_len;
  A.rowpre = c->rowpre;
  A.cta_rb = c->cta_rb;
  A.cols = c->cols;
  A.vals = c->vals;
  A.m_loc = (int)c->m_loc;
  A.row0 = c->row0;
  return A;
}

// Algorithmic bytes of one hess_apply, SURVEY §8(d) / DESIGN.md: CSR with
// int32 columns, 12 nnz + 8 (m + 1) + 16 n, whatever the stored format
// (the bitmap index moves 8 nnz + m nq 16 bytes; ncu traffic shows it).
// With the dense P_rho the product streams every matrix entry once and no column indices:
// 8 m n + 8 (m + 1) + 16 n (fewer than the CSR figure from 2/3 kept on, more below it).
double hv_bytes(const otb_ctx* c) {
  if (c->rho_dense) return 8.0 * (double)c->m_loc * (double)c->n + 8.0 * (c->m_loc + 1) + 16.0 * c->n;
  return 12.0 * c->nnz + 8.0 * (c->m_loc + 1) + 16.0 * c->n;
}

// y = P_rho^T (a * (P_rho v)) reduced to: (mode smem) colpart[hv_grid][n] or
// sendbuf (multi-rank), (mode atomic) cg_y or sendbuf.  Returns via
// ysum/colpart/yatomic the arguments for the column kernels.
struct HvResult {
  const double* colpart;
  int nparts;
  double* yatomic;
  const double* ysum;
};

int run_hv(otb_ctx* c, const double* v_src, const double* r, const double* p_prev, double* p_cur, int update,
           const CgState* st, HvResult* res) {
  const int n = (int)c->n;
  cudaEvent_t e0 = nullptr;
  int hv_parts = c->hv_nb;
  if (c->hv_mode != 1) {
    HvArgs h{csr_view(c), c->a, n, c->hv_ng, v_src, r, p_prev, p_cur, update, st, c->colpart, c->bm, c->nq,
             c->hv_win, c->ld};
    if (c->rho_dense) h.A.vals = c->Pbuf;
    const bool ov = c->hv_mode != 3 && c->rho_dense;                  // dense overlay of a group-kernel context
    const bool wcd = ov || (c->hv_mode == 3 && c->rho_dense && c->hv_wcd);   // dense P_rho: k_hv_wcd (no producer warp)
    if (wcd) h.ng = ov ? c->ov_stages : c->hv_ng_d;
    if (ov) {
      h.A.cta_rb = c->ov_rb;
      h.nwin = c->ov_win;
    }
    hv_parts = ov ? c->ov_ncl : c->hv_nb;
    TRY(prof_begin(c, &e0));
    void* args[1] = {&h};
    if (c->hv_mode == 3 || ov) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(ov ? c->ov_ncl * c->ov_win : c->hv_grid);
      cfg.blockDim = dim3(wcd ? kStConsumers : kStThreads);
      cfg.dynamicSmemBytes = ov ? c->ov_smem : (wcd ? c->hv_smem_d : c->hv_smem);
      cfg.stream = c->stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = (unsigned)(ov ? c->ov_win : c->hv_win);
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      const void* fn = ov ? kWcdFn[c->ov_nq] : (wcd ? kWcdFn[c->hv_var] : kWcFn[c->rho_dense ? 1 : 0][c->hv_var]);
      CUDA_TRY(cudaLaunchKernelExC(&cfg, fn, args));
    } else {
      CUDA_TRY(cudaLaunchKernel(kHvFn[c->hv_var], dim3(c->hv_grid), dim3(c->hv_threads), args, c->hv_smem,
                                c->stream));
    }
    LAUNCH_CHECK();
    TRY(prof_end(c, PC_HV, e0, hv_bytes(c)));
    if (c->nranks > 1) {
      TRY(colreduce(c, hv_parts, nullptr, 0, 0, 0));
      TRY(allreduce(c, c->sendbuf, (size_t)n, kNcclSum));
      *res = {nullptr, 0, nullptr, c->sendbuf};
    } else {
      *res = {c->colpart, hv_parts, nullptr, nullptr};
    }
  } else {
    const double* v = update ? p_cur : v_src;
    if (update) {
      k_cg_p<<<c->colgrid, 256, 0, c->stream>>>(n, r, p_prev, p_cur, st);
      LAUNCH_CHECK();
    }
    HvAtomicArgs h{csr_view(c), c->a, v, c->cg_y, st};
    TRY(prof_begin(c, &e0));
    k_hv_atomic<<<c->hv_grid, 256, 0, c->stream>>>(h);
    LAUNCH_CHECK();
    TRY(prof_end(c, PC_HV, e0, hv_bytes(c)));
    if (c->nranks > 1) {
      CUDA_TRY(cudaMemcpyAsync(c->sendbuf, c->cg_y, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
      CUDA_TRY(cudaMemsetAsync(c->cg_y, 0, sizeof(double) * n, c->stream));
      TRY(allreduce(c, c->sendbuf, (size_t)n, kNcclSum));
      *res = {nullptr, 0, nullptr, c->sendbuf};
    } else {
      *res = {nullptr, 0, c->cg_y, nullptr};
    }
  }
  return OTB_OK;
}

// ------------------------------------------------------------------ CG
int cg_iteration(otb_ctx* c, int64_t k, double* x) {
  const int n = (int)c->n;
  double* pc = c->cg_p[k & 1];
  double* pp = c->cg_p[(k + 1) & 1];
  HvResult hr;
  // p = r + beta p (plain CG) or z + beta p (PCG) inside the hess_apply launch
  TRY(run_hv(c, pc, c->precond ? c->zv : c->cg_r, pp, pc, k > 0 ? 1 : 0, c->cg, &hr));
  cudaEvent_t e0 = nullptr;
  TRY(prof_begin(c, &e0));
  CgApArgs a{n, hr.colpart, hr.nparts, hr.yatomic, hr.ysum, c->d, pc, c->eta, c->cg_ap, c->cg, c->bpart};
  k_cg_ap<<<c->col32, 256, 0, c->stream>>>(a);
  LAUNCH_CHECK();
  k_cg_update<<<c->colgrid, 256, 0, c->stream>>>(n, x, c->cg_r, pc, c->cg_ap, c->cg, c->bpart,
                                                  c->precond ? c->minv : nullptr, c->precond ? c->zv : nullptr);
  LAUNCH_CHECK();
  TRY(prof_end(c, PC_CGVEC, e0, 8.0 * 9 * n));
  return OTB_OK;
}

// Everything a captured CG batch bakes in: the argument blocks of its
// kernels (pointers, eta, kernel variant) and the solution vector.
void cg_graph_key(const otb_ctx* c, const double* x, unsigned char* key) {
  std::memset(key, 0, 160);
  const void* ptrs[14] = {x,      c->vals,  c->cols,   c->Pbuf,  c->a,  c->d,     c->bm,
                          c->row_start, c->row_len, c->cta_rb, c->minv, c->zv, c->colpart, c->sendbuf};
  std::memcpy(key, ptrs, sizeof ptrs);
  const int ints[6] = {c->rho_dense ? 1 : 0, c->precond, c->hv_mode, c->hv_var, c->nranks, c->hv_ng};
  std::memcpy(key + sizeof ptrs, ints, sizeof ints);
  std::memcpy(key + sizeof ptrs + sizeof ints, &c->eta, sizeof(double));
}

// kCgBatch iterations from iteration k0: replayed from a CUDA graph (one
// launch, the NCCL all-reduces inside it on the multi-rank path) unless
// profiling, a local group (its all-reduce synchronises host threads) or
// OTB_CG_GRAPH=0; the graph is captured on first use and again whenever an
// argument it bakes in changes (CSR regrown, dense/bitmap mode, eta).
int cg_batch(otb_ctx* c, int64_t k0, double* x) {
  if (c->prof || c->group || !c->cg_graph) {
    for (int j = 0; j < kCgBatch; ++j) TRY(cg_iteration(c, k0 + j, x));
    return OTB_OK;
  }
  const int which = k0 == 0 ? 0 : 1;   // batches start at even k: the same p-buffer parity
  unsigned char key[160];
  cg_graph_key(c, x, key);
  if (!c->cg_exec[which] || std::memcmp(key, c->cg_key[which], sizeof key) != 0) {
    if (c->cg_exec[which]) {
      cudaGraphExecDestroy(c->cg_exec[which]);
      c->cg_exec[which] = nullptr;
    }
    if (!c->cap_stream) CUDA_TRY(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
    cudaStream_t saved = c->stream;
    const int64_t l0 = c->launches;
    c->stream = c->cap_stream;
    CUDA_TRY(cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal));
    int st = OTB_OK;
    for (int j = 0; j < kCgBatch && st == OTB_OK; ++j) st = cg_iteration(c, k0 + j, x);
    cudaGraph_t g = nullptr;
    const cudaError_t ee = cudaStreamEndCapture(c->cap_stream, &g);
    c->stream = saved;
    const int64_t captured = c->launches - l0;
    c->launches = l0;   // captured, not launched
    if (st != OTB_OK) {
      if (g) cudaGraphDestroy(g);
      return st;
    }
    if (ee != cudaSuccess) return fail(OTB_ERR_CUDA, std::string("CG graph capture: ") + cudaGetErrorString(ee));
    const cudaError_t ei = cudaGraphInstantiate(&c->cg_exec[which], g, 0);
    cudaGraphDestroy(g);
    if (ei != cudaSuccess) {
      c->cg_exec[which] = nullptr;
      return fail(OTB_ERR_CUDA, std::string("CG graph instantiate: ") + cudaGetErrorString(ei));
    }
    std::memcpy(c->cg_key[which], key, sizeof key);
    c->cg_batch_launches[which] = captured;
  }
  CUDA_TRY(cudaGraphLaunch(c->cg_exec[which], c->stream));
  c->launches += c->cg_batch_launches[which];
  return OTB_OK;
}

// The whole CG loop as one cooperative launch (k_cg_fused), after
// k_cg_init; the state is copied to c->hcg asynchronously (read it after the
// next stream synchronisation).  k_cg_fused returns at once when k_cg_init
// already decided (rhs = 0, inconsistent system) or the CSR overflowed.
int cg_fused_launch(otb_ctx* c, double shift, const double* rhs, double rel_tol, int64_t max_iters, double* x,
                    int64_t* rec, const double* neg_of = nullptr, const double* shift_dev = nullptr) {
  const int n = (int)c->n;
  // the persistent CG reduces H v over its own rows only: single rank
  if (c->nranks != 1) return fail(OTB_ERR_ARG, "internal: persistent CG launched with more than one rank");
  // with neg_of the right-hand side -neg_of is formed here into c->rhs (rhs must be c->rhs)
  k_cg_init<<<c->colgrid, 256, 0, c->stream>>>(n, rhs, x, c->cg_r, c->cg_p[0], c->cg, c->bpart, shift, rel_tol,
                                               (long long)max_iters, neg_of, neg_of ? c->rhs : nullptr, shift_dev);
  LAUNCH_CHECK();
  CgFusedArgs fa{csr_view(c), c->a,     c->d,  n,     c->fused_ng, c->eta, x,          rhs, c->cg_ap,
                 c->colpart,  c->scal, c->cg, c->bm, c->nq,       c->cg_trace, &c->ds->flags};
  void* args[1] = {&fa};
  cudaEvent_t e0 = nullptr;
  TRY(prof_begin(c, &e0));
  CUDA_TRY(cudaLaunchCooperativeKernel(kCgFn[c->hv_var], dim3(c->hv_grid), dim3(c->hv_threads), args,
                                       c->fused_smem, c->stream));
  ++c->launches;
  *rec = c->prof ? (int64_t)c->recs.size() : -1;
  TRY(prof_end(c, PC_CGFUSED, e0, 0.0));
  CUDA_TRY(cudaMemcpyAsync(c->hcg, c->cg, sizeof(CgState), cudaMemcpyDeviceToHost, c->stream));
  return OTB_OK;
}

// Host side of a finished CG (c->hcg current).
int cg_finish(otb_ctx* c, int64_t rec, otb_cg_out* out) {
  if (rec >= 0 && rec < (int64_t)c->recs.size()) c->recs[(size_t)rec].bytes = (double)c->hcg->iters * hv_bytes(c);
  if (c->hcg->status == CG_INCONSISTENT)
    return fail(OTB_ERR_INCONSISTENT, "unshifted system with right-hand side outside the range");
  if (c->hcg->status == CG_NOTPD) {
    char buf[96];
    std::snprintf(buf, sizeof buf, "p^T A p = %.3g before convergence", c->hcg->curv);
    return fail(OTB_ERR_NOT_PD, buf);
  }
  if (out) {
    out->iters = c->hcg->iters;
    out->residual = c->hcg->res;
    out->status = c->hcg->status;
  }
  return OTB_OK;
}

int do_cg(otb_ctx* c, double shift, const double* rhs, double rel_tol, int64_t max_iters, double* x, otb_cg_out* out) {
  const int n = (int)c->n;
  if (c->cg_fused && !c->precond) {
    int64_t rec = -1;
    TRY(cg_fused_launch(c, shift, rhs, rel_tol, max_iters, x, &rec));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return cg_finish(c, rec, out);
  }
  const PcgInit pc = c->precond ? PcgInit{c->d, c->jq, c->eta, c->minv, c->zv}
                                : PcgInit{nullptr, nullptr, 1.0, nullptr, nullptr};
  k_cg_init<<<c->colgrid, 256, 0, c->stream>>>(n, rhs, x, c->cg_r, c->cg_p[0], c->cg, c->bpart, shift, rel_tol,
                                               (long long)max_iters, nullptr, nullptr, nullptr, pc);
  LAUNCH_CHECK();
  CUDA_TRY(cudaMemcpyAsync(c->hcg, c->cg, sizeof(CgState), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (c->hcg->status == CG_INCONSISTENT) return cg_finish(c, -1, out);
  int64_t k = 0;
  const size_t rec0 = c->recs.size();
  while (c->hcg->status == CG_RUN) {
    TRY(cg_batch(c, k, x));
    k += kCgBatch;
    CUDA_TRY(cudaMemcpyAsync(c->hcg, c->cg, sizeof(CgState), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
  }
  // profiling: the launches of a batch past convergence return at once;
  // only the iterations that ran count (time and bytes)
  if (c->prof) {
    int64_t hv_seen = 0, vec_seen = 0;
    for (size_t q = rec0; q < c->recs.size(); ++q) {
      auto& r = c->recs[q];
      if (r.cls == PC_HV && ++hv_seen > c->hcg->iters) r.cls = PC_SKIP;
      if (r.cls == PC_CGVEC && ++vec_seen > c->hcg->iters) r.cls = PC_SKIP;
    }
  }
  return cg_finish(c, -1, out);
}

// ------------------------------------------------------ inexact test
int do_round(otb_ctx* c, const double* X, const double* gamma, double* Xout, int recover, int metrics,
             otb_test_out* out) {
  const int n = (int)c->n;
  const double mn = (double)c->m_loc * n;
  // pass A: candidate + row scaling + column sums
  {
    Geom geo = make_geom(c, DK_TESTA, c->C, X);
    if (gamma != nullptr && gamma != c->gev)   // streamed with the rows: the padded copy (-1e300 past n)
      CUDA_TRY(cudaMemcpyAsync(c->gev, gamma, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
    geo.vec[0] = c->gev;
    TestAIO io{gamma,  c->a,     c->log_a, c->lse, c->eta, Xout, c->zrow, c->colpart, c->vpart, recover,
               (metrics && c->ns > OTB_ZETA_A_NS) ? c->czeta : nullptr};   // k_test_c: wide rows take zeta from pass A
    cudaEvent_t e0 = nullptr;
    TRY(prof_begin(c, &e0));
    TRY(launch_dense(c, DK_TESTA, geo, &io));
    TRY(prof_end(c, PC_TESTA, e0, recover ? 24.0 * mn : 16.0 * mn));
    if (c->nranks == 1) {   // y and the two scalars straight from the reduction
      TRY(colreduce(c, c->ncl, c->vpart, c->grid, 2, 2,
                    ColPost{POST_Y, c->b, c->yv, {&c->ds->sumx, &c->ds->scratch[1]}}));
    } else {
      TRY(colreduce(c, c->ncl, c->vpart, c->grid, 2, 2));
      TRY(allreduce(c, c->sendbuf, (size_t)n + 2, kNcclSum));
      k_vec_post<<<c->colgrid, 256, 0, c->stream>>>(POST_Y, n, c->sendbuf, c->b, c->yv, c->ds, c->bpart, nullptr);
      LAUNCH_CHECK();
      CUDA_TRY(cudaMemcpyAsync(&c->ds->sumx, c->sendbuf + n, sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
      CUDA_TRY(cudaMemcpyAsync(&c->ds->scratch[1], c->sendbuf + n + 1, sizeof(double), cudaMemcpyDeviceToDevice,
                               c->stream));
    }
  }
  const double* src = recover ? Xout : X;
  // pass B: F = (X z) y, e_r, e_c, deficit
  {
    Geom geo = make_geom(c, DK_TESTB, src, nullptr);
    geo.vec[0] = c->yv;   // zero padding past n
    TestBIO io{c->zrow, c->yv, c->rowpart, c->colpart};
    cudaEvent_t e0 = nullptr;
    TRY(prof_begin(c, &e0));
    TRY(launch_dense(c, DK_TESTB, geo, &io));
    TRY(prof_end(c, PC_TESTB, e0, 8.0 * mn));
    if (c->nranks == 1 && c->colgrid <= 512) {   // rows, e_c and the deficit in one kernel
      TestFinishIO fi{0,       c->colpart, c->ncl,          (int)n,     c->b,      c->ec,     c->rowpart,
                      (int)c->m_loc, c->cl, c->a,           c->row0,    c->er,     nullptr,   0,
                      c->col32, c->colgrid, c->ds,          c->bpart};
      k_test_finish<<<c->col32 + c->colgrid, 256, 0, c->stream>>>(fi);
      LAUNCH_CHECK();
    } else {
      k_rows_post<<<c->colgrid, 256, 0, c->stream>>>(0, (int)c->m_loc, c->cl, c->rowpart, c->a, c->row0, c->er,
                                                     c->ds, c->bpart, &c->ds->scratch[2]);
      LAUNCH_CHECK();
      TRY(colreduce(c, c->ncl, &c->ds->scratch[2], 1, 1, 1));
      TRY(allreduce(c, c->sendbuf, (size_t)n + 1, kNcclSum));
      k_vec_post<<<c->colgrid, 256, 0, c->stream>>>(POST_EC, n, c->sendbuf, c->b, c->ec, c->ds, c->bpart, nullptr);
      LAUNCH_CHECK();
      CUDA_TRY(cudaMemcpyAsync(&c->ds->deficit, c->sendbuf + n, sizeof(double), cudaMemcpyDeviceToDevice,
                               c->stream));
    }
  }
  // pass C: rank-one correction, Bregman divergence, objective, KKT sums
  {
    const int kind = metrics ? DK_TESTC1 : DK_TESTC0;
    Geom geo = make_geom(c, kind, src, metrics ? c->C : nullptr);
    geo.vec[0] = c->yv;   // zero padding past n
    geo.vec[1] = c->ec;   // zero padding past n
    if (metrics) {        // -1e300 padding past n
      if (gamma != nullptr && gamma != c->gev)
        CUDA_TRY(cudaMemcpyAsync(c->gev, gamma, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
      geo.vec[2] = c->gev;
    }
    TestCIO io{c->zrow, c->yv, c->er, c->ec, &c->ds->deficit, gamma, c->rowpart, c->colpart, c->vpart, c->czeta};
    cudaEvent_t e0 = nullptr;
    TRY(prof_begin(c, &e0));
    TRY(launch_dense(c, kind, geo, &io));
    TRY(prof_end(c, PC_TESTC, e0, metrics ? 16.0 * mn : 8.0 * mn));
    if (c->nranks == 1 && c->colgrid <= 512) {   // rows, columns and the 8 scalars in one kernel
      TestFinishIO fi{1,       c->colpart, c->ncl,          (int)n,     c->b,      nullptr,   c->rowpart,
                      (int)c->m_loc, c->cl, c->a,           c->row0,    nullptr,   c->vpart,  c->grid,
                      c->col32, c->colgrid, c->ds,          c->bpart};
      k_test_finish<<<c->col32 + c->colgrid, 256, 0, c->stream>>>(fi);
      LAUNCH_CHECK();
    } else {
      k_rows_post<<<c->colgrid, 256, 0, c->stream>>>(1, (int)c->m_loc, c->cl, c->rowpart, c->a, c->row0, nullptr,
                                                     c->ds, c->bpart, c->vpart + 7);
      LAUNCH_CHECK();
      TRY(colreduce(c, c->ncl, c->vpart, c->grid, 8, 8));
      TRY(allreduce(c, c->sendbuf, (size_t)n + 8, kNcclSum));
      k_vec_post<<<c->colgrid, 256, 0, c->stream>>>(POST_COLRES, n, c->sendbuf, c->b, nullptr, c->ds, c->bpart,
                                                    &c->ds->col_sq);
      LAUNCH_CHECK();
      CUDA_TRY(cudaMemcpyAsync(c->ds->s8, c->sendbuf + n, 8 * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    }
  }
  TRY(sync_scalars(c));
  c->round_src = src;
  const DevScalars& h = *c->hs;
  if (h.scratch[1] != 0.0) return fail(OTB_ERR_BAD_LOGPLAN, "log plan contains NaN or +inf entries");
  if (out) {
    out->sum_x = h.sumx;
    out->deficit = h.deficit;
    out->bregman = h.s8[0] - h.s8[1] + h.sumx;   // feasibility.py:85
    out->objective = h.s8[2];
    const double cscale = 1.0 + (c->norm_c_dev ? std::sqrt(h.cnorm_sq) : c->norm_c);
    const double row_res = std::sqrt(h.s8[7]) / (1.0 + c->norm_a);
    const double col_res = std::sqrt(h.col_sq) / (1.0 + c->norm_b);
    const double neg = std::sqrt(h.s8[4]) / (1.0 + std::sqrt(h.s8[3]));
    out->delta_p = std::max(std::max(row_res, col_res), neg);
    out->delta_d = std::sqrt(h.s8[5]) / cscale;
    out->delta_c = std::fabs(h.s8[6]) / cscale;
    out->delta_kkt = std::max(std::max(out->delta_p, out->delta_d), out->delta_c);
    if (metrics && !std::isfinite(out->objective)) {
      char buf[64];
      std::snprintf(buf, sizeof buf, "non-finite objective %g", out->objective);
      return fail(OTB_ERR_OBJECTIVE, buf);
    }
  }
  return OTB_OK;
}

}  // namespace

// ------------------------------------------------------------ dense drop-ins
// (dense_api.cuh) Context-free, on `stream`; temporaries from the stream
// allocator; host results after one synchronisation.
namespace {
struct DapiScratch {
  cudaStream_t st;
  std::vector<void*> ptrs;
  ~DapiScratch() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
  int get(double** p, size_t count) {
    cudaError_t e = cudaMallocAsync((void**)p, std::max<size_t>(count, 1) * sizeof(double), st);
    if (e != cudaSuccess) return fail(OTB_ERR_NOMEM, std::string("cudaMallocAsync: ") + cudaGetErrorString(e));
    ptrs.push_back(*p);
    return OTB_OK;
  }
};
int dapi_rows_grid(int64_t m) { return (int)std::max<int64_t>(1, std::min<int64_t>(m, 148 * 8)); }
dim3 dapi_cols_grid(int64_t m, int64_t n) {
  return dim3((unsigned)cdiv(n, kDapiThreads), (unsigned)std::max<int64_t>(1, std::min<int64_t>(m, kDapiRB)));
}
}  // namespace

// ======================================================================
// C ABI
// ======================================================================
extern "C" {

int otb_abi_version(void) { return OTB_ABI_VERSION; }

const char* otb_last_error(void) { return g_err.c_str(); }

int otb_create(otb_ctx** out, int64_t m_global, int64_t n, int64_t row_begin, int64_t row_end, int64_t ld,
               int device, void* stream) {
  if (!out) return fail(OTB_ERR_ARG, "out is null");
  *out = nullptr;
  if (m_global <= 0 || n <= 0) return fail(OTB_ERR_ARG, "empty problem");
  // n <= 65536 where the CSR stores uint16 columns; the window-cluster formats (bitmap words, dense
  // P_rho) store none and go to 16 windows of 8192 columns (checked once the variant is known)
  if (n > (int64_t)kWcMaxW * 1024 * kMaxNQ)
    return fail(OTB_ERR_ARG, "n > 131072 is not supported (16 hess_apply windows of 8192 columns)");
  if (row_begin < 0 || row_end > m_global || row_end <= row_begin) return fail(OTB_ERR_ARG, "bad row range");
  if (ld < n || ld % 32 != 0) return fail(OTB_ERR_ARG, "ld must be >= n and a multiple of 32");
  CUDA_TRY(cudaSetDevice(device));
  otb_ctx* c = new otb_ctx();
  c->device = device;
  c->stream = (cudaStream_t)stream;
  c->m_glob = m_global;
  c->n = n;
  c->row0 = row_begin;
  c->row1 = row_end;
  c->m_loc = row_end - row_begin;
  c->ld = ld;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  c->num_sms = sms;
  // dense geometry: CTAs per SM, cluster size, column window, slices, threads
  // Cluster size: any cl <= 16 whose window fits one CTA (<= kMaxNS slices),
  // chosen for the least time per row block: rows per co-resident cluster x
  // (slices per CTA + the cost of the row exchanges, ~2 slices).  Clusters
  // must fit in a GPC, so the co-resident count is queried: e.g. n = 50000
  // gets cl = 5 (26 clusters, 130 SMs) instead of cl = 8 (15 clusters,
  // 120 SMs).  OTB_DENSE_CL forces the size.  OTB_DENSE_CTAS_PER_SM=2: two
  // CTAs of at most 256 threads per SM (512-column slices, half the shared
  // memory each), so that one CTA's row synchronisation overlaps the other's
  // arithmetic.
  const char* env_cps = std::getenv("OTB_DENSE_CTAS_PER_SM");
  const int per_sm = env_cps ? std::max(1, std::min(2, std::atoi(env_cps))) : 1;
  const int slice_cols = 1024 / per_sm;   // 2 x the most threads per CTA
  int cl = 1;
  {
    const char* env_cl = std::getenv("OTB_DENSE_CL");
    const int force_cl = env_cl ? std::atoi(env_cl) : 0;
    double best = 1e300;
    for (int q = 1; q <= kMaxCluster; ++q) {
      if (force_cl > 0 && q != force_cl) continue;
      const int64_t colw_q = rup(cdiv(n, q), q > 1 ? 64 : 2);
      if (cdiv(colw_q, slice_cols) > kMaxNS) continue;
      const int ns_q = (int)std::max<int64_t>(1, cdiv(colw_q, slice_cols));
      const int nt_q = (int)std::max<int64_t>(32, rup(cdiv(colw_q, 2 * ns_q), 32));
      int fit = sms * per_sm / q;
      if (q > 1) {
        c->nt = nt_q;
        c->ns = ns_q;
        int st = 8;
        while (st > 2 && dense_smem(c, DK_EVAL, st) > kMaxDynSmem / per_sm - kStaticSmem[DK_EVAL] - 1024) --st;
        const void* fn = kDenseFn[DK_EVAL][ns_q];
        int nclus = 0;
        cudaError_t e = allow_max_smem(fn, device);
        if (e == cudaSuccess && q > 8) e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e == cudaSuccess) {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3((unsigned)(q * (sms * per_sm / q)));
          cfg.blockDim = dim3((unsigned)dense_block(DK_EVAL, nt_q));
          cfg.dynamicSmemBytes = dense_smem(c, DK_EVAL, st);
          cudaLaunchAttribute attr[1];
          attr[0].id = cudaLaunchAttributeClusterDimension;
          attr[0].val.clusterDim.x = (unsigned)q;
          attr[0].val.clusterDim.y = 1;
          attr[0].val.clusterDim.z = 1;
          cfg.attrs = attr;
          cfg.numAttrs = 1;
          if (cudaOccupancyMaxActiveClusters(&nclus, fn, &cfg) != cudaSuccess) nclus = 0;
        }
        cudaGetLastError();
        if (nclus < 1) continue;
        fit = std::min(fit, nclus);
      }
      const int64_t ncl_q = std::max<int64_t>(1, std::min<int64_t>(fit, c->m_loc));
      const double cost = (double)cdiv(c->m_loc, ncl_q) * (ns_q + (q > 1 ? 2.0 : 0.0));
      if (cost < best * (1.0 - 1e-9)) {
        best = cost;
        cl = q;
      }
    }
    if (best >= 1e300) {
      delete c;
      return fail(OTB_ERR_ARG, "no dense cluster geometry fits this n");
    }
  }
  c->cl = cl;
  c->per_sm = per_sm;
  c->colw = (int)rup(cdiv(n, cl), cl > 1 ? 64 : 2);   // cluster windows start on 64-column words
  int ns = (int)std::min<int64_t>(kMaxNS, std::max<int64_t>(1, cdiv(c->colw, slice_cols)));
  int nt = (int)rup(cdiv(c->colw, 2 * ns), 32);
  const char* env_nt = std::getenv("OTB_DENSE_NT");
  if (env_nt) {
    const int want = std::atoi(env_nt);
    if (want >= 32 && want <= slice_cols / 2 && want % 32 == 0) {
      nt = want;
      ns = (int)cdiv(c->colw, 2 * nt);
      if (ns > kMaxNS) {
        ns = kMaxNS;
        nt = (int)rup(cdiv(c->colw, 2 * ns), 32);
      }
    }
  }
  c->ns = ns;
  c->nt = std::max(nt, 32);
  // cluster windows are whole slices, so that only the LAST CTA of a cluster
  // can end on a partial slice (whose masked columns lie past n, where the
  // eval's gamma stream is -inf)
  if (cl > 1) c->colw = 2 * c->nt * c->ns;
  c->ncl = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)(sms * per_sm) / cl, c->m_loc));
  c->grid = c->ncl * cl;
  // ring depth: 8 stages unless OTB_DENSE_NSTAGE caps it (a shallower ring
  // leaves more of the SM's 256 KB to L1, where the CTA's window of gamma is
  // re-read every row)
  const char* env_ns = std::getenv("OTB_DENSE_NSTAGE");
  const int max_stage = env_ns ? std::max(2, std::min(8, std::atoi(env_ns))) : 8;
  for (int k = 0; k < DK_COUNT; ++k) {
    const size_t budget = kMaxDynSmem / per_sm - kStaticSmem[k] - 1024;
    int st = kSelfFeed[k] && !env_ns ? kMaxStageSelf : max_stage;   // the self-fed kinds: as deep as fits
    while (st > 2 && dense_smem(c, k, st) > budget) --st;
    c->nstage[k] = st;
    c->smem[k] = dense_smem(c, k, st);
    if (c->smem[k] > budget) {
      if (std::getenv("OTB_DEBUG_GEOM"))
        std::fprintf(stderr, "otb: dense kind %d: %zu B of shared memory > %zu (nt %d, ns %d, cl %d, %d per SM)\n", k,
                     c->smem[k], budget, c->nt, c->ns, cl, per_sm);
      delete c;
      return fail(OTB_ERR_ARG, "dense geometry does not fit shared memory");
    }
    cudaError_t e = allow_max_smem(kDenseFn[k][c->ns], device);
    if (e == cudaSuccess && cl > 8)
      e = cudaFuncSetAttribute(kDenseFn[k][c->ns], cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e == cudaSuccess && env_ns) {   // carve only what the ring needs: the rest is L1
      const int pct = (int)std::min<int64_t>(100, cdiv(100 * (int64_t)(c->smem[k] + kStaticSmem[k] + 1024), 233472));
      e = cudaFuncSetAttribute(kDenseFn[k][c->ns], cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    }
    if (e != cudaSuccess) {
      delete c;
      return fail(OTB_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    }
  }
  // Clusters must fit in a GPC: with cl > 1 fewer than sms / cl clusters may
  // be co-resident, and a second wave would double every dense pass.  Size
  // the row blocks to the clusters that actually run at once.
  if (cl > 1) {
    int fit = c->ncl;
    for (int k = 0; k < DK_COUNT; ++k) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)c->grid);
      cfg.blockDim = dim3((unsigned)dense_block(k, c->nt));
      cfg.dynamicSmemBytes = c->smem[k];
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = (unsigned)cl;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int nclus = 0;
      if (cudaOccupancyMaxActiveClusters(&nclus, kDenseFn[k][c->ns], &cfg) == cudaSuccess && nclus > 0)
        fit = std::min(fit, nclus);
      cudaGetLastError();
    }
    c->ncl = std::max(1, fit);
    c->grid = c->ncl * cl;
  }
  // hess_apply variant: shared-memory group accumulators (NG groups of
  // 512/NG threads, as many as fit) or, for very wide n, global RED.
  const int64_t npad = rup(n, 2);
  const size_t hv_budget = kMaxDynSmem - 16384;   // static smem of k_cg_fused (~14.4 KB)
  int ng = 8;
  const char* env_ng = std::getenv("OTB_HV_GROUPS");
  if (env_ng) ng = std::max(1, std::min(16, std::atoi(env_ng)));
  while (ng > 1 && (size_t)((1 + ng) * npad + 16 * 64) * 8 > hv_budget) ng >>= 1;
  c->hv_ng = ng;
  c->hv_smem = (size_t)((1 + ng) * npad + 16 * 64) * 8;
  const char* env_hv = std::getenv("OTB_HV_MODE");
  c->hv_mode = (c->hv_smem <= hv_budget) ? 0 : 1;
  if (env_hv && std::atoi(env_hv) == 1) c->hv_mode = 1;
  // bitmap hess_apply (sparse.cuh) whenever a thread's columns fit registers
  const int nwords = (int)rup(cdiv(n, 64), 16);   // words per row, zero past n
  const char* env_bm = std::getenv("OTB_HV_BITMAP");
  const char* env_st = std::getenv("OTB_HV_STAGED");
  if (c->hv_mode == 0 && nwords / 16 <= kMaxNQ && !(env_bm && std::atoi(env_bm) == 0)) {
    c->hv_mode = 2;
    c->nq = nwords;
    c->hv_var = nwords / 16;
    c->hv_ng = 0;
    c->hv_smem = (size_t)(npad + 16 * 64) * 8 + kBmSmemBytes;
    if (nwords <= 64 && !(env_st && std::atoi(env_st) == 0)) {   // n <= 4096: TMA-staged values
      c->hv_var = 8 + nwords / 16;
      c->hv_threads = kStThreads;
      c->hv_smem = (size_t)(npad + 16 * 64) * 8 + 2 * (size_t)kStBytes + 32;
    }
  }
  // n > 8192 and too wide for the group accumulators (hv_mode 1): window
  // clusters (sparse.cuh k_hv_wc<NQ>): W CTAs of 1024 NQ columns each,
  // W = ceil(n / (1024 NQ)) <= 16.  NQ is chosen for the least work per SM:
  // rows per co-resident cluster x window width (clusters must fit in a GPC,
  // so e.g. clusters of 13 leave a third of the SMs idle).  OTB_HV_NQ forces
  // NQ; OTB_HV_WC=1 uses the window clusters for any n > 8192.
  const char* env_wc = std::getenv("OTB_HV_WC");
  const bool want_wc = (c->hv_mode == 1 || (env_wc && std::atoi(env_wc) == 1)) && c->hv_mode != 2;
  if (want_wc && n > 8192 && !(env_bm && std::atoi(env_bm) == 0) && !(env_wc && std::atoi(env_wc) == 0) &&
      !(env_hv && std::atoi(env_hv) == 1)) {
    const char* env_nq = std::getenv("OTB_HV_NQ");
    const int force_nq = env_nq ? std::atoi(env_nq) : 0;
    double best = 1e300;
    int best_nq = 0, best_w = 0, best_ncl = 0, best_s = 0;
    for (int nqw = 1; nqw <= kMaxNQ; ++nqw) {
      if (force_nq > 0 && nqw != force_nq) continue;
      const int W = (int)cdiv(n, 1024 * nqw);
      if (W < 2 || W > kWcMaxW) continue;
      const void* fn = kWcFn[0][nqw];
      const int stage = wc_stage_bytes(nqw);
      const int S = (int)std::min<int64_t>(4, (int64_t)(kMaxDynSmem - 8192 - 8192 * nqw) / (stage + 16));
      if (S < 2) continue;
      cudaError_t e = allow_max_smem(fn, device);
      if (e == cudaSuccess) e = allow_max_smem(kWcFn[1][nqw], device);
      if (e == cudaSuccess && W > 8) e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e == cudaSuccess && W > 8)
        e = cudaFuncSetAttribute(kWcFn[1][nqw], cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      int nclusters = 0;
      if (e == cudaSuccess) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(W * (sms / W)));
        cfg.blockDim = dim3(kStThreads);
        cfg.dynamicSmemBytes = wc_smem_bytes(nqw, stage, S);
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = (unsigned)W;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        e = cudaOccupancyMaxActiveClusters(&nclusters, fn, &cfg);
      }
      cudaGetLastError();
      if (e != cudaSuccess || nclusters < 1) continue;
      nclusters = std::min(nclusters, sms / W);
      // rows per cluster x the measured time per row of the dense-P_rho kernel (config 4, n =
      // 16384, profiles/r2/hv_nq_sweep_cfg4.txt): 0.42 us of per-row reduction and exchange plus
      // 0.09 us per 1024 columns (NQ = 2: 0.66, 3: 0.68, 4: 0.75, 6: 0.96 us).  The kernel holds
      // 6 NQ doubles per thread (two rows' values, v, the accumulator) and spills from NQ = 7 on
      // (ptxas: 108 B at 7, 404 B at 8): NQ = 8 measured 2.07 us per row.  So W = 3 x 6144 on 135
      // SMs (1.40 ms per product) beats W = 2 x 8192 on 148 SMs (1.83 ms).
      const double spill = nqw >= 8 ? 1.8 : (nqw == 7 ? 1.3 : 1.0);
      const double cost = (0.42 + 0.09 * nqw) * spill / nclusters;
      if (cost < best * (1.0 - 1e-9)) {
        best = cost;
        best_nq = nqw;
        best_w = W;
        best_ncl = nclusters;
        best_s = S;
      }
    }
    if (best_nq > 0) {
      c->hv_mode = 3;
      c->hv_var = best_nq;
      c->hv_win = best_w;
      c->nq = 16 * best_nq * best_w;   // bitmap words per row
      c->hv_ng = best_s;               // ring stages
      c->hv_smem = wc_smem_bytes(best_nq, wc_stage_bytes(best_nq), best_s);
      c->hv_nb = best_ncl;
      c->hv_grid = best_ncl * best_w;
      const char* env_wcd = std::getenv("OTB_HV_WCD");
      c->hv_wcd = !(env_wcd && std::atoi(env_wcd) == 0);
      // the dense-P_rho kernel: no v window in shared memory, as many stages as fit
      const int stage = wc_stage_bytes(best_nq);
      c->hv_ng_d = (int)std::min<int64_t>(kWcMaxStages, (int64_t)(kMaxDynSmem - 8192) / (stage + 16));
      c->hv_smem_d = (size_t)c->hv_ng_d * stage + 2 * (size_t)c->hv_ng_d * 8;
      const void* fd = kWcdFn[best_nq];
      cudaError_t e = allow_max_smem(fd, device);
      if (e == cudaSuccess && best_w > 8) e = cudaFuncSetAttribute(fd, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      int ncd = 0;
      if (e == cudaSuccess) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)c->hv_grid);
        cfg.blockDim = dim3(kStConsumers);
        cfg.dynamicSmemBytes = c->hv_smem_d;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = (unsigned)best_w;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        e = cudaOccupancyMaxActiveClusters(&ncd, fd, &cfg);
      }
      cudaGetLastError();
      if (e != cudaSuccess || ncd < best_ncl) {   // keep the producer-warp dense kernel
        if (std::getenv("OTB_DEBUG_GEOM"))
          std::fprintf(stderr, "otb: k_hv_wcd<%d> W=%d: %d co-resident clusters (< %d, %s); producer-warp kernel kept\n",
                       best_nq, best_w, ncd, best_ncl, cudaGetErrorString(e));
        c->hv_wcd = false;
      }
    }
  }
  if (n > 65536 && c->hv_mode != 3) {
    delete c;
    return fail(OTB_ERR_ARG, "n > 65536 needs the window-cluster hess_apply (16-bit CSR column indices otherwise)");
  }
  if (c->hv_mode == 0 || c->hv_mode == 2) {
    c->hv_grid = sms;
    const char* env_cgg = std::getenv("OTB_CG_GRID");   // experiments: fewer hess_apply / CG CTAs
    if (env_cgg && std::atoi(env_cgg) > 0) c->hv_grid = std::min(sms, std::atoi(env_cgg));
    c->hv_nb = c->hv_grid;
    cudaError_t e = allow_max_smem(kHvFn[c->hv_var], device);
    if (e == cudaSuccess) e = allow_max_smem(kCgFn[c->hv_var], device);
    if (e != cudaSuccess) {
      delete c;
      return fail(OTB_ERR_CUDA, std::string("cudaFuncSetAttribute(hv): ") + cudaGetErrorString(e));
    }
    // the persistent CG keeps p and r in shared memory as well: (2 + NG) rows
    int fng = c->hv_ng;
    while (fng > 1 && (size_t)((2 + fng) * npad + 16 * 64) * 8 > hv_budget) fng >>= 1;
    c->fused_ng = fng;
    c->fused_smem = (size_t)((2 + fng) * npad + 16 * 64) * 8 +
                    (c->hv_var > kMaxNQ ? 2 * (size_t)kStBytes + 32 : (c->hv_mode == 2 ? kBmSmemBytes : 0));
    int per_sm_fused = 0;
    if (c->fused_smem <= hv_budget)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_fused, kCgFn[c->hv_var], c->hv_threads,
                                                    c->fused_smem);
    const char* env_f = std::getenv("OTB_CG_FUSED");
    c->cg_fused = per_sm_fused >= 1 && !(env_f && std::atoi(env_f) == 0);
  } else if (c->hv_mode == 1) {
    c->hv_grid = sms * 8;
    c->hv_nb = 1;
  }
  // Dense-P_rho overlay of a group-kernel context (8192 < n, e.g. config 3: n = 10000): the
  // dense window-cluster kernel streams P_rho at ~6 TB/s whatever the row's nnz, the CSR group
  // kernel moves 10 B per kept entry at ~2.3 TB/s, so dense wins while a quarter or more is kept
  // (config 3's first Newton steps keep 49%: 212 -> 135 us per product).  Geometry as for the
  // window clusters: the measured time per row x rows per co-resident cluster.
  {
    const char* env_ov = std::getenv("OTB_HV_OVERLAY");
    if (c->hv_mode == 0 && n > 8192 && !(env_ov && std::atoi(env_ov) == 0)) {
      double best = 1e300;
      for (int nqw = 1; nqw <= kMaxNQ; ++nqw) {
        const int W = (int)cdiv(n, 1024 * nqw);
        if (W < 2 || W > kWcMaxW) continue;
        const void* fd = kWcdFn[nqw];
        const int stage = wc_stage_bytes(nqw);
        const int S = (int)std::min<int64_t>(kWcMaxStages, (int64_t)(kMaxDynSmem - 8192) / (stage + 16));
        if (S < 2) continue;
        const size_t smem = (size_t)S * stage + 2 * (size_t)S * 8;
        cudaError_t e = allow_max_smem(fd, device);
        if (e == cudaSuccess && W > 8) e = cudaFuncSetAttribute(fd, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        int ncd = 0;
        if (e == cudaSuccess) {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3((unsigned)(W * (sms / W)));
          cfg.blockDim = dim3(kStConsumers);
          cfg.dynamicSmemBytes = smem;
          cudaLaunchAttribute attr[1];
          attr[0].id = cudaLaunchAttributeClusterDimension;
          attr[0].val.clusterDim.x = (unsigned)W;
          attr[0].val.clusterDim.y = 1;
          attr[0].val.clusterDim.z = 1;
          cfg.attrs = attr;
          cfg.numAttrs = 1;
          e = cudaOccupancyMaxActiveClusters(&ncd, fd, &cfg);
        }
        cudaGetLastError();
        if (e != cudaSuccess || ncd < 1) continue;
        ncd = (int)std::min<int64_t>(std::min(ncd, sms / W), c->m_loc);
        const double spill = nqw >= 8 ? 1.8 : (nqw == 7 ? 1.3 : 1.0);
        const double cost = (0.42 + 0.09 * nqw) * spill / ncd;
        if (cost < best * (1.0 - 1e-9)) {
          best = cost;
          c->ov_ok = true;
          c->ov_nq = nqw;
          c->ov_win = W;
          c->ov_ncl = ncd;
          c->ov_stages = S;
          c->ov_smem = smem;
        }
      }
      if (c->ov_ok) {
        // Which product is faster, from config 3's solve (tools/solve_probe.py, kept density 49% ->
        // 8%): the dense kernel streams m_loc x ld doubles at ~6 TB/s (139 us) whatever is kept; the
        // group kernel costs ~2.2 us per row of a CTA (150 us at 68 rows: latency, not bytes) plus
        // 1.27 us per million kept entries (212 us at 49%, ~165 us at 8-20%).  Dense from the
        // density where it wins — at config 3 always (solve 0.60-0.63 -> 0.53-0.58 s).
        const double dense_us = (double)c->m_loc * (double)ld * 8.0 / 6.0e6 + 5.0;
        const double group_fixed_us = 2.2 * (double)cdiv(c->m_loc, c->hv_grid);
        const double per_entry_us = 1.27e-6;
        c->ov_min_density =
            std::max(0.0, (dense_us - group_fixed_us) / (per_entry_us * (double)c->m_loc * (double)n));
      }
    }
  }
  c->colgrid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 2 * sms));
  c->col32 = (int)cdiv(n, 32);
  // buffers
  const int64_t m_loc = c->m_loc;
  const int64_t nv = npad + 16;
  int st = OTB_OK;
  auto A = [&](double** p, size_t cnt) {
    if (st == OTB_OK) st = dalloc(p, cnt);
  };
  A(&c->rowM, m_loc);
  A(&c->rowS, m_loc);
  A(&c->lse, m_loc);
  A(&c->zrow, m_loc);
  A(&c->czeta, m_loc);
  A(&c->er, m_loc);
  A(&c->rowpart, (size_t)m_loc * cl);
  const int64_t parts = std::max<int64_t>(std::max<int64_t>(2 * c->ncl, c->hv_nb), c->ov_ncl);
  A(&c->colpart, (size_t)parts * n);
  A(&c->vpart, (size_t)std::max(c->grid, c->ncl) * 8 + 8);
  A(&c->sendbuf, nv);
  A(&c->bpart, 4 * (size_t)std::max(c->colgrid, c->col32) + 64);
  A(&c->scal, 2 * (size_t)c->hv_grid + 16);
  for (double** p : {&c->g, &c->d, &c->rhs, &c->dir, &c->cg_r, &c->cg_p[0], &c->cg_p[1], &c->cg_ap, &c->cg_y,
                     &c->gtrial, &c->Mloc, &c->Mglob, &c->Sloc})
    A(p, nv);
  A(&c->ec, (size_t)n + 2 * c->nt + 64);    // + one slice of zero padding (test_c streams e_c)
  A(&c->gev, (size_t)n + 2 * c->nt + 64);   // + one slice of -inf padding
  A(&c->yv, (size_t)n + 2 * c->nt + 64);    // + one slice of zero padding (test_b streams y)
  if (st == OTB_OK) st = dalloc(&c->row_start, m_loc);
  if (st == OTB_OK) st = dalloc(&c->rowpre, m_loc + 1);
  if (st == OTB_OK) st = dalloc(&c->row_len, m_loc);
  if (st == OTB_OK) st = dalloc(&c->cta_rb, (size_t)c->hv_grid + 2);
  if (st == OTB_OK && c->ov_ok) st = dalloc(&c->ov_rb, (size_t)c->ov_ncl + 2);
  if (st == OTB_OK) st = dalloc(&c->ds, 1);
  if (st == OTB_OK) st = dalloc(&c->cg, 1);
  if (st == OTB_OK && (c->hv_mode == 2 || c->hv_mode == 3)) st = dalloc(&c->bm, (size_t)m_loc * c->nq);
  // P of the eval, so that sparsify streams one matrix and does no exp
  // (OTB_STORE_P=0: sparsify recomputes P from C and log X)
  const char* env_p = std::getenv("OTB_STORE_P");
  if (st == OTB_OK && !(env_p && std::atoi(env_p) == 0)) {
    st = dalloc(&c->Pbuf, (size_t)m_loc * ld);
    if (st == OTB_OK) cudaMemset(c->Pbuf, 0, sizeof(double) * (size_t)m_loc * ld);   // padding columns stay 0
  }
  const char* env_cgg2 = std::getenv("OTB_CG_GRAPH");
  c->cg_graph = !(env_cgg2 && std::atoi(env_cgg2) == 0);
  const char* env_fp = std::getenv("OTB_FORCE_EVAL_POST");
  c->force_post = env_fp && std::atoi(env_fp) == 1;
  const char* env_tr = std::getenv("OTB_CG_TRACE");
  if (st == OTB_OK && env_tr && std::atoi(env_tr) == 1) {
    const size_t cnt = (size_t)c->hv_grid * kCgTraceIters * 6;
    if (cudaMalloc((void**)&c->cg_trace, cnt * sizeof(unsigned long long)) != cudaSuccess) st = OTB_ERR_NOMEM;
    else cudaMemset(c->cg_trace, 0, cnt * sizeof(unsigned long long));
  }
  if (st != OTB_OK) {
    otb_destroy(c);
    return st;
  }
  // CSR chunk per bump allocation: large enough that a CTA refills (two
  // named barriers) every ~16 rows, not every ~2 (the slack, at most one
  // chunk per CTA, is part of the capacity)
  c->chunk = rup(std::max<int64_t>(8192, 16 * n), kCsrAlign);
  // first Newton steps keep 50-70% of P: start at 3/4
  int64_t init_cap =
      std::max<int64_t>((int64_t)1 << 20, m_loc * (rup(n, kCsrAlign)) * 3 / 4) + (int64_t)c->ncl * c->chunk;
  // Contexts whose sparsify writes the dense P_rho at every density (window clusters, an overlay that
  // always wins: configs 3-5) never touch the CSR runs: start them at the minimum (config 5: 19 GB of
  // values + columns not allocated); a sparsify in the sparse format (OTB_HV_DENSE=0, OTB_STORE_P=0)
  // grows it through the overflow-and-redo path.
  if (c->Pbuf != nullptr && ((c->hv_mode == 3 && kDenseRhoMin <= 0.0) || (c->ov_ok && c->ov_min_density <= 0.0)))
    init_cap = ((int64_t)1 << 20) + (int64_t)c->ncl * c->chunk;
  const char* env_cap = std::getenv("OTB_CSR_CAP0");   // tests: start small to exercise the overflow path
  if (env_cap && std::atoll(env_cap) > 0) init_cap = std::atoll(env_cap);
  st = grow_csr(c, init_cap);
  if (st != OTB_OK) {
    otb_destroy(c);
    return st;
  }
  if (cudaMallocHost((void**)&c->hs, sizeof(DevScalars)) != cudaSuccess ||
      cudaMallocHost((void**)&c->hcg, sizeof(CgState)) != cudaSuccess ||
      cudaMallocHost((void**)&c->hbuf, 16 * sizeof(double)) != cudaSuccess) {
    otb_destroy(c);
    return fail(OTB_ERR_NOMEM, "cudaMallocHost failed");
  }
  cudaMemset(c->ds, 0, sizeof(DevScalars));
  if (c->hv_mode == 2 || c->hv_mode == 3) {   // equal row counts per hess_apply CTA / cluster, fixed
    Csr A = csr_view(c);
    A.cta_rb = nullptr;
    k_cta_bounds<<<(int)cdiv(c->hv_nb + 1, 256), 256>>>(A, c->hv_nb, c->cta_rb, 1);
  }
  if (c->ov_ok) {   // the overlay's clusters: equal row counts
    Csr A = csr_view(c);
    A.cta_rb = nullptr;
    k_cta_bounds<<<(int)cdiv(c->ov_ncl + 1, 256), 256>>>(A, c->ov_ncl, c->ov_rb, 1);
  }
  cudaMemset(c->cg, 0, sizeof(CgState));
  cudaMemset(c->cg_y, 0, sizeof(double) * nv);
  cudaMemset(c->row_len, 0, sizeof(int) * m_loc);
  {   // padding of the vectors the dense passes stream past n, so that the masked
      // columns of a partial last slice drop out: gamma -1e300 (eval: z = -1e302,
      // exp = 0; test_c: slack +1e300 > 0), y and e_c 0 (f = 0)
    const std::vector<double> pad((size_t)2 * c->nt + 64, -1e300);
    cudaMemcpy(c->gev + n, pad.data(), pad.size() * sizeof(double), cudaMemcpyHostToDevice);
    cudaMemset(c->yv, 0, sizeof(double) * ((size_t)n + 2 * c->nt + 64));
    cudaMemset(c->ec, 0, sizeof(double) * ((size_t)n + 2 * c->nt + 64));
  }
  if (c->bm) cudaMemset(c->bm, 0, sizeof(uint4) * m_loc * c->nq);
  cudaMemset(c->rowpre, 0, sizeof(int64_t) * (m_loc + 1));
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    otb_destroy(c);
    return fail(OTB_ERR_CUDA, std::string("init: ") + cudaGetErrorString(e));
  }
  *out = c;
  return OTB_OK;
}

int otb_destroy(otb_ctx* c) {
  if (!c) return OTB_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (void* p : {(void*)c->rowM, (void*)c->rowS, (void*)c->lse, (void*)c->zrow, (void*)c->czeta, (void*)c->er,
                  (void*)c->rowpart,
                  (void*)c->colpart, (void*)c->vpart, (void*)c->sendbuf, (void*)c->bpart, (void*)c->g, (void*)c->d,
                  (void*)c->rhs, (void*)c->dir, (void*)c->cg_r, (void*)c->cg_p[0], (void*)c->cg_p[1],
                  (void*)c->cg_ap, (void*)c->cg_y, (void*)c->gtrial, (void*)c->yv, (void*)c->ec, (void*)c->Mloc,
                  (void*)c->Mglob, (void*)c->Sloc, (void*)c->gev, (void*)c->row_start, (void*)c->rowpre, (void*)c->row_len, (void*)c->row_nnz,
                  (void*)c->cols, (void*)c->vals, (void*)c->ds, (void*)c->cg, (void*)c->scal, (void*)c->cta_rb,
                  (void*)c->ov_rb, (void*)c->bm, (void*)c->Pbuf, (void*)c->cg_trace, (void*)c->lg_tmp, (void*)c->jq,
                  (void*)c->minv, (void*)c->zv, (void*)c->colpart2})
    if (p) cudaFree(p);
  if (c->hs) cudaFreeHost(c->hs);
  if (c->hcg) cudaFreeHost(c->hcg);
  if (c->hbuf) cudaFreeHost(c->hbuf);
  for (auto& r : c->recs) {
    cudaEventDestroy(r.e0);
    cudaEventDestroy(r.e1);
  }
  for (auto e : c->pool) cudaEventDestroy(e);
  for (auto& e : c->cg_exec)
    if (e) cudaGraphExecDestroy(e);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  if (c->comm && c->nccl.commDestroy) c->nccl.commDestroy(c->comm);
  delete c;
  return OTB_OK;
}

int otb_set_stream(otb_ctx* c, void* stream) {
  if (!c) return fail(OTB_ERR_ARG, "null context");
  c->stream = (cudaStream_t)stream;
  return OTB_OK;
}

int otb_nccl_get_unique_id(const char* nccl_path, void* id128) {
  static Nccl api;
  TRY(load_nccl(nccl_path, api));
  NcclId id;
  const int r = api.getUniqueId(&id);
  if (r != 0) return fail(OTB_ERR_NCCL, "ncclGetUniqueId failed");
  std::memcpy(id128, &id, sizeof id);
  return OTB_OK;
}

int otb_attach_nccl(otb_ctx* c, const char* nccl_path, const void* id128, int nranks, int rank) {
  if (!c) return fail(OTB_ERR_ARG, "null context");
  // OTB_NCCL_SELFTEST=1: a ONE-rank communicator driven through every
  // multi-rank code path (the context behaves as rank 0 of 2: per-iteration
  // CG, fallback reductions, every ncclAllReduce call site, their graph
  // capture), so that a one-GPU box exercises the NCCL binding; the results
  // equal the single-rank ones.
  const char* st = std::getenv("OTB_NCCL_SELFTEST");
  const bool selftest = nranks == 1 && st && st[0] == '1';
  if (nranks <= 1 && !selftest) {
    c->nranks = 1;
    c->rank = 0;
    return OTB_OK;
  }
  TRY(load_nccl(nccl_path, c->nccl));
  NcclId id;
  std::memcpy(&id, id128, sizeof id);
  CUDA_TRY(cudaSetDevice(c->device));
  const int r = c->nccl.commInitRank(&c->comm, nranks, id, rank);
  if (r != 0) return fail(OTB_ERR_NCCL, "ncclCommInitRank failed");
  c->nranks = selftest ? 2 : nranks;
  c->rank = rank;
  c->cg_fused = false;   // the persistent CG has no H v all-reduce (krylov.py:68-84 needs the global H v)
  c->have_eval = false;
  return OTB_OK;
}

int otb_set_cg_precond(otb_ctx* c, int kind) {
  if (!c) return fail(OTB_ERR_ARG, "null context");
  if (kind != 0 && kind != 1) return fail(OTB_ERR_ARG, "preconditioner kind must be 0 (none) or 1 (Jacobi)");
  if (kind == c->precond) return OTB_OK;
  if (kind == 1 && !c->jq) {
    const size_t nv = (size_t)rup(c->n, 2) + 16;
    TRY(dalloc(&c->jq, nv));
    TRY(dalloc(&c->minv, nv));
    TRY(dalloc(&c->zv, nv));
    TRY(dalloc(&c->colpart2, (size_t)c->ncl * c->n));
  }
  c->precond = kind;
  // the sparsify passes carry a second accumulator: re-size their rings
  for (int k : {(int)DK_SPARSIFY, (int)DK_SPARSP, (int)DK_SPDENSE}) {
    const size_t budget = kMaxDynSmem / c->per_sm - kStaticSmem[k] - 1024;
    int st = kSelfFeed[k] ? kMaxStageSelf : 8;
    while (st > 2 && dense_smem(c, k, st) > budget) --st;
    if (dense_smem(c, k, st) > budget) return fail(OTB_ERR_ARG, "PCG accumulator does not fit shared memory");
    c->nstage[k] = st;
    c->smem[k] = dense_smem(c, k, st);
  }
  c->have_eval = false;
  return OTB_OK;
}

int otb_group_create(otb_group** out, int nranks) {
  if (!out) return fail(OTB_ERR_ARG, "out is null");
  *out = nullptr;
  if (nranks < 1 || nranks > kMaxGroup) return fail(OTB_ERR_ARG, "group size must be 1..16");
  otb_group* g = new otb_group();
  g->n = nranks;
  const char* env = std::getenv("OTB_GROUP_TIMEOUT");
  if (env && std::atof(env) > 0) g->timeout_s = std::atof(env);
  *out = g;
  return OTB_OK;
}

int otb_group_abort(otb_group* g) {
  if (!g) return fail(OTB_ERR_ARG, "null group");
  g->abort();
  return OTB_OK;
}

int otb_group_destroy(otb_group* g) {
  if (!g) return OTB_OK;
  for (int q = 0; q < g->n; ++q) {
    if (g->ready[q]) cudaEventDestroy(g->ready[q]);
    if (g->done[q]) cudaEventDestroy(g->done[q]);
  }
  delete g;
  return OTB_OK;
}

int otb_attach_group(otb_ctx* c, otb_group* g, int rank) {
  if (!c || !g) return fail(OTB_ERR_ARG, "null context or group");
  if (rank < 0 || rank >= g->n) return fail(OTB_ERR_ARG, "rank out of range");
  if (c->comm || c->group) return fail(OTB_ERR_ARG, "context already attached");
  CUDA_TRY(cudaSetDevice(c->device));
  {
    std::lock_guard<std::mutex> lk(g->mu);
    if (g->ready[rank]) return fail(OTB_ERR_ARG, "rank already attached");
    CUDA_TRY(cudaEventCreateWithFlags(&g->ready[rank], cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&g->done[rank], cudaEventDisableTiming));
    g->devices[rank] = c->device;
  }
  if (g->n > 1) TRY(dalloc(&c->lg_tmp, (size_t)(rup(c->n, 2) + 16)));
  c->group = g;
  c->nranks = g->n;
  c->rank = rank;
  if (g->n > 1) c->cg_fused = false;
  c->have_eval = false;
  return OTB_OK;
}

int otb_bind(otb_ctx* c, const double* C, const double* a, const double* b, const double* log_a,
             const double* log_b, double eta, int64_t anchor_global, double norm_c, double norm_a, double norm_b) {
  if (!c) return fail(OTB_ERR_ARG, "null context");
  if (!C || !a || !b || !log_a || !log_b) return fail(OTB_ERR_ARG, "null problem array");
  if (!(eta > 0.0)) return fail(OTB_ERR_ARG, "eta must be positive");
  if (anchor_global < 0 || anchor_global >= c->m_glob) return fail(OTB_ERR_ARG, "anchor out of range");
  if (((uintptr_t)C) % 256 != 0) return fail(OTB_ERR_ARG, "C must be 256-byte aligned");
  c->C = C;
  c->a = a;
  c->b = b;
  c->log_a = log_a;
  c->log_b = log_b;
  c->eta = eta;
  c->anchor = anchor_global;
  c->norm_c = norm_c;
  c->norm_c_dev = false;
  c->norm_a = norm_a;
  c->norm_b = norm_b;
  c->bound = true;
  c->have_eval = false;
  return OTB_OK;
}

int otb_eval(otb_ctx* c, const double* logX, const double* gamma, double* lse_out, double* grad_out,
             otb_eval_out* out) {
  TRY(require_bound(c));
  if (((uintptr_t)logX) % 256 != 0) return fail(OTB_ERR_ARG, "logX must be 256-byte aligned");
  TRY(do_eval(c, logX, gamma));
  if (lse_out)
    CUDA_TRY(cudaMemcpyAsync(lse_out, c->lse, sizeof(double) * c->m_loc, cudaMemcpyDeviceToDevice, c->stream));
  if (grad_out)
    CUDA_TRY(cudaMemcpyAsync(grad_out, c->g, sizeof(double) * c->n, cudaMemcpyDeviceToDevice, c->stream));
  if (lse_out || grad_out) CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (out) {
    out->value = c->last_value;
    out->grad_norm = c->last_gnorm;
  }
  return OTB_OK;
}

int otb_sparsify(otb_ctx* c, const double* logX, const double* gamma, double rho, int64_t* nnz_out) {
  TRY(require_bound(c));
  if (!c->have_eval) return fail(OTB_ERR_ARG, "otb_sparsify needs a preceding otb_eval at the same gamma");
  TRY(do_sparsify(c, logX, gamma, rho));
  if (nnz_out) *nnz_out = c->nnz;
  return OTB_OK;
}

int otb_csr_export(otb_ctx* c, int64_t* row_ptr, int32_t* cols, double* vals, double* d) {
  TRY(require_bound(c));
  const bool bitmap = c->hv_mode == 2 || c->hv_mode == 3;   // pair-layout runs, columns in the bitmap words
  if (c->rho_dense) {   // dense P_rho: nonzeros per row (every entry of the anchor row)
    const int64_t anchor_local = (c->anchor >= c->row0 && c->anchor < c->row1) ? c->anchor - c->row0 : -1;
    if (!c->row_nnz) TRY(dalloc(&c->row_nnz, c->m_loc));
    k_dense_rownnz<<<c->num_sms * 8, 256, 0, c->stream>>>(c->Pbuf, c->ld, (int)c->m_loc, (int)c->n, anchor_local,
                                                           c->row_nnz);
    LAUNCH_CHECK();
    k_row_prefix<<<1, 1024, 0, c->stream>>>(c->row_nnz, (int)c->m_loc, c->rowpre);
    LAUNCH_CHECK();
    if (row_ptr)
      CUDA_TRY(cudaMemcpyAsync(row_ptr, c->rowpre, sizeof(int64_t) * (c->m_loc + 1), cudaMemcpyDeviceToDevice,
                               c->stream));
    if (cols && vals) {
      k_dense_export<<<c->num_sms * 8, 256, 0, c->stream>>>(c->Pbuf, c->ld, (int)c->m_loc, (int)c->n, anchor_local,
                                                            c->rowpre, cols, vals);
      LAUNCH_CHECK();
    }
    c->rowpre_valid = false;
    if (d) CUDA_TRY(cudaMemcpyAsync(d, c->d, sizeof(double) * c->n, cudaMemcpyDeviceToDevice, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return OTB_OK;
  }
  if (!c->rowpre_valid && (row_ptr || (cols && vals))) {
    if (bitmap) {
      if (!c->row_nnz) TRY(dalloc(&c->row_nnz, c->m_loc));
      k_bm_rownnz<<<c->num_sms * 8, 256, 0, c->stream>>>(c->bm, c->nq, (int)c->m_loc, c->row_nnz);
      LAUNCH_CHECK();
      k_row_prefix<<<1, 1024, 0, c->stream>>>(c->row_nnz, (int)c->m_loc, c->rowpre);
      LAUNCH_CHECK();
    } else {
      TRY(row_prefix(c));
    }
    c->rowpre_valid = true;
  }
  if (row_ptr)
    CUDA_TRY(cudaMemcpyAsync(row_ptr, c->rowpre, sizeof(int64_t) * (c->m_loc + 1), cudaMemcpyDeviceToDevice,
                             c->stream));
  if (cols && vals) {
    if (bitmap)
      k_bm_export<<<c->num_sms * 8, 256, 0, c->stream>>>(c->bm, c->nq, (int)c->m_loc, c->row_start, c->vals,
                                                         c->rowpre, cols, vals);
    else
      k_csr_compact<<<c->num_sms * 4, 256, 0, c->stream>>>((int)c->m_loc, c->row_start, c->row_len, c->rowpre,
                                                           c->cols, c->vals, cols, vals);
    LAUNCH_CHECK();
  }
  if (d) CUDA_TRY(cudaMemcpyAsync(d, c->d, sizeof(double) * c->n, cudaMemcpyDeviceToDevice, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return OTB_OK;
}

int otb_hess_apply(otb_ctx* c, const double* v, double shift, double* out) {
  TRY(require_bound(c));
  const int n = (int)c->n;
  if (c->hv_mode == 1) CUDA_TRY(cudaMemsetAsync(c->cg_y, 0, sizeof(double) * n, c->stream));
  HvResult hr;
  TRY(run_hv(c, v, nullptr, nullptr, nullptr, 0, nullptr, &hr));
  const double* cp = hr.ysum ? hr.ysum : hr.colpart;
  const int np = hr.ysum ? 1 : hr.nparts;
  k_hv_out<<<c->col32, 256, 0, c->stream>>>(n, cp, np, hr.yatomic, c->d, v, c->eta, shift, out);
  LAUNCH_CHECK();
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return OTB_OK;
}

int otb_cg(otb_ctx* c, double shift, const double* rhs, double rel_tol, int64_t max_iters, double* x_out,
           otb_cg_out* out) {
  TRY(require_bound(c));
  if (max_iters < 0) max_iters = 2 * c->n;
  return do_cg(c, shift, rhs, rel_tol, max_iters, x_out, out);
}

// Armijo backtracking from t0 (whose trial eval is in c->hs when
// `evaluated`), inner_newton.py:74-94.
int armijo(otb_ctx* c, const double* logX, const double* gamma_in, double v0, double slope,
           const otb_newton_params* p, bool evaluated, double* t_out, int64_t* trials_out, double* trial) {
  const int n = (int)c->n;
  double t = 1.0;
  int64_t trials = 0;
  for (int k = 0; k < 200; ++k) {
    if (!(evaluated && k == 0)) {
      k_trial<<<c->colgrid, 256, 0, c->stream>>>(n, gamma_in, c->dir, t, trial);
      LAUNCH_CHECK();
      TRY(do_eval(c, logX, trial));
    }
    ++trials;
    if (c->last_value <= v0 + p->sigma * t * slope) {
      *t_out = t;
      *trials_out = trials;
      return OTB_OK;
    }
    t *= p->beta;
  }
  c->have_eval = false;
  return fail(OTB_ERR_LINESEARCH, "no Armijo step accepted after 200 trials");
}

// The Newton step with the persistent CG (cg_fused): sparsify, CG, slope and
// the t = 1 trial are launched back to back and read with one host
// synchronisation; then Armijo.  With `spec`, the eval at gamma_in was only
// launched (its scalars saved in ds->ev0): rho and the CG shift are read on
// the device, and the host learns L(gamma_in) and ||g|| at the same
// synchronisation.  If that ||g|| is <= floor the step is discarded (the
// eval at gamma_in is redone so that its row state is the cached one) and
// *stepped = false.
int newton_fused(otb_ctx* c, const double* logX, const double* gamma_in, const otb_newton_params* p, bool spec,
                 double floor, double* v0, double* g0, double* rho, otb_cg_out* cgo, double* slope, double* t,
                 int64_t* trials, bool* stepped, double* trial) {
  const int n = (int)c->n;
  const int64_t maxit = (p->cg_max_iters > 0) ? p->cg_max_iters : 2 * c->n;
  *stepped = false;
  for (int attempt = 0; attempt < 8; ++attempt) {
    int64_t sp_rec = -1, cg_rec = -1;
    const double* gdev = spec ? &c->ds->ev0[1] : nullptr;
    TRY(sparsify_launch(c, logX, gamma_in, spec ? 0.0 : *rho, &sp_rec, gdev));
    // inner_newton.py:117: (H + ||g|| I) d = -g  (k_cg_init forms rhs = -g)
    TRY(cg_fused_launch(c, spec ? 0.0 : *g0, c->rhs, p->cg_rel_tol, maxit, c->dir, &cg_rec, c->g, gdev));
    // :118 slope = g . dir, with the t = 1 trial gamma_in + dir in the same pass
    k_dot_trial<<<c->colgrid, 256, 0, c->stream>>>(n, c->g, c->dir, c->ds, c->bpart, &c->ds->slope, gamma_in, 1.0,
                                                   trial);
    LAUNCH_CHECK();
    TRY(eval_launch(c, logX, trial));
    TRY(sync_scalars(c));
    if (spec) {   // the eval at gamma_in, now on the host
      spec = false;
      if (c->hs->ev0[2] != 0.0) {
        c->have_eval = false;
        return fail(OTB_ERR_NONFINITE, "row softmax produced non-finite values after stabilization");
      }
      *v0 = c->hs->ev0[0];
      *g0 = c->hs->ev0[1];
      *rho = c->eta * *g0 / ((double)c->m_glob * (double)c->n);   // inner_newton.py:112-114 (same bits)
      if (*g0 <= floor) {                                          // :205 — nothing to step
        TRY(do_eval(c, logX, gamma_in));
        return OTB_OK;
      }
    }
    bool redo = false;
    TRY(sparsify_finish(c, sp_rec, &redo));
    if (redo) {
      TRY(do_eval(c, logX, gamma_in));   // the trial replaced the row state sparsify reads
      continue;
    }
    c->have_eval = false;   // the row state is the trial's until eval_finish accepts it
    TRY(cg_finish(c, cg_rec, cgo));
    *slope = c->hs->slope;
    TRY(eval_finish(c));
    TRY(armijo(c, logX, gamma_in, *v0, *slope, p, true, t, trials, trial));
    *stepped = true;
    return OTB_OK;
  }
  return fail(OTB_ERR_NOMEM, "CSR capacity could not be grown");
}

void fill_newton_out(const otb_ctx* c, double t, double slope, double rho, double v0, double g0,
                     const otb_cg_out& cgo, int64_t trials, otb_newton_out* out) {
  if (!out) return;
  out->t = t;
  out->slope = slope;
  out->rho = rho;
  out->value_before = v0;
  out->value_after = c->last_value;
  out->grad_norm_before = g0;
  out->grad_norm_after = c->last_gnorm;
  out->cg_iters = cgo.iters;
  out->nnz = c->nnz_glob;   // all ranks' kept entries (the reference's nnz of the global P_rho)
  out->trials = trials;
  out->cg_residual = cgo.residual;
}

int otb_newton_step(otb_ctx* c, const double* logX, const double* gamma_in, double* gamma_out,
                    const otb_newton_params* p, otb_newton_out* out) {
  TRY(require_bound(c));
  if (!p) return fail(OTB_ERR_ARG, "null params");
  if (!c->have_eval) return fail(OTB_ERR_ARG, "otb_newton_step needs a preceding otb_eval at gamma_in");
  const int n = (int)c->n;
  double v0 = c->last_value, g0 = c->last_gnorm;
  // inner_newton.py:112-114
  double rho = (p->rho_override >= 0.0) ? p->rho_override : c->eta * g0 / ((double)c->m_glob * (double)c->n);
  const int64_t maxit = (p->cg_max_iters > 0) ? p->cg_max_iters : 2 * c->n;
  otb_cg_out cgo;
  double slope = 0.0, t = 1.0;
  int64_t trials = 0;
  // trials go straight into gamma_out unless it aliases gamma_in (backtracking re-reads gamma_in)
  double* trial = (gamma_out != gamma_in) ? gamma_out : c->gtrial;
  if (c->cg_fused && !c->precond) {
    bool stepped = false;
    TRY(newton_fused(c, logX, gamma_in, p, false, -1.0, &v0, &g0, &rho, &cgo, &slope, &t, &trials, &stepped,
                     trial));
  } else {
    TRY(do_sparsify(c, logX, gamma_in, rho));
    k_neg<<<c->colgrid, 256, 0, c->stream>>>(n, c->g, c->rhs);
    LAUNCH_CHECK();
    TRY(do_cg(c, g0, c->rhs, p->cg_rel_tol, maxit, c->dir, &cgo));
    k_dot<<<c->colgrid, 256, 0, c->stream>>>(n, c->g, c->dir, c->ds, c->bpart, &c->ds->slope);
    LAUNCH_CHECK();
    TRY(sync_scalars(c));
    slope = c->hs->slope;
    TRY(armijo(c, logX, gamma_in, v0, slope, p, false, &t, &trials, trial));
  }
  // stream-ordered: the caller's later work on this stream sees gamma_out
  if (trial != gamma_out)
    CUDA_TRY(cudaMemcpyAsync(gamma_out, trial, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  fill_newton_out(c, t, slope, rho, v0, g0, cgo, trials, out);
  return OTB_OK;
}

int otb_recover_round(otb_ctx* c, const double* logX, const double* gamma, double* logX_out, int recover,
                      int metrics, otb_test_out* out) {
  TRY(require_bound(c));
  if (recover && !c->have_eval) return fail(OTB_ERR_ARG, "recovery needs a preceding otb_eval at gamma");
  if (recover && (!logX_out || ((uintptr_t)logX_out) % 256 != 0))
    return fail(OTB_ERR_ARG, "logX_out must be a 256-byte aligned buffer");
  return do_round(c, logX, gamma, logX_out, recover, metrics, out);
}

int otb_set_cost_norm_sq(otb_ctx* c, const double* norm_sq) {
  if (!c) return fail(OTB_ERR_ARG, "null context");
  if (!norm_sq) return fail(OTB_ERR_ARG, "null norm");
  CUDA_TRY(cudaMemcpyAsync(&c->ds->cnorm_sq, norm_sq, sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  c->norm_c_dev = true;
  return OTB_OK;
}

int otb_inner_iteration(otb_ctx* c, const double* logX, double* gamma_in, double* gamma_out,
                        const otb_newton_params* p, int eval_first, double floor, double test_below,
                        double* logX_out, const double* gamma_src, otb_inner_out* out) {
  TRY(require_bound(c));
  if (!out) return fail(OTB_ERR_ARG, "out is null");
  if (((uintptr_t)logX) % 256 != 0) return fail(OTB_ERR_ARG, "logX must be 256-byte aligned");
  if (gamma_src && gamma_src != gamma_in)   // the caller's dual, copied into the working buffer
    CUDA_TRY(cudaMemcpyAsync(gamma_in, gamma_src, sizeof(double) * c->n, cudaMemcpyDeviceToDevice, c->stream));
  out->stepped = 0;
  out->tested = 0;
  if (eval_first && c->cg_fused && !c->precond && p && p->rho_override < 0.0) {
    // inner_newton.py:196 + the first step without a synchronisation in
    // between: the eval is launched and its scalars kept on the device
    TRY(eval_launch(c, logX, gamma_in, true));   // its L, ||g||, flag also kept in ds->ev0
    c->p_valid = c->Pbuf != nullptr;   // the stored P is in stream order before sparsify reads it
    double v0 = 0.0, g0 = 0.0, rho = 0.0, slope = 0.0, t = 1.0;
    int64_t trials = 0;
    otb_cg_out cgo{};
    bool stepped = false;
    double* trial = (gamma_out != gamma_in) ? gamma_out : c->gtrial;
    TRY(newton_fused(c, logX, gamma_in, p, true, floor, &v0, &g0, &rho, &cgo, &slope, &t, &trials, &stepped,
                     trial));
    out->value0 = v0;
    out->grad_norm0 = g0;
    if (!stepped) return OTB_OK;                                   // :205 gradient floor
    if (trial != gamma_out)
      CUDA_TRY(cudaMemcpyAsync(gamma_out, trial, sizeof(double) * c->n, cudaMemcpyDeviceToDevice, c->stream));
    fill_newton_out(c, t, slope, rho, v0, g0, cgo, trials, &out->newton);
    out->stepped = 1;
  } else {
    if (eval_first) TRY(do_eval(c, logX, gamma_in));               // inner_newton.py:196
    out->value0 = c->last_value;
    out->grad_norm0 = c->last_gnorm;
    if (c->last_gnorm <= floor) return OTB_OK;                     // :205 gradient floor
    TRY(otb_newton_step(c, logX, gamma_in, gamma_out, p, &out->newton));
    out->stepped = 1;
  }
  if (test_below >= 0.0 && out->newton.grad_norm_after < test_below) {   // :239 pre-check, then the test
    if (!logX_out || ((uintptr_t)logX_out) % 256 != 0)
      return fail(OTB_ERR_ARG, "logX_out must be a 256-byte aligned buffer");
    TRY(do_round(c, logX, gamma_out, logX_out, 1, 1, &out->test));
    out->tested = 1;
  }
  return OTB_OK;
}

int otb_materialize_rounded(otb_ctx* c, double* out, int64_t ldo) {
  TRY(require_bound(c));
  if (!c->round_src) return fail(OTB_ERR_ARG, "no rounding performed yet");
  k_materialize_rounded<<<c->num_sms * 8, 256, 0, c->stream>>>(c->round_src, c->ld, (int)c->m_loc, (int)c->n,
                                                               c->zrow, c->yv, c->er, c->ec, &c->ds->deficit, out,
                                                               ldo);
  LAUNCH_CHECK();
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return OTB_OK;
}

// sinkhorn.py:47-51 + 61-65: zeta sweep fused with the column sums of the
// scaled plan; *err = ||colsum - b|| (host read).
int sweep_zeta(otb_ctx* c, const double* logX, const double* gamma, double* zeta, double* err) {
  const int n = (int)c->n;
  const double mn = (double)c->m_loc * n;
  // sinkhorn.py:47-51 is the eval's row log-sum-exp of logX + (gamma - C)/eta
  // (global row max first, as _lse): the eval kernel without the P store;
  // zeta = eta (log a - lse).  The column sums of the error check
  // (sinkhorn.py:61-65, exp(logX + (zeta + gamma - C)/eta) summed over rows)
  // are then sum_i a_i P_ij, which the eval accumulates anyway (w e_ij with
  // w = a_i / S_i): one pass instead of k_warm_zeta's three divisions and two
  // exps per element; the sums differ from the reference's expression in the
  // last bits and only decide warm_tol.
  if (gamma != c->gev)
    CUDA_TRY(cudaMemcpyAsync(c->gev, gamma, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  Geom geo = make_geom(c, DK_EVAL, c->C, logX);
  geo.vec[0] = c->gev;
  EvalIO io{c->gev, c->a, c->eta, c->rowM, c->rowS, c->lse, c->colpart, c->vpart, nullptr};
  cudaEvent_t e0 = nullptr;
  TRY(prof_begin(c, &e0));
  TRY(launch_dense(c, DK_EVAL, geo, &io));
  TRY(prof_end(c, PC_WARMZ, e0, 16.0 * mn));
  k_zeta_from_lse<<<c->colgrid, 256, 0, c->stream>>>((int)c->m_loc, c->log_a, c->row0, c->lse, c->eta, zeta);
  LAUNCH_CHECK();
  TRY(colreduce(c, c->ncl, nullptr, 0, 0, 0));
  TRY(allreduce(c, c->sendbuf, (size_t)n, kNcclSum));
  k_vec_post<<<c->colgrid, 256, 0, c->stream>>>(POST_WARMERR, n, c->sendbuf, c->b, nullptr, c->ds, c->bpart,
                                                &c->ds->warm_err);
  LAUNCH_CHECK();
  TRY(sync_scalars(c));
  *err = std::sqrt(c->hs->warm_err);
  return OTB_OK;
}

int sweep_gamma(otb_ctx* c, const double* logX, double* gamma, const double* zeta);

int otb_warm_start(otb_ctx* c, const double* logX, double* gamma, double* zeta, double warm_tol, int64_t max_sweeps,
                   otb_warm_out* out) {
  TRY(require_bound(c));
  const int n = (int)c->n;
  int64_t sweeps = 0;
  double err = INFINITY;
  bool done = false;
  for (int64_t s = 0; s < max_sweeps; ++s) {
    TRY(sweep_zeta(c, logX, gamma, zeta, &err));
    sweeps = s + 1;
    if (err < warm_tol) {
      done = true;
      break;
    }
    TRY(sweep_gamma(c, logX, gamma, zeta));
  }
  if (!done) {
    char buf[96];
    std::snprintf(buf, sizeof buf, "warm start did not reach %g in %lld sweeps", warm_tol, (long long)max_sweeps);
    return fail(OTB_ERR_WARMSTART, buf);
  }
  // sinkhorn.py:102-103: recentre gamma onto the zero-sum slice
  k_sum<<<c->colgrid, 256, 0, c->stream>>>(n, gamma, c->ds, c->bpart, &c->ds->drift);
  LAUNCH_CHECK();
  k_shift<<<c->colgrid, 256, 0, c->stream>>>(n, gamma, &c->ds->drift, (double)n, -1.0);
  LAUNCH_CHECK();
  k_shift<<<c->colgrid, 256, 0, c->stream>>>((int)c->m_loc, zeta, &c->ds->drift, (double)n, 1.0);
  LAUNCH_CHECK();
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  c->have_eval = false;
  if (out) {
    out->sweeps = sweeps;
    out->err = err;
  }
  return OTB_OK;
}

// sinkhorn.py:54-58: gamma sweep (column log-sum-exp).
int sweep_gamma(otb_ctx* c, const double* logX, double* gamma, const double* zeta) {
  const int n = (int)c->n;
  const double mn = (double)c->m_loc * n;
  Geom geo = make_geom(c, DK_WARMG, c->C, logX);
  WarmGIO io{zeta, c->eta, c->colpart};
  cudaEvent_t e0 = nullptr;
  TRY(prof_begin(c, &e0));
  TRY(launch_dense(c, DK_WARMG, geo, &io));
  TRY(prof_end(c, PC_WARMG, e0, 16.0 * mn));
  if (c->nranks == 1) {
    k_warm_gamma_combine<<<c->col32, 256, 0, c->stream>>>(1, n, c->colpart, c->ncl, nullptr, nullptr, c->log_b,
                                                            c->eta, gamma);
    LAUNCH_CHECK();
  } else {
    k_warm_gamma_combine<<<c->col32, 256, 0, c->stream>>>(0, n, c->colpart, c->ncl, c->Mloc, c->Sloc, c->log_b,
                                                            c->eta, gamma);
    LAUNCH_CHECK();
    CUDA_TRY(cudaMemcpyAsync(c->Mglob, c->Mloc, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
    TRY(allreduce(c, c->Mglob, (size_t)n, kNcclMax));
    k_warm_rescale<<<c->colgrid, 256, 0, c->stream>>>(n, c->Mloc, c->Mglob, c->Sloc);
    LAUNCH_CHECK();
    TRY(allreduce(c, c->Sloc, (size_t)n, kNcclSum));
    k_warm_gamma_post<<<c->colgrid, 256, 0, c->stream>>>(n, c->Mglob, c->Sloc, c->log_b, c->eta, gamma);
    LAUNCH_CHECK();
  }
  return OTB_OK;
}

int otb_sinkhorn_zeta(otb_ctx* c, const double* logX, const double* gamma, double* zeta, double* col_err) {
  TRY(require_bound(c));
  if (!col_err) return fail(OTB_ERR_ARG, "null");
  TRY(sweep_zeta(c, logX, gamma, zeta, col_err));
  c->have_eval = false;
  return OTB_OK;
}

int otb_sinkhorn_gamma(otb_ctx* c, const double* logX, double* gamma, const double* zeta) {
  TRY(require_bound(c));
  TRY(sweep_gamma(c, logX, gamma, zeta));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  c->have_eval = false;
  return OTB_OK;
}

int otb_scaled_plan(otb_ctx* c, const double* logX, const double* gamma, const double* zeta, double* logX_out) {
  TRY(require_bound(c));
  CUDA_TRY(cudaMemsetAsync(&c->ds->cnt[CNT_SCALED], 0, sizeof(unsigned int), c->stream));
  k_scaled_plan<<<c->num_sms * 8, 256, 0, c->stream>>>(c->C, logX, c->ld, (int)c->m_loc, (int)c->n, zeta, gamma,
                                                       c->eta, logX_out, &c->ds->cnt[CNT_SCALED]);
  LAUNCH_CHECK();
  TRY(sync_scalars(c));
  if (c->hs->cnt[CNT_SCALED] != 0) return fail(OTB_ERR_BAD_LOGPLAN, "log plan contains NaN or +inf entries");
  return OTB_OK;
}

int otb_zeta_from_lse(otb_ctx* c, double* zeta) {
  TRY(require_bound(c));
  if (!c->have_eval) return fail(OTB_ERR_ARG, "no eval cached");
  k_zeta_from_lse<<<c->colgrid, 256, 0, c->stream>>>((int)c->m_loc, c->log_a, c->row0, c->lse, c->eta, zeta);
  LAUNCH_CHECK();
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return OTB_OK;
}

int otb_init_plan(otb_ctx* c, double* logX) {
  TRY(require_bound(c));
  k_init_plan<<<c->num_sms * 8, 256, 0, c->stream>>>(logX, c->ld, (int)c->m_loc, (int)c->n, c->log_a, c->row0,
                                                     c->log_b);
  LAUNCH_CHECK();
  return OTB_OK;
}

int otb_materialize_p(otb_ctx* c, const double* logX, const double* gamma, double* P, int64_t ldp) {
  TRY(require_bound(c));
  if (!c->have_eval) return fail(OTB_ERR_ARG, "no eval cached");
  k_materialize_p<<<c->num_sms * 8, 256, 0, c->stream>>>(c->C, logX, c->ld, (int)c->m_loc, (int)c->n, gamma, c->eta,
                                                         c->rowM, c->rowS, P, ldp);
  LAUNCH_CHECK();
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return OTB_OK;
}

int otb_info(otb_ctx* c, int64_t* o) {
  if (!c || !o) return fail(OTB_ERR_ARG, "null");
  const int64_t v[24] = {c->nt,     c->ns,  c->cl,  c->colw,  c->nstage[DK_EVAL], c->ncl,    c->grid,
                         c->hv_mode, c->hv_grid, c->nnz, c->cap, c->m_loc, c->n, c->ld, c->nranks, c->rank,
                         c->hv_ng,   c->cg_fused ? 1 : 0, (int64_t)c->hv_smem, c->launches,
                         c->rho_dense ? 1 : 0, c->hv_mode == 3 ? c->hv_var : c->ov_nq,
                         c->hv_mode == 3 ? c->hv_win : c->ov_win, c->hv_mode == 3 ? c->hv_nb : c->ov_ncl};
  std::memcpy(o, v, sizeof v);
  return OTB_OK;
}

int otb_selftest_div(const double* x, int64_t n, double y, double* out) {
  if ((!x || !out) && n > 0) return fail(OTB_ERR_ARG, "null");
  if (n <= 0) return OTB_OK;
  k_selftest_div<<<(int)std::min<int64_t>((n + 255) / 256, 4096), 256>>>(x, n, y, out);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaDeviceSynchronize());
  return OTB_OK;
}

int otb_cg_trace(otb_ctx* c, uint64_t* out, int64_t cap, int64_t* count) {
  if (!c || !count) return fail(OTB_ERR_ARG, "null");
  const int64_t cnt = c->cg_trace ? (int64_t)c->hv_grid * kCgTraceIters * 6 : 0;
  *count = cnt;
  if (cnt && out && cap >= cnt) {
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    CUDA_TRY(cudaMemcpy(out, c->cg_trace, (size_t)cnt * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  }
  return OTB_OK;
}

int otb_selftest_exp(const double* x, int64_t n, double* out) {
  if ((!x || !out) && n > 0) return fail(OTB_ERR_ARG, "null");
  if (n <= 0) return OTB_OK;
  k_selftest_exp<<<(int)std::min<int64_t>((n + 255) / 256, 4096), 256>>>(x, n, out);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaDeviceSynchronize());
  return OTB_OK;
}

int otb_selftest_tab(const double* x, int64_t n, double* out) {
  if ((!x || !out) && n > 0) return fail(OTB_ERR_ARG, "null");
  if (n <= 0) return OTB_OK;
  k_selftest_tab<<<(int)std::min<int64_t>((n + 255) / 256, 4096), 256>>>(x, n, out);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaDeviceSynchronize());
  return OTB_OK;
}

int otb_selftest_log(const double* x, int64_t n, double* out) {
  if ((!x || !out) && n > 0) return fail(OTB_ERR_ARG, "null");
  if (n <= 0) return OTB_OK;
  k_selftest_log<<<(int)std::min<int64_t>((n + 255) / 256, 4096), 256>>>(x, n, out);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaDeviceSynchronize());
  return OTB_OK;
}

int otb_sq_dist(const double* x, const double* y, int64_t m_loc, int64_t n, int dim, int64_t row0, double* C,
                int64_t ld, double* local_peak, void* stream) {
  if (!x || !y || !C || !local_peak || dim < 1 || m_loc < 0 || n < 1 || ld < n) return fail(OTB_ERR_ARG, "bad arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned long long* dpeak = nullptr;
  CUDA_TRY(cudaMallocAsync((void**)&dpeak, sizeof(unsigned long long), st));
  CUDA_TRY(cudaMemsetAsync(dpeak, 0, sizeof(unsigned long long), st));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (m_loc > 0) {
    k_sq_dist<<<sms * 8, 256, 0, st>>>(x, y, (int)m_loc, (int)n, dim, row0, C, ld, dpeak);
    CUDA_TRY(cudaGetLastError());
  }
  unsigned long long bits = 0;
  CUDA_TRY(cudaMemcpyAsync(&bits, dpeak, sizeof bits, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  cudaFreeAsync(dpeak, st);
  std::memcpy(local_peak, &bits, sizeof(double));
  return OTB_OK;
}

int otb_scale_cost(double* C, int64_t m_loc, int64_t n, int64_t ld, double peak, void* stream) {
  if (!C || ld < n) return fail(OTB_ERR_ARG, "bad arguments");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (m_loc > 0) {
    k_scale_cost<<<sms * 8, 256, 0, st>>>(C, ld, (int)m_loc, (int)n, peak);
    CUDA_TRY(cudaGetLastError());
  }
  CUDA_TRY(cudaStreamSynchronize(st));
  return OTB_OK;
}

// Counters of otb_check_clamp_plan: a ring of slots so that calls from
// several host threads / streams never share one (no allocation per call).
__device__ unsigned long long g_plan_bad[256];
static std::atomic<unsigned> g_plan_slot{0};

int otb_check_clamp_plan(double* X, int64_t m_loc, int64_t n, int64_t ld, double floor_v, void* stream,
                         int64_t* bad_out) {
  if (!X || !bad_out || ld < n || m_loc < 0 || n < 1) return fail(OTB_ERR_ARG, "bad arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  *bad_out = 0;
  if (m_loc == 0) return OTB_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  unsigned long long* slots = nullptr;
  CUDA_TRY(cudaGetSymbolAddress((void**)&slots, g_plan_bad));
  unsigned long long* dbad = slots + (g_plan_slot.fetch_add(1) & 255u);
  CUDA_TRY(cudaMemsetAsync(dbad, 0, sizeof(unsigned long long), st));
  k_check_clamp<<<sms * 8, 256, 0, st>>>(X, ld, (int)m_loc, (int)n, floor_v, dbad);
  CUDA_TRY(cudaGetLastError());
  unsigned long long hb = 0;
  CUDA_TRY(cudaMemcpyAsync(&hb, dbad, sizeof(hb), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  *bad_out = (int64_t)hb;
  return OTB_OK;
}


int otb_round_dense(const double* x, int64_t m, int64_t n, int64_t ldx, const double* a, const double* b, double* out,
                    int64_t ldo, double* deficit_out, void* stream) {
  if (!x || !a || !b || !out || m < 1 || n < 1 || ldx < n || ldo < n) return fail(OTB_ERR_ARG, "bad arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DapiScratch S{st, {}};
  double *z, *y, *er, *ec, *part, *def;
  TRY(S.get(&z, m));
  TRY(S.get(&y, n));
  TRY(S.get(&er, m));
  TRY(S.get(&ec, n));
  const dim3 cg = dapi_cols_grid(m, n);
  TRY(S.get(&part, (size_t)cg.y * n));
  TRY(S.get(&def, 1));
  const int rg = dapi_rows_grid(m), vg = (int)cdiv(n, kDapiThreads);
  k_dapi_rows<<<rg, kDapiThreads, 0, st>>>(x, ldx, (int)m, (int)n, nullptr, nullptr, a, 1, z);       // :56-58
  k_dapi_cols<<<cg, kDapiThreads, 0, st>>>(x, ldx, (int)m, (int)n, z, nullptr, part);                 // :60
  k_dapi_colfinish<<<vg, kDapiThreads, 0, st>>>(part, (int)cg.y, (int)n, b, 1, y);                   // :61-62
  k_dapi_rows<<<rg, kDapiThreads, 0, st>>>(x, ldx, (int)m, (int)n, z, y, a, 2, er);                   // :64
  k_dapi_cols<<<cg, kDapiThreads, 0, st>>>(x, ldx, (int)m, (int)n, z, y, part);
  k_dapi_colfinish<<<vg, kDapiThreads, 0, st>>>(part, (int)cg.y, (int)n, b, 2, ec);                  // :65
  k_dapi_vsum<<<1, kDapiThreads, 0, st>>>(er, (int)m, 0, def);                                         // :66
  k_dapi_round_out<<<148 * 8, 256, 0, st>>>(x, ldx, (int)m, (int)n, z, y, er, ec, def, out, ldo);     // :67-68
  CUDA_TRY(cudaGetLastError());
  double h = 0.0;
  CUDA_TRY(cudaMemcpyAsync(&h, def, sizeof h, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (deficit_out) *deficit_out = h;
  return OTB_OK;
}

int otb_bregman_dense(const double* x, int64_t ldx, const double* logy, int64_t ldy, int64_t m, int64_t n,
                      double* result, void* stream) {
  if (!x || !logy || !result || m < 1 || n < 1 || ldx < n || ldy < n) return fail(OTB_ERR_ARG, "bad arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DapiScratch S{st, {}};
  double *rows3, *tot;
  TRY(S.get(&rows3, 3 * (size_t)m));
  TRY(S.get(&tot, 3));
  k_dapi_bregman<<<dapi_rows_grid(m), kDapiThreads, 0, st>>>(x, ldx, logy, ldy, (int)m, (int)n, rows3);
  k_dapi_rowstats<<<1, 96, 0, st>>>(rows3, (int)m, 3, nullptr, tot);
  CUDA_TRY(cudaGetLastError());
  double h[3];
  CUDA_TRY(cudaMemcpyAsync(h, tot, sizeof h, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  *result = h[0] - h[1] + h[2];   // feasibility.py:85: terms.sum() - x.sum() + exp(log_y).sum()
  return OTB_OK;
}

int otb_kkt_dense(const double* x, int64_t ldx, const double* C, int64_t ldc, const double* gamma, const double* a,
                  const double* b, int64_t m, int64_t n, double* zeta_out, double* sums8, void* stream) {
  if (!x || !C || !gamma || !a || !b || !sums8 || m < 1 || n < 1 || ldx < n || ldc < n)
    return fail(OTB_ERR_ARG, "bad arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DapiScratch S{st, {}};
  double *zeta = zeta_out, *rows6, *tot, *part, *cs;
  if (!zeta) TRY(S.get(&zeta, m));
  TRY(S.get(&rows6, 6 * (size_t)m));
  TRY(S.get(&tot, 8));
  const dim3 cg = dapi_cols_grid(m, n);
  TRY(S.get(&part, (size_t)cg.y * n));
  TRY(S.get(&cs, n));
  k_dapi_kkt<<<dapi_rows_grid(m), kDapiThreads, 0, st>>>(x, ldx, C, ldc, gamma, (int)m, (int)n, zeta, rows6);
  k_dapi_rowstats<<<1, 224, 0, st>>>(rows6, (int)m, 6, a, tot);   // tot[0..5] sums, tot[6] = sum (rowsum - a)^2
  k_dapi_cols<<<cg, kDapiThreads, 0, st>>>(x, ldx, (int)m, (int)n, nullptr, nullptr, part);
  k_dapi_colfinish<<<(int)cdiv(n, kDapiThreads), kDapiThreads, 0, st>>>(part, (int)cg.y, (int)n, b, 0, cs);
  k_dapi_sqdiff<<<1, kDapiThreads, 0, st>>>(cs, b, (int)n, tot + 7);
  CUDA_TRY(cudaGetLastError());
  double h[8];
  CUDA_TRY(cudaMemcpyAsync(h, tot, sizeof h, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  // [row_res_sq, col_res_sq, neg_sq, x_sq, dslack_sq, comp, <C,x>, sum x]
  sums8[0] = h[6];
  sums8[1] = h[7];
  sums8[2] = h[1];
  sums8[3] = h[2];
  sums8[4] = h[3];
  sums8[5] = h[4];
  sums8[6] = h[5];
  sums8[7] = h[0];
  return OTB_OK;
}

int otb_hessian_dense(const double* P, int64_t ld, int64_t m, int64_t n, const double* a, const double* v, double eta,
                      double* out, void* stream) {
  if (!P || !a || !v || !out || m < 1 || n < 1 || ld < n || !(eta > 0.0)) return fail(OTB_ERR_ARG, "bad arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DapiScratch S{st, {}};
  double *w, *p0, *p1;
  TRY(S.get(&w, m));
  const dim3 cg = dapi_cols_grid(m, n);
  TRY(S.get(&p0, (size_t)cg.y * n));
  TRY(S.get(&p1, (size_t)cg.y * n));
  k_dapi_rowdot<<<dapi_rows_grid(m), kDapiThreads, 0, st>>>(P, ld, (int)m, (int)n, v, a, w);
  k_dapi_cols2<<<cg, kDapiThreads, 0, st>>>(P, ld, (int)m, (int)n, a, w, p0, p1);
  k_dapi_hv_out<<<(int)cdiv(n, kDapiThreads), kDapiThreads, 0, st>>>(p0, p1, (int)cg.y, (int)n, v, eta, out);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(st));
  return OTB_OK;
}

int otb_launch_count(otb_ctx* c, int64_t* out) {
  if (!c || !out) return fail(OTB_ERR_ARG, "null");
  *out = c->launches;
  return OTB_OK;
}

int otb_prof_enable(otb_ctx* c, int on) {
  if (!c) return fail(OTB_ERR_ARG, "null context");
  TRY(prof_collect(c));
  c->prof = on != 0;
  return OTB_OK;
}

int otb_prof_read(otb_ctx* c, double* ms16, int64_t* launches16, double* bytes16, int reset) {
  if (!c) return fail(OTB_ERR_ARG, "null context");
  TRY(prof_collect(c));
  for (int k = 0; k < PC_N; ++k) {
    if (ms16) ms16[k] = c->prof_ms[k];
    if (launches16) launches16[k] = c->prof_cnt[k];
    if (bytes16) bytes16[k] = c->prof_bytes[k];
  }
  if (reset) {
    std::fill(c->prof_ms, c->prof_ms + PC_N, 0.0);
    std::fill(c->prof_bytes, c->prof_bytes + PC_N, 0.0);
    std::fill(c->prof_cnt, c->prof_cnt + PC_N, (int64_t)0);
  }
  return OTB_OK;
}

}  // extern "C"
