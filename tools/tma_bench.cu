// Stand-alone probe: streaming read bandwidth of (a) 1-D TMA bulk copies
// through a shared-memory ring (one producer lane, consumers release), and
// (b) plain 16-byte vector loads, on this B200.  Debug tool for the
// dense/CSR streaming design (profiles/ notes).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2603_07156_b200/csrc/common.cuh"
using namespace otb;

__global__ void k_tma(const double* src, size_t per_cta_bytes, int stage_bytes, int S, double* sink, int spin,
                      int chunks = 1) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)S * stage_bytes);
  uint64_t* empty = full + S;
  const int nt = blockDim.x - 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], nt / 32); }
    fence_mbar_init();
  }
  __syncthreads();
  const char* base = reinterpret_cast<const char*>(src) + (size_t)blockIdx.x * per_cta_bytes;
  const int nseg = (int)(per_cta_bytes / stage_bytes);
  double acc = 0.0;
  if (threadIdx.x >= nt) {
    if ((threadIdx.x & 31) == 0) {
      int st = 0; uint32_t ph = 0;
      for (int k = 0; k < nseg; ++k) {
        mbar_wait(&empty[st], ph ^ 1u);
        mbar_arrive_expect_tx(&full[st], stage_bytes);
        const int cb = stage_bytes / chunks;
        for (int q = 0; q < chunks; ++q)
          bulk_g2s(sm + (size_t)st * stage_bytes + (size_t)q * cb, base + (size_t)k * stage_bytes + (size_t)q * cb, cb,
                   &full[st]);
        if (++st == S) { st = 0; ph ^= 1u; }
      }
    }
  } else {
    int st = 0; uint32_t ph = 0;
    for (int k = 0; k < nseg; ++k) {
      mbar_wait(&full[st], ph);
      const double* buf = reinterpret_cast<const double*>(sm + (size_t)st * stage_bytes);
      for (int i = 0; i < spin; ++i) acc += buf[(threadIdx.x + i * nt) % (stage_bytes / 8)];
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[st]);
      if (++st == S) { st = 0; ph ^= 1u; }
    }
  }
  if (acc == 12345.678) sink[0] = acc;
}

__global__ void k_ldg(const double2* src, size_t n2, double* sink) {
  double acc = 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldg(src + i);
    acc += v.x + v.y;
  }
  if (acc == 12345.678) sink[0] = acc;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t total = (size_t)1 << 31;    // 2 GiB
  double* src; cudaMalloc(&src, total); cudaMemset(src, 0, total);
  double* sink; cudaMalloc(&sink, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (int blocks_per_sm = 1; blocks_per_sm <= 2; ++blocks_per_sm)
  for (int stage_kb : {8, 16, 32}) for (int S : {2, 4, 8, 12}) {
    const int stage = stage_kb * 1024;
    const size_t smem = (size_t)S * stage + 2 * S * 8;
    if (smem * blocks_per_sm > 227 * 1024) continue;
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = sms * blocks_per_sm;
    const size_t per = (total / grid) / stage * stage;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      k_tma<<<grid, 512 + 32, smem>>>(src, per, stage, S, sink, 0);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1);
    printf("TMA  cta/sm=%d stage=%2dKB S=%2d inflight=%3dKB/SM : %7.0f GB/s  err=%s\n", blocks_per_sm, stage_kb, S,
           stage_kb * S * blocks_per_sm, per * grid / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  // large stages (one row window per stage, as the window-cluster hess_apply), 1 or several copies each
  for (int grid_sms : {135, 148})
  for (int stage_kb : {48, 64}) for (int S : {2, 3, 4}) for (int chunks : {1, 4, 12}) {
    const int stage = stage_kb * 1024;
    const size_t smem = (size_t)S * stage + 2 * S * 8;
    if (smem > 227 * 1024) continue;
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = grid_sms;
    const size_t per = (total / grid) / stage * stage;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      k_tma<<<grid, 512 + 32, smem>>>(src, per, stage, S, sink, 0, chunks);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1);
    printf("TMA  ctas=%d stage=%2dKB S=%d copies/stage=%2d : %7.0f GB/s  err=%s\n", grid, stage_kb, S, chunks,
           per * grid / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  for (int bpsm : {1, 2, 4, 8}) for (int th : {256, 512, 1024}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      k_ldg<<<sms * bpsm, th>>>(reinterpret_cast<const double2*>(src), total / 16, sink);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1);
    printf("LDG  blocks/sm=%d threads=%4d : %7.0f GB/s\n", bpsm, th, total / (ms * 1e-3) / 1e9);
  }
  return 0;
}
