// Probe: achievable HBM read bandwidth of a bulk-copy (TMA) fed smem ring on
// B200, vs tile size / stages / CTAs per SM, and of plain vectorised loads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tma_bw.cu -o tma_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2412_04964_b200/csrc/fc_tma.cuh"
using namespace fc;

__global__ void k_tma(const uint8_t* src, size_t bytes, int tile, int S, uint32_t* sink) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t sb = smem_u32(smem), full0 = sb + S * tile, empty0 = full0 + 8 * S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x / 32 - 1;
  const int items = (int)(bytes / tile), per = (items + gridDim.x - 1) / gridDim.x;
  const int b = min(items, (int)blockIdx.x * per), e = min(items, b + per);
  if (threadIdx.x == 0) { for (int s = 0; s < S; ++s) { mbar_init(full0 + 8 * s, 1); mbar_init(empty0 + 8 * s, nwarps); } fence_mbar_init(); }
  __syncthreads();
  if (warp == nwarps) {
    if (lane == 0) {
      int st = 0; uint32_t ph = 0;
      for (int i = b; i < e; ++i) {
        if (i - b >= S) mbar_wait(empty0 + 8 * st, ph ^ 1);
        mbar_arrive_expect_tx(full0 + 8 * st, tile);
        bulk_g2s(sb + st * tile, src + (size_t)i * tile, tile, full0 + 8 * st);
        if (++st == S) { st = 0; ph ^= 1; }
      }
    }
    return;
  }
  uint32_t acc = 0; int st = 0; uint32_t ph = 0;
  for (int i = b; i < e; ++i) {
    mbar_wait(full0 + 8 * st, ph);
    for (int o = threadIdx.x * 16; o < tile; o += nwarps * 32 * 16) { uint4 v = lds128_(sb + st * tile + o); acc ^= v.x ^ v.w; }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * st);
    if (++st == S) { st = 0; ph ^= 1; }
  }
  if (acc == 0x12345678) sink[0] = acc;
}

__global__ void k_ldg(const uint4* src, size_t n16, uint32_t* sink) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldg(src + i); acc ^= v.x ^ v.w;
  }
  if (acc == 0x12345678) sink[0] = acc;
}
__global__ void k_copy(const uint4* src, uint4* dst, size_t n16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) dst[i] = __ldg(src + i);
}

// write probes: plain 16-B stores vs bulk (TMA) shared->global stores of whole tiles
__global__ void k_stg(uint4* dst, size_t n16) {
  const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) dst[i] = v;
}
__global__ void k_bulk_store(uint8_t* dst, size_t bytes, int tile, int depth) {
  extern __shared__ __align__(128) uint8_t smem[];
  for (int i = threadIdx.x * 16; i < tile; i += blockDim.x * 16) *reinterpret_cast<uint4*>(smem + i) = make_uint4(i, 1, 2, 3);
  fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int items = (int)(bytes / tile);
  int n = 0;
  for (int i = blockIdx.x; i < items; i += gridDim.x) {
    bulk_s2g(dst + (size_t)i * tile, smem_u32(smem), tile);
    bulk_commit();
    if (++n >= depth) bulk_wait_read<4>();
  }
  bulk_wait<0>();
}

int main() {
  const size_t bytes = 1ull << 30;
  uint8_t *src, *dst; uint32_t* sink;
  cudaMalloc(&src, bytes); cudaMalloc(&dst, bytes); cudaMalloc(&sink, 4);
  cudaMemset(src, 1, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, z; cudaEventCreate(&a); cudaEventCreate(&z);
  auto timeit = [&](auto fn) { fn(); cudaEventRecord(a); for (int r = 0; r < 10; ++r) fn(); cudaEventRecord(z); cudaEventSynchronize(z); float ms; cudaEventElapsedTime(&ms, a, z); return ms / 10; };
  cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int tile : {4096, 8192, 16384, 32768}) for (int S : {2, 4, 6, 8}) for (int threads : {288, 160}) {
    const int smem = S * tile + 16 * S; if (smem > 220 * 1024) continue;
    int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tma, threads, smem);
    for (int cps : {1, 2, 4}) {
      if (cps > occ) continue;
      float ms = timeit([&] { k_tma<<<sms * cps, threads, smem>>>(src, bytes, tile, S, sink); });
      printf("{\"probe\":\"tma_read\",\"tile\":%d,\"stages\":%d,\"threads\":%d,\"ctas_per_sm\":%d,\"GBs\":%.0f}\n", tile, S, threads, cps, bytes / ms / 1e6);
    }
  }
  for (int bl : {1, 2, 4, 8}) {
    float ms = timeit([&] { k_ldg<<<sms * bl * 2, 1024>>>((const uint4*)src, bytes / 16, sink); });
    printf("{\"probe\":\"ldg_read\",\"blocks_per_sm\":%d,\"GBs\":%.0f}\n", bl * 2, bytes / ms / 1e6);
  }
  float ms = timeit([&] { k_copy<<<sms * 4, 1024>>>((const uint4*)src, (uint4*)dst, bytes / 16); });
  printf("{\"probe\":\"copy\",\"GBs\":%.0f}\n", 2.0 * bytes / ms / 1e6);
  for (int bl : {1, 2, 4, 8}) {
    float w = timeit([&] { k_stg<<<sms * bl, 1024>>>((uint4*)dst, bytes / 16); });
    printf("{\"probe\":\"stg_write\",\"blocks_per_sm\":%d,\"GBs\":%.0f}\n", bl, bytes / w / 1e6);
  }
  cudaFuncSetAttribute(k_bulk_store, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int tile : {4096, 16384, 32768}) for (int cps : {1, 2, 4, 8}) {
    float w = timeit([&] { k_bulk_store<<<sms * cps, 128, tile>>>(dst, bytes, tile, 8); });
    printf("{\"probe\":\"bulk_write\",\"tile\":%d,\"ctas_per_sm\":%d,\"GBs\":%.0f}\n", tile, cps, bytes / w / 1e6);
  }
  printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
