// Flash All-Reduce device code (Alg. 1 of arXiv 2412.04964; reference
// collectives.py:321-402), B200 form.
//
// Per rank r and round (a sub-range [sub_off, sub_off+sub_len) of every rank
// segment; rounds are result-transparent, collectives.py:14-16):
//   scatter(r->j, t): quantize tile t of r's segment j with stage 1 and store
//                     it straight into rank j's receive slot [r] (NVLink P2P /
//                     IPC-mapped stores), then raise rflag[j][r][t].
//   reduce(j, t):     wait rflag[j][*][t]; dequantize the N-1 peer tiles and
//                     QDQ the own tile in registers; fp32 sum in ascending
//                     source rank (collectives.py:182-187); stage-2 quantize;
//                     store to every peer's gather slot [j]; decode the own
//                     output; raise gflag[p][j][t].
//   gather(r, j, t):  wait gflag[r][j][t]; decode into out[j*seg + ...].
// Own pieces never touch HBM as codes (collectives.py:364-365,378 are done in
// registers).
#pragma once

#include <cooperative_groups.h>

#include "fc_codec_dev.cuh"
#include "fc_lane.cuh"
#include "fc_stage.cuh"

namespace fc {

struct FlashArgs {
  int world;
  int rank_lo, rank_hi;     // ranks handled by this launch
  int ctas_per_rank;        // fused kernel
  int lag;                  // fused schedule lag (steps)
  int tiles;                // ceil(sub_len / kTileElems)
  uint32_t epoch;           // host epoch of this round (used when epoch_dev is null)
  const uint32_t* epoch_dev;  // device epoch counter of the launching rank (CUDA-graph safe), bumped per round
  int64_t M;                // elements per rank (unpadded)
  int64_t seg;              // ceil(M / world)
  int64_t sub_off, sub_len; // this round's sub-range of every segment
  int64_t slot_bytes;
  int64_t flags_cap;
  uint64_t timeout_ns;
  int stages;               // cp.async ring depth of the phase-split kernels
  int stage_hint;           // host-side override of the reduce ring depth (0 = auto)
  int q_hint, d_hint;       // ring depths of the streaming scatter / gather kernels (0 = auto)
  int cta_cap;              // resident CTAs per SM cap for the streaming kernels (0 = occupancy)
  int fp_chunk;             // fused stream kernel: tiles per schedule chunk
  int fp_dctas;             // fused stream kernel: CTAs [0, fp_dctas) run the gather role
  uint64_t* tprof;          // fused stream kernel: per-CTA role timeline (measurement; null = off)
  int fp_bars;              // fused stream kernel: byte offset of the barrier region in shared memory
  int fp_meta;              // fused stream kernel: byte offset of the DynIter id ring in shared memory
  int q_stages_f, d_stages_f;  // fused stream kernel ring depths of the scatter / gather roles
  int r_ring_f;             // fused stream kernel: piece-slot ring depth of the reduce role
  int ownq;                 // 1: the scatter also stage-1 quantizes the own piece into recv_slot[r][r]
                            // (the group-lane reduce reads every source from the slots)
  int sys_scope;            // flags cross GPUs: system-scope fences; else gpu scope (one GPU)
  int dbg;                  // FC_OPT_STREAM_MASK A/B bits (include/flashcomm.h)
  DevCodec c1, c2;
  int mode;                 // 0: flash all-reduce; 1: single-GPU codec job (in[0] -> out[0], c1)
  uint32_t* cerr;           // mode 1: error word
  const void* in[kMaxRanks];
  void* out[kMaxRanks];
  uint8_t* blk[kMaxRanks];  // every rank's block, addressable from the launching device
};

// block layout (host mirror in fc_api.cu)
__host__ __device__ inline int64_t blk_flags_off(int world, int64_t slot_bytes) { return 2 * (int64_t)world * slot_bytes; }
__host__ __device__ inline int64_t blk_misc_off(int world, int64_t slot_bytes, int64_t flags_cap) {
  return blk_flags_off(world, slot_bytes) + 2 * (int64_t)world * flags_cap * 4;
}
// err word @0, barrier flags @64: [2][kMaxRanks] u32; fused-kernel work counters @512:
// [3 roles][kFusedMaxChunks] u32 + one launch-done counter
constexpr int kFusedMaxChunks = 1024;
constexpr int64_t kMiscBytes = 512 + (3 * kFusedMaxChunks + 32) * 4;

__device__ __forceinline__ uint8_t* recv_slot(const FlashArgs& a, int owner, int src) {
  return a.blk[owner] + (int64_t)src * a.slot_bytes;
}
__device__ __forceinline__ uint8_t* gath_slot(const FlashArgs& a, int owner, int src) {
  return a.blk[owner] + (int64_t)(a.world + src) * a.slot_bytes;
}
__device__ __forceinline__ uint32_t* rflag(const FlashArgs& a, int owner, int src) {
  return reinterpret_cast<uint32_t*>(a.blk[owner] + blk_flags_off(a.world, a.slot_bytes)) + (int64_t)src * a.flags_cap;
}
__device__ __forceinline__ uint32_t* gflag(const FlashArgs& a, int owner, int src) {
  return reinterpret_cast<uint32_t*>(a.blk[owner] + blk_flags_off(a.world, a.slot_bytes)) +
         (int64_t)(a.world + src) * a.flags_cap;
}
__device__ __forceinline__ uint32_t* errw(const FlashArgs& a, int owner) {
  return reinterpret_cast<uint32_t*>(a.blk[owner] + blk_misc_off(a.world, a.slot_bytes, a.flags_cap));
}
__device__ __forceinline__ uint32_t* fctr(const FlashArgs& a, int owner) { return errw(a, owner) + 128; }

// a wait of `rank` on `peer` timed out: latch the ProtocolError in the rank's own error word
// and propagate the same word into every other rank's (peer memory, system scope), so their
// waits give up at once instead of each running into its own timeout -- the reference's
// fabric abort (fabric.py:140, 168-172, 203-205); every rank then reports the originator
static __device__ __noinline__ void raise_timeout(const FlashArgs& a, int rank, int peer, uint32_t phase) {
  const uint32_t w = make_err(kErrTimeout, phase, peer, rank);
  atomicCAS(errw(a, rank), 0u, w);
  for (int p = 0; p < a.world; ++p)
    if (p != rank && a.blk[p]) atomicCAS_system(errw(a, p), 0u, w);
  __threadfence_system();
}
__device__ __forceinline__ uint32_t* barflag(const FlashArgs& a, int owner, int phase, int src) {
  return errw(a, owner) + 16 + phase * kMaxRanks + src;
}

// epoch of this round: read from the device counter (bumped by k_epoch_bump
// earlier on the same stream, so every CTA of the launch reads the same value
// and a replayed CUDA graph advances it) or the host value
__device__ __forceinline__ uint32_t flag_epoch(const FlashArgs& a) {
  return a.epoch_dev ? *reinterpret_cast<const volatile uint32_t*>(a.epoch_dev) : a.epoch;
}

static __global__ void k_epoch_bump(uint32_t* e) { *e += 1u; }

enum Phase : uint32_t { kPhScatter = 1, kPhReduce = 2, kPhGather = 3, kPhBarrier = 4 };

// ---------------------------------------------------------------- work items

template <typename Tin, int CW, class S1>
__device__ __forceinline__ void do_scatter(const FlashArgs& a, int r, int j, int t) {
  const int lane = threadIdx.x & 31;
  const int64_t p0 = (int64_t)t * kTileElems + (int64_t)threadIdx.x * kLaneElems;
  const int nvalid = (int)max((int64_t)0, min(a.sub_len - p0, (int64_t)kLaneElems));
  LaneOf<Tin> v;
  load_lane_src(reinterpret_cast<const Tin*>(a.in[r]), (int64_t)j * a.seg + a.sub_off + p0, a.M, nvalid, v);
  LaneQuant<CW> q;
  const bool bad = quantize_lane<S1>(a.c1, v, nvalid, q);
  store_lane(a.c1, recv_slot(a, j, r), p0, nvalid, q, lane);
  if (bad) atomicOr(errw(a, r), make_err(kErrNonFinite, kPhScatter, j, r));
}

template <typename Tin, typename Tout, int CW, class S1, class S2>
__device__ __forceinline__ void do_reduce(const FlashArgs& a, int j, int t) {
  const int lane = threadIdx.x & 31;
  const int64_t p0 = (int64_t)t * kTileElems + (int64_t)threadIdx.x * kLaneElems;
  const int nvalid = (int)max((int64_t)0, min(a.sub_len - p0, (int64_t)kLaneElems));
  const int64_t idx0 = (int64_t)j * a.seg + a.sub_off + p0;
  bool bad = false;
  FloatLane acc;
  for (int s = 0; s < a.world; ++s) {
    LaneCodes<CW> L;
    if (s == j) {
      LaneOf<Tin> v;
      load_lane_src(reinterpret_cast<const Tin*>(a.in[j]), idx0, a.M, nvalid, v);
      LaneQuant<CW> q;
      bad |= quantize_lane<S1>(a.c1, v, nvalid, q);  // own piece: QDQ in registers (collectives.py:364-365)
      lane_codes_from(a.c1, q, L);
    } else if (nvalid > 0) {
      load_lane(a.c1, recv_slot(a, j, s), p0, L);
    } else {
#pragma unroll
      for (int i = 0; i < CW; ++i) L.w[i] = 0;
      L.s = 0.0f;
      L.mz = 0.0f;
    }
    if (s == 0)
      decode_lane<S1, false>(a.c1, L, acc.v);  // ascending source rank (collectives.py:182-187)
    else
      decode_lane<S1, true>(a.c1, L, acc.v);
  }
  LaneQuant<CW> q2;
  bad |= quantize_lane<S2>(a.c2, acc, nvalid, q2);
  for (int pp = 1; pp < a.world; ++pp) {
    const int p = (j + pp) % a.world;
    store_lane(a.c2, gath_slot(a, p, j), p0, nvalid, q2, lane);
  }
  LaneCodes<CW> L2;
  lane_codes_from(a.c2, q2, L2);
  float o[kLaneElems];
  decode_lane<S2, false>(a.c2, L2, o);  // owner decodes its own payload too (collectives.py:378)
  if (nvalid > 0) store_chunk(reinterpret_cast<Tout*>(a.out[j]), idx0, a.M, nvalid, o);
  if (bad) atomicOr(errw(a, j), make_err(kErrNonFinite, kPhReduce, j, j));
}

template <typename Tout, int CW, class S2>
__device__ __forceinline__ void do_gather(const FlashArgs& a, int r, int j, int t) {
  const int64_t p0 = (int64_t)t * kTileElems + (int64_t)threadIdx.x * kLaneElems;
  const int nvalid = (int)max((int64_t)0, min(a.sub_len - p0, (int64_t)kLaneElems));
  if (nvalid <= 0) return;
  LaneCodes<CW> L;
  load_lane(a.c2, gath_slot(a, r, j), p0, L);
  float o[kLaneElems];
  decode_lane<S2, false>(a.c2, L, o);
  store_chunk(reinterpret_cast<Tout*>(a.out[r]), (int64_t)j * a.seg + a.sub_off + p0, a.M, nvalid, o);
}

// ---------------------------------------------------------------- flags

// Threads [0, nflags) each wait for one flag to reach the epoch. Returns true
// if the CTA must abort (timeout here -> error word; or an error elsewhere).
__device__ __forceinline__ bool wait_flags(const FlashArgs& a, int rank, uint32_t* const* flags, const int* peers,
                                           int nflags, uint32_t phase, int* s_abort) {
  if ((int)threadIdx.x < nflags) {
    const uint32_t* f = flags[threadIdx.x];
    const uint32_t ep = flag_epoch(a);
    const uint64_t t0 = globaltimer();
    volatile uint32_t* ew = errw(a, rank);
    uint32_t spins = 0;
    while ((int32_t)(ld_acquire_sys(f) - ep) < 0) {
      if ((*ew >> 28) == kErrTimeout) {  // another CTA of this rank gave up
        *s_abort = 1;
        break;
      }
      if ((++spins & 63u) == 0 && globaltimer() - t0 > a.timeout_ns) {
        raise_timeout(a, rank, peers[threadIdx.x], phase);
        *s_abort = 1;
        break;
      }
      __nanosleep(32);
    }
  }
  __syncthreads();
  return *s_abort != 0;
}

// All threads' prior stores (incl. to peer memory) are published before the
// flag: bar.sync orders them before thread 0's system-scope fence.
__device__ __forceinline__ void raise_flags(uint32_t* const* flags, int nflags, uint32_t epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int i = 0; i < nflags; ++i) st_relaxed_sys(flags[i], epoch);
  }
}

// ---------------------------------------------------------------- kernels

// One persistent kernel per rank (or all ranks of one GPU in one grid):
// item i -> CTA i % ctas_per_rank, items in increasing order. Schedule step k
// holds P scatter items for tile k, the reduce of tile k-lag and P gathers of
// tile k-2*lag. Every wait targets an item of a strictly earlier position, so
// with all CTAs resident the schedule cannot deadlock.
template <typename Tin, typename Tout, int CW, class S1, class S2>
__global__ void __launch_bounds__(kThreads, 2) k_flash_fused(FlashArgs a) {
  __shared__ int s_abort;
  __shared__ uint32_t* s_flags[kMaxRanks];
  __shared__ int s_peers[kMaxRanks];
  const int rank = a.rank_lo + (int)(blockIdx.x / a.ctas_per_rank);
  const int cta = (int)(blockIdx.x % a.ctas_per_rank);
  const int P = a.world - 1;
  const int per_step = 2 * P + 1;
  const int64_t total = (int64_t)(a.tiles + 2 * a.lag) * per_step;
  if (threadIdx.x == 0) s_abort = 0;
  __syncthreads();
  for (int64_t i = cta; i < total; i += a.ctas_per_rank) {
    const int64_t k = i / per_step;
    const int slot = (int)(i % per_step);
    if (slot < P) {
      const int64_t t = k;
      if (t >= a.tiles) continue;
      const int j = (rank + 1 + slot) % a.world;
      do_scatter<Tin, CW, S1>(a, rank, j, (int)t);
      if (threadIdx.x == 0) s_flags[0] = rflag(a, j, rank) + t;
      raise_flags(s_flags, 1, flag_epoch(a));
    } else if (slot == P) {
      const int64_t t = k - a.lag;
      if (t < 0 || t >= a.tiles) continue;
      if (threadIdx.x < P) {
        const int s = (rank + 1 + threadIdx.x) % a.world;
        s_flags[threadIdx.x] = rflag(a, rank, s) + t;
        s_peers[threadIdx.x] = s;
      }
      __syncthreads();
      if (wait_flags(a, rank, s_flags, s_peers, P, kPhReduce, &s_abort)) return;
      __syncthreads();
      do_reduce<Tin, Tout, CW, S1, S2>(a, rank, (int)t);
      __syncthreads();
      if (threadIdx.x < P) s_flags[threadIdx.x] = gflag(a, (rank + 1 + threadIdx.x) % a.world, rank) + t;
      raise_flags(s_flags, P, flag_epoch(a));
    } else {
      const int64_t t = k - 2 * a.lag;
      if (t < 0 || t >= a.tiles) continue;
      const int j = (rank + 1 + (slot - P - 1)) % a.world;
      if (threadIdx.x == 0) {
        s_flags[0] = gflag(a, rank, j) + t;
        s_peers[0] = j;
      }
      __syncthreads();
      if (wait_flags(a, rank, s_flags, s_peers, 1, kPhGather, &s_abort)) return;
      do_gather<Tout, CW, S2>(a, rank, j, (int)t);
    }
    __syncthreads();
  }
}

// Phase-split kernels (no flags): ordering comes from kernel boundaries
// (one GPU), stream events (several GPUs, one process) or k_barrier (IPC).
// Grids are 2-D: blockIdx.y names the (rank, peer) pair or the owning rank,
// blockIdx.x strides over tiles, so no item index is ever divided. Each
// thread streams its operands through a cp.async ring of a.stages tiles
// (fc_stage.cuh), keeping that many tiles of HBM traffic in flight.

// blockIdx.y -> (r, j) with j = r+1+jj (mod world), for ranks [rank_lo, rank_hi)
__device__ __forceinline__ void pair_of(const FlashArgs& a, int y, int& r, int& j) {
  const int P = a.world - 1;
  r = a.rank_lo + y / P;
  j = r + 1 + y % P;
  if (j >= a.world) j -= a.world;
}

// scatter job y -> (rank r, destination j): with ownq every rank has world jobs,
// the last one its own piece (j == r), else world - 1 (peers only)
__device__ __forceinline__ void qpair_of(const FlashArgs& a, int y, int& r, int& j) {
  const int P = a.world - 1 + a.ownq;
  r = a.rank_lo + y / P;
  j = r + 1 + y % P;
  if (j >= a.world) j -= a.world;
}
__device__ __forceinline__ int q_jobs(const FlashArgs& a) { return (a.rank_hi - a.rank_lo) * (a.world - 1 + a.ownq); }

__device__ __forceinline__ int lane_valid(int64_t len, int64_t p0) {
  const int64_t d = len - p0;
  return d <= 0 ? 0 : (d >= kLaneElems ? kLaneElems : (int)d);
}

// Small messages on one GPU (decode regime, C4): the three phases in one
// cooperative launch separated by grid-wide barriers, every item a direct
// (register) lane codec call — no staging rings, no per-tile flags, one launch
// instead of three.
template <typename Tin, typename Tout, int CW, class S1, class S2>
__global__ void __launch_bounds__(kThreads) k_oneshot(FlashArgs a) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int P = a.world - 1, nr = a.rank_hi - a.rank_lo;
  for (int i = blockIdx.x; i < nr * P * a.tiles; i += gridDim.x) {
    const int y = i / a.tiles, t = i - y * a.tiles;
    int r, j;
    pair_of(a, y, r, j);
    do_scatter<Tin, CW, S1>(a, r, j, t);
  }
  grid.sync();
  for (int i = blockIdx.x; i < nr * a.tiles; i += gridDim.x) {
    const int y = i / a.tiles, t = i - y * a.tiles;
    do_reduce<Tin, Tout, CW, S1, S2>(a, a.rank_lo + y, t);
  }
  grid.sync();
  for (int i = blockIdx.x; i < nr * P * a.tiles; i += gridDim.x) {
    const int y = i / a.tiles, t = i - y * a.tiles;
    int r, j;
    pair_of(a, y, r, j);
    do_gather<Tout, CW, S2>(a, r, j, t);
  }
}


template <typename Tin, int CW, class S1>
__global__ void __launch_bounds__(kThreads) k_scatter(FlashArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int CB = Chunk<Tin>::kBytes;
  const int lane = threadIdx.x & 31;
  const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(smem) + threadIdx.x * CB;
  const int S = a.stages;
  int r, j;
  pair_of(a, blockIdx.y, r, j);
  const Tin* src = reinterpret_cast<const Tin*>(a.in[r]) + (int64_t)j * a.seg + a.sub_off;
  const int64_t Mrel = a.M - ((int64_t)j * a.seg + a.sub_off);  // elements of `src` before the padding
  uint8_t* dst = recv_slot(a, j, r);
  const int tx = threadIdx.x * kLaneElems;
  auto issue = [&](int t, int st) {
    if (t < a.tiles) {
      const int64_t p0 = (int64_t)t * kTileElems + tx;
      chunk_issue<Tin>(s0 + st * kThreads * CB, src, p0, Mrel, lane_valid(a.sub_len, p0), lane);
    }
    cp_async_commit();
  };
  for (int k = 0; k < S - 1; ++k) issue(blockIdx.x + k * gridDim.x, k);
  int st = 0;
  bool bad = false;
  for (int t = blockIdx.x; t < a.tiles; t += gridDim.x) {
    issue(t + (S - 1) * gridDim.x, st == 0 ? S - 1 : st - 1);
    cp_async_wait_dyn(S - 1);
    const int64_t p0 = (int64_t)t * kTileElems + tx;
    const int nvalid = lane_valid(a.sub_len, p0);
    LaneOf<Tin> v;
    chunk_read_src<Tin>(s0 + st * kThreads * CB, lane, v);
    LaneQuant<CW> q;
    bad |= quantize_lane<S1>(a.c1, v, nvalid, q);
    store_lane(a.c1, dst, p0, nvalid, q, lane);
    st = (st + 1 == S) ? 0 : st + 1;
  }
  if (bad) atomicOr(errw(a, r), make_err(kErrNonFinite, kPhScatter, j, r));
}

// bytes of one thread's reduce stage: own input chunk + (world-1) code chunks
template <typename Tin>
__host__ __device__ inline int reduce_thread_bytes(const DevCodec& c1, int world) {
  return Chunk<Tin>::kBytes + (world - 1) * code_chunk_bytes(c1);
}

template <typename Tin, typename Tout, int CW, class S1, class S2>
__global__ void __launch_bounds__(kThreads) k_reduce(FlashArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  const int TB = reduce_thread_bytes<Tin>(a.c1, a.world);
  const int CCB = code_chunk_bytes(a.c1);
  const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(smem) + threadIdx.x * TB;
  const int S = a.stages;
  const int j = a.rank_lo + blockIdx.y;  // owner of the segment
  const int64_t seg0 = (int64_t)j * a.seg + a.sub_off;
  const Tin* own = reinterpret_cast<const Tin*>(a.in[j]) + seg0;
  const int64_t Mrel = a.M - seg0;
  const int tx = threadIdx.x * kLaneElems;
  auto issue = [&](int t, int st) {
    if (t < a.tiles) {
      const int64_t p0 = (int64_t)t * kTileElems + tx;
      const int nvalid = lane_valid(a.sub_len, p0);
      const uint32_t base = s0 + st * kThreads * TB;
      chunk_issue<Tin>(base, own, p0, Mrel, nvalid, lane);
      if (nvalid > 0) {
        uint32_t off = base + Chunk<Tin>::kBytes;
        for (int s = 0; s < a.world; ++s) {
          if (s == j) continue;
          code_issue(a.c1, off, recv_slot(a, j, s), p0);
          off += CCB;
        }
      }
    }
    cp_async_commit();
  };
  for (int k = 0; k < S - 1; ++k) issue(blockIdx.x + k * gridDim.x, k);
  int st = 0;
  bool bad = false;
  for (int t = blockIdx.x; t < a.tiles; t += gridDim.x) {
    issue(t + (S - 1) * gridDim.x, st == 0 ? S - 1 : st - 1);
    cp_async_wait_dyn(S - 1);
    const int64_t p0 = (int64_t)t * kTileElems + tx;
    const int nvalid = lane_valid(a.sub_len, p0);
    const uint32_t base = s0 + st * kThreads * TB;
    // own piece: stage-1 QDQ in registers (collectives.py:364-365)
    FloatLane mine;
    {
      LaneOf<Tin> v;
      chunk_read_src<Tin>(base, lane, v);
      LaneQuant<CW> q;
      bad |= quantize_lane<S1>(a.c1, v, nvalid, q);
      LaneCodes<CW> L;
      lane_codes_from(a.c1, q, L);
      decode_lane<S1, false>(a.c1, L, mine.v);
    }
    // fp32 sum in ascending source rank (collectives.py:182-187)
    FloatLane acc;
    if (j == 0) {
#pragma unroll
      for (int k = 0; k < kLaneElems; ++k) acc.v[k] = mine.v[k];
    }
    uint32_t off = base + Chunk<Tin>::kBytes;
    for (int s = 0; s < a.world; ++s) {
      if (s == j) {
        if (s != 0) {
#pragma unroll
          for (int k = 0; k < kLaneElems; ++k) acc.v[k] += mine.v[k];
        }
        continue;
      }
      LaneCodes<CW> L;
      if (nvalid > 0) {
        code_read(a.c1, off, p0, L);
      } else {
#pragma unroll
        for (int w = 0; w < CW; ++w) L.w[w] = 0;
        L.s = 0.0f;
        L.mz = 0.0f;
      }
      off += CCB;
      if (s == 0)
        decode_lane<S1, false>(a.c1, L, acc.v);
      else
        decode_lane<S1, true>(a.c1, L, acc.v);
    }
    LaneQuant<CW> q2;
    bad |= quantize_lane<S2>(a.c2, acc, nvalid, q2);
    for (int p = j + 1;; ++p) {  // every peer's gather slot [j]
      if (p == a.world) p = 0;
      if (p == j) break;
      store_lane(a.c2, gath_slot(a, p, j), p0, nvalid, q2, lane);
    }
    LaneCodes<CW> L2;
    lane_codes_from(a.c2, q2, L2);
    float o[kLaneElems];
    decode_lane<S2, false>(a.c2, L2, o);  // owner decodes its own payload too (collectives.py:378)
    if (nvalid > 0) store_chunk(reinterpret_cast<Tout*>(a.out[j]), seg0 + p0, a.M, nvalid, o);
    st = (st + 1 == S) ? 0 : st + 1;
  }
  if (bad) atomicOr(errw(a, j), make_err(kErrNonFinite, kPhReduce, j, j));
}

template <typename Tout, int CW, class S2>
__global__ void __launch_bounds__(kThreads) k_gather(FlashArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int CB = code_chunk_bytes(a.c2);
  const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(smem) + threadIdx.x * CB;
  const int S = a.stages;
  int r, j;
  pair_of(a, blockIdx.y, r, j);
  const uint8_t* src = gath_slot(a, r, j);
  const int64_t seg0 = (int64_t)j * a.seg + a.sub_off;
  Tout* out = reinterpret_cast<Tout*>(a.out[r]);
  const int tx = threadIdx.x * kLaneElems;
  auto issue = [&](int t, int st) {
    if (t < a.tiles) {
      const int64_t p0 = (int64_t)t * kTileElems + tx;
      if (p0 < a.sub_len) code_issue(a.c2, s0 + st * kThreads * CB, src, p0);
    }
    cp_async_commit();
  };
  for (int k = 0; k < S - 1; ++k) issue(blockIdx.x + k * gridDim.x, k);
  int st = 0;
  for (int t = blockIdx.x; t < a.tiles; t += gridDim.x) {
    issue(t + (S - 1) * gridDim.x, st == 0 ? S - 1 : st - 1);
    cp_async_wait_dyn(S - 1);
    const int64_t p0 = (int64_t)t * kTileElems + tx;
    const int nvalid = lane_valid(a.sub_len, p0);
    if (nvalid > 0) {
      LaneCodes<CW> L;
      code_read(a.c2, s0 + st * kThreads * CB, p0, L);
      float o[kLaneElems];
      decode_lane<S2, false>(a.c2, L, o);
      store_chunk(out, seg0 + p0, a.M, nvalid, o);
    }
    st = (st + 1 == S) ? 0 : st + 1;
  }
}

// Cross-process barrier between phases (IPC world, phase-split/generic):
// one warp; lane p != rank raises barflag[p][phase][rank], then waits on its own.
static __global__ void k_barrier(FlashArgs a, int rank, int phase) {
  const int p = threadIdx.x;
  __threadfence_system();
  __syncwarp();
  const uint32_t ep = flag_epoch(a);
  if (p < a.world && p != rank) st_relaxed_sys(barflag(a, p, phase, rank), ep);
  if (p < a.world && p != rank) {
    const uint32_t* f = barflag(a, rank, phase, p);
    const uint64_t t0 = globaltimer();
    volatile uint32_t* ew = errw(a, rank);
    while ((int32_t)(ld_acquire_sys(f) - ep) < 0) {
      if ((*ew >> 28) == kErrTimeout) break;
      if (globaltimer() - t0 > a.timeout_ns) {
        raise_timeout(a, rank, p, kPhBarrier);
        break;
      }
      __nanosleep(100);
    }
  }
  __syncwarp();
  __threadfence_system();
}

// ---------------------------------------------------------------- generic path

// scratch[i] = sum_s dequant(recv_slot[owner][s])[i], ascending s
static __global__ void k_gen_sum(FlashArgs a, int owner, float* scratch) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.sub_len;
       i += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.0f;
    for (int s = 0; s < a.world; ++s) {
      const float d = gen_value_at(a.c1, recv_slot(a, owner, s), i);
      acc = (s == 0) ? d : acc + d;
    }
    scratch[i] = acc;
  }
}

// copy owner's own gather slot [owner] to every peer's gather slot [owner]
static __global__ void k_gen_bcast(FlashArgs a, int owner, int64_t bytes) {
  const uint8_t* src = gath_slot(a, owner, owner);
  const int64_t n16 = bytes / 16;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 v = ld_v4(src + 16 * i);
    for (int pp = 1; pp < a.world; ++pp) st_v4(gath_slot(a, (owner + pp) % a.world, owner) + 16 * i, v);
  }
}

template <typename Tin, typename Tout>
__global__ void k_convert(const Tin* __restrict__ in, Tout* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = DT<Tout>::from_f(DT<Tin>::to_f(in[i]));
}

}  // namespace fc
