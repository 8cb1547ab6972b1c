// Small-message (decode regime, C4) Flash All-Reduce in ONE launch per rank
// (or one for all logical ranks of a GPU), synchronised only by per-tile
// epoch flags in the ranks' blocks -- no grid barrier, so the same kernel runs
// across GPUs / processes (peer memory over NVLink, system-scope fences).
//
// Items, in this order: scatter (rank r, piece j, tile t) -> rflag[j][r][t];
// reduce (owner j, tile t) waits rflag[j][s][t] for every peer s, sums the
// N-1 received pieces and its own QDQ'd piece in ascending source rank
// (collectives.py:182-187, 364-365), stage-2 quantizes, stores into every
// peer's gather slot [j] and decodes its own output (collectives.py:378) ->
// gflag[p][j][t]; gather (rank r, owner j, tile t) waits gflag[r][j][t] and
// decodes into the output. A CTA takes items i = blockIdx.x, +gridDim.x, ...
// in that order and all CTAs are co-resident (cooperative launch), so every
// wait targets an item some CTA reaches without waiting on a later one: no
// deadlock. At decode sizes every item gets its own CTA and the three phases
// overlap; the critical path is one scatter item, one flag hop, one reduce
// item, one flag hop and one gather item.
//
// The epoch is bumped in-kernel: every CTA reads the rank's counter at entry
// and the launch's last CTA writes counter + 1 at exit (after every CTA read
// it), so a CUDA-graph replay needs no separate k_epoch_bump launch.
#pragma once

#include "fc_flash.cuh"

namespace fc {

constexpr int kSmallBatch = 8;  // sources whose codes are in flight together in the reduce

// codes, scale and decode bias of one lane of a stored stage-1 piece (compile-time width)
template <int CW, class S>
__device__ __forceinline__ void load_lane_s(const DevCodec& c, const uint8_t* buf, int64_t p0, LaneCodes<CW>& L) {
  const uint8_t* cp = buf + p0 * S::SB / 8;
#pragma unroll
  for (int i = 0; i < S::SB / 4; ++i) {
    const uint4 u = ld_cg_v4(cp + 16 * i);
    L.w[4 * i] = u.x;
    L.w[4 * i + 1] = u.y;
    L.w[4 * i + 2] = u.z;
    L.w[4 * i + 3] = u.w;
  }
  const int64_t grp = p0 >> c.gshift;
  // raw scale / zero bits parked in the float slots (bit casts, no use of the loaded values
  // here): fixed up by lane_meta_fix once every source's loads are in flight
  L.s = __uint_as_float((uint32_t)__ldcg(reinterpret_cast<const unsigned short*>(buf + c.scales_off) + grp));
  L.mz = S::SYM ? 0.0f : __uint_as_float((uint32_t)__ldcg(buf + c.zeros_off + grp));
  if constexpr (S::SYM) {
    const uint32_t xr = rep_xor(c);
#pragma unroll
    for (int i = 0; i < S::SB; ++i) L.w[i] ^= xr;
  }
}

// turn load_lane_s's raw scale / zero bits into the decode's scale and bias
template <int CW, class S>
__device__ __forceinline__ void lane_meta_fix(const DevCodec& c, LaneCodes<CW>& L) {
  L.s = __half2float(__ushort_as_half((unsigned short)__float_as_uint(L.s)));
  L.mz = 8388608.0f + (S::SYM ? (float)(1 << (c.bits - 1)) : (float)__float_as_uint(L.mz));
}

// thread-level wait for one flag to reach the epoch (timeout -> error word, false)
__device__ __forceinline__ bool small_wait(const FlashArgs& a, int rank, const uint32_t* f, int peer, uint32_t ep,
                                           uint32_t phase) {
  const uint64_t t0 = globaltimer();
  volatile uint32_t* ew = errw(a, rank);
  uint32_t spins = 0;
  while ((int32_t)((a.sys_scope ? ld_acquire_sys(f) : ld_acquire_gpu(f)) - ep) < 0) {
    if ((*ew >> 28) == kErrTimeout) return false;
    if ((++spins & 63u) == 0 && globaltimer() - t0 > a.timeout_ns) {
      raise_timeout(a, rank, peer, phase);
      return false;
    }
    __nanosleep(32);
  }
  return true;
}

// publish after a CTA barrier: every thread's stores of the item happen before the flag
__device__ __forceinline__ void small_publish(const FlashArgs& a, uint32_t* f, uint32_t ep) {
  if (a.sys_scope) {
    __threadfence_system();
    st_relaxed_sys(f, ep);
  } else {
    st_release_gpu(f, ep);
  }
}

// reduce item: the peers' codes of a batch of sources are loaded before any is decoded, so
// their L2 / NVLink round trips overlap (do_reduce walks them one by one)
template <typename Tin, typename Tout, int CW, class S1, class S2>
__device__ __forceinline__ void do_reduce_small(const FlashArgs& a, int j, int t, uint32_t ep, uint64_t* tpr = nullptr) {
  const int lane = threadIdx.x & 31;
  const int64_t p0 = (int64_t)t * kTileElems + (int64_t)threadIdx.x * kLaneElems;
  const int nvalid = (int)max((int64_t)0, min(a.sub_len - p0, (int64_t)kLaneElems));
  const int64_t idx0 = (int64_t)j * a.seg + a.sub_off + p0;
  bool bad = false;
  // the own piece does not depend on any flag: its load and stage-1 QDQ (collectives.py:364-365)
  // run while the peers' scatter items are still in flight (one copy of the codec code: a
  // per-source copy made the kernel cold-instruction-cache bound)
  LaneCodes<CW> own;
  {
    LaneOf<Tin> v;
    load_lane_src(reinterpret_cast<const Tin*>(a.in[j]), idx0, a.M, nvalid, v);
    LaneQuant<CW> qq;
    bad |= quantize_lane<S1>(a.c1, v, nvalid, qq);
    lane_codes_from(a.c1, qq, own);
  }
  // thread s waits for rank s's stage-1 piece of this tile (rflag[j][s][t])
  if ((int)threadIdx.x < a.world && (int)threadIdx.x != j)
    small_wait(a, j, rflag(a, j, threadIdx.x) + t, threadIdx.x, ep, kPhReduce);
  __syncthreads();
  if (tpr) tpr[3] = globaltimer();
  FloatLane acc;
#pragma unroll
  for (int e = 0; e < kLaneElems; ++e) acc.v[e] = 0.0f;  // 0 + (c - z) s is exact and never -0
  for (int b0 = 0; b0 < a.world; b0 += kSmallBatch) {
    LaneCodes<CW> L[kSmallBatch];
#pragma unroll
    for (int q = 0; q < kSmallBatch; ++q) {
      const int s = b0 + q;
      if (s < a.world && s != j && nvalid > 0) load_lane_s<CW, S1>(a.c1, recv_slot(a, j, s), p0, L[q]);
    }
    if (tpr && b0 == 0) tpr[10] = globaltimer();
#pragma unroll
    for (int q = 0; q < kSmallBatch; ++q) {
      const int s = b0 + q;
      if (s >= a.world) break;
      if (tpr && b0 == 0 && q == 1) tpr[11] = globaltimer();
      LaneCodes<CW> C = L[q];
      if (s != j && nvalid > 0) lane_meta_fix<CW, S1>(a.c1, C);
      if (s == j) C = own;  // register select, ascending source rank (collectives.py:182-187)
      if (nvalid > 0) decode_lane<S1, true>(a.c1, C, acc.v);
    }
  }
  if (tpr) tpr[6] = globaltimer();
  LaneQuant<CW> q2;
  bad |= quantize_lane<S2>(a.c2, acc, nvalid, q2);
  if (tpr) tpr[7] = globaltimer();
  for (int pp = 1; pp < a.world; ++pp) {
    int p = j + pp;
    if (p >= a.world) p -= a.world;
    store_lane(a.c2, gath_slot(a, p, j), p0, nvalid, q2, lane);
  }
  if (tpr) tpr[8] = globaltimer();
  LaneCodes<CW> L2;
  lane_codes_from(a.c2, q2, L2);
  float o[kLaneElems];
  decode_lane<S2, false>(a.c2, L2, o);  // owner decodes its own payload too (collectives.py:378)
  if (nvalid > 0) store_chunk(reinterpret_cast<Tout*>(a.out[j]), idx0, a.M, nvalid, o);
  if (tpr) tpr[9] = globaltimer();
  if (bad) atomicOr(errw(a, j), make_err(kErrNonFinite, kPhReduce, j, j));
}

template <typename Tin, typename Tout, int CW, class S1, class S2>
__global__ void __launch_bounds__(kThreads) k_small(FlashArgs a) {
  __shared__ uint32_t s_ep;
  __shared__ int s_last;
  const int P = a.world - 1, nr = a.rank_hi - a.rank_lo, T = a.tiles;
  const int nS = nr * P * T, nR = nr * T, nG = nr * P * T;
  uint32_t* ectr = const_cast<uint32_t*>(a.epoch_dev);
  if (threadIdx.x == 0) s_ep = *reinterpret_cast<volatile uint32_t*>(ectr) + 1u;
  __syncthreads();
  const uint32_t ep = s_ep;
  // measurement (FC_OPT_ROLE_PROFILE): entry, first item's kind / start / after-wait / end, exit
  uint64_t* tp = a.tprof ? a.tprof + (int64_t)blockIdx.x * FC_ROLE_PROFILE_U64 : nullptr;
  if (tp && threadIdx.x == 0) tp[0] = globaltimer();
  for (int i = blockIdx.x; i < nS + nR + nG; i += gridDim.x) {
    const bool prof = tp && threadIdx.x == 0 && i == (int)blockIdx.x;
    if (prof) {
      tp[1] = i < nS ? 0 : (i < nS + nR ? 1 : 2);
      tp[2] = globaltimer();
    }
    if (i < nS) {  // ---- scatter (r, j, t) -> rflag[j][r][t]
      const int y = i / T, t = i - y * T;
      int r, j;
      pair_of(a, y, r, j);
      do_scatter<Tin, CW, S1>(a, r, j, t);
      __syncthreads();
      if (threadIdx.x == 0) small_publish(a, rflag(a, j, r) + t, ep);
    } else if (i < nS + nR) {  // ---- reduce (j, t): N-1 peers' pieces -> gflag[p][j][t]
      const int y = (i - nS) / T, t = (i - nS) - y * T;
      const int j = a.rank_lo + y;
      do_reduce_small<Tin, Tout, CW, S1, S2>(a, j, t, ep, prof ? tp : nullptr);
      __syncthreads();
      if (threadIdx.x < a.world && threadIdx.x != j) {
        if (a.sys_scope) __threadfence_system();
        else __threadfence();
        st_relaxed_sys(gflag(a, threadIdx.x, j) + t, ep);
      }
    } else {  // ---- gather (r, j, t)
      const int i2 = i - nS - nR;
      const int y = i2 / T, t = i2 - y * T;
      int r, j;
      pair_of(a, y, r, j);
      if (threadIdx.x == 0) small_wait(a, r, gflag(a, r, j) + t, j, ep, kPhGather);
      __syncthreads();
      if (prof) tp[3] = globaltimer();
      do_gather<Tout, CW, S2>(a, r, j, t);
    }
    if (tp) {  // (measurement only) the item's stores are issued by every thread
      __syncthreads();
      if (prof) tp[4] = globaltimer();
    }
  }
  if (tp && threadIdx.x == 0) tp[5] = globaltimer();
  // the launch's last CTA advances the epoch counter (every CTA has read it)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    uint32_t* done = fctr(a, a.rank_lo) + 3 * kFusedMaxChunks + 1;
    s_last = atomicAdd(done, 1u) == gridDim.x - 1;
    if (s_last) {
      *done = 0u;
      *reinterpret_cast<volatile uint32_t*>(ectr) = ep;
      __threadfence();
    }
  }
}

}  // namespace fc
