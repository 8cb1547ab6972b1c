// Streaming phase kernels of the Flash All-Reduce (and the single-GPU codec)
// for the compile-time lane codecs of fc_lane.cuh and 16-bit inputs.
//
// Work is a flat list of items (job, 8192-element tile) walked by persistent
// CTAs. Quantize-type kernels (k_qstream: stage-1 scatter / codec quantize,
// k_rstream: reduce) are fed by a dedicated producer warp that issues bulk
// copies (cp.async.bulk, TMA engine) of whole tiles into an S-stage
// shared-memory ring guarded by full/empty mbarriers; the 8 consumer warps
// only compute. A consumer thread owns 32 contiguous elements (a group of
// g elements spans g/32 lanes); it reads its 64 B from shared memory as four
// 16-B vectors in a lane-rotated order (vector (q + rot) & 3 at step q,
// rot = (lane >> 1) & 3), which makes every LDS.128 conflict-free; the
// rotation is undone on the 4 (INT4) / 8 (INT8) packed code words, or on the
// input words when decoded values must line up with other ranks' (reduce).
// Codes leave as one/two coalesced 16-B stores per lane (a warp writes 512 B
// contiguous), straight into the destination rank's slot (peer memory over
// NVLink when the ranks are different GPUs).
//
// The dequantize-type kernel (k_dstream: all-gather decode / codec
// dequantize) needs no group statistics, so it uses the transposed mapping:
// thread t decodes 8-element blocks t, t+256, t+512, t+768 of a tile, which
// makes both the code loads and the 16-B output stores coalesced.
#pragma once

#include "fc_flash.cuh"
#include "fc_lane.cuh"
#include "fc_tma.cuh"

namespace fc {

constexpr int kConsumerWarps = kThreads / 32;  // 8
constexpr int kStreamThreads = kThreads + 32;  // + one producer warp

// ------------------------------------------------------------------ jobs

// quantize job y: source elements, element limit (elements at or past it
// read as 0, collectives.py:145-149), destination slot, error word
template <typename Tin>
struct QJob {
  const Tin* src;
  int64_t limit;
  uint8_t* dst;
  uint32_t* err;
  uint32_t ecode;
};

template <typename Tin>
__device__ __forceinline__ QJob<Tin> qjob(const FlashArgs& a, int y) {
  QJob<Tin> q;
  if (a.mode == 1) {
    q.src = reinterpret_cast<const Tin*>(a.in[0]);
    q.limit = a.M;
    q.dst = reinterpret_cast<uint8_t*>(a.out[0]);
    q.err = a.cerr;
    q.ecode = make_err(kErrNonFinite, 0, 0, 0);
    return q;
  }
  int r, j;
  qpair_of(a, y, r, j);
  const int64_t off = (int64_t)j * a.seg + a.sub_off;
  q.src = reinterpret_cast<const Tin*>(a.in[r]) + off;
  q.limit = a.M - off;
  q.dst = recv_slot(a, j, r);
  q.err = errw(a, r);
  q.ecode = make_err(kErrNonFinite, kPhScatter, j, r);
  return q;
}

__device__ __forceinline__ int64_t clamp0(int64_t v) { return v < 0 ? 0 : v; }

// elements of tile t of a job that are real data (inside the round and below the limit)
__device__ __forceinline__ int64_t tile_valid(int64_t len, int64_t limit, int64_t e0) {
  return clamp0(min((int64_t)kTileElems, min(len - e0, limit - e0)));
}

// ------------------------------------------------------------------ stores

// predicated global stores (no divergent branches around the stores)
__device__ __forceinline__ void st_v4_if(void* p, uint4 v, bool pred) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %5, 0;\n @q st.global.v4.u32 [%0], {%1,%2,%3,%4};\n}" ::"l"(p),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"((uint32_t)pred)
               : "memory");
}
__device__ __forceinline__ void st_u16_if(void* p, unsigned short v, bool pred) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q st.global.u16 [%0], %1;\n}" ::"l"(p), "h"(v),
               "r"((uint32_t)pred)
               : "memory");
}
__device__ __forceinline__ void st_u8_if(void* p, uint32_t v, bool pred) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q st.global.u8 [%0], %1;\n}" ::"l"(p), "r"(v),
               "r"((uint32_t)pred)
               : "memory");
}

// where a lane chunk's codes and its group's metadata live inside a slot
struct CodeDst {
  uint32_t codes;       // byte offset of the chunk's packed codes
  int64_t scale, zero;  // byte offsets of the group's fp16 scale / zero byte
  bool any, meta;       // chunk holds elements / this lane writes the group metadata
};
template <class Spec>
__device__ __forceinline__ CodeDst code_dst(const DevCodec& c, int64_t p0, int nvalid, int lane) {
  CodeDst d;
  d.codes = (uint32_t)(p0 * Spec::SB / 8);
  const int64_t grp = p0 >> c.gshift;
  d.scale = c.scales_off + 2 * grp;
  d.zero = c.zeros_off + grp;
  d.any = nvalid > 0;
  d.meta = d.any && (lane & (c.lpg - 1)) == 0;
  return d;
}
template <class Spec>
__device__ __forceinline__ void store_codes_at(uint8_t* buf, const CodeDst& d, const LaneQuant<8>& q) {
  st_v4_if(buf + d.codes, make_uint4(q.w[0], q.w[1], q.w[2], q.w[3]), d.any);
  if constexpr (Spec::SB == 8) st_v4_if(buf + d.codes + 16, make_uint4(q.w[4], q.w[5], q.w[6], q.w[7]), d.any);
  st_u16_if(buf + d.scale, __half_as_ushort(q.s16), d.meta);
  if constexpr (!Spec::SYM) st_u8_if(buf + d.zero, q.z8, d.meta);
}
template <class Spec>
__device__ __forceinline__ void store_codes(const DevCodec& c, uint8_t* buf, int64_t p0, int nvalid,
                                            const LaneQuant<8>& q, int lane) {
  store_codes_at<Spec>(buf, code_dst<Spec>(c, p0, nvalid, lane), q);
}

// undo the lane rotation of packed code words
template <class Spec>
__device__ __forceinline__ void unrotate_codes(uint32_t* w, int rot) {
  if constexpr (Spec::SB == 4) {
    unrotate4(w, rot);
  } else {
    uint32_t e[4] = {w[0], w[2], w[4], w[6]}, o[4] = {w[1], w[3], w[5], w[7]};
    unrotate4(e, rot);
    unrotate4(o, rot);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      w[2 * i] = e[i];
      w[2 * i + 1] = o[i];
    }
  }
}

// read this thread's 64-B input chunk (rotated order) from a staged tile
template <typename Tin>
__device__ __forceinline__ void read_rotated(uint32_t tile, const uint32_t qoff[4], PackedLane<Tin>& L) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint4 u = lds128_(tile + qoff[q]);
    L.w[4 * q] = u.x;
    L.w[4 * q + 1] = u.y;
    L.w[4 * q + 2] = u.z;
    L.w[4 * q + 3] = u.w;
  }
}

// put rotated input words back in element order (16 words = 4 vectors)
template <typename Tin>
__device__ __forceinline__ void unrotate_input(PackedLane<Tin>& L, int rot) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t v[4] = {L.w[c], L.w[4 + c], L.w[8 + c], L.w[12 + c]};
    unrotate4(v, rot);
    L.w[c] = v[0];
    L.w[4 + c] = v[1];
    L.w[8 + c] = v[2];
    L.w[12 + c] = v[3];
  }
}

// bytes of one peer's staged piece of a tile: codes, scales, zeros (16-B aligned parts)
__host__ __device__ inline uint32_t peer_codes_bytes(const DevCodec& c) { return kTileElems * c.sb / 8; }
__host__ __device__ inline uint32_t peer_scale_bytes(const DevCodec& c) { return ((kTileElems / c.g) * 2 + 15) & ~15u; }
__host__ __device__ inline uint32_t peer_meta_bytes(const DevCodec& c) {
  const uint32_t groups = kTileElems / c.g;
  return peer_scale_bytes(c) + (c.sym ? 0u : ((groups + 15) & ~15u));
}
__host__ __device__ inline uint32_t rstage_bytes(const DevCodec& c1, int world) {
  return kTileElems * 2 + (uint32_t)(world - 1) * (peer_codes_bytes(c1) + peer_meta_bytes(c1));
}

__device__ __forceinline__ uint32_t up16(int64_t v) { return (uint32_t)((v + 15) & ~(int64_t)15); }

// one received stage-1 lane chunk from the staged peer region `src`
template <class S1>
__device__ __forceinline__ void read_peer(const DevCodec& c1, uint32_t src, uint32_t PC, uint32_t SCB, uint32_t gl,
                                          LaneCodes<8>& C) {
  const uint32_t cp = src + threadIdx.x * (kLaneElems * S1::SB / 8);
  const uint4 u = lds128_(cp);
  C.w[0] = u.x;
  C.w[1] = u.y;
  C.w[2] = u.z;
  C.w[3] = u.w;
  if constexpr (S1::SB == 8) {
    const uint4 u2 = lds128_(cp + 16);
    C.w[4] = u2.x;
    C.w[5] = u2.y;
    C.w[6] = u2.z;
    C.w[7] = u2.w;
  }
  unsigned short sh;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(sh) : "r"(src + PC + 2 * gl) : "memory");
  C.s = __half2float(__ushort_as_half(sh));
  float zf;
  if constexpr (S1::SYM) {
    zf = (float)(1 << (c1.bits - 1));
    const uint32_t xr = rep_xor(c1);
#pragma unroll
    for (int w = 0; w < S1::SB; ++w) C.w[w] ^= xr;
  } else {
    uint32_t zz;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(zz) : "r"(src + PC + SCB + gl) : "memory");
    zf = (float)zz;
  }
  C.mz = 8388608.0f + zf;
}

// ------------------------------------------------------------------ item iterators

// Phase-split kernels: each CTA walks a contiguous range of the job-major item
// list, so (job y, tile t) advance by increment and consecutive items of a CTA
// are consecutive tiles of one job.
struct RangeIter {
  int i, end, y, t, tiles;
  int t0;
  __device__ __forceinline__ RangeIter(int items, int tiles_, int cta, int nctas, int t0_ = 0) : tiles(tiles_), t0(t0_) {
    const int per = (items + nctas - 1) / nctas;
    i = min(items, cta * per);
    end = min(items, i + per);
    y = i / tiles;
    t = i - y * tiles + t0;
  }
  __device__ __forceinline__ bool ok() const { return i < end; }
  __device__ __forceinline__ void next() {
    ++i;
    if (++t == tiles + t0) {
      t = t0;
      ++y;
    }
  }
};

// Fused kernel: tile-major items (t = i / P, y = i % P) dealt round-robin to the
// CTAs of a role, so every role sweeps the tiles in step and a tile's
// producers run ahead of its consumers.
struct RoundIter {
  int i, items, y, t, P, dy, dt, step;
  __device__ __forceinline__ RoundIter(int items_, int P_, int first, int step_, int t0 = 0)
      : i(first), items(items_), P(P_), step(step_) {
    t = first / P;
    y = first - t * P;
    t += t0;
    dt = step / P;
    dy = step - dt * P;
  }
  __device__ __forceinline__ bool ok() const { return i < items; }
  __device__ __forceinline__ void next() {
    i += step;
    t += dt;
    y += dy;
    if (y >= P) {
      y -= P;
      ++t;
    }
  }
};

// ------------------------------------------------------------------ cross-CTA / cross-GPU flags (fused)

// lanes [0, n) of the calling warp each wait for flags[lane] to reach the
// epoch; a wait past the timeout (or an error raised elsewhere) latches a
// ProtocolError in the error word and gives up (results then are garbage,
// the call reports the error). Returns false when aborted.
__device__ __forceinline__ bool warp_wait_flags(const FlashArgs& a, int rank, const uint32_t* flag, int peer,
                                                bool active, uint32_t phase) {
  bool ok = true;
  if (active && !(a.dbg & 256)) {  // dbg 256: measurement only, no waits (results are garbage)
    const uint64_t t0 = globaltimer();
    volatile uint32_t* ew = errw(a, rank);
    uint32_t spins = 0;
    const uint32_t ep = flag_epoch(a);
    while ((int32_t)((a.sys_scope ? ld_acquire_sys(flag) : ld_acquire_gpu(flag)) - ep) < 0) {
      if ((*ew >> 28) == kErrTimeout) {
        ok = false;
        break;
      }
      if ((++spins & 63u) == 0 && globaltimer() - t0 > a.timeout_ns) {
        raise_timeout(a, rank, peer, phase);
        ok = false;
        break;
      }
      __nanosleep(64);
    }
  }
  ok = __all_sync(0xffffffffu, ok);
  // the data behind the flags is read by bulk copies (async proxy)
  asm volatile("fence.proxy.async.global;" ::: "memory");
  return ok;
}

// consumer warps only (named barrier 1): every consumer thread's stores of this
// item happen before thread 0's system-scope fence and flag stores
template <int NT = kThreads>
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory"); }

// publish one per-tile flag after a named-barrier sync of the threads whose
// stores it covers: system scope (fence.sc.sys, then a relaxed sys store) when
// the flag crosses GPUs, else a gpu-scope release store
__device__ __forceinline__ void publish_flag(const FlashArgs& a, uint32_t* f, uint32_t ep) {
  if (a.sys_scope) {
    __threadfence_system();
    st_relaxed_sys(f, ep);
  } else {
    st_release_gpu(f, ep);
  }
}

// fused kernels publish a tile's flags from the PRODUCER warp once the tile's
// consumers have handed its ring stage back: the consumers issue all of the
// tile's global stores before they arrive on the stage's empty barrier
// (mbarrier.arrive: release.cta; the producer's try_wait: acquire.cta), so the
// producer's gpu/system-scope release covers them by cumulativity -- the same
// argument as a bar.sync before a publishing thread, but the fence stalls
// only the producer (which has S stages of bulk copies queued), not a
// consumer warp in the middle of its tiles.
__device__ __forceinline__ void publish_scatter(const FlashArgs& a, int y, int t, uint32_t ep) {
  if (a.dbg & 512) return;  // measurement only
  int r, j;
  qpair_of(a, y, r, j);
  publish_flag(a, rflag(a, j, r) + t, ep);
}
__device__ __forceinline__ void publish_reduce(const FlashArgs& a, int y, int t, uint32_t ep) {
  if (a.dbg & 512) return;
  const int j = a.rank_lo + y;
  if (a.sys_scope) __threadfence_system();
  else __threadfence();
  for (int p = 0; p < a.world; ++p)
    if (p != j) st_relaxed_sys(gflag(a, p, j) + t, ep);
}

__device__ __forceinline__ void mbar_inval(uint32_t bar) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}

// ------------------------------------------------------------------ ring setup

__device__ __forceinline__ void ring_init(uint32_t full0, uint32_t empty0, int S) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
}
__device__ __forceinline__ void ring_next(int& st, uint32_t& ph, int S) {
  if (++st == S) {
    st = 0;
    ph ^= 1;
  }
}

// ------------------------------------------------------------------ quantize role

// stage-1 scatter (mode 0: (rank, peer) job y of [rank_lo, rank_hi)) or codec
// quantize (mode 1). FUSED: raise rflag[j][r][t] after each tile's stores.
template <typename Tin, class S1, bool FUSED, class Iter>
__device__ __forceinline__ void q_role(const FlashArgs& a, uint32_t sbase, int S, Iter it0) {
  static_assert(sizeof(Tin) == 2, "16-bit inputs");
  constexpr uint32_t STAGE = kTileElems * 2;
  const uint32_t full0 = sbase + S * STAGE, empty0 = full0 + 8 * S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  ring_init(full0, empty0, S);
  if (warp == kConsumerWarps) {  // producer warp: one lane issues the bulk copies
    if (lane == 0) {
      int st = 0, k = 0, cy = -1;
      uint32_t ph = 0;
      QJob<Tin> jb;
      for (Iter it = it0; it.ok(); it.next(), ++k) {
        if (k >= S) mbar_wait(empty0 + 8 * st, ph ^ 1);
        if (it.y != cy) {
          jb = qjob<Tin>(a, it.y);
          cy = it.y;
        }
        const int64_t e0 = (int64_t)it.t * kTileElems;
        const uint32_t bytes = (uint32_t)(tile_valid(a.sub_len, jb.limit, e0) * 2) & ~15u;
        mbar_arrive_expect_tx(full0 + 8 * st, bytes);
        if (bytes) bulk_g2s(sbase + st * STAGE, jb.src + e0, bytes, full0 + 8 * st);
        ring_next(st, ph, S);
      }
    }
    return;
  }
  const int rot = (lane >> 1) & 3;
  uint32_t qoff[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) qoff[q] = threadIdx.x * 64 + 16 * ((q + rot) & 3);
  int st = 0, cy = -1;
  uint32_t ph = 0;
  QJob<Tin> jb;
  for (Iter it = it0; it.ok(); it.next()) {
    if (it.y != cy) {
      jb = qjob<Tin>(a, it.y);
      cy = it.y;
    }
    const int64_t p0 = (int64_t)it.t * kTileElems + threadIdx.x * kLaneElems;
    const int nvalid = lane_valid(a.sub_len, p0);
    const bool staged = nvalid == kLaneElems && p0 + kLaneElems <= jb.limit;
    PackedLane<Tin> L;
    mbar_wait(full0 + 8 * st, ph);
    if (staged)
      read_rotated(sbase + st * STAGE, qoff, L);
    else
      load_lane_src(jb.src, p0, jb.limit, nvalid, L);
    LaneQuant<8> q;
    const bool bad = quantize_lane<S1>(a.c1, L, nvalid, q);
    // release the stage only after the shared loads were consumed: an LDS still
    // in flight at the arrive could otherwise read the next tile's bulk copy
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * st);
    if (staged) unrotate_codes<S1>(q.w, rot);
    store_codes<S1>(a.c1, jb.dst, p0, nvalid, q, lane);
    if (bad && jb.err) atomicOr(jb.err, jb.ecode);
    if constexpr (FUSED) {
      consumers_sync();
      if (threadIdx.x == 0) {
        int r, j;
        qpair_of(a, it.y, r, j);
        if (a.sys_scope) {
          __threadfence_system();
          st_relaxed_sys(rflag(a, j, r) + it.t, flag_epoch(a));
        } else {
          st_release_gpu(rflag(a, j, r) + it.t, flag_epoch(a));  // bar.sync + release: cumulative over the CTA's stores
        }
      }
    }
    ring_next(st, ph, S);
  }
}

// ------------------------------------------------------------------ fused kernel: dynamic item dealing

// One (role, chunk) of the fused kernel: its items are dealt dynamically. The
// producer warp of a CTA grabs item ids from a global counter (tile-major:
// t = t0 + id / per, y = id % per) and writes each id beside its ring stage in
// shared memory; the consumer warps read it after the stage's full barrier; a
// negative id ends the role. Faster CTAs take more items, so the CTAs leave a
// role together (a static round-robin deal left 50-100 us of per-role tails
// at C2 on one GPU). The counters are zeroed by the last CTA of the launch.
struct DynIter {
  uint32_t* ctr;  // this (role, chunk)'s counter
  int items, per, t0;
  uint32_t meta;  // shared-memory id ring, one int per stage
  uint32_t ep;    // the round's flag epoch
  __device__ __forceinline__ int grab() const { return (int)atomicAdd(ctr, 1u); }
  __device__ __forceinline__ void decode(int id, int& y, int& t) const {
    t = id / per;
    y = id - t * per;
    t += t0;
  }
};
__device__ __forceinline__ void sts32(uint32_t addr, int v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ int lds_id(uint32_t addr) {
  int v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}

// ------------------------------------------------------------------ group-per-lane quantize role

// g = 128 quantize with one lane per whole group (k_qstream_gpl). The
// 32-element lane layout above spreads a group over 4 lanes, so every lane
// repeats the group's statistics tail, the float64 scale and the zero point
// (SIMT: one pass computes 8 groups per warp); with one lane per group the
// same pass serves 32 groups, and no shuffles are needed. A lane reads its
// 256-B group as 16 vectors in XOR-swizzled order (vector k ^ (lane & 7) at
// step k: the 8 lanes of each quarter-warp hit 8 distinct bank groups), keeps
// the 64 input words in registers, and undoes the swizzle on the 16 (INT4) /
// 32 (INT8) code words with three conditional-swap layers. Same numerics as
// lane_quantize_fast (identical group_params, per-element rounding, packing).
constexpr int kGplG = 128;
constexpr int kGplWarps = 4;                         // consumer warps
constexpr int kGplThreads = (kGplWarps + 1) * 32;    // + the producer warp
constexpr int kGplWpt = kTileElems / (32 * kGplG);   // warps per tile (2)
constexpr int kGplSlots = kGplWarps / kGplWpt;       // tiles in flight across the consumers (2)

// element e (0..7) of an 8-element chunk held as 4 packed 16-bit pairs, as fp32 bits
template <typename Tin>
__device__ __forceinline__ uint32_t chunk_elem(const uint32_t x[4], int e) {
  const uint32_t w = x[e >> 1];
  if constexpr (std::is_same<Tin, __nv_bfloat16>::value) {
    return (e & 1) ? (w & 0xFFFF0000u) : (w << 16);
  } else {
    const __half h = __ushort_as_half((unsigned short)((e & 1) ? (w >> 16) : (w & 0xFFFFu)));
    return __float_as_uint(__half2float(h));
  }
}
template <typename Tin>
__device__ __forceinline__ uint64_t chunk_pair(const uint32_t x[4], int a, int b) {
  uint64_t r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "r"(chunk_elem<Tin>(x, a)), "r"(chunk_elem<Tin>(x, b)));
  return r;
}

// offset-binary codes of one 8-element chunk (1 word INT4, 2 words INT8); requires g.normal
template <class Spec, typename Tin>
__device__ __forceinline__ void chunk_codes_packed(const uint32_t x[4], const GroupQ& g, uint32_t qmax, uint32_t* w) {
  const uint64_t R2 = f2_splat(g.r), NS2 = f2_splat(-g.s), C2 = f2_splat(12582912.0f);
  const uint32_t Z2 = g.z * 0x00010001u, Q2 = qmax * 0x00010001u;
  auto code_pair = [&](int a, int b) -> uint32_t {
    const uint64_t X = chunk_pair<Tin>(x, a, b);
    const uint64_t T = f2_mul(X, R2);
    const uint64_t Q = f2_fma(f2_fma(T, NS2, X), R2, T);
    const uint64_t Y = Spec::CEIL ? f2_add_rp(Q, C2) : f2_add(Q, C2);
    uint32_t ya, yb;
    f2_bits(Y, ya, yb);
    const uint32_t p = __byte_perm(ya, yb, 0x5410);
    const uint32_t c = __viaddmax_s16x2(p, Z2, 0u);
    return __vimin3_s16x2(c, Q2, Q2);
  };
  if constexpr (Spec::SB == 4) {
    w[0] = code_pair(0, 4) + (code_pair(1, 5) << 4) + (code_pair(2, 6) << 8) + (code_pair(3, 7) << 12);
  } else {
    w[0] = code_pair(0, 2) + (code_pair(1, 3) << 8);
    w[1] = code_pair(4, 6) + (code_pair(5, 7) << 8);
  }
}

// the float-clamp path of lane_codes (fc_common.cuh) for one chunk: |x/s| may exceed 16 bits
template <class Spec, typename Tin>
__device__ __forceinline__ void chunk_codes_clamped(const uint32_t x[4], float s, int z, int qmax, uint32_t* w) {
  const float r = __frcp_rn(s);
  const float C0 = 12582912.0f;
  const float lob = -(float)z, hib = (float)(qmax - z);
  const int zb = z - 0x4B400000;
  w[0] = 0;
  if constexpr (Spec::SB == 8) w[1] = 0;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const float xv = __uint_as_float(chunk_elem<Tin>(x, e));
    const float t = xv * r;
    const float q1 = fmaf(fmaf(-t, s, xv), r, t);
    const float qc = fminf(fmaxf(q1, lob), hib);
    const float y = Spec::CEIL ? __fadd_ru(qc, C0) : __fadd_rn(qc, C0);
    const uint32_t code = (uint32_t)(__float_as_int(y) + zb);
    if constexpr (Spec::SB == 4)
      w[0] |= code << (4 * e);
    else
      w[e >> 2] |= code << (8 * (e & 3));
  }
}

// minifloat codes of one 8-element chunk: RN32(x / s) by reciprocal + one FMA correction, then
// cvt.rn.satfinite pairwise (mf_enc2: +0 for zero magnitudes); INT8-like byte storage (e4m3 /
// e5m2: w[0] = elements 0..3, w[1] = 4..7) or nibbles little-nibble-first (e2m1: w[0])
template <class Spec, typename Tin>
__device__ __forceinline__ void chunk_codes_mf(const uint32_t x[4], const GroupQ& g, uint32_t* w) {
  const uint64_t R2 = f2_splat(g.r), NS2 = f2_splat(-g.s);
  uint32_t two[4];
#pragma unroll
  for (int p = 0; p < 4; ++p) {  // the quotient pairwise (FMUL2 / FFMA2: the same roundings as fmaf)
    const uint64_t X = chunk_pair<Tin>(x, 2 * p, 2 * p + 1);
    const uint64_t T = f2_mul(X, R2);
    float q0, q1;
    f2_unpack(f2_fma(f2_fma(T, NS2, X), R2, T), q0, q1);
    two[p] = mf_enc2_raw(Spec::FMT, q0, q1);
  }
  if constexpr (Spec::SB == 8) {
    w[0] = mf_fix_zero<Spec::FMT>(two[0] | (two[1] << 16));
    w[1] = mf_fix_zero<Spec::FMT>(two[2] | (two[3] << 16));
  } else {
    w[0] = mf_fix_zero<Spec::FMT>(two[0] | (two[1] << 8) | (two[2] << 16) | (two[3] << 24));
  }
}

// 16-bit packed min / max (NaN-propagating), bf16x2 or f16x2
template <typename Tin>
__device__ __forceinline__ uint32_t h2min(uint32_t a, uint32_t b) {
  uint32_t r;
  if constexpr (std::is_same<Tin, __nv_bfloat16>::value)
    asm("min.NaN.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  else
    asm("min.NaN.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
template <typename Tin>
__device__ __forceinline__ uint32_t h2max(uint32_t a, uint32_t b) {
  uint32_t r;
  if constexpr (std::is_same<Tin, __nv_bfloat16>::value)
    asm("max.NaN.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  else
    asm("max.NaN.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
template <typename Tin>
__device__ __forceinline__ float h_lo(uint32_t w) {
  if constexpr (std::is_same<Tin, __nv_bfloat16>::value) return __uint_as_float(w << 16);
  else return __half2float(__ushort_as_half((unsigned short)(w & 0xFFFFu)));
}
template <typename Tin>
__device__ __forceinline__ float h_hi(uint32_t w) {
  if constexpr (std::is_same<Tin, __nv_bfloat16>::value) return __uint_as_float(w & 0xFFFF0000u);
  else return __half2float(__ushort_as_half((unsigned short)(w >> 16)));
}

// words w[k * CWPC + i] of chunk k -> chunk k ^ m (three conditional-swap layers)
template <int NC, int CWPC>
__device__ __forceinline__ void unswizzle_chunks(uint32_t* w, int m) {
#pragma unroll
  for (int b = 1; b < 8; b <<= 1) {
    const bool sw = (m & b) != 0;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      if (k & b) continue;
#pragma unroll
      for (int i = 0; i < CWPC; ++i) {
        const uint32_t u = w[k * CWPC + i], v = w[(k ^ b) * CWPC + i];
        w[k * CWPC + i] = sw ? v : u;
        w[(k ^ b) * CWPC + i] = sw ? u : v;
      }
    }
  }
}

template <typename Tin, class S1, bool FUSED, class Iter, int G = 128>
__device__ __forceinline__ void q_role_gpl(const FlashArgs& a, uint32_t sbase, int S, Iter it0, uint32_t bars = 0) {
  static_assert(sizeof(Tin) == 2, "16-bit inputs");
  static_assert(G == 32 || G == 64 || G == 128 || G == 256, "a lane's 128-element slice holds 4, 2, 1 or half a group");
  constexpr uint32_t STAGE = kTileElems * 2;
  constexpr int NC = kGplG / 8;      // 8-element chunks per group
  constexpr int CWPC = S1::SB / 4;   // code words per chunk
  const uint32_t full0 = bars ? bars : sbase + S * STAGE, empty0 = full0 + 8 * S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, kGplWpt * 32);  // every consumer thread releases its own reads
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == kGplWarps) {  // producer warp: one lane issues the bulk copies (as in q_role)
    if (lane == 0) {
      int st = 0, k = 0, cy = -1;
      uint32_t ph = 0;
      QJob<Tin> jb;
      auto issue = [&](int y, int t) {
        if (y != cy) {
          jb = qjob<Tin>(a, y);
          cy = y;
        }
        const int64_t e0 = (int64_t)t * kTileElems;
        const uint32_t bytes = (uint32_t)(tile_valid(a.sub_len, jb.limit, e0) * 2) & ~15u;
        mbar_arrive_expect_tx(full0 + 8 * st, bytes);
        if (bytes) bulk_g2s(sbase + st * STAGE, jb.src + e0, bytes, full0 + 8 * st);
      };
      if constexpr (!FUSED) {
        for (Iter it = it0; it.ok(); it.next(), ++k) {
          if (k >= S) mbar_wait(empty0 + 8 * st, ph ^ 1);
          issue(it.y, it.t);
          ring_next(st, ph, S);
        }
      } else {
        // dynamic dealing (DynIter): grab ids until the (role, chunk) is exhausted; a recycled
        // stage's previous item has its stores issued: publish its flag (publish_scatter)
        const DynIter& D = it0;
        // flags of recycled items are published in batches of kPubBatch behind ONE release fence
        // (a gpu/system-scope release per item stalled this thread ~3 us each -- it waits for the
        // consumers' code stores -- and left the ring idle: fused scatter role 290 vs 233 us)
        constexpr int kPubBatch = 8;
        int pend[kPubBatch];
        int npend = 0;
        auto flush = [&]() {
          if (npend == 0 || (a.dbg & 512)) {
            npend = 0;
            return;
          }
          if (a.sys_scope) __threadfence_system();
          else __threadfence();
#pragma unroll
          for (int i = 0; i < kPubBatch; ++i)
            if (i < npend) {
              int y, t, r, j;
              D.decode(pend[i], y, t);
              qpair_of(a, y, r, j);
              st_relaxed_sys(rflag(a, j, r) + t, D.ep);
            }
          npend = 0;
        };
        auto publish_id = [&](int old) {
          pend[npend++] = old;
          if (npend == kPubBatch) flush();
        };
        auto recycle = [&]() {
          mbar_wait(empty0 + 8 * st, ph ^ 1);
          publish_id(lds_id(D.meta + 4 * st));
        };
        int id = D.grab();
        for (;; ++k) {
          const int nid = id < D.items ? D.grab() : id;  // the next id is in flight during this item
          if (k >= S) recycle();
          if (id >= D.items) break;
          sts32(D.meta + 4 * st, id);
          int y, t;
          D.decode(id, y, t);
          issue(y, t);
          ring_next(st, ph, S);
          id = nid;
        }
        // one end sentinel per consumer slot (the first one takes the stage recycled above)
        const int K = k;
        for (int n = 0; n < kGplSlots; ++n, ++k) {
          if (n > 0 && k >= S) recycle();
          sts32(D.meta + 4 * st, -1);
          mbar_arrive(full0 + 8 * st);
          ring_next(st, ph, S);
        }
        // the real items whose stages were not recycled: wait for their hand-back, publish
        for (int kp = k > S ? k - S : 0; kp < K; ++kp) {
          mbar_wait(empty0 + 8 * (kp % S), (uint32_t)(kp / S) & 1u);
          publish_id(lds_id(D.meta + 4 * (kp % S)));
        }
        flush();
      }
    }
    return;
  }
  const int slot = warp / kGplWpt, part = warp % kGplWpt;
  const int m = lane & 7;
  const int gi = part * 32 + lane;  // this lane's group within a tile
  int cy = -1;
  QJob<Tin> jb;
  auto item = [&](int y, int t, int st, uint32_t ph) {
      if (y != cy) {
        jb = qjob<Tin>(a, y);
        cy = y;
      }
      const int64_t p0 = (int64_t)t * kTileElems + gi * kGplG;
      const bool whole = p0 + kGplG <= a.sub_len && p0 + kGplG <= jb.limit;
      mbar_wait(full0 + 8 * st, ph);
      if (__all_sync(0xffffffffu, whole)) {
        const uint32_t gb = sbase + st * STAGE + gi * (kGplG * 2);
        uint32_t x[NC][4];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const uint4 u = lds128_(gb + 16 * (c ^ m));
          x[c][0] = u.x;
          x[c][1] = u.y;
          x[c][2] = u.z;
          x[c][3] = u.w;
        }
        // group bounds in 16-bit packed arithmetic (exact), then fp32. The slice holds NG groups
        // of CPG chunks (G = 32: four; 64: two; 128: one; 256: half a group, the partner lane --
        // the adjacent slice -- holds the other half: one shuffle). x[c] is physical chunk c ^ m
        // (m < 8), whose group is (c / CPG) ^ (m / CPG): the "virtual" group c / CPG of the
        // step order (equal to the physical one for CPG >= 8) maps to physical group v ^ mg.
        constexpr int NG = G >= 128 ? 1 : 128 / G;
        constexpr int CPG = NC / NG;
        GroupQ gq[NG];
        bool bad = false;
#pragma unroll
        for (int v = 0; v < NG; ++v) {
          uint32_t mn, mx;
          if constexpr (S1::SYM) {
            mx = x[v * CPG][0] & 0x7FFF7FFFu;
#pragma unroll
            for (int c = v * CPG; c < (v + 1) * CPG; ++c)
#pragma unroll
              for (int i = 0; i < 4; ++i)
                if (c != v * CPG || i) mx = h2max<Tin>(mx, x[c][i] & 0x7FFF7FFFu);
            mn = mx;
          } else {
            mn = h2min<Tin>(x[v * CPG][0], x[v * CPG][1]);
            mx = h2max<Tin>(x[v * CPG][0], x[v * CPG][1]);
#pragma unroll
            for (int c = v * CPG; c < (v + 1) * CPG; ++c)
#pragma unroll
              for (int i = 0; i < 4; ++i)
                if (c > v * CPG || i > 1) {
                  mn = h2min<Tin>(mn, x[c][i]);
                  mx = h2max<Tin>(mx, x[c][i]);
                }
          }
          float hi = fmax_nan(h_lo<Tin>(mx), h_hi<Tin>(mx));
          float lo = S1::SYM ? -hi : fmin_nan(h_lo<Tin>(mn), h_hi<Tin>(mn));
          if constexpr (G == 256) {
            hi = fmax_nan(hi, __shfl_xor_sync(0xffffffffu, hi, 1));
            lo = S1::SYM ? -hi : fmin_nan(lo, __shfl_xor_sync(0xffffffffu, lo, 1));
          }
          const bool bv = !(fabsf(lo) <= 3.402823466e38f && fabsf(hi) <= 3.402823466e38f);
          bad |= bv;
          if constexpr (S1::MF) {  // scale = absmax / max_finite (codec.py:345), no zero point
            gq[v].s16 = __half_as_ushort(snap_scale((double)hi / a.c1.qdiv, a.c1.floor));
            gq[v].s = __half2float(__ushort_as_half(gq[v].s16));
            gq[v].r = __frcp_rn(gq[v].s);
            gq[v].z = 0u;
            gq[v].normal = true;
          } else {
            group_params<S1>(a.c1, lo, hi, gq[v]);
            if (bv) gq[v].z = S1::SYM ? gq[v].z : 0u;
          }
        }
        const uint32_t qmax = (1u << a.c1.bits) - 1u;
        uint32_t w[NC * CWPC];
#pragma unroll
        for (int v = 0; v < NG; ++v) {
          const GroupQ& g = gq[v];
          if constexpr (S1::MF) {
#pragma unroll
            for (int c = v * CPG; c < (v + 1) * CPG; ++c) chunk_codes_mf<S1, Tin>(x[c], g, w + c * CWPC);
            continue;
          }
          if (g.normal) {
#pragma unroll
            for (int c = v * CPG; c < (v + 1) * CPG; ++c) chunk_codes_packed<S1, Tin>(x[c], g, qmax, w + c * CWPC);
          } else {
#pragma unroll
            for (int c = v * CPG; c < (v + 1) * CPG; ++c)
              chunk_codes_clamped<S1, Tin>(x[c], g.s, (int)g.z, (int)qmax, w + c * CWPC);
          }
        }
        if constexpr (S1::SYM && !S1::MF) {
          const uint32_t xr = rep_xor(a.c1);
#pragma unroll
          for (int i = 0; i < NC * CWPC; ++i) w[i] ^= xr;
        }
        unswizzle_chunks<NC, CWPC>(w, m);
        constexpr int NV = NC * CWPC / 4;      // 16-B code vectors per lane
        constexpr int CB = 16 * NV;            // code bytes per lane (group)
        if (!(a.dbg & 32)) {
          // coalesced code stores: the warp's 32 groups of codes are contiguous in the slot;
          // stage them in the lanes' own (consumed) input regions, vector v at slot v ^ m,
          // then copy the warp's 32 * CB bytes out 512 B per instruction
          __syncwarp();  // every lane's shared loads of its group are consumed
#pragma unroll
          for (int v = 0; v < NV; ++v)
            asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(gb + 16 * (v ^ m)), "r"(w[4 * v]),
                         "r"(w[4 * v + 1]), "r"(w[4 * v + 2]), "r"(w[4 * v + 3])
                         : "memory");
          __syncwarp();
          const uint32_t wb = sbase + st * STAGE + part * 32 * (kGplG * 2);
          fence_proxy_async_smem();  // generic st.shared before the stage's next bulk (async-proxy) fill
          uint8_t* cw0 = jb.dst + ((int64_t)t * kTileElems + part * 32 * kGplG) * S1::SB / 8;
#pragma unroll
          for (int r = 0; r < NV; ++r) {
            const int x = 512 * r + 16 * lane, l = x / CB, v = (x % CB) / 16;
            st_v4(cw0 + x, lds128_(wb + l * (kGplG * 2) + 16 * (v ^ (l & 7))));
          }
        } else {
          uint8_t* cd = jb.dst + p0 * S1::SB / 8;
#pragma unroll
          for (int v = 0; v < NV; ++v)
            *reinterpret_cast<uint4*>(cd + 16 * v) = make_uint4(w[4 * v], w[4 * v + 1], w[4 * v + 2], w[4 * v + 3]);
        }
        const int64_t grp = p0 >> a.c1.gshift;  // the slice's first group
        const int mg = G == 32 ? (m >> 2) : 0;   // virtual -> physical group (G = 32)
        if (G != 256 || (lane & 1) == 0) {
#pragma unroll
          for (int v = 0; v < NG; ++v) {
            const int64_t gp = grp + (v ^ mg);
            *reinterpret_cast<unsigned short*>(jb.dst + a.c1.scales_off + 2 * gp) = gq[v].s16;
            if constexpr (!S1::SYM) jb.dst[a.c1.zeros_off + gp] = (uint8_t)gq[v].z;
          }
        }
        // the tile's stores are issued (each store consumed the thread's shared loads): every
        // thread hands the stage back for its own reads (FUSED: the producer then publishes rflag)
        mbar_arrive(empty0 + 8 * st);
        if (bad && jb.err) atomicOr(jb.err, jb.ecode);
      } else {
        // ragged tail: the 32-element lane codec over this warp's 4096 elements, 1024 at a time
        bool bad = false;
        for (int sub = 0; sub < kGplG / 32; ++sub) {
          const int64_t q0 = (int64_t)t * kTileElems + part * (32 * kGplG) + sub * (32 * kLaneElems) + lane * kLaneElems;
          const int nvalid = lane_valid(a.sub_len, q0);
          PackedLane<Tin> L;
          load_lane_src(jb.src, q0, jb.limit, nvalid, L);
          LaneQuant<8> q;
          bad |= quantize_lane<S1>(a.c1, L, nvalid, q);
          store_codes<S1>(a.c1, jb.dst, q0, nvalid, q, lane);
        }
        mbar_arrive(empty0 + 8 * st);
        if (bad && jb.err) atomicOr(jb.err, jb.ecode);
      }
  };
  if constexpr (!FUSED) {
    int st = 0, k = 0;
    uint32_t ph = 0;
    for (Iter it = it0; it.ok(); it.next(), ++k) {
      if (k % kGplSlots == slot) item(it.y, it.t, st, ph);  // S is a multiple of the slot count
      ring_next(st, ph, S);
    }
  } else {
    const DynIter& D = it0;
    for (int k = slot;; k += kGplSlots) {
      const int st = k % S;
      const uint32_t ph = (uint32_t)(k / S) & 1u;
      mbar_wait(full0 + 8 * st, ph);
      const int id = lds_id(D.meta + 4 * st);
      if (id < 0) break;
      int y, t;
      D.decode(id, y, t);
      item(y, t, st, ph);
    }
  }
}

// ------------------------------------------------------------------ group-lane quantize, any g in {32..256}

// Quantize with a lane per 128-element slice for group sizes 32, 64, 128 and
// 256 and both storage widths (k_qstream_gq: the single-GPU codec and the
// INT8 scatter). Same CTA shape, producer ring and coalesced staged code
// stores as q_role_gpl, but two passes over the staged slice: pass 1 reads the
// 16 XOR-swizzled vectors for the group bounds only, pass 2 reads them again
// and encodes chunk by chunk, so the 64 input words never sit in registers
// (INT8: no spills, 4 CTAs per SM). A slice holds 128 / g groups (g <= 128) or
// half a group (g = 256: the partner lane's bounds come over one shuffle). At
// step c a lane reads physical chunk c ^ m, whose group is (c / CPG) ^ (m /
// CPG): bounds and parameters are kept per step-order ("virtual") group and
// the metadata goes to the physical group's address.
template <typename Tin, class S1, int G, bool FUSED, class Iter>
__device__ __forceinline__ void q_role_gq(const FlashArgs& a, uint32_t sbase, int S, Iter it0, uint32_t bars = 0) {
  static_assert(sizeof(Tin) == 2, "16-bit inputs");
  static_assert(G == 32 || G == 64 || G == 128 || G == 256, "group size");
  static_assert(!FUSED, "the fused kernel uses q_role_gpl");
  constexpr uint32_t STAGE = kTileElems * 2;
  constexpr int SL = 128;                      // elements per lane slice
  constexpr int NC = SL / 8;                   // 8-element chunks per slice
  constexpr int NGL = G >= SL ? 1 : SL / G;    // groups per slice
  constexpr int CPG = NC / NGL;                // chunks per (virtual) group
  constexpr int CWPC = S1::SB / 4;             // code words per chunk
  constexpr int MSH = CPG >= 8 ? 0 : (CPG == 4 ? 2 : 1);  // m >> MSH: the swizzle's group-index bits
  const uint32_t full0 = bars ? bars : sbase + S * STAGE, empty0 = full0 + 8 * S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, kGplWpt);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == kGplWarps) {
    if (lane == 0) {
      int st = 0, k = 0, cy = -1;
      uint32_t ph = 0;
      QJob<Tin> jb;
      for (Iter it = it0; it.ok(); it.next(), ++k) {
        if (k >= S) mbar_wait(empty0 + 8 * st, ph ^ 1);
        if (it.y != cy) {
          jb = qjob<Tin>(a, it.y);
          cy = it.y;
        }
        const int64_t e0 = (int64_t)it.t * kTileElems;
        const uint32_t bytes = (uint32_t)(tile_valid(a.sub_len, jb.limit, e0) * 2) & ~15u;
        mbar_arrive_expect_tx(full0 + 8 * st, bytes);
        if (bytes) bulk_g2s(sbase + st * STAGE, jb.src + e0, bytes, full0 + 8 * st);
        ring_next(st, ph, S);
      }
    }
    return;
  }
  const int slot = warp / kGplWpt, part = warp % kGplWpt;
  const int m = lane & 7;
  const int mg = CPG >= 8 ? 0 : (m >> MSH);  // physical group = virtual ^ mg
  const int li = part * 32 + lane;           // this lane's slice within a tile
  const uint32_t qmax = (1u << a.c1.bits) - 1u;
  int st = 0, cy = -1, k = 0;
  uint32_t ph = 0;
  QJob<Tin> jb;
  for (Iter it = it0; it.ok(); it.next(), ++k) {
    if (k % kGplSlots == slot) {
      if (it.y != cy) {
        jb = qjob<Tin>(a, it.y);
        cy = it.y;
      }
      const int64_t p0 = (int64_t)it.t * kTileElems + li * SL;
      const bool whole = p0 + SL <= a.sub_len && p0 + SL <= jb.limit;
      mbar_wait(full0 + 8 * st, ph);
      if (__all_sync(0xffffffffu, whole)) {
        const uint32_t gb = sbase + st * STAGE + li * (SL * 2);
        // ---- pass 1: bounds per virtual group (16-bit packed, exact)
        uint32_t mn[NGL], mx[NGL];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const uint4 u = lds128_(gb + 16 * (c ^ m));
          const int v = c / CPG;
          const uint32_t xs[4] = {u.x, u.y, u.z, u.w};
          if constexpr (S1::SYM) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const uint32_t ab = xs[i] & 0x7FFF7FFFu;
              mx[v] = (c % CPG == 0 && i == 0) ? ab : h2max<Tin>(mx[v], ab);
            }
          } else {
            if (c % CPG == 0) {
              mn[v] = h2min<Tin>(xs[0], xs[1]);
              mx[v] = h2max<Tin>(xs[0], xs[1]);
            } else {
              mn[v] = h2min<Tin>(mn[v], xs[0]);
              mx[v] = h2max<Tin>(mx[v], xs[0]);
              mn[v] = h2min<Tin>(mn[v], xs[1]);
              mx[v] = h2max<Tin>(mx[v], xs[1]);
            }
            mn[v] = h2min<Tin>(mn[v], xs[2]);
            mx[v] = h2max<Tin>(mx[v], xs[2]);
            mn[v] = h2min<Tin>(mn[v], xs[3]);
            mx[v] = h2max<Tin>(mx[v], xs[3]);
          }
        }
        GroupQ gq[NGL];
        bool bad = false;
#pragma unroll
        for (int v = 0; v < NGL; ++v) {
          float hi = fmax_nan(h_lo<Tin>(mx[v]), h_hi<Tin>(mx[v]));
          float lo = S1::SYM ? -hi : fmin_nan(h_lo<Tin>(mn[v]), h_hi<Tin>(mn[v]));
          if constexpr (G > SL) {  // the partner lane holds the other half of the group
            hi = fmax_nan(hi, __shfl_xor_sync(0xffffffffu, hi, 1));
            lo = S1::SYM ? -hi : fmin_nan(lo, __shfl_xor_sync(0xffffffffu, lo, 1));
          }
          const bool b = !(fabsf(lo) <= 3.402823466e38f && fabsf(hi) <= 3.402823466e38f);
          group_params<S1>(a.c1, lo, hi, gq[v]);
          if (b) gq[v].z = S1::SYM ? gq[v].z : 0u;
          bad |= b;
        }
        // ---- pass 2: re-read each chunk and encode it with its group's parameters
        uint32_t w[NC * CWPC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const uint4 u = lds128_(gb + 16 * (c ^ m));
          const uint32_t xs[4] = {u.x, u.y, u.z, u.w};
          const GroupQ& g = gq[c / CPG];
          if (g.normal)
            chunk_codes_packed<S1, Tin>(xs, g, qmax, w + c * CWPC);
          else
            chunk_codes_clamped<S1, Tin>(xs, g.s, (int)g.z, (int)qmax, w + c * CWPC);
        }
        if constexpr (S1::SYM) {
          const uint32_t xr = rep_xor(a.c1);
#pragma unroll
          for (int i = 0; i < NC * CWPC; ++i) w[i] ^= xr;
        }
        unswizzle_chunks<NC, CWPC>(w, m);
        constexpr int NV = NC * CWPC / 4;  // 16-B code vectors per lane
        constexpr int CB = 16 * NV;        // code bytes per lane
        __syncwarp();  // every lane's shared loads of its slice are consumed
#pragma unroll
        for (int v = 0; v < NV; ++v)
          asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(gb + 16 * (v ^ m)), "r"(w[4 * v]),
                       "r"(w[4 * v + 1]), "r"(w[4 * v + 2]), "r"(w[4 * v + 3])
                       : "memory");
        __syncwarp();
        const uint32_t wb = sbase + st * STAGE + part * 32 * (SL * 2);
        fence_proxy_async_smem();
        uint8_t* cw0 = jb.dst + ((int64_t)it.t * kTileElems + part * 32 * SL) * S1::SB / 8;
#pragma unroll
        for (int r = 0; r < NV; ++r) {
          const int x = 512 * r + 16 * lane, l = x / CB, v = (x % CB) / 16;
          st_v4(cw0 + x, lds128_(wb + l * (SL * 2) + 16 * (v ^ (l & 7))));
        }
        // ---- metadata of the slice's groups (physical group v ^ mg)
        if constexpr (G > SL) {
          if ((lane & 1) == 0) {
            const int64_t grp = p0 / G;
            *reinterpret_cast<unsigned short*>(jb.dst + a.c1.scales_off + 2 * grp) = gq[0].s16;
            if constexpr (!S1::SYM) jb.dst[a.c1.zeros_off + grp] = (uint8_t)gq[0].z;
          }
        } else {
          const int64_t grp0 = p0 / G;
#pragma unroll
          for (int v = 0; v < NGL; ++v) {
            const int64_t grp = grp0 + (v ^ mg);
            *reinterpret_cast<unsigned short*>(jb.dst + a.c1.scales_off + 2 * grp) = gq[v].s16;
            if constexpr (!S1::SYM) jb.dst[a.c1.zeros_off + grp] = (uint8_t)gq[v].z;
          }
        }
        // every store of the slice is issued: hand the stage back (FUSED: the producer publishes)
        __syncwarp();
        if (lane == 0) mbar_arrive(empty0 + 8 * st);
        if (bad && jb.err) atomicOr(jb.err, jb.ecode);
      } else {
        // ragged tail: the 32-element lane codec over this warp's 4096 elements, 1024 at a time
        bool bad = false;
        for (int sub = 0; sub < SL / 32; ++sub) {
          const int64_t q0 = (int64_t)it.t * kTileElems + part * (32 * SL) + sub * (32 * kLaneElems) + lane * kLaneElems;
          const int nvalid = lane_valid(a.sub_len, q0);
          PackedLane<Tin> L;
          load_lane_src(jb.src, q0, jb.limit, nvalid, L);
          LaneQuant<8> q;
          bad |= quantize_lane<S1>(a.c1, L, nvalid, q);
          store_codes<S1>(a.c1, jb.dst, q0, nvalid, q, lane);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty0 + 8 * st);
        if (bad && jb.err) atomicOr(jb.err, jb.ecode);
      }
    }
    ring_next(st, ph, S);
  }
}

// ------------------------------------------------------------------ group-per-lane reduce role

// acc (+)= (c - z) * s for NW code words (8 offset-binary INT4 codes each),
// into pairs in the INT4 pairing (8i+a, 8i+a+4): decode_pairs over NW words
template <int NW>
__device__ __forceinline__ void decode_words4(const uint32_t* cw, float s, float mz, uint64_t* acc) {
  const uint64_t S2 = f2_splat(s), NMZ2 = f2_splat(-mz);
  const uint64_t S16 = f2_splat(s * 0.0625f), NMZ16 = f2_splat(-fmaf(mz, 16.0f, -125829120.0f));
  auto emit = [&](int idx, uint32_t va, uint32_t vb, uint64_t nmz, uint64_t sc) {
    uint64_t M;
    asm("mov.b64 %0, {%1,%2};" : "=l"(M) : "r"(va), "r"(vb));
    acc[idx] = f2_fma(f2_add(M, nmz), sc, acc[idx]);
  };
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    const uint32_t lo = cw[i] & 0x0F0F0F0Fu, hi = cw[i] & 0xF0F0F0F0u;
    emit(4 * i + 0, __byte_perm(lo, 0x4B000000u, 0x7440u), __byte_perm(lo, 0x4B000000u, 0x7442u), NMZ2, S2);
    emit(4 * i + 2, __byte_perm(lo, 0x4B000000u, 0x7441u), __byte_perm(lo, 0x4B000000u, 0x7443u), NMZ2, S2);
    emit(4 * i + 1, __byte_perm(hi, 0x4B000000u, 0x7440u), __byte_perm(hi, 0x4B000000u, 0x7442u), NMZ16, S16);
    emit(4 * i + 3, __byte_perm(hi, 0x4B000000u, 0x7441u), __byte_perm(hi, 0x4B000000u, 0x7443u), NMZ16, S16);
  }
}

// the same for NW INT8 code words (4 codes each) into the INT8 pairing (4i+a, 4i+a+2)
template <int NW>
__device__ __forceinline__ void decode_words8(const uint32_t* cw, float s, float mz, uint64_t* acc) {
  const uint64_t S2 = f2_splat(s), NMZ2 = f2_splat(-mz);
  auto emit = [&](int idx, uint32_t va, uint32_t vb) {
    uint64_t M;
    asm("mov.b64 %0, {%1,%2};" : "=l"(M) : "r"(va), "r"(vb));
    acc[idx] = f2_fma(f2_add(M, NMZ2), S2, acc[idx]);
  };
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    emit(2 * i + 0, __byte_perm(cw[i], 0x4B000000u, 0x7440u), __byte_perm(cw[i], 0x4B000000u, 0x7442u));
    emit(2 * i + 1, __byte_perm(cw[i], 0x4B000000u, 0x7441u), __byte_perm(cw[i], 0x4B000000u, 0x7443u));
  }
}
template <int SB, int NW>
__device__ __forceinline__ void decode_words(const uint32_t* cw, float s, float mz, uint64_t* acc) {
  if constexpr (SB == 4)
    decode_words4<NW>(cw, s, mz, acc);
  else
    decode_words8<NW>(cw, s, mz, acc);
}

// acc (+)= grid * s for NW minifloat code words into the pairing of the storage width (e4m3 /
// e5m2 bytes: (4i+a, 4i+a+2); e2m1 nibbles: (8i+a, 8i+a+4)). grid * s is exact (a few-bit
// grid value times an fp16 scale), so the FFMA2 rounds once like the reference's add
template <class Spec, int NW>
__device__ __forceinline__ void decode_words_mf(const uint32_t* cw, float s, uint64_t* acc) {
  const uint64_t S2 = f2_splat(s);
  auto emit = [&](int idx, uint32_t two) {
    float v0, v1;
    mf_dec2(Spec::FMT, two, v0, v1);
    uint64_t M;
    asm("mov.b64 %0, {%1,%2};" : "=l"(M) : "f"(v0), "f"(v1));
    acc[idx] = f2_fma(M, S2, acc[idx]);
  };
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    if constexpr (Spec::SB == 8) {
      emit(2 * i + 0, __byte_perm(cw[i], 0u, 0x0020u) & 0xFFFFu);  // elements 4i, 4i+2
      emit(2 * i + 1, __byte_perm(cw[i], 0u, 0x0031u) & 0xFFFFu);  // 4i+1, 4i+3
    } else {
      const uint32_t lo = cw[i] & 0x0F0F0F0Fu, hi = (cw[i] >> 4) & 0x0F0F0F0Fu;
      const uint32_t t = lo | (lo >> 12), u = hi | (hi >> 12);  // byte 0: (a, a+4), byte 1: (a+2, a+6)
      emit(4 * i + 0, t & 0xFFu);
      emit(4 * i + 2, (t >> 8) & 0xFFu);
      emit(4 * i + 1, u & 0xFFu);
      emit(4 * i + 3, (u >> 8) & 0xFFu);
    }
  }
}

// element e of accumulators held in the pairing of storage width SB
template <int SB = 4>
__device__ __forceinline__ float acc_get(const uint64_t* acc, int e) {
  float a, b;
  if constexpr (SB == 4) {
    f2_unpack(acc[(e >> 3) * 4 + (e & 3)], a, b);
    return (e & 4) ? b : a;
  } else {
    f2_unpack(acc[(e >> 2) * 2 + (e & 1)], a, b);
    return (e & 2) ? b : a;
  }
}

// g = 128 reduce with 64 elements per lane, 2 lanes per group (k_rstream_gpl).
// Every source piece -- the own one included -- comes from the receive slots:
// with FlashArgs::ownq the scatter also stage-1 quantizes the rank's own piece
// into recv_slot[j][j] (collectives.py:364-365: the own piece is QDQ'd like
// the others), so the reduce never reads the bf16 input and never repeats the
// stage-1 group statistics; it decodes N pieces in ascending source rank
// (collectives.py:182-187), stage-2 quantizes the fp32 sum, stores the codes
// into every peer's gather slot [j] and decodes its own output
// (collectives.py:378). The 32-element layout of r_role spreads a group over 4
// lanes; here a lane pair shares a group (one shuffle step) and a lane keeps
// its 64 fp32 accumulators as 32 register pairs in the codec's pairing
// (decode, accumulate and re-encode never move registers).
// Shared memory: a ring of R piece slots (codes | fp16 scales | zeros, one
// source's share of a tile, full/empty mbarrier per slot) that the producer
// warp streams continuously -- piece (item k, source s) lands in slot
// (k N + s) % R and is handed back by the 4 consumer warps as soon as they
// decoded it, so the next tile's pieces land during this tile's sum, stage-2
// quantize and stores -- plus a 4-KB output staging buffer per warp (the
// output leaves as one coalesced 512-B store per warp instruction).
// FUSED: the producer waits for every source's rflag of the tile before its
// copies and publishes gflag of item k-2 once the consumers' done barrier of
// that item completed (every stage-2 store into a peer's gather slot issued).
// Whole tiles only (launch_rstream falls back to r_role otherwise).
constexpr int kRgEpl = 64;                              // elements per lane
constexpr int kRgLpg = kGplG / kRgEpl;                  // lanes per group (2)
constexpr int kRgWpt = kTileElems / (32 * kRgEpl);      // warps per tile (4)
constexpr uint32_t kRgStage = kTileElems * 2;           // output staging bytes (4 KB per warp)
constexpr int kRgMaxRing = 32;                          // piece slots at most
constexpr int kRgDone = 4;                              // FUSED: done-barrier ring (publish lag 2)

// bytes of one piece slot, the barrier region, the whole layout for a ring of R slots
__host__ __device__ inline uint32_t rg_piece_bytes(const DevCodec& c1) { return peer_codes_bytes(c1) + peer_meta_bytes(c1); }
__host__ __device__ inline uint32_t rg_bars_off(const DevCodec& c1, int R) { return kRgStage + (uint32_t)R * rg_piece_bytes(c1); }
__host__ __device__ inline uint32_t rg_smem_bytes(const DevCodec& c1, int R) {
  return rg_bars_off(c1, R) + 8 * (2 * R + kRgDone) + 4 * (R + kRgDone);
}
// ring depth for a per-CTA shared-memory budget (at least 2)
__host__ __device__ inline int rg_ring_for(const DevCodec& c1, uint32_t budget) {
  const uint32_t per = rg_piece_bytes(c1) + 8 * 2 + 4;
  const uint32_t fixed = kRgStage + 12 * kRgDone;
  int R = budget > fixed ? (int)((budget - fixed) / per) : 0;
  return R < 2 ? 2 : (R > kRgMaxRing ? kRgMaxRing : R);
}

template <typename Tin, typename Tout, class S1, class S2, bool FUSED, class Iter>
__device__ __forceinline__ void r_role_gpl(const FlashArgs& a, uint32_t sbase, int R, Iter it0, uint32_t bars_in = 0) {
  static_assert(sizeof(Tin) == 2 && (sizeof(Tout) == 2 || sizeof(Tout) == 4), "16-bit inputs, 16/32-bit outputs");
  static_assert(S1::SB == S2::SB, "one storage width for both stages");
  static_assert(kGplWarps == kRgWpt, "one tile per pass of the consumer warps");
  constexpr int SB = S1::SB;
  constexpr int NC = kRgEpl / 8;         // 8-element chunks per lane
  constexpr int CWPC = SB / 4;           // code words per chunk
  constexpr int NW = NC * CWPC;          // code words per lane
  const uint32_t PC = peer_codes_bytes(a.c1), PM = peer_meta_bytes(a.c1), SCB = peer_scale_bytes(a.c1);
  const uint32_t PB = rg_piece_bytes(a.c1);
  const int NP = a.world;
  const uint32_t ring0 = sbase + kRgStage;
  const uint32_t bars = bars_in ? bars_in : sbase + rg_bars_off(a.c1, R);
  const uint32_t full0 = bars, empty0 = bars + 8 * R, done0 = bars + 16 * R;
  const uint32_t meta = done0 + 8 * kRgDone;  // FUSED: item id beside the slot of its first piece
  const uint32_t hist = meta + 4 * R;         // FUSED: ids of the last kRgDone items (producer)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < R; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, kRgWpt * 32);  // every consumer thread releases its own reads
    }
    for (int s = 0; s < kRgDone; ++s) mbar_init(done0 + 8 * s, kRgWpt);
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == kGplWarps) {  // producer (lane 0 issues; FUSED: the warp waits for the tile's rflags)
    // ring position of the next piece: slot, phase, whether the slot was used before
    // (incremental: a runtime modulo costs ~20 instructions per piece)
    uint32_t psl = 0, pph = 0;
    bool pused = false;
    auto slot_acquire = [&]() -> uint32_t {  // lane 0: the next ring slot, once handed back
      const uint32_t sl = psl;
      if (pused) mbar_wait(empty0 + 8 * sl, pph ^ 1u);
      if (++psl == (uint32_t)R) {
        psl = 0;
        pph ^= 1u;
        pused = true;
      }
      return sl;
    };
    auto issue = [&](int y, int t, int id) {
      const int j = a.rank_lo + y;
      const int64_t e0 = (int64_t)t * kTileElems;
      const int64_t grp0 = e0 >> a.c1.gshift;
      if constexpr (FUSED)  // lane s waits for rank s's stage-1 piece of tile t (rflag[j][s][t])
        warp_wait_flags(a, j, rflag(a, j, lane) + t, lane, lane < a.world, kPhReduce);
      if (lane == 0) {
        const uint32_t zb = S1::SYM ? 0u : PM - SCB;
        for (int s = 0; s < NP; ++s) {
          const uint32_t sl = slot_acquire();
          if (FUSED && s == 0) sts32(meta + 4 * sl, id);
          const uint32_t bar = full0 + 8 * sl, dst = ring0 + sl * PB;
          const uint8_t* src = recv_slot(a, j, s);
          mbar_arrive_expect_tx(bar, PC + SCB + zb);
          bulk_g2s(dst, src + e0 * SB / 8, PC, bar);
          bulk_g2s(dst + PC, src + a.c1.scales_off + grp0 * 2, SCB, bar);
          if (zb) bulk_g2s(dst + PC + SCB, src + a.c1.zeros_off + grp0, zb, bar);
        }
      }
      __syncwarp();
    };
    if constexpr (!FUSED) {
      for (Iter it = it0; it.ok(); it.next()) issue(it.y, it.t, 0);
    } else {
      // dynamic dealing (DynIter); after issuing item k, wait for item k-2's done barrier (its
      // stage-2 codes are stored into every peer's gather slot) and publish its gflags
      const DynIter& D = it0;
      int id = 0, k = 0;
      if (lane == 0) id = D.grab();
      id = __shfl_sync(0xffffffffu, id, 0);
      auto publish_k = [&](int kk) {
        if (lane == 0) {
          mbar_wait(done0 + 8 * (kk % kRgDone), (uint32_t)(kk / kRgDone) & 1u);
          int y, t;
          D.decode(lds_id(hist + 4 * (kk % kRgDone)), y, t);
          publish_reduce(a, y, t, D.ep);
        }
      };
      for (;; ++k) {
        int nid = 0;
        if (lane == 0 && id < D.items) nid = D.grab();  // the next id is in flight during this item
        if (id >= D.items) break;
        int y, t;
        D.decode(id, y, t);
        if (lane == 0) sts32(hist + 4 * (k % kRgDone), id);
        issue(y, t, id);
        if (k >= 2) publish_k(k - 2);
        id = __shfl_sync(0xffffffffu, nid, 0);
      }
      if (lane == 0) {  // end sentinel in the slot of the next item's first piece
        const uint32_t sl = slot_acquire();
        sts32(meta + 4 * sl, -1);
        mbar_arrive(full0 + 8 * sl);
      }
      for (int kk = k >= 2 ? k - 2 : 0; kk < k; ++kk) publish_k(kk);
      __syncwarp();
    }
    return;
  }
  const int m = lane & 7;
  const int li = warp * 32 + lane;         // lane slice of the tile: elements [li*64, li*64+64)
  const int gt = li / kRgLpg;              // tile-local group
  const bool lead = (li & (kRgLpg - 1)) == 0;
  const uint32_t xr1 = S1::MF ? 0u : rep_xor(a.c1), xr2 = S2::MF ? 0u : rep_xor(a.c2);
  const uint32_t qmax2 = (1u << a.c2.bits) - 1u;
  const uint32_t lb = sbase + li * (kRgEpl * 2);  // the lane's 128-B region of the output staging
  const uint32_t dep_zero = (uint32_t)a.tiles >> 31;  // 0 at run time, opaque to the compiler
  uint32_t csl = 0, cph = 0;                      // ring position of the next piece to consume
  auto item = [&](int k, int y, int t) {
    const int j = a.rank_lo + y;
    const int64_t seg0 = (int64_t)j * a.seg + a.sub_off;
    const int64_t e0 = (int64_t)t * kTileElems;
    const int64_t p0 = e0 + li * kRgEpl;  // lane slice start in the round
    // ---- fp32 sum of the N stage-1 pieces in ascending source rank
    uint64_t acc[4 * NC];
#pragma unroll
    for (int e = 0; e < 4 * NC; ++e) acc[e] = 0ull;
    for (int s = 0; s < NP; ++s) {
      mbar_wait(full0 + 8 * csl, cph);
      const uint32_t src = ring0 + csl * PB;
      uint32_t cw[NW];
#pragma unroll
      for (int v = 0; v < NW / 4; ++v) {
        const uint4 u = lds128_(src + li * (kRgEpl * SB / 8) + 16 * v);
        cw[4 * v] = u.x;
        cw[4 * v + 1] = u.y;
        cw[4 * v + 2] = u.z;
        cw[4 * v + 3] = u.w;
      }
      unsigned short sh;
      asm volatile("ld.shared.u16 %0, [%1];" : "=h"(sh) : "r"(src + PC + 2 * gt) : "memory");
      float zf;
      if constexpr (S1::MF) {  // minifloat codes: no zero point, stored as is
        zf = 0.0f;
      } else if constexpr (S1::SYM) {
        zf = (float)(1 << (a.c1.bits - 1));
#pragma unroll
        for (int w = 0; w < NW; ++w) cw[w] ^= xr1;
      } else {
        uint32_t zz;
        asm volatile("ld.shared.u8 %0, [%1];" : "=r"(zz) : "r"(src + PC + SCB + gt) : "memory");
        zf = (float)zz;
      }
      // hand the slot back, each thread for its own reads (release.cta per thread), with a data
      // dependency on every loaded vector and the metadata: the arrive cannot issue before the
      // loads have returned. (The shared loads carry "memory" clobbers so the compiler cannot
      // hoist them above the full-barrier wait: an INT8-sym build that did read stale pieces at
      // four CTAs per SM, tools/dbg_sym8b.py.)
      uint32_t dep = (uint32_t)sh ^ __float_as_uint(zf);
#pragma unroll
      for (int v = 0; v < NW / 4; ++v) dep ^= cw[4 * v];
      mbar_arrive_dep(empty0 + 8 * csl, dep, dep_zero);
      if constexpr (S1::MF)
        decode_words_mf<S1, NW>(cw, __half2float(__ushort_as_half(sh)), acc);
      else
        decode_words<SB, NW>(cw, __half2float(__ushort_as_half(sh)), 8388608.0f + zf, acc);
      if (++csl == (uint32_t)R) {
        csl = 0;
        cph ^= 1u;
      }
    }
    // ---- stage-2 quantize of the sum
    float lo2, hi2;
    {
      float a0 = acc_get<SB>(acc, 0), b0 = S2::SYM ? fabsf(a0) : a0;
#pragma unroll
      for (int e = 1; e < kRgEpl; e += 2) {
        const float u = acc_get<SB>(acc, e), v = e + 1 < kRgEpl ? acc_get<SB>(acc, e + 1) : u;
        if constexpr (S2::SYM) {
          b0 = fmax3_nan(b0, fabsf(u), fabsf(v));
        } else {
          a0 = fmin3_nan(a0, u, v);
          b0 = fmax3_nan(b0, u, v);
        }
      }
      b0 = fmax_nan(b0, __shfl_xor_sync(0xffffffffu, b0, 1));
      if constexpr (!S2::SYM) a0 = fmin_nan(a0, __shfl_xor_sync(0xffffffffu, a0, 1));
      hi2 = b0;
      lo2 = S2::SYM ? -b0 : a0;
    }
    const bool bad = !(fabsf(lo2) <= 3.402823466e38f && fabsf(hi2) <= 3.402823466e38f);
    GroupQ g2;
    if constexpr (S2::MF) {  // scale = absmax / max_finite (codec.py:345), no zero point
      g2.s16 = __half_as_ushort(snap_scale((double)hi2 / a.c2.qdiv, a.c2.floor));
      g2.s = __half2float(__ushort_as_half(g2.s16));
      g2.r = __frcp_rn(g2.s);
      g2.z = 0u;
      g2.normal = true;
    } else {
      group_params<S2>(a.c2, lo2, hi2, g2);
      if (bad) g2.z = S2::SYM ? g2.z : 0u;
    }
    uint32_t w2[NW];
    if constexpr (S2::MF) {
      // RN32(x / s) by reciprocal + one FMA correction (pairwise), then cvt.rn.satfinite
      const uint64_t R2 = f2_splat(g2.r), NS2 = f2_splat(-g2.s);
      auto quo = [&](uint64_t X, float& qa, float& qb) {
        const uint64_t T = f2_mul(X, R2);
        f2_unpack(f2_fma(f2_fma(T, NS2, X), R2, T), qa, qb);
      };
#pragma unroll
      for (int i = 0; i < NW; ++i) {
        if constexpr (SB == 8) {
          float q0, q1, q2, q3;
          quo(acc[2 * i], q0, q2);
          quo(acc[2 * i + 1], q1, q3);
          w2[i] = mf_fix_zero<S2::FMT>(mf_enc2_raw(S2::FMT, q0, q1) | (mf_enc2_raw(S2::FMT, q2, q3) << 16));
        } else {
          float q[8];
#pragma unroll
          for (int aa = 0; aa < 4; ++aa) quo(acc[4 * i + aa], q[aa], q[aa + 4]);
          w2[i] = mf_fix_zero<S2::FMT>(mf_enc2_raw(S2::FMT, q[0], q[1]) | (mf_enc2_raw(S2::FMT, q[2], q[3]) << 8) |
                                       (mf_enc2_raw(S2::FMT, q[4], q[5]) << 16) |
                                       (mf_enc2_raw(S2::FMT, q[6], q[7]) << 24));
        }
      }
    } else if (g2.normal) {
      const uint64_t R2 = f2_splat(g2.r), NS2 = f2_splat(-g2.s), C2 = f2_splat(12582912.0f);
      const uint32_t Z2 = g2.z * 0x00010001u, Q2 = qmax2 * 0x00010001u;
      auto code_pair = [&](uint64_t X) -> uint32_t {
        const uint64_t T = f2_mul(X, R2);
        const uint64_t Q = f2_fma(f2_fma(T, NS2, X), R2, T);
        const uint64_t Y = S2::CEIL ? f2_add_rp(Q, C2) : f2_add(Q, C2);
        uint32_t ya, yb;
        f2_bits(Y, ya, yb);
        const uint32_t pp = __byte_perm(ya, yb, 0x5410);
        const uint32_t c = __viaddmax_s16x2(pp, Z2, 0u);
        return __vimin3_s16x2(c, Q2, Q2);
      };
      if constexpr (SB == 4) {
#pragma unroll
        for (int i = 0; i < NW; ++i)
          w2[i] = code_pair(acc[4 * i]) + (code_pair(acc[4 * i + 1]) << 4) + (code_pair(acc[4 * i + 2]) << 8) +
                  (code_pair(acc[4 * i + 3]) << 12);
      } else {
#pragma unroll
        for (int i = 0; i < NW; ++i) w2[i] = code_pair(acc[2 * i]) + (code_pair(acc[2 * i + 1]) << 8);
      }
    } else {  // float clamp before rounding (the lane_codes path)
      const float r = __frcp_rn(g2.s);
      const float lob = -(float)g2.z, hib = (float)(qmax2 - g2.z);
      const int zb = (int)g2.z - 0x4B400000;
      constexpr int EPW = 32 / SB;  // elements per code word
#pragma unroll
      for (int i = 0; i < NW; ++i) {
        uint32_t wv = 0;
#pragma unroll
        for (int e = 0; e < EPW; ++e) {
          const float xv = acc_get<SB>(acc, EPW * i + e);
          const float tq = xv * r;
          const float q1 = fmaf(fmaf(-tq, g2.s, xv), r, tq);
          const float qc = fminf(fmaxf(q1, lob), hib);
          const float yv = S2::CEIL ? __fadd_ru(qc, 12582912.0f) : __fadd_rn(qc, 12582912.0f);
          wv |= (uint32_t)(__float_as_int(yv) + zb) << (SB * e);
        }
        w2[i] = wv;
      }
    }
    // ---- every peer's gather slot [j] (stored codes: offset binary ^ xr for sym)
    {
      const int64_t slot_off = (int64_t)(a.world + j) * a.slot_bytes;
      const int64_t grp = p0 >> a.c2.gshift;
      uint4 cv[NW / 4];
#pragma unroll
      for (int v = 0; v < NW / 4; ++v)
        cv[v] = make_uint4(w2[4 * v] ^ xr2, w2[4 * v + 1] ^ xr2, w2[4 * v + 2] ^ xr2, w2[4 * v + 3] ^ xr2);
      for (int p = j + 1;; ++p) {
        if (p == a.world) p = 0;
        if (p == j) break;
        uint8_t* b = a.blk[p] + slot_off;
        uint8_t* cd = b + p0 * SB / 8;
#pragma unroll
        for (int v = 0; v < NW / 4; ++v) *reinterpret_cast<uint4*>(cd + 16 * v) = cv[v];
        if (lead) {
          *reinterpret_cast<unsigned short*>(b + a.c2.scales_off + 2 * grp) = g2.s16;
          if constexpr (!S2::SYM) b[a.c2.zeros_off + grp] = (uint8_t)g2.z;
        }
      }
    }
    if constexpr (FUSED) {  // this item's gather-slot stores are issued (the producer publishes gflag)
      __syncwarp();
      if (lane == 0) mbar_arrive(done0 + 8 * (k % kRgDone));
    }
    // ---- own output: the owner decodes its own payload (collectives.py:378), staged
    // through the warp's own 4-KB buffer (swizzled), then one coalesced copy
    {
#pragma unroll
      for (int e = 0; e < 4 * NC; ++e) acc[e] = 0ull;
      if constexpr (S2::MF)
        decode_words_mf<S2, NW>(w2, g2.s, acc);  // 0 + grid s: exact, +0 for the +0 code
      else
        decode_words<SB, NW>(w2, g2.s, 8388608.0f + (float)g2.z, acc);  // 0 + (c - z) s: exact, never -0
      if constexpr (sizeof(Tout) == 4) {
        // fp32 outputs: the lane's 64 elements (256 contiguous bytes) as 16-B stores; a warp
        // instruction covers half of 32 sectors, the next one the other half (merged in L2)
        float* ob = reinterpret_cast<float*>(a.out[j]) + seg0 + p0;
#pragma unroll
        for (int c = 0; c < 2 * NC; ++c)
          st_v4(ob + 4 * c, make_uint4(__float_as_uint(acc_get<SB>(acc, 4 * c)), __float_as_uint(acc_get<SB>(acc, 4 * c + 1)),
                                       __float_as_uint(acc_get<SB>(acc, 4 * c + 2)),
                                       __float_as_uint(acc_get<SB>(acc, 4 * c + 3))));
      } else {
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          uint32_t h[4];
#pragma unroll
          for (int qq = 0; qq < 4; ++qq)
            h[qq] = pack2(acc_get<SB>(acc, 8 * c + 2 * qq), acc_get<SB>(acc, 8 * c + 2 * qq + 1), (Tout*)nullptr);
          asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(lb + 16 * (c ^ m)), "r"(h[0]), "r"(h[1]),
                       "r"(h[2]), "r"(h[3])
                       : "memory");
        }
        __syncwarp();
        const uint32_t wbase = sbase + warp * (32 * kRgEpl * 2);
        uint8_t* ob = reinterpret_cast<uint8_t*>(reinterpret_cast<Tout*>(a.out[j]) + seg0 + e0 + warp * (32 * kRgEpl));
        // byte 512 v + 16 lane of the warp's output = chunk qq = lane % 8 of slice l = 4 v + lane / 8,
        // stored at l * 128 + 16 (qq ^ (l & 7)) (conflict-free for each 8-lane phase)
#pragma unroll
        for (int v = 0; v < NC; ++v) {
          const int l = 4 * v + (lane >> 3), qq = lane & 7;
          st_v4(ob + 512 * v + 16 * lane, lds128_(wbase + l * (kRgEpl * 2) + 16 * (qq ^ (l & 7))));
        }
        __syncwarp();  // the staging buffer's loads are complete before the next item rewrites it
      }
    }
    if (bad) atomicOr(errw(a, j), make_err(kErrNonFinite, kPhReduce, j, j));
    if (a.dbg & 4096) consumers_sync<kRgWpt * 32>();  // A/B: consumer warps in lockstep per tile
  };
  if constexpr (!FUSED) {
    int k = 0;
    for (Iter it = it0; it.ok(); it.next(), ++k) item(k, it.y, it.t);
  } else {
    const DynIter& D = it0;
    for (int k = 0;; ++k) {
      mbar_wait(full0 + 8 * csl, cph);
      const int id = lds_id(meta + 4 * csl);
      if (id < 0) break;
      int y, t;
      D.decode(id, y, t);
      item(k, y, t);
    }
  }
}

// ------------------------------------------------------------------ reduce role

// owner j = rank_lo + y: own segment QDQ + N-1 received pieces -> fp32 sum
// (ascending source rank) -> stage-2 quantize -> every peer's gather slot [j]
// + own output. FUSED: wait rflag[j][*][t] before the copies, raise
// gflag[p][j][t] for every peer p after the stores.
template <typename Tin, typename Tout, class S1, class S2, bool FUSED, class Iter>
__device__ __forceinline__ void r_role(const FlashArgs& a, uint32_t sbase, int S, Iter it0) {
  static_assert(sizeof(Tin) == 2, "16-bit inputs");
  const uint32_t SBY = rstage_bytes(a.c1, a.world);
  const uint32_t PC = peer_codes_bytes(a.c1), PM = peer_meta_bytes(a.c1), SCB = peer_scale_bytes(a.c1);
  // one full barrier per piece of a stage (own input, then the N-1 peers in rank
  // order), so consumers start on the own tile and each peer as soon as it lands
  const int NP = a.world;
  const uint32_t full0 = sbase + S * SBY, empty0 = full0 + 8 * S * NP;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S * NP; ++s) mbar_init(full0 + 8 * s, 1);
    for (int s = 0; s < S; ++s) mbar_init(empty0 + 8 * s, kConsumerWarps);
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == kConsumerWarps) {
    int st = 0, k = 0;
    uint32_t ph = 0;
    for (Iter it = it0; it.ok(); it.next(), ++k) {
      const int j = a.rank_lo + it.y;
      if constexpr (FUSED) {  // lanes s != j wait for rank s's stage-1 piece of tile t
        warp_wait_flags(a, j, rflag(a, j, lane) + it.t, lane, lane < a.world && lane != j, kPhReduce);
      }
      if (lane == 0) {
        if (k >= S) mbar_wait(empty0 + 8 * st, ph ^ 1);
        const int64_t e0 = (int64_t)it.t * kTileElems;
        const int64_t seg0 = (int64_t)j * a.seg + a.sub_off;
        const uint32_t own = (uint32_t)(tile_valid(a.sub_len, a.M - seg0, e0) * 2) & ~15u;
        const int64_t v = clamp0(min((int64_t)kTileElems, a.sub_len - e0));
        const int64_t grp0 = e0 >> a.c1.gshift, ng = (v + a.c1.g - 1) >> a.c1.gshift;
        const uint32_t cb = v > 0 ? up16(v * a.c1.sb / 8) : 0u;
        const uint32_t sb = v > 0 ? up16(ng * 2) : 0u;
        const uint32_t zb = (v > 0 && !a.c1.sym) ? up16(ng) : 0u;
        const uint32_t st_base = sbase + st * SBY;
        const uint32_t bar0 = full0 + 8 * (st * NP);
        mbar_arrive_expect_tx(bar0, own);
        if (own) bulk_g2s(st_base, reinterpret_cast<const Tin*>(a.in[j]) + seg0 + e0, own, bar0);
        uint32_t dst = st_base + kTileElems * 2;
        int piece = 1;
        for (int s = 0; s < a.world; ++s) {
          if (s == j) continue;
          const uint32_t bar = bar0 + 8 * piece++;
          const uint8_t* slot = recv_slot(a, j, s);
          mbar_arrive_expect_tx(bar, cb + sb + zb);
          if (cb) bulk_g2s(dst, slot + e0 * a.c1.sb / 8, cb, bar);
          if (sb) bulk_g2s(dst + PC, slot + a.c1.scales_off + grp0 * 2, sb, bar);
          if (zb) bulk_g2s(dst + PC + SCB, slot + a.c1.zeros_off + grp0, zb, bar);
          dst += PC + PM;
        }
      }
      __syncwarp();
      ring_next(st, ph, S);
    }
    return;
  }
  const int rot = (lane >> 1) & 3;
  uint32_t qoff[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) qoff[q] = threadIdx.x * 64 + 16 * ((q + rot) & 3);
  const uint32_t gl = (uint32_t)((threadIdx.x * kLaneElems) >> a.c1.gshift);
  int st = 0;
  uint32_t ph = 0;
  for (Iter it = it0; it.ok(); it.next()) {
    const int j = a.rank_lo + it.y;
    const int64_t p0 = (int64_t)it.t * kTileElems + threadIdx.x * kLaneElems;
    const int64_t seg0 = (int64_t)j * a.seg + a.sub_off;
    const int nvalid = lane_valid(a.sub_len, p0);
    const bool staged = nvalid == kLaneElems && seg0 + p0 + kLaneElems <= a.M;
    const uint32_t st_base = sbase + st * SBY;
    const uint32_t bar0 = full0 + 8 * (st * NP);
    // fp32 sum in ascending source rank (collectives.py:182-187): acc = ((0 + d_0) + d_1) + ...
    // (0 + x == x exactly for every decoded x, none is -0); the own piece is
    // QDQ'd in registers at its rank position (collectives.py:364-365) and
    // accumulated straight from its codes (acc + (c - z) * s, one rounding)
    PairLane<S1::SB> acc;
#pragma unroll
    for (int e = 0; e < 16; ++e) acc.p[e] = 0ull;
    bool bad = false;
    uint32_t src = st_base + kTileElems * 2;
    uint32_t pbar = bar0;
    for (int s = 0; s < a.world; ++s) {
      LaneCodes<8> C;
      if (s == j) {  // uniform
        mbar_wait(bar0, ph);
        PackedLane<Tin> L;
        if (staged) {
          read_rotated(st_base, qoff, L);
          unrotate_input(L, rot);
        } else {
          load_lane_src(reinterpret_cast<const Tin*>(a.in[j]) + seg0, p0, a.M - seg0, nvalid, L);
        }
        LaneQuant<8> q;
        bad = quantize_lane<S1>(a.c1, L, nvalid, q);
        lane_codes_from(a.c1, q, C);
      } else {
        pbar += 8;
        mbar_wait(pbar, ph);
        read_peer<S1>(a.c1, src, PC, SCB, gl, C);  // lanes past the round read stale bytes (never stored)
        src += PC + PM;
      }
      decode_pairs<S1, true>(C, acc);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * st);
    LaneQuant<8> q2;
    bad |= quantize_lane<S2>(a.c2, acc, nvalid, q2);
    {
      const CodeDst cd = code_dst<S2>(a.c2, p0, nvalid, lane);
      const int64_t slot_off = (int64_t)(a.world + j) * a.slot_bytes;  // gather slot [j] (gath_slot)
      for (int p = j + 1;; ++p) {  // every peer's gather slot [j], starting after the owner
        if (p == a.world) p = 0;
        if (p == j) break;
        store_codes_at<S2>(a.blk[p] + slot_off, cd, q2);
      }
    }
    LaneCodes<8> L2;
    lane_codes_from(a.c2, q2, L2);
    PairLane<S2::SB> o;
    decode_pairs<S2, false>(L2, o);  // owner decodes its own payload too (collectives.py:378)
    if (nvalid > 0) {
      float ov[kLaneElems];
#pragma unroll
      for (int e = 0; e < kLaneElems; ++e) ov[e] = o.get(e);
      store_chunk(reinterpret_cast<Tout*>(a.out[j]), seg0 + p0, a.M, nvalid, ov);
    }
    if (bad) atomicOr(errw(a, j), make_err(kErrNonFinite, kPhReduce, j, j));
    if constexpr (FUSED) {
      consumers_sync();
      if (threadIdx.x == 0) {
        if (a.sys_scope) {
          __threadfence_system();
          for (int p = 0; p < a.world; ++p)
            if (p != j) st_relaxed_sys(gflag(a, p, j) + it.t, flag_epoch(a));
        } else {
          __threadfence();
          for (int p = 0; p < a.world; ++p)
            if (p != j) st_relaxed_sys(gflag(a, p, j) + it.t, flag_epoch(a));
        }
      }
    }
    ring_next(st, ph, S);
  }
}

// ------------------------------------------------------------------ dequantize role

template <typename Tout>
__device__ __forceinline__ void store8(Tout* p, const float v[8]) {
  if constexpr (sizeof(Tout) == 4) {
    st_v4(p, make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]), __float_as_uint(v[2]), __float_as_uint(v[3])));
    st_v4(p + 4, make_uint4(__float_as_uint(v[4]), __float_as_uint(v[5]), __float_as_uint(v[6]), __float_as_uint(v[7])));
  } else {
    st_v4(p, make_uint4(pack2(v[0], v[1], (Tout*)nullptr), pack2(v[2], v[3], (Tout*)nullptr),
                        pack2(v[4], v[5], (Tout*)nullptr), pack2(v[6], v[7], (Tout*)nullptr)));
  }
}

// decode the 8 stored codes of one block into v[0..7] (element order)
template <class Spec>
__device__ __forceinline__ void decode8(uint2 cw, float s, float mz, float v[8]) {
  if constexpr (Spec::MF) {  // minifloat codes: exact fp16 grid values, times the scale (exact)
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const uint32_t two = Spec::SB == 8 ? (((p < 2 ? cw.x : cw.y) >> (16 * (p & 1))) & 0xFFFFu) : ((cw.x >> (8 * p)) & 0xFFu);
      mf_dec2(Spec::FMT, two, v[2 * p], v[2 * p + 1]);
      v[2 * p] *= s;
      v[2 * p + 1] *= s;
    }
    return;
  }
  const uint64_t S2 = f2_splat(s), NMZ2 = f2_splat(-mz);
  auto two = [&](uint32_t ma, uint32_t mb, float& x, float& y) {
    uint64_t M;
    asm("mov.b64 %0, {%1,%2};" : "=l"(M) : "r"(ma), "r"(mb));
    f2_unpack(f2_mul(f2_add(M, NMZ2), S2), x, y);
  };
  if constexpr (Spec::SB == 4) {
    const uint32_t lo = cw.x & 0x0F0F0F0Fu, hi = (cw.x >> 4) & 0x0F0F0F0Fu;
    two(__byte_perm(lo, 0x4B000000u, 0x7440u), __byte_perm(hi, 0x4B000000u, 0x7440u), v[0], v[1]);
    two(__byte_perm(lo, 0x4B000000u, 0x7441u), __byte_perm(hi, 0x4B000000u, 0x7441u), v[2], v[3]);
    two(__byte_perm(lo, 0x4B000000u, 0x7442u), __byte_perm(hi, 0x4B000000u, 0x7442u), v[4], v[5]);
    two(__byte_perm(lo, 0x4B000000u, 0x7443u), __byte_perm(hi, 0x4B000000u, 0x7443u), v[6], v[7]);
  } else {
    two(__byte_perm(cw.x, 0x4B000000u, 0x7440u), __byte_perm(cw.x, 0x4B000000u, 0x7441u), v[0], v[1]);
    two(__byte_perm(cw.x, 0x4B000000u, 0x7442u), __byte_perm(cw.x, 0x4B000000u, 0x7443u), v[2], v[3]);
    two(__byte_perm(cw.y, 0x4B000000u, 0x7440u), __byte_perm(cw.y, 0x4B000000u, 0x7441u), v[4], v[5]);
    two(__byte_perm(cw.y, 0x4B000000u, 0x7442u), __byte_perm(cw.y, 0x4B000000u, 0x7443u), v[6], v[7]);
  }
}

// The write-dominated gather runs fastest with ~26-42 KB of code reads in flight per SM
// from a single CTA: more CTAs / deeper rings put more concurrent read streams against
// its output writes (C2: 198-201 µs at 1 CTA x 6-7 stages vs 222 µs at 3 x 6; tools/gather_sweep.sh)
constexpr int kDCtasPerSm = 1;
constexpr int64_t kDSmallItems = 4096;  // gather items (tiles) at most for the small-round CTA count
template <class S2>
constexpr int dstream_stages() { return S2::SB == 4 ? 7 : 5; }

// dequantize job y: quantized source, output span
template <typename Tout>
struct DJob {
  const uint8_t* src;
  Tout* out;
  int64_t limit;  // valid output elements from `out`
};

template <typename Tout>
__device__ __forceinline__ DJob<Tout> djob(const FlashArgs& a, int y) {
  DJob<Tout> d;
  if (a.mode == 1) {
    d.src = reinterpret_cast<const uint8_t*>(a.in[0]);
    d.out = reinterpret_cast<Tout*>(a.out[0]);
    d.limit = a.M;
    return d;
  }
  int r, j;
  pair_of(a, y, r, j);
  const int64_t off = (int64_t)j * a.seg + a.sub_off;
  d.src = gath_slot(a, r, j);
  d.out = reinterpret_cast<Tout*>(a.out[r]) + off;
  d.limit = a.M - off;
  return d;
}

// bytes of one staged code tile of the decode stream: codes, scales, zeros
__host__ __device__ inline uint32_t dstage_bytes(const DevCodec& c) {
  return peer_codes_bytes(c) + peer_meta_bytes(c);
}

// all-gather decode (mode 0: rank r's gather slot [j] -> out[r][segment j],
// job y = (r, j) of [rank_lo, rank_hi)) or codec dequantize (mode 1). A
// producer warp bulk-copies each tile's codes/scales/zeros into the ring;
// consumer thread t decodes 8-element blocks t + 256*b (b = 0..3) of the
// tile: conflict-free shared loads and coalesced 16-B output stores.
// FUSED: wait gflag[r][j][t] before the copies.
template <typename Tout, class S2, bool FUSED, class Iter, int NCW = kConsumerWarps>
__device__ __forceinline__ void d_role(const FlashArgs& a, uint32_t sbase, int S, Iter it0, uint32_t bars = 0) {
  constexpr int NT = NCW * 32;                    // consumer threads
  constexpr int kBlocks = kTileElems / 8 / NT;    // 8-element blocks per thread and tile (4 or 8)
  constexpr int kHalf = kBlocks < 4 ? kBlocks : 4;  // blocks decoded per pass (register budget)
  const DevCodec& c = a.c2;
  const uint32_t SBY = dstage_bytes(c), PC = peer_codes_bytes(c), SCB = peer_scale_bytes(c);
  const uint32_t full0 = bars ? bars : sbase + S * SBY, empty0 = full0 + 8 * S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gs = c.gshift;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, NCW * 32);  // every consumer thread releases its own reads
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == NCW) {
    int st = 0, k = 0, cy = -1;
    uint32_t ph = 0;
    DJob<Tout> d;
    auto issue = [&](int y, int t, bool wait_empty) {  // lane 0
      if (wait_empty) mbar_wait(empty0 + 8 * st, ph ^ 1);
      if (y != cy) {
        d = djob<Tout>(a, y);
        cy = y;
      }
      const int64_t e0 = (int64_t)t * kTileElems;
      const int64_t v = clamp0(min((int64_t)kTileElems, min(a.sub_len - e0, d.limit - e0)));
      const int64_t grp0 = e0 >> gs, ng = (v + c.g - 1) >> gs;
      const uint32_t cb = v > 0 ? up16(v * S2::SB / 8) : 0u, sb = v > 0 ? up16(ng * 2) : 0u;
      const uint32_t zb = (v > 0 && !S2::SYM) ? up16(ng) : 0u;
      const uint32_t dst = sbase + st * SBY, bar = full0 + 8 * st;
      mbar_arrive_expect_tx(bar, cb + sb + zb);
      if (cb) bulk_g2s(dst, d.src + e0 * S2::SB / 8, cb, bar);
      if (sb) bulk_g2s(dst + PC, d.src + c.scales_off + grp0 * 2, sb, bar);
      if (zb) bulk_g2s(dst + PC + SCB, d.src + c.zeros_off + grp0, zb, bar);
    };
    if constexpr (!FUSED) {
      for (Iter it = it0; it.ok(); it.next(), ++k) {
        if (lane == 0) issue(it.y, it.t, k >= S);
        __syncwarp();
        ring_next(st, ph, S);
      }
    } else {
      const DynIter& D = it0;  // dynamic dealing; the owner's gflag is awaited before the copies
      int id = 0;
      if (lane == 0) id = D.grab();
      id = __shfl_sync(0xffffffffu, id, 0);
      for (;; ++k) {
        if (id >= D.items) break;
        int nid = 0;
        if (lane == 0) nid = D.grab();  // the next id is in flight during this item
        int y, t, r, j;
        D.decode(id, y, t);
        pair_of(a, y, r, j);
        warp_wait_flags(a, r, gflag(a, r, j) + t, j, lane == 0, kPhGather);
        if (lane == 0) {
          if (k >= S) mbar_wait(empty0 + 8 * st, ph ^ 1);
          sts32(D.meta + 4 * st, id);
          issue(y, t, false);
        }
        __syncwarp();
        ring_next(st, ph, S);
        id = __shfl_sync(0xffffffffu, nid, 0);
      }
      if (lane == 0) {  // end sentinel
        if (k >= S) mbar_wait(empty0 + 8 * st, ph ^ 1);
        sts32(D.meta + 4 * st, -1);
        mbar_arrive(full0 + 8 * st);
      }
      __syncwarp();
    }
    return;
  }
  const uint32_t xr = rep_xor(c);
  const uint32_t dep_zero = (uint32_t)a.tiles >> 31;  // 0 at run time, opaque to the compiler
  const float zsym = S2::SYM ? 8388608.0f + (float)(1 << (c.bits - 1)) : 0.0f;
  const uint32_t code_off = threadIdx.x * S2::SB;                // bytes of 8 codes of SB bits
  const uint32_t grp_off = (uint32_t)(threadIdx.x * 8) >> gs;    // tile-local group of block 0
  const uint32_t grp_step = (uint32_t)(NT * 8) >> gs;            // groups per block step
  int cy = -1;
  DJob<Tout> d;
  auto item = [&](int y, int t, int st, uint32_t ph) {
    if (y != cy) {
      d = djob<Tout>(a, y);
      cy = y;
    }
    const int64_t e0 = (int64_t)t * kTileElems;
    const int64_t v = min(a.sub_len - e0, d.limit - e0);  // valid elements from e0
    const uint32_t tile = sbase + st * SBY;
    Tout* obase = d.out + e0 + threadIdx.x * 8;
    mbar_wait(full0 + 8 * st, ph);
#pragma unroll
    for (int h = 0; h < kBlocks; h += kHalf) {
      uint2 cw[kHalf];
      float sc[kHalf], mz[kHalf];
#pragma unroll
      for (int b = 0; b < kHalf; ++b) {
        const uint32_t ca = tile + code_off + (h + b) * NT * S2::SB;
        if constexpr (S2::SB == 4) {
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(cw[b].x) : "r"(ca) : "memory");
          cw[b].y = 0;
        } else {
          asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(cw[b].x), "=r"(cw[b].y) : "r"(ca) : "memory");
        }
        const uint32_t g = grp_off + (h + b) * grp_step;
        unsigned short sh;
        asm volatile("ld.shared.u16 %0, [%1];" : "=h"(sh) : "r"(tile + PC + 2 * g) : "memory");
        sc[b] = __half2float(__ushort_as_half(sh));
        if constexpr (S2::SYM) {
          mz[b] = zsym;
        } else {
          uint32_t zz;
          asm volatile("ld.shared.u8 %0, [%1];" : "=r"(zz) : "r"(tile + PC + SCB + g) : "memory");
          mz[b] = __uint_as_float(0x4B000000u | zz);
        }
      }
      float val[kHalf][8];
#pragma unroll
      for (int b = 0; b < kHalf; ++b) {
        uint2 w = cw[b];
        if constexpr (S2::SYM && !S2::MF) {
          w.x ^= xr;
          w.y ^= xr;
        }
        decode8<S2>(w, sc[b], mz[b], val[b]);
      }
      if (h + kHalf >= kBlocks) {
        // release the stage per thread, the arrive's address data-dependent on every value this
        // thread loaded from it (see r_role_gpl: an arrive ahead of an outstanding LDS races the
        // stage's next bulk fill)
        uint32_t dep = 0;
#pragma unroll
        for (int b = 0; b < kHalf; ++b) dep ^= cw[b].x ^ cw[b].y ^ __float_as_uint(sc[b]) ^ __float_as_uint(mz[b]);
        mbar_arrive_dep(empty0 + 8 * st, dep, dep_zero);
      }
      if (v >= kTileElems) {  // whole tile: no per-block checks
#pragma unroll
        for (int b = 0; b < kHalf; ++b) store8(obase + (h + b) * NT * 8, val[b]);
      } else {
#pragma unroll
        for (int b = 0; b < kHalf; ++b) {
          const int64_t e = (int64_t)(threadIdx.x + (h + b) * NT) * 8;
          Tout* o = obase + (h + b) * NT * 8;
          if (e + 8 <= v) {
            store8(o, val[b]);
          } else {
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (e + q < v) o[q] = DT<Tout>::from_f(val[b][q]);
          }
        }
      }
    }
  };
  int st = 0;
  uint32_t ph = 0;
  if constexpr (!FUSED) {
    for (Iter it = it0; it.ok(); it.next()) {
      item(it.y, it.t, st, ph);
      ring_next(st, ph, S);
    }
  } else {
    const DynIter& D = it0;
    for (;;) {
      mbar_wait(full0 + 8 * st, ph);
      const int id = lds_id(D.meta + 4 * st);
      if (id < 0) break;
      int y, t;
      D.decode(id, y, t);
      item(y, t, st, ph);
      ring_next(st, ph, S);
    }
  }
}

// ------------------------------------------------------------------ phase-split kernels

// Programmatic dependent launch (the phase kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization): a CTA waits for the previous kernel's
// completion (and the visibility of its memory) before its first global access, and lets the
// next kernel launch once all its warps are done -- the next phase's launch and CTA
// scheduling overlap this phase's last CTAs. (Triggering earlier -- at entry, or from the
// producer warp, which finishes issuing long before the consumers -- placed the next
// kernel's CTAs on the SMs that drained first and unbalanced its persistent grid: C2
// 535 -> 617-742 us, tools/pdl_probe.py.) Both are no-ops for plain launches.
__device__ __forceinline__ void pdl_enter() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_exit() {
  __syncthreads();  // one trigger per CTA, after every warp's work (the producer warp ends early)
  if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename Tin, class S1>
__global__ void __launch_bounds__(kStreamThreads) k_qstream(FlashArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  pdl_enter();
  const int njobs = a.mode == 1 ? 1 : q_jobs(a);
  q_role<Tin, S1, false>(a, smem_u32(smem), a.stages, RangeIter(njobs * a.tiles, a.tiles, blockIdx.x, gridDim.x));
  pdl_exit();
}

// g = 128 scatter / codec quantize, one lane per group (q_role_gpl)
template <typename Tin, class S1, int G = 128>
__global__ void __launch_bounds__(kGplThreads, 3) k_qstream_gpl(FlashArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  pdl_enter();
  const int njobs = a.mode == 1 ? 1 : q_jobs(a);
  q_role_gpl<Tin, S1, false, RangeIter, G>(a, smem_u32(smem), a.stages,
                                          RangeIter(njobs * a.tiles, a.tiles, blockIdx.x, gridDim.x));
  pdl_exit();
}

// any g in {32, 64, 128, 256}, INT4 or INT8, one lane per 128-element slice (q_role_gq)
template <typename Tin, class S1, int G>
__global__ void __launch_bounds__(kGplThreads, 4) k_qstream_gq(FlashArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  pdl_enter();
  const int njobs = a.mode == 1 ? 1 : q_jobs(a);
  q_role_gq<Tin, S1, G, false>(a, smem_u32(smem), a.stages, RangeIter(njobs * a.tiles, a.tiles, blockIdx.x, gridDim.x));
  pdl_exit();
}

template <typename Tin, typename Tout, class S1, class S2>
__global__ void __launch_bounds__(kStreamThreads, 2) k_rstream(FlashArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  pdl_enter();
  r_role<Tin, Tout, S1, S2, false>(a, smem_u32(smem), a.stages,
                                   RangeIter((a.rank_hi - a.rank_lo) * a.tiles, a.tiles, blockIdx.x, gridDim.x));
  pdl_exit();
}

// g = 128 reduce, two lanes per group (r_role_gpl, a.stages piece slots); one storage width, whole tiles only
template <typename Tin, typename Tout, class S1, class S2>
__global__ void __launch_bounds__(kGplThreads, 4) k_rstream_gpl(FlashArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  pdl_enter();
  if constexpr ((sizeof(Tout) == 2 || sizeof(Tout) == 4) && S1::SB == S2::SB)
    r_role_gpl<Tin, Tout, S1, S2, false>(a, smem_u32(smem), a.stages,
                                  RangeIter((a.rank_hi - a.rank_lo) * a.tiles, a.tiles, blockIdx.x, gridDim.x));
  pdl_exit();
}

template <typename Tout, class S2>
__global__ void __launch_bounds__(kStreamThreads) k_dstream(FlashArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  pdl_enter();
  const int njobs = a.mode == 1 ? 1 : (a.rank_hi - a.rank_lo) * (a.world - 1);
  d_role<Tout, S2, false>(a, smem_u32(smem), a.stages, RangeIter(njobs * a.tiles, a.tiles, blockIdx.x, gridDim.x));
  pdl_exit();
}

// ------------------------------------------------------------------ fused kernel

// smem layout of the fused kernel: one data region (the largest role's rings)
// and one barrier region behind it, so a role's barriers never overlay
// another role's data
struct FusedSmem {
  int q_stages, d_stages, r_ring, data_bytes, bars_off, max_bars, meta_off, total;
};
__host__ __device__ inline FusedSmem fused_smem(const DevCodec& c1, const DevCodec& c2, int qs, int ds, int rr) {
  FusedSmem f;
  f.q_stages = qs;
  f.d_stages = ds;
  f.r_ring = rr;
  const int q = qs * kTileElems * 2;
  const int r = (int)rg_bars_off(c1, rr);
  const int d = ds * (int)dstage_bytes(c2);
  f.data_bytes = q > r ? (q > d ? q : d) : (r > d ? r : d);
  f.bars_off = (f.data_bytes + 127) & ~127;
  // the reduce role keeps its item-id ring (one int per piece slot) behind its barriers
  const int nq = 2 * qs, nr = 2 * rr + kRgDone + (rr + kRgDone + 1) / 2, nd = 2 * ds;
  f.max_bars = nq > nr ? (nq > nd ? nq : nd) : (nr > nd ? nr : nd);
  f.meta_off = f.bars_off + 8 * f.max_bars;  // DynIter id ring: one int per stage (<= 16)
  f.total = f.meta_off + 64;
  return f;
}

// hand the CTA's shared memory from one role to the next: every thread's
// generic shared stores are ordered before later bulk (async-proxy) fills, all
// of the previous role's waits are over, its barriers are invalidated
__device__ __forceinline__ void fused_role_switch(uint32_t bars, int nb) {
  fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x == 0)
    for (int i = 0; i < nb; ++i) mbar_inval(bars + 8 * i);
}

// One cooperative launch per rank (or one for all logical ranks of a GPU):
// the paper's fused kernel. Every CTA runs the three roles
// of the group-lane codec — scatter (q_role_gpl: stage-1 quantize, codes
// stored straight into the owners' receive slots, peer memory over NVLink),
// reduce (r_role_gpl: the N stage-1 pieces, own one included -> fp32 rank-ordered sum ->
// stage-2 quantize -> every peer's gather slot) and gather (d_role: decode the
// owners' stage-2 pieces) — synchronised only by per-tile epoch flags (rflag /
// gflag: published by a role's producer warp once the tile's stores are
// issued, acquired before the tile's bulk copies).
// The segment's tiles are cut into chunks of a.fp_chunk tiles; at step s a CTA
// scatters chunk s, reduces chunk s-1 and gathers chunk s-2, so NVLink-bound
// scatter/reduce traffic of one chunk overlaps the HBM-bound gather of an
// earlier one. Items of a (role, chunk) are dealt dynamically (DynIter: a
// global counter per (role, chunk), tile-major ids). A CTA enters a role only
// after every item of the previous (role, chunk) was taken, every wait
// targets an item of an earlier step (on any rank), and all CTAs are
// co-resident (cooperative launch), so the schedule cannot deadlock. The
// launch's last CTA zeroes the counters for the next launch.
template <typename Tin, typename Tout, class S1, class S2>
__global__ void __launch_bounds__(kGplThreads, 3) k_fstream(const __grid_constant__ FlashArgs a) {
  if constexpr (sizeof(Tin) == 2 && (sizeof(Tout) == 2 || sizeof(Tout) == 4) && S1::SB == S2::SB) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ int s_last;
    const uint32_t sb = smem_u32(smem);
    const uint32_t bars = sb + (uint32_t)a.fp_bars;
    const int G = (int)gridDim.x, cta = (int)blockIdx.x;
    const int nr = a.rank_hi - a.rank_lo;
    const int P = nr * (a.world - 1);   // gather jobs (peers' pieces)
    const int PQ = nr * (a.world - 1 + a.ownq);  // scatter jobs (ownq: the own piece too)
    const int B = a.fp_chunk;
    const int nch = (a.tiles + B - 1) / B;
    uint32_t* ctr = fctr(a, a.rank_lo);
    const uint32_t ep = flag_epoch(a);  // the round's epoch (k_epoch_bump ran before this launch)
    int nb = 0;
    uint64_t* tp = a.tprof ? a.tprof + (int64_t)cta * FC_ROLE_PROFILE_U64 : nullptr;
    if (tp && threadIdx.x == 0) tp[9] = globaltimer();
#pragma unroll 1
    for (int s = 0; s < nch + 2; ++s) {
#pragma unroll 1
      for (int role = 0; role < 3; ++role) {
        const int c = s - role;
        if (c < 0 || c >= nch) continue;
        if (role == 2 && cta >= a.fp_dctas) continue;  // measurement option: fewer gather CTAs
        const int t0 = c * B, bt = min(B, a.tiles - t0);
        const int per = role == 0 ? PQ : role == 1 ? nr : P;
        fused_role_switch(bars, nb);
        const uint64_t r0 = tp ? globaltimer() : 0;
        const DynIter it{ctr + role * kFusedMaxChunks + c, per * bt, per, t0, sb + (uint32_t)a.fp_meta, ep};
        if (role == 0) q_role_gpl<Tin, S1, true>(a, sb, a.q_stages_f, it, bars);
        else if (role == 1) r_role_gpl<Tin, Tout, S1, S2, true>(a, sb, a.r_ring_f, it, bars);
        else d_role<Tout, S2, true, DynIter, kGplWarps>(a, sb, a.d_stages_f, it, bars);
        nb = role == 0 ? 2 * a.q_stages_f : role == 1 ? 2 * a.r_ring_f + kRgDone : 2 * a.d_stages_f;
        if (tp) {
          __syncthreads();
          if (threadIdx.x == 0) {
            const uint64_t r1 = globaltimer();
            if (!tp[role]) tp[role] = r0;
            tp[3 + role] = r1;
            tp[6 + role] += r1 - r0;
          }
        }
      }
    }
    // the last CTA to finish zeroes the (role, chunk) counters for the next launch
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      s_last = atomicAdd(ctr + 3 * kFusedMaxChunks, 1u) == (uint32_t)(G - 1);
    }
    __syncthreads();
    if (s_last) {
      for (int i = threadIdx.x; i < 3 * nch; i += blockDim.x) ctr[(i / nch) * kFusedMaxChunks + i % nch] = 0u;
      if (threadIdx.x == 0) ctr[3 * kFusedMaxChunks] = 0u;
    }
    if (tp) {
      __syncthreads();
      if (threadIdx.x == 0) tp[10] = globaltimer();
    }
  }
}

}  // namespace fc
