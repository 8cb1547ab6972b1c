// Flash all-reduce orchestration (host): round planning, launch of the fused
// or phase-split kernels, the generic path and IPC barriers. Included by the
// per-dtype translation units fc_run_*.cu, which instantiate run_typed.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <numeric>

#include "fc_comm.h"
#include "fc_flash.cuh"
#include "fc_stream.cuh"

namespace fc {


constexpr int kSpecGen = 0, kSpecA4 = 1, kSpecA8 = 2;
inline int spec_id(const fc_codec& c) {
  if (c.kind != FC_KIND_INT || c.symmetric || c.rounding != FC_ROUND_NEAREST_EVEN) return kSpecGen;
  if (c.group_size != 32 && c.group_size != 64 && c.group_size != 128 && c.group_size != 256) return kSpecGen;
  return storage_bits(c) == 4 ? kSpecA4 : kSpecA8;
}

struct Plan {
  int64_t seg = 0, R = 0, rounds = 0;
  bool fast = false;
  fc_layout L1{}, L2{};
};

inline fc_status make_plan(const fc_comm* c, const fc_flash_cfg* cfg, int64_t n, bool aligned, Plan* p) {
  const int N = c->world;
  p->seg = ceil_div(n, N);
  p->fast = c->fast && fast_group(cfg->stage1) && fast_group(cfg->stage2) && (p->seg % 8 == 0) && aligned;
  int64_t unit = std::lcm(group_of(cfg->stage1), group_of(cfg->stage2));
  if (p->fast) unit = std::lcm(unit, (int64_t)kTileElems);
  // largest multiple of `unit` whose two slot layouts fit and whose tiles fit the flags
  const int sbmax = std::max(storage_bits(cfg->stage1), storage_bits(cfg->stage2));
  int64_t rmax = (c->slot_bytes * 8 / sbmax) / unit * unit;
  while (rmax > 0 && (layout_of(cfg->stage1, rmax).total_bytes > c->slot_bytes ||
                      layout_of(cfg->stage2, rmax).total_bytes > c->slot_bytes ||
                      ceil_div(rmax, kTileElems) > c->flags_cap))
    rmax -= unit;
  if (rmax <= 0 && p->seg > 0) {
    // a single round of the whole segment may still fit (seg < unit)
    if (layout_of(cfg->stage1, p->seg).total_bytes <= c->slot_bytes &&
        layout_of(cfg->stage2, p->seg).total_bytes <= c->slot_bytes && ceil_div(p->seg, kTileElems) <= c->flags_cap)
      rmax = p->seg;
    else
      return fail(FC_ERR_CONFIG, "communicator slots (%lld B) too small for group lcm %lld",
                  (long long)c->slot_bytes, (long long)unit);
  }
  p->R = std::min(p->seg, rmax);
  p->rounds = ceil_div(p->seg, p->R);
  p->L1 = layout_of(cfg->stage1, p->R);
  p->L2 = layout_of(cfg->stage2, p->R);
  return FC_OK;
}

inline uint8_t* h_recv_slot(const fc_comm* c, int owner, int src) { return c->blk[owner] + (int64_t)src * c->slot_bytes; }
inline uint8_t* h_gath_slot(const fc_comm* c, int owner, int src) {
  return c->blk[owner] + (int64_t)(c->world + src) * c->slot_bytes;
}

template <typename Tin, typename Tout, int CW, class S1, class S2>
fc_status launch_fused(const fc_comm* c, FlashArgs a, int rank_lo, int rank_hi, int device, cudaStream_t st) {
  auto kern = k_flash_fused<Tin, Tout, CW, S1, S2>;
  int occ = 0;
  FC_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, 0));
  const int cap = std::max(1, occ) * num_sms(device);
  const int nr = rank_hi - rank_lo;
  int C = c->ctas > 0 ? (int)c->ctas : cap / nr;
  C = std::max(1, std::min(C, cap / nr));
  a.rank_lo = rank_lo;
  a.rank_hi = rank_hi;
  a.ctas_per_rank = C;
  const int per_step = 2 * (a.world - 1) + 1;
  a.lag = c->lag > 0 ? (int)c->lag : (C + per_step - 1) / per_step + 1;
  void* args[] = {&a};
  FC_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)kern, dim3(nr * C), dim3(kThreads), args, 0, st));
  ++g_launch_count;
  return FC_OK;
}

inline unsigned grid_for(int device, int64_t items) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(items, (int64_t)num_sms(device) * 8));
}

// order every rank's stream after every other rank's work so far (one process, several GPUs)
inline fc_status cross_sync(fc_comm* c, cudaStream_t* st) {
  for (int r = 0; r < c->world; ++r) {
    FC_CUDA_TRY(cudaSetDevice(c->devices[r]));
    FC_CUDA_TRY(cudaEventRecord(c->ev[r], st[r]));
  }
  for (int r = 0; r < c->world; ++r) {
    FC_CUDA_TRY(cudaSetDevice(c->devices[r]));
    for (int q = 0; q < c->world; ++q)
      if (q != r) FC_CUDA_TRY(cudaStreamWaitEvent(st[r], c->ev[q], 0));
  }
  return FC_OK;
}

inline fc_status ensure_scratch(fc_comm* c, int r, int64_t elems) {
  if (c->scratch_elems[r] >= elems) return FC_OK;
  FC_CUDA_TRY(cudaSetDevice(c->devices[r]));
  if (c->scratch[r]) {
    FC_CUDA_TRY(cudaDeviceSynchronize());
    cudaFree(c->scratch[r]);
  }
  FC_CUDA_TRY(cudaMalloc(&c->scratch[r], (size_t)elems * 4));
  c->scratch_elems[r] = elems;
  return FC_OK;
}

// generic (any group size) phases for rank r ------------------------------------
template <typename Tin>
fc_status gen_phase_scatter(fc_comm* c, const FlashArgs& a, int r, cudaStream_t st) {
  const int dev = c->devices[r];
  for (int j = 0; j < c->world; ++j) {
    SrcSeg<Tin> src{reinterpret_cast<const Tin*>(a.in[r]), (int64_t)j * a.seg + a.sub_off, a.M};
    uint8_t* dst = h_recv_slot(c, j, r);
    uint32_t* ew = reinterpret_cast<uint32_t*>(c->blk[r] + blk_misc_off(c->world, c->slot_bytes, c->flags_cap));
    if (a.c1.kind == FC_KIND_INT) {
      k_gen_params<<<grid_for(dev, ceil_div(ceil_div(a.sub_len, a.c1.g), 256)), 256, 0, st>>>(src, a.sub_len, a.c1, dst,
                                                                                            ew, r);
      ++g_launch_count;
    }
    k_gen_codes<<<grid_for(dev, ceil_div(gen_code_units(a.c1, a.sub_len), 256)), 256, 0, st>>>(src, a.sub_len, a.c1,
                                                                                             dst, ew, r);
    ++g_launch_count;
  }
  FC_CUDA_TRY(cudaGetLastError());
  return FC_OK;
}

inline fc_status gen_phase_reduce(fc_comm* c, const FlashArgs& a, int j, cudaStream_t st, int64_t L2_bytes) {
  const int dev = c->devices[j];
  FC_TRY(ensure_scratch(c, j, a.sub_len));
  FC_CUDA_TRY(cudaSetDevice(dev));
  uint32_t* ew = reinterpret_cast<uint32_t*>(c->blk[j] + blk_misc_off(c->world, c->slot_bytes, c->flags_cap));
  k_gen_sum<<<grid_for(dev, ceil_div(a.sub_len, 256)), 256, 0, st>>>(a, j, c->scratch[j]); ++g_launch_count;
  SrcF32 src{c->scratch[j]};
  uint8_t* dst = h_gath_slot(c, j, j);
  if (a.c2.kind == FC_KIND_INT) {
    k_gen_params<<<grid_for(dev, ceil_div(ceil_div(a.sub_len, a.c2.g), 256)), 256, 0, st>>>(src, a.sub_len, a.c2, dst,
                                                                                          ew, j);
    ++g_launch_count;
  }
  k_gen_codes<<<grid_for(dev, ceil_div(gen_code_units(a.c2, a.sub_len), 256)), 256, 0, st>>>(src, a.sub_len, a.c2, dst,
                                                                                           ew, j);
  ++g_launch_count;
  k_gen_bcast<<<grid_for(dev, ceil_div(L2_bytes / 16, 256)), 256, 0, st>>>(a, j, L2_bytes); ++g_launch_count;
  FC_CUDA_TRY(cudaGetLastError());
  return FC_OK;
}

template <typename Tout>
fc_status gen_phase_gather(fc_comm* c, const FlashArgs& a, int r, cudaStream_t st) {
  const int dev = c->devices[r];
  for (int j = 0; j < c->world; ++j) {
    k_gen_dequant<Tout><<<grid_for(dev, ceil_div(a.sub_len, 256)), 256, 0, st>>>(
        h_gath_slot(c, r, j), a.sub_len, a.c2, reinterpret_cast<Tout*>(a.out[r]), (int64_t)j * a.seg + a.sub_off, a.M);
    ++g_launch_count;
  }
  FC_CUDA_TRY(cudaGetLastError());
  return FC_OK;
}

// IPC barrier between phases
inline fc_status ipc_barrier(fc_comm* c, const FlashArgs& a, int rank, int phase, cudaStream_t st) {
  k_barrier<<<1, 32, 0, st>>>(a, rank, phase); ++g_launch_count;
  FC_CUDA_TRY(cudaGetLastError());
  return FC_OK;
}


// ---------------------------------------------------------------- staged launches

inline fc_status ensure_smem(const void* kern, int dev, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;
  std::lock_guard<std::mutex> lock(mu);
  int& have = done[{kern, dev}];
  if (bytes > have) {
    FC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    have = bytes;
  }
  return FC_OK;
}

inline unsigned persistent_grid(const void* kern, int dev, int smem, int64_t items) {
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, smem) != cudaSuccess || occ < 1) occ = 1;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(items, (int64_t)occ * num_sms(dev)));
}

// 2-D grid: y = ydim (rank pairs / owners), x strides over tiles; all CTAs resident
inline dim3 grid2d(const void* kern, int dev, int smem, int tiles, int ydim) {
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, smem) != cudaSuccess || occ < 1) occ = 1;
  const int64_t total = (int64_t)occ * num_sms(dev);
  const int64_t gx = std::max<int64_t>(1, std::min<int64_t>(tiles, total / ydim));  // one wave, never a ragged second
  return dim3((unsigned)gx, (unsigned)ydim);
}

constexpr int kStageBudget = 200 * 1024;  // dynamic smem per CTA for the cp.async rings

template <typename Tin, int CW, class S1>
fc_status launch_scatter(FlashArgs a, int dev, cudaStream_t st, int64_t items) {
  const void* kern = (const void*)k_scatter<Tin, CW, S1>;
  a.stages = Chunk<Tin>::kBytes <= 64 ? 4 : 3;
  const int smem = a.stages * kThreads * Chunk<Tin>::kBytes;
  FC_TRY(ensure_smem(kern, dev, smem));
  k_scatter<Tin, CW, S1><<<grid2d(kern, dev, smem, a.tiles, (a.rank_hi - a.rank_lo) * (a.world - 1)), kThreads, smem, st>>>(a);
  ++g_launch_count;
  return FC_OK;
}

template <typename Tin, typename Tout, int CW, class S1, class S2>
fc_status launch_reduce(FlashArgs a, int dev, cudaStream_t st, int64_t items) {
  const void* kern = (const void*)k_reduce<Tin, Tout, CW, S1, S2>;
  const int tb = reduce_thread_bytes<Tin>(a.c1, a.world) * kThreads;
  a.stages = a.stage_hint > 0 ? a.stage_hint : std::max(1, std::min(3, kStageBudget / tb));
  const int smem = a.stages * tb;
  FC_TRY(ensure_smem(kern, dev, smem));
  k_reduce<Tin, Tout, CW, S1, S2><<<grid2d(kern, dev, smem, a.tiles, a.rank_hi - a.rank_lo), kThreads, smem, st>>>(a);
  ++g_launch_count;
  return FC_OK;
}

template <typename Tout, int CW, class S2>
fc_status launch_gather(FlashArgs a, int dev, cudaStream_t st, int64_t items) {
  const void* kern = (const void*)k_gather<Tout, CW, S2>;
  a.stages = 4;
  const int smem = a.stages * kThreads * code_chunk_bytes(a.c2);
  FC_TRY(ensure_smem(kern, dev, smem));
  k_gather<Tout, CW, S2><<<grid2d(kern, dev, smem, a.tiles, (a.rank_hi - a.rank_lo) * (a.world - 1)), kThreads, smem, st>>>(a);
  ++g_launch_count;
  return FC_OK;
}

// ---------------------------------------------------------------- stream launches (fc_stream.cuh)

inline unsigned stream_grid(const void* kern, int dev, int threads, int smem, int64_t items, int cap = 0) {
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem) != cudaSuccess || occ < 1) occ = 1;
  if (cap > 0) occ = std::min(occ, cap);
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(items, (int64_t)occ * num_sms(dev)));
}

constexpr int kQStages = 4;
constexpr int kDStages = 6;

template <typename Tin, class S1>
fc_status launch_qstream(FlashArgs a, int dev, cudaStream_t st, int64_t items) {
  if constexpr (sizeof(Tin) != 2 || !S1::kFast) {
    return fail(FC_ERR_CONFIG, "stream kernels need 16-bit inputs and a compile-time codec");
  } else {
  const void* kern = (const void*)k_qstream<Tin, S1>;
  a.stages = a.q_hint > 0 ? a.q_hint : kQStages;
  const int smem = a.stages * (kTileElems * 2 + 16);
  FC_TRY(ensure_smem(kern, dev, smem));
  k_qstream<Tin, S1><<<stream_grid(kern, dev, kStreamThreads, smem, items, a.cta_cap), kStreamThreads, smem, st>>>(a);
  ++g_launch_count;
  return FC_OK;
  }
}

// two stages when that lets two CTAs share an SM, else as many as fit (<= 4)
inline int rstream_stages(const FlashArgs& a) {
  const int sb = (int)rstage_bytes(a.c1, a.world) + 16;
  if (2 * (2 * sb + 1024) <= 228 * 1024) return 2;
  return std::min(4, kStageBudget / sb);
}

template <typename Tin, typename Tout, class S1, class S2>
fc_status launch_rstream(FlashArgs a, int dev, cudaStream_t st, int64_t items) {
  if constexpr (sizeof(Tin) != 2 || !S1::kFast || !S2::kFast) {
    return fail(FC_ERR_CONFIG, "stream kernels need 16-bit inputs and a compile-time codec");
  } else {
  const void* kern = (const void*)k_rstream<Tin, Tout, S1, S2>;
  a.stages = a.stage_hint > 0 ? (int)a.stage_hint : rstream_stages(a);
  const int smem = a.stages * ((int)rstage_bytes(a.c1, a.world) + 16);
  FC_TRY(ensure_smem(kern, dev, smem));
  k_rstream<Tin, Tout, S1, S2><<<stream_grid(kern, dev, kStreamThreads, smem, items, a.cta_cap), kStreamThreads, smem, st>>>(a);
  ++g_launch_count;
  return FC_OK;
  }
}

template <typename Tout, class S2>
fc_status launch_dstream(FlashArgs a, int dev, cudaStream_t st, int64_t items) {
  if constexpr (!S2::kFast) {
    return fail(FC_ERR_CONFIG, "stream kernels need a compile-time codec");
  } else {
    const void* kern = (const void*)k_dstream<Tout, S2>;
    a.stages = a.d_hint > 0 ? a.d_hint : kDStages;
    const int smem = a.stages * ((int)dstage_bytes(a.c2) + 16);
    FC_TRY(ensure_smem(kern, dev, smem));
    k_dstream<Tout, S2><<<stream_grid(kern, dev, kStreamThreads, smem, items, a.cta_cap), kStreamThreads, smem, st>>>(a);
    ++g_launch_count;
    return FC_OK;
  }
}

// Fused streaming kernel (fc_stream.cuh k_fstream): role pattern from weights
// (scatter : reduce : gather CTAs), interleaved over the period.
inline void role_pattern(int wq, int wr, int wd, FlashArgs& a) {
  const int w[3] = {std::max(0, wq), std::max(0, wr), std::max(0, wd)};
  int per = w[0] + w[1] + w[2];
  if (per <= 0 || per > 16) {
    per = 8;
  }
  const int ww[3] = {per == w[0] + w[1] + w[2] ? w[0] : 3, per == w[0] + w[1] + w[2] ? w[1] : 2,
                     per == w[0] + w[1] + w[2] ? w[2] : 3};
  // largest-remainder interleave: slot k gets the role furthest behind its share
  double acc[3] = {0, 0, 0};
  uint32_t pat = 0;
  for (int k = 0; k < per; ++k) {
    int best = -1;
    double bv = -1e9;
    for (int r = 0; r < 3; ++r) {
      if (ww[r] == 0) continue;
      const double v = (double)ww[r] * (k + 1) / per - acc[r];
      if (v > bv) {
        bv = v;
        best = r;
      }
    }
    acc[best] += 1.0;
    pat |= (uint32_t)best << (2 * k);
  }
  a.role_period = per;
  a.role_pat = pat;
}

template <typename Tin, typename Tout, class S1, class S2>
fc_status launch_fstream(const fc_comm* c, FlashArgs a, int rank_lo, int rank_hi, int dev, cudaStream_t st) {
  if constexpr (sizeof(Tin) != 2 || !S1::kFast || !S2::kFast) {
    return fail(FC_ERR_CONFIG, "stream kernels need 16-bit inputs and a compile-time codec");
  } else {
    const void* kern = (const void*)k_fstream<Tin, Tout, S1, S2>;
    a.rank_lo = rank_lo;
    a.rank_hi = rank_hi;
    a.sys_scope = 0;
    for (int r = 0; r < c->world; ++r) a.sys_scope |= (c->ipc || c->devices[r] != dev) ? 1 : 0;
    const int rsb = (int)rstage_bytes(a.c1, a.world) + 16;
    a.r_stages_f = a.stage_hint > 0 ? a.stage_hint : 2;
    const int budget = std::max(a.r_stages_f * rsb, 64 * 1024);
    a.q_stages_f = a.q_hint > 0 ? a.q_hint : std::max(2, std::min(6, budget / (kTileElems * 2 + 16)));
    a.d_stages_f = a.d_hint > 0 ? a.d_hint : std::max(2, std::min(8, budget / ((int)dstage_bytes(a.c2) + 16)));
    const int smem = std::max({a.r_stages_f * rsb, a.q_stages_f * (kTileElems * 2 + 16),
                               a.d_stages_f * ((int)dstage_bytes(a.c2) + 16)});
    FC_TRY(ensure_smem(kern, dev, smem));
    const int64_t w = c->role_weights;
    role_pattern((int)(w & 0xFF), (int)((w >> 8) & 0xFF), (int)((w >> 16) & 0xFF), a);
    int occ = 0;
    FC_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kStreamThreads, smem));
    if (a.cta_cap > 0) occ = std::min(occ, a.cta_cap);
    if (occ < 1) return fail(FC_ERR_CUDA, "fused stream kernel does not fit on an SM");
    int grid = occ * num_sms(dev);
    grid = std::max(a.role_period, grid / a.role_period * a.role_period);
    void* args[] = {&a};
    FC_CUDA_TRY(cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(kStreamThreads), args, smem, st));
    ++g_launch_count;
    return FC_OK;
  }
}

template <typename Tin, typename Tout, int CW, class S1, class S2>
fc_status run_typed_cw(fc_comm* c, const void* const* ins, void* const* outs, int64_t n, const fc_flash_cfg* cfg,
                       cudaStream_t* st, int only_rank /* -1: local world */) {
  const int N = c->world;
  bool aligned = true;
  for (int r = 0; r < N; ++r) {
    if (only_rank >= 0 && r != only_rank) continue;
    aligned &= ((uintptr_t)ins[r] % 16 == 0) && ((uintptr_t)outs[r] % 16 == 0);
  }
  Plan p;
  FC_TRY(make_plan(c, cfg, n, aligned, &p));
  g_launch_count = 0;
  FlashArgs a{};
  a.world = N;
  a.M = n;
  a.seg = p.seg;
  a.slot_bytes = c->slot_bytes;
  a.flags_cap = c->flags_cap;
  a.timeout_ns = (uint64_t)c->timeout_ms * 1000000ull;
  a.stage_hint = (int)c->reduce_stages;
  a.q_hint = (int)c->q_stages;
  a.d_hint = (int)c->d_stages;
  a.cta_cap = (int)c->ctas_per_sm;
  a.dbg = (int)c->stream_mask;
  a.c1 = dev_codec(cfg->stage1, p.L1);
  a.c2 = dev_codec(cfg->stage2, p.L2);
  for (int r = 0; r < N; ++r) {
    a.in[r] = ins[r];
    a.out[r] = outs[r];
    a.blk[r] = c->blk[r];
  }
  a.mode = 0;
  a.cerr = nullptr;
  bool single_dev = true;
  for (int r = 1; r < N; ++r) single_dev &= c->devices[r] == c->devices[0];
  // streaming kernels (bulk-copy fed, fc_stream.cuh) for compile-time schemes and 16-bit inputs;
  // fast == 2 keeps the cp.async-staged kernels (A/B testing)
  bool use_stream = false;
  if constexpr (S1::kFast && S2::kFast && sizeof(Tin) == 2) {
    use_stream = p.fast && c->fast == 1;
    if (use_stream) {
      FlashArgs t = a;
      t.world = N;
      use_stream = rstream_stages(t) >= 2;
    }
  }

  for (int64_t k = 0; k < p.rounds; ++k) {
    a.sub_off = k * p.R;
    a.sub_len = std::min(p.R, p.seg - a.sub_off);
    a.tiles = (int)ceil_div(a.sub_len, kTileElems);
    a.epoch = ++c->epoch;
    if (only_rank >= 0) {
      // ---------------- IPC world: this process is rank `only_rank`
      const int r = only_rank;
      const int dev = c->devices[r];
      FC_CUDA_TRY(cudaSetDevice(dev));
      cudaStream_t s = st[r];
      if (use_stream && c->fused != 0) {
        FC_TRY((launch_fstream<Tin, Tout, S1, S2>(c, a, r, r + 1, dev, s)));
      } else if (p.fast && c->fused != 0) {
        FC_TRY((launch_fused<Tin, Tout, CW, S1, S2>(c, a, r, r + 1, dev, s)));
      } else if (p.fast) {
        a.rank_lo = r;
        a.rank_hi = r + 1;
        if (use_stream) {
          FC_TRY((launch_qstream<Tin, S1>(a, dev, s, (int64_t)(N - 1) * a.tiles)));
          FC_TRY(ipc_barrier(c, a, r, 0, s));
          FC_TRY((launch_rstream<Tin, Tout, S1, S2>(a, dev, s, a.tiles)));
          FC_TRY(ipc_barrier(c, a, r, 1, s));
          FC_TRY((launch_dstream<Tout, S2>(a, dev, s, (int64_t)(N - 1) * a.tiles)));
        } else {
          FC_TRY((launch_scatter<Tin, CW, S1>(a, dev, s, (int64_t)(N - 1) * a.tiles)));
          FC_TRY(ipc_barrier(c, a, r, 0, s));
          FC_TRY((launch_reduce<Tin, Tout, CW, S1, S2>(a, dev, s, a.tiles)));
          FC_TRY(ipc_barrier(c, a, r, 1, s));
          FC_TRY((launch_gather<Tout, CW, S2>(a, dev, s, (int64_t)(N - 1) * a.tiles)));
        }
      } else {
        FC_TRY(gen_phase_scatter<Tin>(c, a, r, s));
        FC_TRY(ipc_barrier(c, a, r, 0, s));
        FC_TRY(gen_phase_reduce(c, a, r, s, p.L2.total_bytes));
        FC_TRY(ipc_barrier(c, a, r, 1, s));
        FC_TRY(gen_phase_gather<Tout>(c, a, r, s));
      }
      FC_CUDA_TRY(cudaGetLastError());
      continue;
    }
    // ---------------- local world: this process drives every rank
    // default (-1): phase-split when every rank shares one GPU (nothing crosses a link, and the
    // per-tile flag chains of the fused kernel cost more than the two kernel boundaries); fused
    // across GPUs so NVLink stores overlap the HBM streaming
    if (use_stream && (c->fused == 1 || (c->fused == -1 && !single_dev))) {
      if (single_dev) {
        FC_CUDA_TRY(cudaSetDevice(c->devices[0]));
        FC_TRY((launch_fstream<Tin, Tout, S1, S2>(c, a, 0, N, c->devices[0], st[0])));
      } else {
        for (int r = 0; r < N; ++r) {
          FC_CUDA_TRY(cudaSetDevice(c->devices[r]));
          FC_TRY((launch_fstream<Tin, Tout, S1, S2>(c, a, r, r + 1, c->devices[r], st[r])));
        }
      }
    } else if (p.fast && (c->fused == 1 || (c->fused == -1 && !single_dev))) {
      if (single_dev) {
        FC_CUDA_TRY(cudaSetDevice(c->devices[0]));
        FC_TRY((launch_fused<Tin, Tout, CW, S1, S2>(c, a, 0, N, c->devices[0], st[0])));
      } else {
        for (int r = 0; r < N; ++r) {
          FC_CUDA_TRY(cudaSetDevice(c->devices[r]));
          FC_TRY((launch_fused<Tin, Tout, CW, S1, S2>(c, a, r, r + 1, c->devices[r], st[r])));
        }
      }
    } else if (p.fast && single_dev) {
      const int dev = c->devices[0];
      FC_CUDA_TRY(cudaSetDevice(dev));
      a.rank_lo = 0;
      a.rank_hi = N;
      const int64_t dm = c->stream_mask;  // testing: bit k keeps phase k on the staged kernel
      const int64_t pm = c->phases ? c->phases : 7;  // measurement: run only the selected phases
      if (pm & 1) {
        if (use_stream && !(dm & 1))
          FC_TRY((launch_qstream<Tin, S1>(a, dev, st[0], (int64_t)N * (N - 1) * a.tiles)));
        else
          FC_TRY((launch_scatter<Tin, CW, S1>(a, dev, st[0], (int64_t)N * (N - 1) * a.tiles)));
      }
      if (pm & 2) {
        if (use_stream && !(dm & 2))
          FC_TRY((launch_rstream<Tin, Tout, S1, S2>(a, dev, st[0], (int64_t)N * a.tiles)));
        else
          FC_TRY((launch_reduce<Tin, Tout, CW, S1, S2>(a, dev, st[0], (int64_t)N * a.tiles)));
      }
      if (pm & 4) {
        if (use_stream && !(dm & 4))
          FC_TRY((launch_dstream<Tout, S2>(a, dev, st[0], (int64_t)N * (N - 1) * a.tiles)));
        else
          FC_TRY((launch_gather<Tout, CW, S2>(a, dev, st[0], (int64_t)N * (N - 1) * a.tiles)));
      }
    } else if (p.fast) {
      for (int r = 0; r < N; ++r) {
        FC_CUDA_TRY(cudaSetDevice(c->devices[r]));
        a.rank_lo = r;
        a.rank_hi = r + 1;
        if (use_stream)
          FC_TRY((launch_qstream<Tin, S1>(a, c->devices[r], st[r], (int64_t)(N - 1) * a.tiles)));
        else
          FC_TRY((launch_scatter<Tin, CW, S1>(a, c->devices[r], st[r], (int64_t)(N - 1) * a.tiles)));
      }
      FC_TRY(cross_sync(c, st));
      for (int r = 0; r < N; ++r) {
        FC_CUDA_TRY(cudaSetDevice(c->devices[r]));
        a.rank_lo = r;
        a.rank_hi = r + 1;
        if (use_stream)
          FC_TRY((launch_rstream<Tin, Tout, S1, S2>(a, c->devices[r], st[r], a.tiles)));
        else
          FC_TRY((launch_reduce<Tin, Tout, CW, S1, S2>(a, c->devices[r], st[r], a.tiles)));
      }
      FC_TRY(cross_sync(c, st));
      for (int r = 0; r < N; ++r) {
        FC_CUDA_TRY(cudaSetDevice(c->devices[r]));
        a.rank_lo = r;
        a.rank_hi = r + 1;
        if (use_stream)
          FC_TRY((launch_dstream<Tout, S2>(a, c->devices[r], st[r], (int64_t)(N - 1) * a.tiles)));
        else
          FC_TRY((launch_gather<Tout, CW, S2>(a, c->devices[r], st[r], (int64_t)(N - 1) * a.tiles)));
      }
    } else {
      for (int r = 0; r < N; ++r) {
        FC_CUDA_TRY(cudaSetDevice(c->devices[r]));
        FC_TRY(gen_phase_scatter<Tin>(c, a, r, single_dev ? st[0] : st[r]));
      }
      if (!single_dev) FC_TRY(cross_sync(c, st));
      for (int r = 0; r < N; ++r) {
        FC_CUDA_TRY(cudaSetDevice(c->devices[r]));
        FC_TRY(gen_phase_reduce(c, a, r, single_dev ? st[0] : st[r], p.L2.total_bytes));
      }
      if (!single_dev) FC_TRY(cross_sync(c, st));
      for (int r = 0; r < N; ++r) {
        FC_CUDA_TRY(cudaSetDevice(c->devices[r]));
        FC_TRY(gen_phase_gather<Tout>(c, a, r, single_dev ? st[0] : st[r]));
      }
    }
    FC_CUDA_TRY(cudaGetLastError());
  }
  c->last_launches = g_launch_count;
  c->last_c1 = cfg->stage1;
  c->last_c2 = cfg->stage2;
  c->last_R = p.R;
  c->last_sub_len = std::min(p.R, p.seg - (p.rounds - 1) * p.R);
  return FC_OK;
}

// kernels keep 8 code words per lane unless a stage is the fp16 passthrough
template <typename Tin, typename Tout>
fc_status run_typed(fc_comm* c, const void* const* ins, void* const* outs, int64_t n, const fc_flash_cfg* cfg,
                    cudaStream_t* st, int only_rank) {
  if (cfg->stage1.kind == FC_KIND_FP16 || cfg->stage2.kind == FC_KIND_FP16)
    return run_typed_cw<Tin, Tout, 16, GenSpec, GenSpec>(c, ins, outs, n, cfg, st, only_rank);
  if (c->fast) {  // compile-time schemes of the FlashConfig presets (from_bits 4 / 8 / 6)
    const int a = spec_id(cfg->stage1), b = spec_id(cfg->stage2);
    if (a == kSpecA4 && b == kSpecA4) return run_typed_cw<Tin, Tout, 8, SpecA4, SpecA4>(c, ins, outs, n, cfg, st, only_rank);
    if (a == kSpecA8 && b == kSpecA8) return run_typed_cw<Tin, Tout, 8, SpecA8, SpecA8>(c, ins, outs, n, cfg, st, only_rank);
    if (a == kSpecA4 && b == kSpecA8) return run_typed_cw<Tin, Tout, 8, SpecA4, SpecA8>(c, ins, outs, n, cfg, st, only_rank);
  }
  return run_typed_cw<Tin, Tout, 8, GenSpec, GenSpec>(c, ins, outs, n, cfg, st, only_rank);
}

template <typename Tin, typename Tout>
fc_status identity_typed(const void* in, void* out, int64_t n, int device, cudaStream_t st) {
  FC_CUDA_TRY(cudaSetDevice(device));
  k_convert<Tin, Tout><<<grid_for(device, ceil_div(n, 256)), 256, 0, st>>>(reinterpret_cast<const Tin*>(in),
                                                                          reinterpret_cast<Tout*>(out), n);
  FC_CUDA_TRY(cudaGetLastError());
  return FC_OK;
}


}  // namespace fc
