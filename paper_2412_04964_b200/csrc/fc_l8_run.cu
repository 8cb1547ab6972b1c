// Host side of the lane-8 path (fc_l8.cuh): minifloat stage codecs and the
// fused Hadamard rotation, on the local (one process, N devices) and the IPC
// (one process per rank) communicators. Three phase launches per round,
// ordered like the generic path: cross-device events or IPC barrier kernels.
#include "fc_l8.cuh"
#include "fc_run.cuh"

namespace fc {

namespace {

inline bool l8_group_ok(const fc_codec& c) {
  if (c.kind == FC_KIND_FP16) return false;
  const int g = c.group_size;
  return g >= kL8 && g <= 256 && (g & (g - 1)) == 0;
}

inline unsigned l8_grid(int dev, int64_t lanes, int ydim) {
  const int64_t blocks = ceil_div(ceil_div(lanes, 32) * 32, (int64_t)kL8Threads);
  const int64_t cap = std::max<int64_t>(1, (int64_t)num_sms(dev) * 8 / std::max(1, ydim));
  return (unsigned)std::max<int64_t>(1, std::min(blocks, cap));
}

template <typename Tin, typename Tout, int F>
fc_status run_l8_typed(fc_comm* c, const void* const* ins, void* const* outs, int64_t n, const fc_flash_cfg* cfg,
                       cudaStream_t* st, int only_rank) {
  const int N = c->world;
  Plan p;
  FC_TRY(make_plan(c, cfg, n, false, &p));
  g_launch_count = 0;
  FlashArgs a{};
  a.world = N;
  a.M = n;
  a.seg = p.seg;
  a.slot_bytes = c->slot_bytes;
  a.flags_cap = c->flags_cap;
  a.timeout_ns = (uint64_t)c->timeout_ms * 1000000ull;
  a.c1 = dev_codec(cfg->stage1, p.L1);
  a.c2 = dev_codec(cfg->stage2, p.L2);
  for (int r = 0; r < N; ++r) {
    a.in[r] = ins[r];
    a.out[r] = outs[r];
    a.blk[r] = c->blk[r];
  }
  bool single_dev = true;
  for (int r = 1; r < N; ++r) single_dev &= c->devices[r] == c->devices[0];
  auto rot_of = [&](int r) {
    L8Rot rot{c->rot_dim, c->rot_normalize, c->rot_dim ? c->rot_signs[r] : nullptr};
    return rot;
  };
  // one launch per phase for ranks [lo, hi) on device dev
  auto scatter = [&](int lo, int hi, int dev, cudaStream_t s) -> fc_status {
    FlashArgs b = a;
    b.rank_lo = lo;
    b.rank_hi = hi;
    const int ny = (hi - lo) * (N - 1);
    k_l8_scatter<Tin, F><<<dim3(l8_grid(dev, ceil_div(b.sub_len, kL8), ny), ny), kL8Threads, 0, s>>>(b, rot_of(lo));
    ++g_launch_count;
    return FC_OK;
  };
  auto reduce = [&](int lo, int hi, int dev, cudaStream_t s) -> fc_status {
    FlashArgs b = a;
    b.rank_lo = lo;
    b.rank_hi = hi;
    const int ny = hi - lo;
    k_l8_reduce<Tin, Tout, F><<<dim3(l8_grid(dev, ceil_div(b.sub_len, kL8), ny), ny), kL8Threads, 0, s>>>(b, rot_of(lo));
    ++g_launch_count;
    return FC_OK;
  };
  auto gather = [&](int lo, int hi, int dev, cudaStream_t s) -> fc_status {
    FlashArgs b = a;
    b.rank_lo = lo;
    b.rank_hi = hi;
    const int ny = (hi - lo) * (N - 1);
    k_l8_gather<Tout, F><<<dim3(l8_grid(dev, ceil_div(b.sub_len, kL8), ny), ny), kL8Threads, 0, s>>>(b, rot_of(lo));
    ++g_launch_count;
    return FC_OK;
  };
  // one minifloat format in both stages, g = 128, 16-bit inputs, 16-bit or fp32 outputs, no rotation: the
  // TMA-fed streaming kernels (k_qstream_gpl / k_rstream_gpl / k_dstream on MfSpec) take every
  // round of whole tiles; the lane-8 kernels the rest (bit 10 of FC_OPT_STREAM_MASK: A/B off)
  bool stream_ok = false;
  if constexpr (F != 0 && sizeof(Tin) == 2 && (sizeof(Tout) == 2 || sizeof(Tout) == 4)) {
    stream_ok = c->fast == 1 && c->rot_dim == 0 && !(c->stream_mask & 1024);
    // rounds of whole tiles: the plan unit of a minifloat codec is its group, so round the
    // round size down to a tile multiple when a segment spans several rounds (decided before
    // the buffers' alignment, which may differ between IPC ranks: every rank keeps one slot
    // layout)
    if (stream_ok && p.R > kTileElems && p.R % kTileElems) {
      p.R = p.R / kTileElems * kTileElems;
      p.rounds = ceil_div(p.seg, p.R);
      p.L1 = layout_of(cfg->stage1, p.R);
      p.L2 = layout_of(cfg->stage2, p.R);
      a.c1 = dev_codec(cfg->stage1, p.L1);
      a.c2 = dev_codec(cfg->stage2, p.L2);
    }
    for (int r = 0; r < N && stream_ok; ++r) {
      if (only_rank >= 0 && r != only_rank) continue;
      stream_ok = (uintptr_t)ins[r] % 16 == 0 && (uintptr_t)outs[r] % 16 == 0;
    }
    a.stage_hint = (int)c->reduce_stages;
    a.q_hint = (int)c->q_stages;
    a.d_hint = (int)c->d_stages;
    a.cta_cap = (int)c->ctas_per_sm;
    a.dbg = (int)c->stream_mask;
  }
  const int64_t span_lo = c->span_hi >= 0 ? c->span_lo : 0;
  const int64_t span_hi = c->span_hi >= 0 ? std::min(c->span_hi, p.seg) : p.seg;
  const int64_t rounds = ceil_div(span_hi - span_lo, p.R);
  // the three streaming phase launches for ranks [lo, hi) on device dev (ownq: the scatter
  // stage-1 quantizes the own piece into the receive slot too, the reduce reads it there)
  auto stream_phase = [&](int ph, int lo, int hi, int dev, cudaStream_t s) -> fc_status {
    if constexpr (F != 0 && sizeof(Tin) == 2 && (sizeof(Tout) == 2 || sizeof(Tout) == 4)) {
      using MS = MfSpec<F - 1>;
      FlashArgs b = a;
      b.rank_lo = lo;
      b.rank_hi = hi;
      b.ownq = 1;
      const int64_t nr = hi - lo;
      if (ph == 0) return launch_qstream<Tin, MS>(b, dev, s, nr * N * b.tiles);
      if (ph == 1) return launch_rstream<Tin, Tout, MS, MS>(b, dev, s, nr * b.tiles);
      return launch_dstream<Tout, MS>(b, dev, s, nr * (N - 1) * b.tiles);
    } else {
      return fail(FC_ERR_CONFIG, "internal: minifloat streaming phase without a compile-time format");
    }
  };
  for (int64_t k = 0; k < rounds; ++k) {
    a.sub_off = span_lo + k * p.R;
    a.sub_len = std::min(p.R, span_hi - a.sub_off);
    a.tiles = (int)ceil_div(a.sub_len, kTileElems);
    a.epoch = ++c->epoch;
    a.epoch_dev = nullptr;
    bool strm = false;
    if constexpr (F != 0 && sizeof(Tin) == 2 && (sizeof(Tout) == 2 || sizeof(Tout) == 4)) {
      FlashArgs t = a;  // every rank decides alike: the last owner's segment bounds the round
      t.rank_lo = 0;
      t.rank_hi = N;
      strm = stream_ok && rgpl_ok<Tin, Tout, MfSpec<F - 1>, MfSpec<F - 1>>(t);
    }
    // across GPUs / processes (FC_OPT_FUSED -1) or when forced (1): the single-launch fused
    // streaming kernel (k_fstream on MfSpec), like the integer codecs' default there
    const bool fused = strm && (c->fused == 1 || (c->fused < 0 && (!single_dev || only_rank >= 0))) &&
                       fused_eligible(a);
    if (fused) {
      if constexpr (F != 0 && sizeof(Tin) == 2 && (sizeof(Tout) == 2 || sizeof(Tout) == 4)) {
        using MS = MfSpec<F - 1>;
        if (only_rank >= 0) {
          const int r = only_rank, dev = c->devices[r];
          FC_CUDA_TRY(cudaSetDevice(dev));
          FC_TRY(bump_epoch(c, a, r, st[r]));
          FC_TRY((launch_fstream<Tin, Tout, MS, MS>(c, a, r, r + 1, dev, st[r])));
        } else if (single_dev) {
          FC_CUDA_TRY(cudaSetDevice(c->devices[0]));
          FC_TRY(bump_epoch(c, a, 0, st[0]));
          FC_TRY((launch_fstream<Tin, Tout, MS, MS>(c, a, 0, N, c->devices[0], st[0])));
        } else {
          for (int r = 0; r < N; ++r) {
            FC_CUDA_TRY(cudaSetDevice(c->devices[r]));
            FC_TRY(bump_epoch(c, a, r, st[r]));
            FC_TRY((launch_fstream<Tin, Tout, MS, MS>(c, a, r, r + 1, c->devices[r], st[r])));
          }
        }
      }
      FC_CUDA_TRY(cudaGetLastError());
      continue;
    }
    if (strm) {
      if (only_rank >= 0) {
        const int r = only_rank, dev = c->devices[r];
        FC_CUDA_TRY(cudaSetDevice(dev));
        FC_TRY(bump_epoch(c, a, r, st[r]));
        FC_TRY(stream_phase(0, r, r + 1, dev, st[r]));
        FC_TRY(ipc_barrier(c, a, r, 0, st[r]));
        FC_TRY(stream_phase(1, r, r + 1, dev, st[r]));
        FC_TRY(ipc_barrier(c, a, r, 1, st[r]));
        FC_TRY(stream_phase(2, r, r + 1, dev, st[r]));
      } else if (single_dev) {
        const int dev = c->devices[0];
        FC_CUDA_TRY(cudaSetDevice(dev));
        for (int ph = 0; ph < 3; ++ph) FC_TRY(stream_phase(ph, 0, N, dev, st[0]));
      } else {
        for (int ph = 0; ph < 3; ++ph) {
          if (ph) FC_TRY(cross_sync(c, st));
          for (int r = 0; r < N; ++r) {
            FC_CUDA_TRY(cudaSetDevice(c->devices[r]));
            FC_TRY(stream_phase(ph, r, r + 1, c->devices[r], st[r]));
          }
        }
      }
      FC_CUDA_TRY(cudaGetLastError());
      continue;
    }
    if (only_rank >= 0) {
      const int r = only_rank, dev = c->devices[r];
      FC_CUDA_TRY(cudaSetDevice(dev));
      FC_TRY(bump_epoch(c, a, r, st[r]));
      FC_TRY(scatter(r, r + 1, dev, st[r]));
      FC_TRY(ipc_barrier(c, a, r, 0, st[r]));
      FC_TRY(reduce(r, r + 1, dev, st[r]));
      FC_TRY(ipc_barrier(c, a, r, 1, st[r]));
      FC_TRY(gather(r, r + 1, dev, st[r]));
    } else if (single_dev) {
      const int dev = c->devices[0];
      FC_CUDA_TRY(cudaSetDevice(dev));
      FC_TRY(scatter(0, N, dev, st[0]));
      FC_TRY(reduce(0, N, dev, st[0]));
      FC_TRY(gather(0, N, dev, st[0]));
    } else {
      for (int r = 0; r < N; ++r) {
        FC_CUDA_TRY(cudaSetDevice(c->devices[r]));
        FC_TRY(scatter(r, r + 1, c->devices[r], st[r]));
      }
      FC_TRY(cross_sync(c, st));
      for (int r = 0; r < N; ++r) {
        FC_CUDA_TRY(cudaSetDevice(c->devices[r]));
        FC_TRY(reduce(r, r + 1, c->devices[r], st[r]));
      }
      FC_TRY(cross_sync(c, st));
      for (int r = 0; r < N; ++r) {
        FC_CUDA_TRY(cudaSetDevice(c->devices[r]));
        FC_TRY(gather(r, r + 1, c->devices[r], st[r]));
      }
    }
    FC_CUDA_TRY(cudaGetLastError());
  }
  c->last_launches = g_launch_count;
  c->last_c1 = cfg->stage1;
  c->last_c2 = cfg->stage2;
  c->last_R = p.R;
  c->last_sub_len = std::min(p.R, span_hi - span_lo - (rounds - 1) * p.R);
  return FC_OK;
}

}  // namespace

// the lane-8 path takes a round when a stage is a minifloat codec or a rotation is set, both
// stages are group-scaled (g = 8..256, power of two) and, with a rotation, its blocks tile
// every round (seg and the round size multiples of dim <= 256)
bool l8_wanted(const fc_comm* c, const fc_flash_cfg* cfg, int64_t n) {
  const bool mf = cfg->stage1.kind == FC_KIND_MINIFLOAT || cfg->stage2.kind == FC_KIND_MINIFLOAT;
  if (!mf && c->rot_dim == 0) return false;
  if (!c->fast || !l8_group_ok(cfg->stage1) || !l8_group_ok(cfg->stage2)) return false;
  const int64_t seg = ceil_div(n, (int64_t)c->world);
  if (seg % kL8) return false;
  if (c->rot_dim) {
    Plan p;
    if (make_plan(c, cfg, n, false, &p) != FC_OK) return false;
    if (c->rot_dim < kL8 || c->rot_dim > kL8MaxRot || seg % c->rot_dim || p.R % c->rot_dim) return false;
  }
  return true;
}

template <typename Tin, typename Tout>
fc_status run_l8_f(fc_comm* c, const void* const* ins, void* const* outs, int64_t n, const fc_flash_cfg* cfg,
                   cudaStream_t* st, int only_rank) {
  switch (l8_f_of(cfg->stage1, cfg->stage2)) {  // both stages one minifloat format: compile-time codec
    case 1: return run_l8_typed<Tin, Tout, 1>(c, ins, outs, n, cfg, st, only_rank);
    case 2: return run_l8_typed<Tin, Tout, 2>(c, ins, outs, n, cfg, st, only_rank);
    case 3: return run_l8_typed<Tin, Tout, 3>(c, ins, outs, n, cfg, st, only_rank);
    default: return run_l8_typed<Tin, Tout, 0>(c, ins, outs, n, cfg, st, only_rank);
  }
}

fc_status run_l8(int in_dt, int out_dt, fc_comm* c, const void* const* ins, void* const* outs, int64_t n,
                 const fc_flash_cfg* cfg, cudaStream_t* st, int only_rank) {
  switch (in_dt * 3 + out_dt) {
    case FC_DTYPE_F32 * 3 + FC_DTYPE_F32: return run_l8_f<float, float>(c, ins, outs, n, cfg, st, only_rank);
    case FC_DTYPE_F16 * 3 + FC_DTYPE_F32: return run_l8_f<__half, float>(c, ins, outs, n, cfg, st, only_rank);
    case FC_DTYPE_F16 * 3 + FC_DTYPE_F16: return run_l8_f<__half, __half>(c, ins, outs, n, cfg, st, only_rank);
    case FC_DTYPE_BF16 * 3 + FC_DTYPE_F32:
      return run_l8_f<__nv_bfloat16, float>(c, ins, outs, n, cfg, st, only_rank);
    case FC_DTYPE_BF16 * 3 + FC_DTYPE_BF16:
      return run_l8_f<__nv_bfloat16, __nv_bfloat16>(c, ins, outs, n, cfg, st, only_rank);
    default: return fail(FC_ERR_CONFIG, "output dtype must equal the input dtype or be float32");
  }
}

// single-GPU minifloat codec (fc_quantize / fc_dequantize): compile-time format
template <int F>
static fc_status l8_quant_f(const void* x, int in_dt, int64_t n, const DevCodec& dc, void* dst, uint32_t* err,
                            cudaStream_t st, unsigned grid) {
  switch (in_dt) {
    case FC_DTYPE_F32: k_l8_quant<float, F><<<grid, kL8Threads, 0, st>>>((const float*)x, n, dc, (uint8_t*)dst, err); break;
    case FC_DTYPE_F16: k_l8_quant<__half, F><<<grid, kL8Threads, 0, st>>>((const __half*)x, n, dc, (uint8_t*)dst, err); break;
    default:
      k_l8_quant<__nv_bfloat16, F><<<grid, kL8Threads, 0, st>>>((const __nv_bfloat16*)x, n, dc, (uint8_t*)dst, err);
  }
  FC_CUDA_TRY(cudaGetLastError());
  return FC_OK;
}
template <int F>
static fc_status l8_dequant_f(const void* src, int64_t n, const DevCodec& dc, void* out, int out_dt, cudaStream_t st,
                              unsigned grid) {
  switch (out_dt) {
    case FC_DTYPE_F32: k_l8_dequant<float, F><<<grid, kL8Threads, 0, st>>>((const uint8_t*)src, n, dc, (float*)out); break;
    case FC_DTYPE_F16: k_l8_dequant<__half, F><<<grid, kL8Threads, 0, st>>>((const uint8_t*)src, n, dc, (__half*)out); break;
    default:
      k_l8_dequant<__nv_bfloat16, F><<<grid, kL8Threads, 0, st>>>((const uint8_t*)src, n, dc, (__nv_bfloat16*)out);
  }
  FC_CUDA_TRY(cudaGetLastError());
  return FC_OK;
}

fc_status l8_codec_quantize(const void* x, int in_dt, int64_t n, const DevCodec& dc, void* dst, uint32_t* err,
                            cudaStream_t st) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned grid = l8_grid(dev, ceil_div(n, (int64_t)kL8), 1);
  switch (dc.mf_fmt) {
    case FC_FMT_E4M3: return l8_quant_f<1>(x, in_dt, n, dc, dst, err, st, grid);
    case FC_FMT_E5M2: return l8_quant_f<2>(x, in_dt, n, dc, dst, err, st, grid);
    default: return l8_quant_f<3>(x, in_dt, n, dc, dst, err, st, grid);
  }
}
fc_status l8_codec_dequantize(const void* src, int64_t n, const DevCodec& dc, void* out, int out_dt, cudaStream_t st) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned grid = l8_grid(dev, ceil_div(n, (int64_t)kL8), 1);
  switch (dc.mf_fmt) {
    case FC_FMT_E4M3: return l8_dequant_f<1>(src, n, dc, out, out_dt, st, grid);
    case FC_FMT_E5M2: return l8_dequant_f<2>(src, n, dc, out, out_dt, st, grid);
    default: return l8_dequant_f<3>(src, n, dc, out, out_dt, st, grid);
  }
}

}  // namespace fc
