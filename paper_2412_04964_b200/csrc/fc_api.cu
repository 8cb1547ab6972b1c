// C ABI of the B200 Flash All-Reduce: codec entry points, the communicator
// (CUDA-IPC / P2P peer-buffer manager + topology discovery) and the
// flash_all_reduce orchestration. See include/flashcomm.h.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>

#include "fc_comm.h"
#include "fc_flash.cuh"

namespace fc {

// the flash all-reduce instantiations live in the generated fc_run_*.cu units
#define FC_EXTERN_RUN(TI, TO)                                                                                    \
  extern template fc_status run_typed<TI, TO>(fc_comm*, const void* const*, void* const*, int64_t, const fc_flash_cfg*, \
                                               cudaStream_t*, int);
FC_EXTERN_RUN(float, float)
FC_EXTERN_RUN(__half, float)
FC_EXTERN_RUN(__half, __half)
FC_EXTERN_RUN(__nv_bfloat16, float)
FC_EXTERN_RUN(__nv_bfloat16, __nv_bfloat16)
#undef FC_EXTERN_RUN

static thread_local std::string g_err;
thread_local int64_t g_launch_count = 0;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
}

fc_status fail(fc_status s, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

// codec.py:61-73
fc_status validate_codec(const fc_codec* c) {
  if (!c) return fail(FC_ERR_CONFIG, "codec is NULL");
  if (c->kind == FC_KIND_FP16) return FC_OK;
  if (c->kind == FC_KIND_MINIFLOAT) {
    if (c->reserved < FC_FMT_E4M3 || c->reserved > FC_FMT_E2M1)
      return fail(FC_ERR_CONFIG, "minifloat format must be one of ('e4m3', 'e5m2', 'e2m1')");
    if (c->group_size < 1) return fail(FC_ERR_CONFIG, "group_size must be >= 1");
    if (!(c->scale_floor > 0)) return fail(FC_ERR_CONFIG, "scale_floor must be positive");
    return FC_OK;
  }
  if (c->kind != FC_KIND_INT) return fail(FC_ERR_CONFIG, "unknown codec kind %d", c->kind);
  if (c->bits < 2 || c->bits > 8) return fail(FC_ERR_CONFIG, "bits must be in 2..8, got %d", c->bits);
  if (c->group_size < 1) return fail(FC_ERR_CONFIG, "group_size must be >= 1");
  if (c->rounding != FC_ROUND_NEAREST_EVEN && c->rounding != FC_ROUND_CEIL)
    return fail(FC_ERR_CONFIG, "rounding must be one of ('nearest-even', 'ceil')");
  if (!(c->scale_floor > 0)) return fail(FC_ERR_CONFIG, "scale_floor must be positive");
  return FC_OK;
}

int64_t group_of(const fc_codec& c) { return c.kind == FC_KIND_FP16 ? 1 : c.group_size; }

// collectives.py:56-75
static fc_status resolve_chunk(const fc_flash_cfg* cfg, int world, int64_t* out) {
  const int64_t mult = std::lcm(group_of(cfg->stage1), group_of(cfg->stage2));
  const int64_t unit = (int64_t)world * mult;
  const int64_t dflt = 64 * 1024;
  if (cfg->chunk_elems <= 0) {
    *out = std::max<int64_t>(1, ceil_div(dflt, unit)) * unit;
    return FC_OK;
  }
  if (cfg->chunk_elems % unit != 0)
    return fail(FC_ERR_CONFIG, "chunk_size %lld must be a multiple of world_size*group lcm = %lld",
                (long long)cfg->chunk_elems, (long long)unit);
  *out = cfg->chunk_elems;
  return FC_OK;
}

}  // namespace fc

using namespace fc;

// ============================================================================
// communicator


static int64_t block_bytes_for(int world, int64_t slot_bytes, int64_t flags_cap) {
  return blk_misc_off(world, slot_bytes, flags_cap) + kMiscBytes;
}

static fc_status comm_init_common(fc_comm* c, int world, int64_t slot_bytes) {
  if (world < 1 || world > kMaxRanks) return fail(FC_ERR_CONFIG, "world_size must be in 1..%d, got %d", kMaxRanks, world);
  if (slot_bytes < 4096) return fail(FC_ERR_CONFIG, "slot_bytes must be >= 4096");
  c->world = world;
  c->slot_bytes = align_up(slot_bytes, 256);
  c->flags_cap = align_up(c->slot_bytes / 2048 + 16, 64);
  c->block_bytes = block_bytes_for(world, c->slot_bytes, c->flags_cap);
  return FC_OK;
}

static fc_status alloc_block(fc_comm* c, int r) {
  FC_CUDA_TRY(cudaSetDevice(c->devices[r]));
  void* p = nullptr;
  FC_CUDA_TRY(cudaMalloc(&p, (size_t)c->block_bytes));
  FC_CUDA_TRY(cudaMemset(p, 0, (size_t)c->block_bytes));
  FC_CUDA_TRY(cudaDeviceSynchronize());
  c->blk[r] = (uint8_t*)p;
  c->owned[r] = true;
  FC_CUDA_TRY(cudaEventCreateWithFlags(&c->ev[r], cudaEventDisableTiming));
  return FC_OK;
}

extern "C" {

const char* fc_version(void) { return "flashcomm 0.1.0 (sm_100a)"; }
const char* fc_last_error(void) { return g_err.c_str(); }

fc_status fc_codec_validate(const fc_codec* codec) { return validate_codec(codec); }

fc_status fc_codec_layout(const fc_codec* codec, int64_t n, fc_layout* out) {
  FC_TRY(validate_codec(codec));
  if (n < 0 || !out) return fail(FC_ERR_DOMAIN, "invalid element count");
  *out = layout_of(*codec, n);
  return FC_OK;
}

fc_status fc_hadamard(const void* x, int32_t in_dtype, int64_t n, int64_t n_padded, int32_t dim, int32_t normalize,
                      const float* signs, int32_t inverse, void* out, int32_t out_dtype, int64_t n_out, void* stream) {
  if (!x || !out) return fail(FC_ERR_CONFIG, "NULL buffer");
  if (!dtype_ok(in_dtype) || !dtype_ok(out_dtype)) return fail(FC_ERR_CONFIG, "unsupported dtype");
  if (dim < 1 || (dim & (dim - 1)) != 0) return fail(FC_ERR_CONFIG, "dimension must be a power of two >= 1, got %d", dim);
  if (dim > 8192) return fail(FC_ERR_CONFIG, "Hadamard block dimension %d exceeds 8192 on the GPU path", dim);
  if (n < 0 || n_padded < n || n_out < 0 || n_out > n_padded)
    return fail(FC_ERR_DOMAIN, "invalid lengths (n=%lld, padded=%lld)", (long long)n, (long long)n_padded);
  if (n_padded % dim != 0)  // rotation.py:53-58
    return fail(FC_ERR_DOMAIN, "length %lld is not divisible by block dimension %d", (long long)n_padded, dim);
  if (n_padded == 0) return FC_OK;
  return launch_hadamard(x, in_dtype, n, n_padded, dim, normalize, signs, inverse, out, out_dtype, n_out,
                         (cudaStream_t)stream);
}

fc_status fc_flash_resolve_chunk(const fc_flash_cfg* cfg, int32_t world, int64_t* chunk_out) {
  if (!cfg || !chunk_out) return fail(FC_ERR_CONFIG, "NULL argument");
  FC_TRY(validate_codec(&cfg->stage1));
  FC_TRY(validate_codec(&cfg->stage2));
  if (world < 1) return fail(FC_ERR_CONFIG, "world_size must be >= 1");
  return resolve_chunk(cfg, world, chunk_out);
}

fc_status fc_quantize(const void* x, int32_t in_dtype, int64_t n, const fc_codec* codec, void* dst,
                      uint32_t* err_word, void* stream) {
  FC_TRY(validate_codec(codec));
  if (!dtype_ok(in_dtype)) return fail(FC_ERR_CONFIG, "unsupported dtype %d", in_dtype);
  if (n <= 0) return fail(FC_ERR_DOMAIN, "input tensor is empty");
  if (!x || !dst) return fail(FC_ERR_DOMAIN, "NULL buffer");
  return launch_quantize(x, in_dtype, n, *codec, dst, err_word, (cudaStream_t)stream, true);
}

fc_status fc_dequantize(const void* src, int64_t n, const fc_codec* codec, void* out, int32_t out_dtype,
                        void* stream) {
  FC_TRY(validate_codec(codec));
  if (!dtype_ok(out_dtype)) return fail(FC_ERR_CONFIG, "unsupported dtype %d", out_dtype);
  if (n <= 0) return fail(FC_ERR_DOMAIN, "input tensor is empty");
  if (!src || !out) return fail(FC_ERR_DOMAIN, "NULL buffer");
  return launch_dequantize(src, n, *codec, out, out_dtype, (cudaStream_t)stream, true);
}

static fc_status decode_err_word(uint32_t w) {
  if (w == 0) return FC_OK;
  const uint32_t kind = w >> 28, phase = (w >> 20) & 0xFF, peer = (w >> 10) & 0x3FF, rank = w & 0x3FF;
  static const char* names[] = {"?", "scatter", "reduce", "gather", "barrier"};
  if (kind == kErrNonFinite) return fail(FC_ERR_DOMAIN, "input contains NaN or infinity (rank %u)", rank);
  if (kind == kErrTimeout)
    return fail(FC_ERR_PROTOCOL, "deadlock: rank %u timed out waiting on rank %u (%s)", rank, peer,
                names[phase < 5 ? phase : 0]);
  return fail(FC_ERR_PROTOCOL, "device error word 0x%08x", w);
}

fc_status fc_error_word_check(const uint32_t* err_word, void* stream) {
  FC_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  if (!err_word) return FC_OK;
  uint32_t w = 0;
  FC_CUDA_TRY(cudaMemcpy(&w, err_word, 4, cudaMemcpyDeviceToHost));
  return decode_err_word(w);
}

fc_status fc_comm_create_local(int32_t world, const int32_t* devices, int64_t slot_bytes, fc_comm** out) {
  if (!out || !devices) return fail(FC_ERR_CONFIG, "NULL argument");
  fc_comm* c = new fc_comm();
  fc_status s = comm_init_common(c, world, slot_bytes);
  if (s != FC_OK) {
    delete c;
    return s;
  }
  c->ipc = false;
  for (int r = 0; r < world; ++r) c->devices[r] = devices[r];
  for (int r = 0; r < world; ++r) {
    s = alloc_block(c, r);
    if (s != FC_OK) {
      fc_comm_destroy(c);
      return s;
    }
  }
  // P2P between distinct devices (NVLink through NVSwitch on one B200 box)
  for (int a = 0; a < world; ++a)
    for (int b = 0; b < world; ++b) {
      if (c->devices[a] == c->devices[b]) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, c->devices[a], c->devices[b]);
      if (!can) {
        fc_comm_destroy(c);
        return fail(FC_ERR_CONFIG, "device %d cannot access peer device %d", c->devices[a], c->devices[b]);
      }
      cudaSetDevice(c->devices[a]);
      cudaError_t e = cudaDeviceEnablePeerAccess(c->devices[b], 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
        fc_comm_destroy(c);
        return fail(FC_ERR_CUDA, "cudaDeviceEnablePeerAccess(%d->%d): %s", c->devices[a], c->devices[b],
                    cudaGetErrorString(e));
      }
      cudaGetLastError();
    }
  *out = c;
  return FC_OK;
}

fc_status fc_comm_create_ipc(int32_t world, int32_t rank, int32_t device, int64_t slot_bytes, fc_comm** out) {
  if (!out) return fail(FC_ERR_CONFIG, "NULL argument");
  if (rank < 0 || rank >= world) return fail(FC_ERR_CONFIG, "rank %d outside world of size %d", rank, world);
  fc_comm* c = new fc_comm();
  fc_status s = comm_init_common(c, world, slot_bytes);
  if (s != FC_OK) {
    delete c;
    return s;
  }
  c->ipc = true;
  c->my_rank = rank;
  for (int r = 0; r < world; ++r) c->devices[r] = device;
  s = alloc_block(c, rank);
  if (s != FC_OK) {
    fc_comm_destroy(c);
    return s;
  }
  *out = c;
  return FC_OK;
}

fc_status fc_comm_ipc_handle(fc_comm* c, void* handle_out) {
  if (!c || !c->ipc || !handle_out) return fail(FC_ERR_CONFIG, "not an IPC communicator");
  FC_CUDA_TRY(cudaSetDevice(c->devices[c->my_rank]));
  cudaIpcMemHandle_t h;
  FC_CUDA_TRY(cudaIpcGetMemHandle(&h, c->blk[c->my_rank]));
  static_assert(sizeof(h) == FC_IPC_HANDLE_BYTES, "IPC handle size");
  memcpy(handle_out, &h, sizeof h);
  return FC_OK;
}

fc_status fc_comm_ipc_open(fc_comm* c, const void* handles) {
  if (!c || !c->ipc || !handles) return fail(FC_ERR_CONFIG, "not an IPC communicator");
  FC_CUDA_TRY(cudaSetDevice(c->devices[c->my_rank]));
  for (int p = 0; p < c->world; ++p) {
    if (p == c->my_rank || c->opened[p]) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, (const uint8_t*)handles + (size_t)p * FC_IPC_HANDLE_BYTES, sizeof h);
    void* ptr = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess)
      return fail(FC_ERR_PROTOCOL, "rank %d cannot map rank %d's buffers: %s", c->my_rank, p, cudaGetErrorString(e));
    c->blk[p] = (uint8_t*)ptr;
    c->opened[p] = true;
  }
  return FC_OK;
}

fc_status fc_comm_destroy(fc_comm* c) {
  if (!c) return FC_OK;
  for (int r = 0; r < kMaxRanks; ++r) {
    if (c->owned[r] && c->blk[r]) {
      cudaSetDevice(c->devices[r]);
      cudaDeviceSynchronize();
      cudaFree(c->blk[r]);
    }
    if (c->opened[r] && c->blk[r]) cudaIpcCloseMemHandle(c->blk[r]);
    if (c->scratch[r]) cudaFree(c->scratch[r]);
    if (c->tprof[r]) cudaFree(c->tprof[r]);
    if (c->ev[r]) cudaEventDestroy(c->ev[r]);
    if (c->hs_in[r] || c->hs_out[r] || c->hs_h2d[r]) cudaSetDevice(c->devices[r]);
    if (c->hs_in[r]) cudaFree(c->hs_in[r]);
    if (c->hs_out[r]) cudaFree(c->hs_out[r]);
    if (c->hs_h2d[r]) cudaStreamDestroy(c->hs_h2d[r]);
    if (c->hs_comp[r]) cudaStreamDestroy(c->hs_comp[r]);
    if (c->hs_d2h[r]) cudaStreamDestroy(c->hs_d2h[r]);
  }
  for (cudaEvent_t e : c->hs_ev)
    if (e) cudaEventDestroy(e);
  cudaGetLastError();
  delete c;
  return FC_OK;
}

fc_status fc_comm_set_option(fc_comm* c, int32_t option, int64_t value) {
  if (!c) return fail(FC_ERR_CONFIG, "NULL communicator");
  switch (option) {
    case FC_OPT_FUSED: c->fused = value < 0 ? -1 : (value != 0); break;
    case FC_OPT_CTAS: c->ctas = std::max<int64_t>(0, value); break;
    case FC_OPT_TIMEOUT_MS:
      if (value <= 0) return fail(FC_ERR_CONFIG, "timeout must be positive");
      c->timeout_ms = value;
      break;
    case FC_OPT_LAG: c->lag = std::max<int64_t>(0, value); break;
    case FC_OPT_FAST: c->fast = value < 0 ? 0 : (value > 2 ? 2 : value); break;
    case FC_OPT_REDUCE_STAGES: c->reduce_stages = std::max<int64_t>(0, std::min<int64_t>(32, value)); break;
    case FC_OPT_SCATTER_STAGES: c->q_stages = std::max<int64_t>(0, std::min<int64_t>(8, value)); break;
    case FC_OPT_GATHER_STAGES: c->d_stages = std::max<int64_t>(0, std::min<int64_t>(12, value)); break;
    case FC_OPT_CTAS_PER_SM: c->ctas_per_sm = std::max<int64_t>(0, std::min<int64_t>(16, value)); break;
    case FC_OPT_STREAM_MASK: c->stream_mask = value & 65535; break;
    case FC_OPT_PHASES: c->phases = value & 7; break;
    case FC_OPT_ONESHOT: c->oneshot = value < 0 ? 0 : (value > 2 ? 2 : value); break;
    case FC_OPT_FUSED_CHUNK: c->fused_chunk = std::max<int64_t>(0, value); break;
    case FC_OPT_HOST_CHUNK_BYTES: c->host_chunk_bytes = std::max<int64_t>(0, value); break;
    case FC_OPT_FUSED_GATHER_CTAS: c->fused_gather_ctas = std::max<int64_t>(0, std::min<int64_t>(16, value)); break;
    case FC_OPT_ROLE_PROFILE: c->role_profile = value != 0; break;
    default: return fail(FC_ERR_CONFIG, "unknown option %d", option);
  }
  return FC_OK;
}

fc_status fc_comm_get_option(fc_comm* c, int32_t option, int64_t* value) {
  if (!c || !value) return fail(FC_ERR_CONFIG, "NULL argument");
  switch (option) {
    case FC_OPT_FUSED: *value = c->fused; break;
    case FC_OPT_CTAS: *value = c->ctas; break;
    case FC_OPT_TIMEOUT_MS: *value = c->timeout_ms; break;
    case FC_OPT_LAG: *value = c->lag; break;
    case FC_OPT_FAST: *value = c->fast; break;
    case FC_OPT_LAST_LAUNCHES: *value = c->last_launches; break;
    case FC_OPT_REDUCE_STAGES: *value = c->reduce_stages; break;
    case FC_OPT_SCATTER_STAGES: *value = c->q_stages; break;
    case FC_OPT_GATHER_STAGES: *value = c->d_stages; break;
    case FC_OPT_CTAS_PER_SM: *value = c->ctas_per_sm; break;
    case FC_OPT_STREAM_MASK: *value = c->stream_mask; break;
    case FC_OPT_PHASES: *value = c->phases; break;
    case FC_OPT_ONESHOT: *value = c->oneshot; break;
    case FC_OPT_FUSED_CHUNK: *value = c->fused_chunk; break;
    case FC_OPT_HOST_CHUNK_BYTES: *value = c->host_chunk_bytes; break;
    case FC_OPT_FUSED_GATHER_CTAS: *value = c->fused_gather_ctas; break;
    case FC_OPT_ROLE_PROFILE: *value = c->role_profile; break;
    default: return fail(FC_ERR_CONFIG, "unknown option %d", option);
  }
  return FC_OK;
}

}  // extern "C"

// ============================================================================
// flash all-reduce orchestration

namespace {

#define FC_DISPATCH2(IN_DT, OUT_DT, FN, ...)                                                     \
  [&]() -> fc_status {                                                                           \
    switch ((IN_DT) * 3 + (OUT_DT)) {                                                            \
      case FC_DTYPE_F32 * 3 + FC_DTYPE_F32: return FN<float, float>(__VA_ARGS__);                \
      case FC_DTYPE_F32 * 3 + FC_DTYPE_F16: return FN<float, __half>(__VA_ARGS__);               \
      case FC_DTYPE_F32 * 3 + FC_DTYPE_BF16: return FN<float, __nv_bfloat16>(__VA_ARGS__);       \
      case FC_DTYPE_F16 * 3 + FC_DTYPE_F32: return FN<__half, float>(__VA_ARGS__);               \
      case FC_DTYPE_F16 * 3 + FC_DTYPE_F16: return FN<__half, __half>(__VA_ARGS__);              \
      case FC_DTYPE_F16 * 3 + FC_DTYPE_BF16: return FN<__half, __nv_bfloat16>(__VA_ARGS__);      \
      case FC_DTYPE_BF16 * 3 + FC_DTYPE_F32: return FN<__nv_bfloat16, float>(__VA_ARGS__);       \
      case FC_DTYPE_BF16 * 3 + FC_DTYPE_F16: return FN<__nv_bfloat16, __half>(__VA_ARGS__);      \
      default: return FN<__nv_bfloat16, __nv_bfloat16>(__VA_ARGS__);                              \
    }                                                                                            \
  }()

// flash kernels exist for out dtype == in dtype, or float32 out
#define FC_DISPATCH_RUN(IN_DT, OUT_DT, ...)                                                      \
  [&]() -> fc_status {                                                                           \
    switch ((IN_DT) * 3 + (OUT_DT)) {                                                            \
      case FC_DTYPE_F32 * 3 + FC_DTYPE_F32: return run_typed<float, float>(__VA_ARGS__);         \
      case FC_DTYPE_F16 * 3 + FC_DTYPE_F32: return run_typed<__half, float>(__VA_ARGS__);        \
      case FC_DTYPE_F16 * 3 + FC_DTYPE_F16: return run_typed<__half, __half>(__VA_ARGS__);       \
      case FC_DTYPE_BF16 * 3 + FC_DTYPE_F32: return run_typed<__nv_bfloat16, float>(__VA_ARGS__); \
      case FC_DTYPE_BF16 * 3 + FC_DTYPE_BF16:                                                    \
        return run_typed<__nv_bfloat16, __nv_bfloat16>(__VA_ARGS__);                             \
      default:                                                                                   \
        return fail(FC_ERR_CONFIG, "output dtype must equal the input dtype or be float32");    \
    }                                                                                            \
  }()

inline bool dispatch_ok(int in_dt, int out_dt) { return in_dt == out_dt || out_dt == FC_DTYPE_F32; }

inline fc_status check_call(const fc_comm* c, int64_t n, int in_dt, int out_dt, const fc_flash_cfg* cfg) {
  if (!c) return fail(FC_ERR_CONFIG, "NULL communicator");
  if (!cfg) return fail(FC_ERR_CONFIG, "flash method needs a FlashConfig");
  FC_TRY(validate_codec(&cfg->stage1));
  FC_TRY(validate_codec(&cfg->stage2));
  if (!dtype_ok(in_dt) || !dtype_ok(out_dt)) return fail(FC_ERR_CONFIG, "unsupported dtype");
  if (n <= 0) return fail(FC_ERR_DOMAIN, "rank tensors must be nonempty");
  int64_t chunk = 0;
  return resolve_chunk(cfg, c->world, &chunk);
}

}  // namespace

extern "C" {

fc_status fc_flash_all_reduce_local(fc_comm* c, const void* const* ins, void* const* outs, int64_t n, int32_t in_dtype,
                                    int32_t out_dtype, const fc_flash_cfg* cfg, void* const* streams) {
  FC_TRY(check_call(c, n, in_dtype, out_dtype, cfg));
  if (c->ipc) return fail(FC_ERR_CONFIG, "fc_flash_all_reduce_local needs a local communicator");
  if (!ins || !outs) return fail(FC_ERR_DOMAIN, "NULL buffer list");
  for (int r = 0; r < c->world; ++r)
    if (!ins[r] || !outs[r]) return fail(FC_ERR_DOMAIN, "NULL buffer for rank %d", r);
  cudaStream_t st[kMaxRanks];
  for (int r = 0; r < c->world; ++r) st[r] = streams ? (cudaStream_t)streams[r] : (cudaStream_t)0;
  if (c->world == 1) return FC_DISPATCH2(in_dtype, out_dtype, identity_typed, ins[0], outs[0], n, c->devices[0], st[0]);
  if (l8_wanted(c, cfg, n)) return run_l8(in_dtype, out_dtype, c, ins, outs, n, cfg, st, -1);
  if (c->rot_dim) return fail(FC_ERR_CONFIG, "rotation cannot be fused at this size / codec");
  return FC_DISPATCH_RUN(in_dtype, out_dtype, c, ins, outs, n, cfg, st, -1);
}

fc_status fc_flash_all_reduce(fc_comm* c, const void* in, void* out, int64_t n, int32_t in_dtype, int32_t out_dtype,
                              const fc_flash_cfg* cfg, void* stream) {
  FC_TRY(check_call(c, n, in_dtype, out_dtype, cfg));
  if (!c->ipc) return fail(FC_ERR_CONFIG, "fc_flash_all_reduce needs an IPC communicator");
  if (!in || !out) return fail(FC_ERR_DOMAIN, "NULL buffer");
  // every rank must take the same kernel path (flags / barriers, slot layouts); the path
  // depends on buffer alignment, which one process cannot see for its peers
  if ((uintptr_t)in % 16 || (uintptr_t)out % 16)
    return fail(FC_ERR_DOMAIN, "IPC all-reduce buffers must be 16-byte aligned");
  const int r = c->my_rank;
  if (c->world == 1) return FC_DISPATCH2(in_dtype, out_dtype, identity_typed, in, out, n, c->devices[r], (cudaStream_t)stream);
  for (int p = 0; p < c->world; ++p)
    if (!c->blk[p]) return fail(FC_ERR_PROTOCOL, "rank %d has not mapped rank %d (call fc_comm_ipc_open)", r, p);
  const void* ins[kMaxRanks] = {nullptr};
  void* outs[kMaxRanks] = {nullptr};
  cudaStream_t st[kMaxRanks] = {nullptr};
  ins[r] = in;
  outs[r] = out;
  st[r] = (cudaStream_t)stream;
  if (l8_wanted(c, cfg, n)) return run_l8(in_dtype, out_dtype, c, ins, outs, n, cfg, st, r);
  if (c->rot_dim) return fail(FC_ERR_CONFIG, "rotation cannot be fused at this size / codec");
  return FC_DISPATCH_RUN(in_dtype, out_dtype, c, ins, outs, n, cfg, st, r);
}

fc_status fc_comm_teardown_check(fc_comm* c) {
  if (!c) return fail(FC_ERR_CONFIG, "NULL communicator");
  if (!c->ipc) return FC_OK;  // one process drives every rank: the ranks run in lockstep
  FC_CUDA_TRY(cudaSetDevice(c->devices[c->my_rank]));
  FC_CUDA_TRY(cudaDeviceSynchronize());
  uint32_t ep[kMaxRanks] = {0};
  for (int r = 0; r < c->world; ++r) {
    if (!c->blk[r]) return fail(FC_ERR_PROTOCOL, "rank %d has not mapped rank %d", c->my_rank, r);
    const uint32_t* e = reinterpret_cast<const uint32_t*>(c->blk[r] + blk_misc_off(c->world, c->slot_bytes, c->flags_cap)) + 8;
    FC_CUDA_TRY(cudaMemcpy(&ep[r], e, 4, cudaMemcpyDeviceToHost));
  }
  std::string un;
  for (int r = 0; r < c->world; ++r)
    if (ep[r] != ep[c->my_rank]) {
      char b[96];
      snprintf(b, sizeof b, "%s(rank %d: %u rounds, rank %d: %u)", un.empty() ? "" : ", ", c->my_rank,
               ep[c->my_rank], r, ep[r]);
      un += b;
    }
  if (!un.empty()) return fail(FC_ERR_PROTOCOL, "unconsumed messages at teardown: %s", un.c_str());
  return FC_OK;
}

fc_status fc_comm_set_rotation(fc_comm* c, int32_t rank, int32_t dim, int32_t normalize, const float* signs) {
  if (!c) return fail(FC_ERR_CONFIG, "NULL communicator");
  if (dim < 0 || (dim & (dim - 1)) != 0) return fail(FC_ERR_CONFIG, "rotation dimension must be a power of two");
  if (rank < -1 || rank >= c->world) return fail(FC_ERR_CONFIG, "rank %d outside world %d", rank, c->world);
  c->rot_dim = dim;
  c->rot_normalize = normalize ? 1 : 0;
  for (int r = 0; r < c->world; ++r)
    if (rank < 0 || r == rank) c->rot_signs[r] = dim ? signs : nullptr;
  return FC_OK;
}

int32_t fc_flash_rotation_fusable(fc_comm* c, int64_t n, const fc_flash_cfg* cfg, int32_t dim) {
  if (!c || !cfg || dim <= 0) return 0;
  const int32_t keep = c->rot_dim;
  c->rot_dim = dim;
  const bool ok = l8_wanted(c, cfg, n);
  c->rot_dim = keep;
  return ok ? 1 : 0;
}

fc_status fc_comm_check(fc_comm* c, int32_t rank) {
  if (!c) return fail(FC_ERR_CONFIG, "NULL communicator");
  fc_status first = FC_OK;
  std::string msg;
  for (int r = 0; r < c->world; ++r) {
    if (rank >= 0 && r != rank) continue;
    if (c->ipc && r != c->my_rank) continue;
    FC_CUDA_TRY(cudaSetDevice(c->devices[r]));
    FC_CUDA_TRY(cudaDeviceSynchronize());
    uint32_t* ew = reinterpret_cast<uint32_t*>(c->blk[r] + blk_misc_off(c->world, c->slot_bytes, c->flags_cap));
    uint32_t w = 0;
    FC_CUDA_TRY(cudaMemcpy(&w, ew, 4, cudaMemcpyDeviceToHost));
    if (w) {
      FC_CUDA_TRY(cudaMemset(ew, 0, 4));  // latch consumed; the comm stays usable
      fc_status s = decode_err_word(w);
      if (first == FC_OK) {
        first = s;
        msg = g_err;
      }
    }
  }
  if (first != FC_OK) g_err = msg;
  return first;
}

}  // extern "C"

// ============================================================================
// host-buffer pipeline (fc_flash_all_reduce_host)

namespace {

// grow-only device staging of `bytes` on rank r's device
fc_status ensure_stage(fc_comm* c, int r, void** buf, int64_t* have, int64_t bytes) {
  if (*have >= bytes) return FC_OK;
  FC_CUDA_TRY(cudaSetDevice(c->devices[r]));
  if (*buf) {
    FC_CUDA_TRY(cudaDeviceSynchronize());
    FC_CUDA_TRY(cudaFree(*buf));
    *buf = nullptr;
    *have = 0;
  }
  FC_CUDA_TRY(cudaMalloc(buf, (size_t)bytes));
  *have = bytes;
  return FC_OK;
}

// copy the rows of one chunk: element span [lo, hi) of every segment j of a
// rank tensor of n elements (segment j starts at j*seg; the tail past n is padding)
fc_status copy_rows(void* dst, const void* src, int64_t n, int64_t seg, int world, int64_t lo, int64_t hi, int e,
                    cudaMemcpyKind kind, cudaStream_t st) {
  int full = 0;  // rows wholly inside the tensor
  while (full < world && (int64_t)full * seg + hi <= n) ++full;
  const size_t pitch = (size_t)(seg * e);
  if (full > 0)
    FC_CUDA_TRY(cudaMemcpy2DAsync((char*)dst + lo * e, pitch, (const char*)src + lo * e, pitch, (size_t)((hi - lo) * e),
                                  (size_t)full, kind, st));
  if (full < world) {
    const int64_t a = (int64_t)full * seg + lo, b = std::min(n, (int64_t)full * seg + hi);
    if (b > a) FC_CUDA_TRY(cudaMemcpyAsync((char*)dst + a * e, (const char*)src + a * e, (size_t)((b - a) * e), kind, st));
  }
  return FC_OK;
}

// only_rank >= 0: IPC world, this process is that rank (its buffers at index only_rank)
fc_status host_pipeline(fc_comm* c, const void* const* hin, void* const* hout, int64_t n, int in_dt, int out_dt,
                        const fc_flash_cfg* cfg, int only_rank) {
  const int N = c->world;
  auto active = [&](int r) { return only_rank < 0 || r == only_rank; };
  const int ein = dtype_size(in_dt), eout = dtype_size(out_dt);
  int lead[kMaxRanks];  // the first active rank on each rank's device owns that device's streams
  for (int r = 0; r < N; ++r) {
    lead[r] = active(r) ? r : -1;
    if (!active(r)) continue;
    for (int q = 0; q < r; ++q)
      if (active(q) && c->devices[q] == c->devices[r]) {
        lead[r] = q;
        break;
      }
  }
  for (int r = 0; r < N; ++r) {
    if (!active(r)) continue;
    FC_TRY(ensure_stage(c, r, &c->hs_in[r], &c->hs_in_bytes[r], n * ein));
    FC_TRY(ensure_stage(c, r, &c->hs_out[r], &c->hs_out_bytes[r], n * eout));
    if (lead[r] == r && !c->hs_h2d[r]) {
      FC_CUDA_TRY(cudaSetDevice(c->devices[r]));
      FC_CUDA_TRY(cudaStreamCreateWithFlags(&c->hs_h2d[r], cudaStreamNonBlocking));
      FC_CUDA_TRY(cudaStreamCreateWithFlags(&c->hs_comp[r], cudaStreamNonBlocking));
      FC_CUDA_TRY(cudaStreamCreateWithFlags(&c->hs_d2h[r], cudaStreamNonBlocking));
    }
  }
  const void* din[kMaxRanks] = {nullptr};
  void* dout[kMaxRanks] = {nullptr};
  cudaStream_t st[kMaxRanks] = {nullptr};
  for (int r = 0; r < N; ++r) {
    if (!active(r)) continue;
    din[r] = c->hs_in[r];
    dout[r] = c->hs_out[r];
    st[r] = c->hs_comp[lead[r]];
  }
  // chunk span: a multiple of the plan unit (group lcm, and the tile for the tiled
  // kernels) so every chunk run quantizes the same groups as one whole call
  const int64_t seg = (n + N - 1) / N;
  int64_t unit = std::lcm(group_of(cfg->stage1), group_of(cfg->stage2));
  if (fast_group(cfg->stage1) && fast_group(cfg->stage2)) unit = std::lcm(unit, (int64_t)kTileElems);
  // 12 MiB of H2D per rank per chunk: large enough for full-rate 2-D copies, small enough that
  // the tail after the last H2D (its all-reduce + D2H) stays short (tools/e2e_probe.py)
  const int64_t target = c->host_chunk_bytes > 0 ? c->host_chunk_bytes : (int64_t)12 << 20;
  int64_t span = std::max<int64_t>(1, target / ((int64_t)N * ein));
  span = std::max(unit, span / unit * unit);
  if (N == 1) span = seg;
  const int64_t chunks = (seg + span - 1) / span;
  const size_t need = (size_t)(chunks * N * 2);
  if (c->hs_ev.size() < need) {
    const size_t have = c->hs_ev.size();
    c->hs_ev.resize(need, nullptr);
    for (size_t i = have; i < need; ++i) {
      const int r = (int)((i / 2) % N);
      FC_CUDA_TRY(cudaSetDevice(c->devices[r]));
      FC_CUDA_TRY(cudaEventCreateWithFlags(&c->hs_ev[i], cudaEventDisableTiming));
    }
  }
  // events are created on the device of rank (i / 2) % N; the layout is fixed per comm
  auto ev = [&](int64_t k, int r, int which) { return c->hs_ev[(size_t)((k * N + r) * 2 + which)]; };
  fc_status status = FC_OK;
  for (int64_t k = 0; k < chunks && status == FC_OK; ++k) {
    const int64_t lo = k * span, hi = std::min(seg, lo + span);
    for (int r = 0; r < N; ++r) {
      if (!active(r)) continue;
      FC_CUDA_TRY(cudaSetDevice(c->devices[r]));
      FC_TRY(copy_rows(c->hs_in[r], hin[r], n, seg, N, lo, hi, ein, cudaMemcpyHostToDevice, c->hs_h2d[lead[r]]));
      FC_CUDA_TRY(cudaEventRecord(ev(k, r, 0), c->hs_h2d[lead[r]]));
    }
    // every rank's chunk must have landed before any rank's run of it
    for (int r = 0; r < N; ++r) {
      if (lead[r] != r || !active(r)) continue;
      FC_CUDA_TRY(cudaSetDevice(c->devices[r]));
      for (int q = 0; q < N; ++q) {
        if (!active(q)) continue;
        bool last_of_dev = true;  // one wait per (device, source device): the last copy queued there
        for (int q2 = q + 1; q2 < N; ++q2) last_of_dev &= !(active(q2) && lead[q2] == lead[q]);
        if (last_of_dev) FC_CUDA_TRY(cudaStreamWaitEvent(c->hs_comp[r], ev(k, q, 0), 0));
      }
    }
    if (N == 1) {
      status = FC_DISPATCH2(in_dt, out_dt, identity_typed, din[0], dout[0], n, c->devices[0], st[0]);
    } else {
      c->span_lo = lo;
      c->span_hi = hi;
      if (only_rank >= 0) FC_CUDA_TRY(cudaSetDevice(c->devices[only_rank]));
      status = l8_wanted(c, cfg, n) ? run_l8(in_dt, out_dt, c, din, dout, n, cfg, st, only_rank)
                                    : FC_DISPATCH_RUN(in_dt, out_dt, c, din, dout, n, cfg, st, only_rank);
      c->span_lo = 0;
      c->span_hi = -1;
    }
    if (status != FC_OK) break;
    for (int r = 0; r < N; ++r) {
      if (!active(r) || !hout[r]) continue;
      FC_CUDA_TRY(cudaSetDevice(c->devices[r]));
      FC_CUDA_TRY(cudaEventRecord(ev(k, r, 1), st[r]));
      FC_CUDA_TRY(cudaStreamWaitEvent(c->hs_d2h[lead[r]], ev(k, r, 1), 0));
      FC_TRY(copy_rows(hout[r], c->hs_out[r], n, seg, N, lo, hi, eout, cudaMemcpyDeviceToHost, c->hs_d2h[lead[r]]));
    }
  }
  for (int r = 0; r < N; ++r) {
    if (lead[r] != r || !active(r)) continue;
    FC_CUDA_TRY(cudaSetDevice(c->devices[r]));
    FC_CUDA_TRY(cudaStreamSynchronize(c->hs_h2d[r]));
    FC_CUDA_TRY(cudaStreamSynchronize(c->hs_comp[r]));
    FC_CUDA_TRY(cudaStreamSynchronize(c->hs_d2h[r]));
  }
  return status;
}

}  // namespace

extern "C" {

fc_status fc_flash_all_reduce_host(fc_comm* c, const void* const* host_ins, void* const* host_outs, int64_t n,
                                   int32_t in_dtype, int32_t out_dtype, const fc_flash_cfg* cfg) {
  FC_TRY(check_call(c, n, in_dtype, out_dtype, cfg));
  if (c->ipc) return fail(FC_ERR_CONFIG, "fc_flash_all_reduce_host needs a local communicator");
  if (!host_ins || !host_outs) return fail(FC_ERR_DOMAIN, "NULL buffer list");
  for (int r = 0; r < c->world; ++r)
    if (!host_ins[r]) return fail(FC_ERR_DOMAIN, "NULL input buffer for rank %d", r);
  if (c->world > 1 && !dispatch_ok(in_dtype, out_dtype))
    return fail(FC_ERR_CONFIG, "output dtype must equal the input dtype or be float32");
  FC_TRY(host_pipeline(c, host_ins, host_outs, n, in_dtype, out_dtype, cfg, -1));
  return fc_comm_check(c, -1);
}

fc_status fc_flash_all_reduce_host_rank(fc_comm* c, const void* host_in, void* host_out, int64_t n, int32_t in_dtype,
                                        int32_t out_dtype, const fc_flash_cfg* cfg) {
  FC_TRY(check_call(c, n, in_dtype, out_dtype, cfg));
  if (!c->ipc) return fail(FC_ERR_CONFIG, "fc_flash_all_reduce_host_rank needs an IPC communicator");
  if (!host_in) return fail(FC_ERR_DOMAIN, "NULL input buffer");
  if (c->world > 1 && !dispatch_ok(in_dtype, out_dtype))
    return fail(FC_ERR_CONFIG, "output dtype must equal the input dtype or be float32");
  const int r = c->my_rank;
  for (int p = 0; p < c->world; ++p)
    if (!c->blk[p]) return fail(FC_ERR_PROTOCOL, "rank %d has not mapped rank %d (call fc_comm_ipc_open)", r, p);
  const void* ins[kMaxRanks] = {nullptr};
  void* outs[kMaxRanks] = {nullptr};
  ins[r] = host_in;
  outs[r] = host_out;
  FC_TRY(host_pipeline(c, ins, outs, n, in_dtype, out_dtype, cfg, r));
  return fc_comm_check(c, r);
}

fc_status fc_comm_slot(fc_comm* c, int32_t rank, int32_t stage, int32_t src, void* dst, fc_layout* layout) {
  if (!c || !layout) return fail(FC_ERR_CONFIG, "NULL argument");
  if (rank < 0 || rank >= c->world || src < 0 || src >= c->world || !c->blk[rank])
    return fail(FC_ERR_DOMAIN, "rank/src out of range");
  if (stage != 1 && stage != 2) return fail(FC_ERR_DOMAIN, "stage must be 1 or 2");
  if (c->last_R <= 0) return fail(FC_ERR_PROTOCOL, "no flash_all_reduce has run on this communicator");
  const fc_codec& cc = stage == 1 ? c->last_c1 : c->last_c2;
  fc_layout L = layout_of(cc, c->last_R);
  const fc_layout Ln = layout_of(cc, c->last_sub_len);
  L.elements = Ln.elements;  // offsets follow the round capacity, counts the last round
  L.groups = Ln.groups;
  L.codes_bytes = Ln.codes_bytes;
  L.wire_bytes = Ln.wire_bytes;
  *layout = L;
  if (dst) {
    const uint8_t* p = stage == 1 ? h_recv_slot(c, rank, src) : h_gath_slot(c, rank, src);
    FC_CUDA_TRY(cudaSetDevice(c->devices[c->ipc ? c->my_rank : rank]));
    FC_CUDA_TRY(cudaDeviceSynchronize());
    FC_CUDA_TRY(cudaMemcpy(dst, p, (size_t)L.total_bytes, cudaMemcpyDefault));
  }
  return FC_OK;
}

fc_status fc_comm_role_profile(fc_comm* c, int32_t rank, uint64_t* host_dst, int32_t max_ctas, int32_t* ctas) {
  if (!c || !host_dst) return fail(FC_ERR_CONFIG, "NULL argument");
  if (rank < 0 || rank >= c->world) return fail(FC_ERR_DOMAIN, "rank out of range");
  if (!c->tprof[rank] || c->tprof_ctas[rank] <= 0)
    return fail(FC_ERR_PROTOCOL, "no profiled fused launch on rank %d (set FC_OPT_ROLE_PROFILE)", rank);
  const int n = std::min(max_ctas, c->tprof_ctas[rank]);
  FC_CUDA_TRY(cudaSetDevice(c->devices[rank]));
  FC_CUDA_TRY(cudaDeviceSynchronize());
  FC_CUDA_TRY(cudaMemcpy(host_dst, c->tprof[rank], (size_t)n * FC_ROLE_PROFILE_U64 * 8, cudaMemcpyDeviceToHost));
  if (ctas) *ctas = c->tprof_ctas[rank];
  return FC_OK;
}

fc_status fc_comm_topology(fc_comm* c, int32_t* can_access, int32_t* multicast) {
  if (!c) return fail(FC_ERR_CONFIG, "NULL communicator");
  const int N = c->world;
  if (can_access) {
    for (int a = 0; a < N; ++a)
      for (int b = 0; b < N; ++b) {
        int v = 1;
        if (c->devices[a] != c->devices[b]) cudaDeviceCanAccessPeer(&v, c->devices[a], c->devices[b]);
        can_access[a * N + b] = v;
      }
  }
  if (multicast) {
    *multicast = 0;
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuDeviceGetAttribute", &fn, cudaEnableDefault, &q) == cudaSuccess && fn &&
        q == cudaDriverEntryPointSuccess) {
      typedef CUresult (*GetAttr)(int*, CUdevice_attribute, CUdevice);
      int v = 0;
      if (((GetAttr)fn)(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, c->devices[c->ipc ? c->my_rank : 0]) ==
          CUDA_SUCCESS)
        *multicast = v;
    }
    cudaGetLastError();
  }
  return FC_OK;
}

}  // extern "C"
