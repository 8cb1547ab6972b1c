// Host-side helpers shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdarg>
#include <cmath>
#include <cstdio>
#include <map>
#include <mutex>
#include <tuple>
#include <string>

#include "../../include/flashcomm.h"
#include "fc_common.cuh"

namespace fc {

void set_error(const char* fmt, ...);

#define FC_CUDA_TRY(expr)                                                             \
  do {                                                                                \
    cudaError_t e_ = (expr);                                                          \
    if (e_ != cudaSuccess) {                                                          \
      ::fc::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__); \
      return FC_ERR_CUDA;                                                             \
    }                                                                                 \
  } while (0)

#define FC_TRY(expr)                  \
  do {                                \
    fc_status s_ = (expr);            \
    if (s_ != FC_OK) return s_;       \
  } while (0)

inline int64_t align_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }
inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// minifloat.py:40-45: (exp bits, mantissa bits, bias, max finite)
struct MiniFmt {
  int e, m, bias;
  double max_finite;
};
inline MiniFmt minifloat_format(int id) {
  switch (id) {
    case FC_FMT_E5M2: return {5, 2, 15, 57344.0};
    case FC_FMT_E2M1: return {2, 1, 1, 6.0};
    default: return {4, 3, 7, 448.0};
  }
}

inline int storage_bits(const fc_codec& c) {
  if (c.kind == FC_KIND_FP16) return 16;
  if (c.kind == FC_KIND_MINIFLOAT) {
    const MiniFmt f = minifloat_format(c.reserved);
    return 1 + f.e + f.m <= 4 ? 4 : 8;
  }
  return c.bits <= 4 ? 4 : 8;
}

// Device layout of `n` quantized elements (see fc_layout in flashcomm.h).
// The codes region holds whole 32-element lane chunks so vector stores of a
// ragged tail stay inside the region.
inline fc_layout layout_of(const fc_codec& c, int64_t n) {
  fc_layout L{};
  const int sb = storage_bits(c);
  L.elements = n;
  L.groups = (c.kind == FC_KIND_FP16) ? 0 : ceil_div(n, c.group_size);
  L.codes_bytes = (n * sb + 7) / 8;
  const int64_t code_cap = align_up(align_up(n, kLaneElems) * sb / 8, 16);
  L.scales_offset = code_cap;
  L.zeros_offset = L.scales_offset + align_up(L.groups * 2, 16);
  const bool has_zero = c.kind == FC_KIND_INT && !c.symmetric;
  L.total_bytes = L.zeros_offset + (has_zero ? align_up(L.groups, 16) : 0);
  if (L.total_bytes == 0) L.total_bytes = 16;
  const int meta = (c.kind == FC_KIND_FP16) ? 0 : ((c.kind == FC_KIND_INT && !c.symmetric) ? 3 : 2);
  L.wire_bytes = L.codes_bytes + L.groups * meta;
  return L;
}

inline bool fast_group(const fc_codec& c) {
  if (c.kind == FC_KIND_FP16) return true;
  if (c.kind == FC_KIND_MINIFLOAT) return false;  // minifloat codes run on the generic kernels
  return c.group_size == 32 || c.group_size == 64 || c.group_size == 128 || c.group_size == 256;
}

inline double half_bits_value(uint32_t b) {
  const int e = (int)((b >> 10) & 31u), m = (int)(b & 1023u);
  return e == 0 ? std::ldexp((double)m, -24) : std::ldexp((double)(1024 + m), e - 25);
}
// smallest positive-or-zero fp16 pattern whose value is >= floor (0x7C00 = inf if none):
// the reference's "nextafter(h, +inf) while h < floor" (codec.py:246-247) after RN16
inline uint32_t floor16_of(double floor) {
  uint32_t lo = 0, hi = 0x7C00;  // answer in [lo, hi]
  while (lo < hi) {
    const uint32_t mid = (lo + hi) / 2;
    if (half_bits_value(mid) >= floor) hi = mid; else lo = mid + 1;
  }
  return lo;
}

inline DevCodec dev_codec(const fc_codec& c, const fc_layout& L) {
  DevCodec d{};
  d.kind = c.kind;
  d.bits = c.bits;
  d.g = c.group_size;
  d.sym = c.symmetric;
  d.ceil_mode = c.rounding == FC_ROUND_CEIL;
  d.sb = storage_bits(c);
  d.lpg = (c.kind == FC_KIND_INT && fast_group(c)) ? c.group_size / kLaneElems : 1;
  d.gshift = -1;
  for (int b = 0; b < 31; ++b)  // integer and minifloat groups (the streaming codec kernels index by shift)
    if ((c.kind == FC_KIND_INT || c.kind == FC_KIND_MINIFLOAT) && c.group_size == (1 << b)) d.gshift = b;
  if (c.kind == FC_KIND_INT) {
    if (c.symmetric) {
      d.qmax_f = (float)((1 << (c.bits - 1)) - 1);
      d.qmin_f = -(float)(1 << (c.bits - 1));
      d.qdiv = (double)((1 << (c.bits - 1)) - 1);
    } else {
      d.qmax_f = (float)((1 << c.bits) - 1);
      d.qmin_f = 0.0f;
      d.qdiv = (double)((1 << c.bits) - 1);
    }
  }
  d.qinv = d.qdiv > 0 ? 1.0 / d.qdiv : 0.0;
  if (c.kind == FC_KIND_MINIFLOAT) {
    const MiniFmt f = minifloat_format(c.reserved);
    d.mf_exp = f.e;
    d.mf_mant = f.m;
    d.mf_bias = f.bias;
    d.mf_fmt = c.reserved;
    d.mf_max = f.max_finite;
    d.qdiv = f.max_finite;  // raw scale = absmax / max_finite (codec.py:345)
    d.bits = 1 + f.e + f.m;
  }
  d.floor = c.scale_floor;
  d.floor16 = floor16_of(c.scale_floor);
  d.scales_off = L.scales_offset;
  d.zeros_off = L.zeros_offset;
  return d;
}

inline int dtype_size(int dt) { return dt == FC_DTYPE_F32 ? 4 : 2; }
inline bool dtype_ok(int dt) { return dt == FC_DTYPE_F32 || dt == FC_DTYPE_F16 || dt == FC_DTYPE_BF16; }

fc_status validate_codec(const fc_codec* c);
// lane-8 path (fc_l8_run.cu): minifloat stages / fused Hadamard rotation
bool l8_wanted(const fc_comm* c, const fc_flash_cfg* cfg, int64_t n);
fc_status run_l8(int in_dt, int out_dt, fc_comm* c, const void* const* ins, void* const* outs, int64_t n,
                 const fc_flash_cfg* cfg, cudaStream_t* st, int only_rank);
fc_status l8_codec_quantize(const void* x, int in_dt, int64_t n, const DevCodec& dc, void* dst, uint32_t* err,
                            cudaStream_t st);
fc_status l8_codec_dequantize(const void* src, int64_t n, const DevCodec& dc, void* out, int out_dt, cudaStream_t st);

// kernels (fc_codec.cu)
fc_status launch_quantize(const void* x, int in_dtype, int64_t n, const fc_codec& c, void* dst,
                          uint32_t* err, cudaStream_t st, bool allow_fast);
fc_status launch_dequantize(const void* src, int64_t n, const fc_codec& c, void* out, int out_dtype,
                            cudaStream_t st, bool allow_fast);

int num_sms(int device);

// cudaOccupancyMaxActiveBlocksPerMultiprocessor, memoised per (kernel, threads,
// smem, device): the query costs microseconds of host time per launch, which
// starves the GPU between short kernels (mid-size messages)
inline int occupancy(const void* kern, int threads, int smem, int dev) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int, int>, int> memo;
  const auto key = std::make_tuple(kern, threads, smem, dev);
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = memo.find(key);
    if (it != memo.end()) return it->second;
  }
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem) != cudaSuccess) occ = 0;
  std::lock_guard<std::mutex> lock(mu);
  memo[key] = occ;
  return occ;
}
fc_status launch_hadamard(const void* x, int in_dtype, int64_t n, int64_t n_padded, int dim, int normalize,
                          const float* signs, int inverse, void* out, int out_dtype, int64_t n_out, cudaStream_t st);

}  // namespace fc
