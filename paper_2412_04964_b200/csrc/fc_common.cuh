// Device-side building blocks of the B200 Flash All-Reduce (sm_100a).
//
// Numerics follow the reference group codec bit-exactly
// (/root/reference/pkg/src/qcollectives/codec.py:235-248,292-329,354-384):
//   * group min/max (absmax) over fp32 values;
//   * raw scale in float64, ONE cvt.rn.f16.f64 rounding, inf -> 65504, a
//     result below the floor moves one fp16 ulp up (codec.py:242-248);
//   * asym zero point ceil(-min/s) in float64, clamped (codec.py:321);
//   * per-element code = clamp(round(x/s) + z) with an IEEE fp32 divide
//     (x/s never lands within half an fp32 ulp of a rounding boundary when s
//     is an fp16 value, so fp32 and float64 division agree);
//   * dequant (c - z) * s is exact in fp32 (<= 9-bit int x 11-bit scale).
// Never compile with -use_fast_math.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/flashcomm.h"

namespace fc {

constexpr int kLaneElems = 32;                          // elements per thread chunk
constexpr int kThreads = 256;                           // threads per CTA
constexpr int kTileElems = kLaneElems * kThreads;       // 8192 elements per CTA tile
constexpr int kMaxRanks = FC_MAX_RANKS;

// error word layout (device): [31:28] kind, [27:20] phase, [19:10] peer, [9:0] rank
constexpr uint32_t kErrTimeout = 1u;
constexpr uint32_t kErrNonFinite = 2u;
__host__ __device__ inline uint32_t make_err(uint32_t kind, uint32_t phase, uint32_t peer, uint32_t rank) {
  return (kind << 28) | ((phase & 0xFF) << 20) | ((peer & 0x3FF) << 10) | (rank & 0x3FF);
}

// Codec as seen by kernels. Layout of a quantized buffer: codes at byte 0,
// fp16 scales at scales_off, uint8 zeros at zeros_off (both 16-B aligned).
struct DevCodec {
  int kind;        // FC_KIND_INT / FC_KIND_FP16
  int bits;        // 2..8
  int g;           // group size
  int sym;         // symmetric?
  int ceil_mode;   // rounding == ceil
  int sb;          // storage bits: 4, 8 or 16 (fp16 passthrough)
  int lpg;         // lanes per group in the fast path (g / 32), 0 if not fast
  int pad_;
  float qmax_f;    // asym: 2^b-1 ; sym: 2^(b-1)-1
  float qmin_f;    // asym: 0     ; sym: -2^(b-1)
  double qdiv;     // divisor of the raw scale: 2^b-1 (asym) or 2^(b-1)-1 (sym)
  double floor;    // scale_floor
  int64_t scales_off;
  int64_t zeros_off;
};

// --------------------------------------------------------------------------
// dtype helpers

template <typename T> struct DT;
template <> struct DT<float> {
  static __device__ __forceinline__ float to_f(float v) { return v; }
  static __device__ __forceinline__ float from_f(float v) { return v; }
};
template <> struct DT<__half> {
  static __device__ __forceinline__ float to_f(__half v) { return __half2float(v); }
  static __device__ __forceinline__ __half from_f(float v) { return __float2half_rn(v); }
};
template <> struct DT<__nv_bfloat16> {
  static __device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
  static __device__ __forceinline__ __nv_bfloat16 from_f(float v) { return __float2bfloat16_rn(v); }
};

__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ld_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p) : "memory");
  return r;
}
// L2-only load (bypasses L1): data written by other SMs / GPUs during this launch
__device__ __forceinline__ uint4 ld_cg_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ void st_v4(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

__device__ __forceinline__ void unpack2(uint32_t w, float& a, float& b, __nv_bfloat16*) {
  a = __uint_as_float(w << 16);
  b = __uint_as_float(w & 0xFFFF0000u);
}
__device__ __forceinline__ void unpack2(uint32_t w, float& a, float& b, __half*) {
  __half2 h = *reinterpret_cast<__half2*>(&w);
  float2 f = __half22float2(h);
  a = f.x;
  b = f.y;
}

// Load the 32-element lane chunk starting at element index idx0 of `base`.
// Elements k >= nvalid are outside the segment (value irrelevant; excluded by
// the caller); elements with idx0+k >= M are the zero padding of
// collectives.py:145-149.
template <typename T>
__device__ __forceinline__ void load_chunk(const T* __restrict__ base, int64_t idx0, int64_t M, int nvalid,
                                           float v[kLaneElems]) {
  if (nvalid == kLaneElems && idx0 + kLaneElems <= M) {
    if constexpr (sizeof(T) == 4) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        uint4 u = ld_nc_v4(reinterpret_cast<const float*>(base) + idx0 + 4 * q);
        v[4 * q + 0] = __uint_as_float(u.x);
        v[4 * q + 1] = __uint_as_float(u.y);
        v[4 * q + 2] = __uint_as_float(u.z);
        v[4 * q + 3] = __uint_as_float(u.w);
      }
    } else {
      uint4 u[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) u[q] = ld_nc_v4(base + idx0 + 8 * q);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        unpack2(u[q].x, v[8 * q + 0], v[8 * q + 1], (T*)nullptr);
        unpack2(u[q].y, v[8 * q + 2], v[8 * q + 3], (T*)nullptr);
        unpack2(u[q].z, v[8 * q + 4], v[8 * q + 5], (T*)nullptr);
        unpack2(u[q].w, v[8 * q + 6], v[8 * q + 7], (T*)nullptr);
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < kLaneElems; ++k) {
      int64_t i = idx0 + k;
      v[k] = (k < nvalid && i < M) ? DT<T>::to_f(base[i]) : 0.0f;
    }
  }
}

__device__ __forceinline__ uint32_t pack2(float a, float b, __nv_bfloat16*) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ uint32_t pack2(float a, float b, __half*) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

template <typename T>
__device__ __forceinline__ void store_chunk(T* __restrict__ base, int64_t idx0, int64_t M, int nvalid,
                                            const float v[kLaneElems]) {
  if (nvalid == kLaneElems && idx0 + kLaneElems <= M) {
    if constexpr (sizeof(T) == 4) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        uint4 u = make_uint4(__float_as_uint(v[4 * q]), __float_as_uint(v[4 * q + 1]),
                             __float_as_uint(v[4 * q + 2]), __float_as_uint(v[4 * q + 3]));
        st_v4(reinterpret_cast<float*>(base) + idx0 + 4 * q, u);
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 u = make_uint4(pack2(v[8 * q + 0], v[8 * q + 1], (T*)nullptr), pack2(v[8 * q + 2], v[8 * q + 3], (T*)nullptr),
                             pack2(v[8 * q + 4], v[8 * q + 5], (T*)nullptr), pack2(v[8 * q + 6], v[8 * q + 7], (T*)nullptr));
        st_v4(base + idx0 + 8 * q, u);
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < kLaneElems; ++k) {
      int64_t i = idx0 + k;
      if (k < nvalid && i < M) base[i] = DT<T>::from_f(v[k]);
    }
  }
}

// --------------------------------------------------------------------------
// scale snapping: codec.py:235-248

__device__ __forceinline__ __half snap_scale(double raw, double floor) {
  double r = raw > floor ? raw : floor;  // np.maximum(raw, floor); raw never NaN here
  __half h = __double2half(r);           // cvt.rn.f16.f64: one rounding
  unsigned short bits = __half_as_ushort(h);
  if ((bits & 0x7FFFu) == 0x7C00u) bits = 0x7BFFu;                 // inf -> 65504
  if ((double)__half2float(__ushort_as_half(bits)) < floor) bits += 1;  // nextafter(+inf)
  return __ushort_as_half(bits);
}

// --------------------------------------------------------------------------
// lane quantizer: one 32-element chunk, group of `lpg` consecutive lanes.
//
// All 32 lanes of the warp must call this together (shuffles). Elements
// k >= nvalid are excluded from the statistics and produce code 0.
// Outputs: packed codes in w[] (INT4: w[0..3], INT8: w[0..7], fp16: w[0..15]),
// the group's fp16 scale, fp32 scale and zero; returns true if a valid
// element was non-finite.

struct LaneQuant {
  uint32_t w[16];
  __half s16;
  float s;
  float zf;   // zero point as float (0 for symmetric)
  uint8_t z8;
};

__device__ __forceinline__ float group_allreduce_min(float v, int lpg) {
  for (int o = 1; o < lpg; o <<= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float group_allreduce_max(float v, int lpg) {
  for (int o = 1; o < lpg; o <<= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ bool lane_quantize(const DevCodec& c, const float v[kLaneElems], int nvalid,
                                              LaneQuant& q) {
  // non-finite detection: x*0 is NaN iff x is inf/NaN
  float probe = 0.0f;
#pragma unroll
  for (int k = 0; k < kLaneElems; ++k)
    if (k < nvalid) probe = fmaf(v[k], 0.0f, probe);
  const bool bad = probe != probe;

  if (c.kind == FC_KIND_FP16) {
#pragma unroll
    for (int k = 0; k < kLaneElems; k += 2) {
      __half2 h = __floats2half2_rn(k < nvalid ? v[k] : 0.0f, k + 1 < nvalid ? v[k + 1] : 0.0f);
      q.w[k / 2] = *reinterpret_cast<uint32_t*>(&h);
    }
    q.s16 = __ushort_as_half(0);
    q.s = 1.0f;
    q.zf = 0.0f;
    q.z8 = 0;
    return bad;
  }

  float lo = INFINITY, hi = -INFINITY;
  if (c.sym) {
#pragma unroll
    for (int k = 0; k < kLaneElems; ++k)
      if (k < nvalid) hi = fmaxf(hi, fabsf(v[k]));
    hi = group_allreduce_max(hi, c.lpg);
    q.s16 = snap_scale((double)hi / c.qdiv, c.floor);
    q.zf = 0.0f;
    q.z8 = 0;
  } else {
#pragma unroll
    for (int k = 0; k < kLaneElems; ++k)
      if (k < nvalid) {
        lo = fminf(lo, v[k]);
        hi = fmaxf(hi, v[k]);
      }
    lo = group_allreduce_min(lo, c.lpg);
    hi = group_allreduce_max(hi, c.lpg);
    q.s16 = snap_scale(((double)hi - (double)lo) / c.qdiv, c.floor);
    double z = ceil(-(double)lo / (double)__half2float(q.s16));
    z = fmin(fmax(z, 0.0), (double)c.qmax_f);
    q.zf = (float)z;
    q.z8 = (uint8_t)(int)z;
  }
  q.s = __half2float(q.s16);

  const uint32_t mask = (1u << c.bits) - 1u;
#pragma unroll
  for (int k = 0; k < kLaneElems; ++k) {
    float t = __fdiv_rn(v[k], q.s);
    t = c.ceil_mode ? ceilf(t) : rintf(t);
    t = fminf(fmaxf(t + q.zf, c.qmin_f), c.qmax_f);
    uint32_t code = (k < nvalid) ? ((uint32_t)(int)t & mask) : 0u;
    if (c.sb == 4) {
      if ((k & 7) == 0) q.w[k >> 3] = 0;
      q.w[k >> 3] |= code << (4 * (k & 7));
    } else {
      if ((k & 3) == 0) q.w[k >> 2] = 0;
      q.w[k >> 2] |= code << (8 * (k & 3));
    }
  }
  return bad;
}

// bytes of packed codes per 32-element lane chunk
__device__ __forceinline__ int lane_code_bytes(const DevCodec& c) { return c.sb * 4; }

// Store a quantized lane chunk into a buffer (local or peer memory).
// p0: element offset of the chunk within the quantized range.
__device__ __forceinline__ void store_lane(const DevCodec& c, uint8_t* buf, int64_t p0, int nvalid,
                                           const LaneQuant& q, int lane) {
  if (nvalid <= 0) return;  // chunk lies past the end of the range
  uint8_t* cp = buf + p0 * c.sb / 8;
  const int nq = c.sb / 4;  // number of 16-B vectors: 1 (int4), 2 (int8), 4 (fp16)
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (i < nq) st_v4(cp + 16 * i, make_uint4(q.w[4 * i], q.w[4 * i + 1], q.w[4 * i + 2], q.w[4 * i + 3]));
  if (c.kind == FC_KIND_INT && nvalid > 0 && (lane % c.lpg) == 0) {
    int64_t grp = p0 / c.g;
    reinterpret_cast<__half*>(buf + c.scales_off)[grp] = q.s16;
    if (!c.sym) buf[c.zeros_off + grp] = q.z8;
  }
}

// Decode helpers ------------------------------------------------------------

// float(code) via the 2^23 magic: exact for 0 <= c < 2^23 (LOP3 + FADD)
__device__ __forceinline__ float u2f_magic(uint32_t c) { return __uint_as_float(0x4B000000u | c) - 8388608.0f; }

struct LaneCodes {
  uint32_t w[16];
  float s;
  float zf;
};

__device__ __forceinline__ void load_lane(const DevCodec& c, const uint8_t* buf, int64_t p0, LaneCodes& L) {
  const uint8_t* cp = buf + p0 * c.sb / 8;
  const int nq = c.sb / 4;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (i >= nq) break;
    uint4 u = ld_cg_v4(cp + 16 * i);
    L.w[4 * i] = u.x;
    L.w[4 * i + 1] = u.y;
    L.w[4 * i + 2] = u.z;
    L.w[4 * i + 3] = u.w;
  }
  if (c.kind == FC_KIND_INT) {
    int64_t grp = p0 / c.g;
    L.s = __half2float(__ldcg(reinterpret_cast<const __half*>(buf + c.scales_off) + grp));
    L.zf = c.sym ? 0.0f : (float)__ldcg(buf + c.zeros_off + grp);
  } else {
    L.s = 1.0f;
    L.zf = 0.0f;
  }
}

// element k of a loaded lane: (c - z) * s (asym), signext(c) * s (sym), fp16 value
__device__ __forceinline__ float lane_value(const DevCodec& c, const LaneCodes& L, int k) {
  if (c.kind == FC_KIND_FP16) {
    uint32_t h = (L.w[k >> 1] >> (16 * (k & 1))) & 0xFFFFu;
    return __half2float(__ushort_as_half((unsigned short)h));
  }
  uint32_t code = (c.sb == 4) ? (L.w[k >> 3] >> (4 * (k & 7))) & 0xFu : (L.w[k >> 2] >> (8 * (k & 3))) & 0xFFu;
  float cf;
  if (c.sym) {
    int sh = 32 - c.bits;
    cf = (float)(((int)(code << sh)) >> sh);
  } else {
    cf = u2f_magic(code);
  }
  return (cf - L.zf) * L.s;
}

// --------------------------------------------------------------------------
// memory-model helpers for cross-GPU flags

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

}  // namespace fc
