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

#include <type_traits>

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
  int gshift;      // log2(g) when g is a power of two (fast path), else -1
  float qmax_f;    // asym: 2^b-1 ; sym: 2^(b-1)-1
  float qmin_f;    // asym: 0     ; sym: -2^(b-1)
  double qdiv;     // divisor of the raw scale: 2^b-1 (asym) or 2^(b-1)-1 (sym)
  double qinv;     // RN64(1 / qdiv)
  double floor;    // scale_floor
  uint32_t floor16;  // bit pattern of the smallest fp16 >= floor (0x7C00 if none)
  int64_t scales_off;
  int64_t zeros_off;
  // minifloat (FC_KIND_MINIFLOAT): e/m bits, bias, largest finite magnitude
  int mf_exp, mf_mant, mf_bias;
  int mf_fmt;      // fc_minifloat_format
  double mf_max;
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
// k >= nvalid are excluded from the statistics and produce stored code 0.
//
// Per element the code is round(x / s) + z, clamped (codec.py:324), computed
// without a divide instruction:
//   r  = RN(1/s) (once per lane), t = RN(x * r),
//   q1 = RN(t + r * RN(x - t*s))            (two FMAs)
// is the correctly rounded fp32 quotient RN(x/s) for every finite x and every
// fp16 scale s (one Newton step from a correctly rounded reciprocal —
// Markstein's theorem; tools/probes/div_check.cu checked 1e11 (x, s) pairs
// bit-for-bit against __fdiv_rn with no mismatch). RN(x/s) never crosses a
// half-integer or integer that the float64 quotient of the reference does not
// (x/s lies at least 2^-24 |x/s| away from any boundary it is not exactly on),
// so rounding q1 is exactly numpy's round / ceil of x/s. Then clamp in float
// to [-z, qmax-z] (monotone, integral bounds: commutes with rounding), round
// by the magic add y = q1c + 1.5*2^23 (RN: ties-to-even; RU: ceil) whose low
// mantissa bits hold the integer, and add z as an integer.
// Symmetric codes are computed in offset binary (z = 2^(b-1)) and XOR-ed back
// to two's complement, so both schemes share one decoder.

template <int CW>
struct LaneQuant {
  uint32_t w[CW];  // packed codes: INT4 w[0..3], INT8 w[0..7], fp16 bits w[0..15]
  __half s16;
  float s;         // scale (exact fp16 value as fp32)
  float mz;        // decode bias 2^23 + zero (asym) or 2^23 + 2^(b-1) (sym)
  uint32_t xr;     // per-word XOR taking stored codes to offset binary
  uint8_t z8;
};

template <int CW>
struct LaneCodes {
  uint32_t w[CW];  // offset-binary codes (xr already applied) or fp16 bits
  float s;
  float mz;
};

__device__ __forceinline__ float fmin_nan(float a, float b) {
  float r;
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

__device__ __forceinline__ uint32_t rep_xor(const DevCodec& c) {
  if (!c.sym) return 0u;
  const uint32_t h = 1u << (c.bits - 1);
  return c.sb == 4 ? h * 0x11111111u : h * 0x01010101u;
}

// Lane sources: element k of the chunk as fp32. FloatLane holds fp32 values;
// PackedLane<T> holds 32 raw 16-bit values (bf16/fp16), unpacked on use so the
// statistics can run on packed pairs.
struct FloatLane {
  float v[kLaneElems];
  __device__ __forceinline__ float get(int k) const { return v[k]; }
};
template <typename T>
struct PackedLane {
  uint32_t w[kLaneElems / 2];
  __device__ __forceinline__ float get(int k) const {
    if constexpr (std::is_same<T, __nv_bfloat16>::value) {
      return (k & 1) ? __uint_as_float(w[k >> 1] & 0xFFFF0000u) : __uint_as_float(w[k >> 1] << 16);
    } else {
      const __half2 h = *reinterpret_cast<const __half2*>(&w[k >> 1]);
      return (k & 1) ? __high2float(h) : __low2float(h);
    }
  }
};

// Statistics of the lane's valid elements, NaN-propagating (NaN and +-inf
// surface as a non-finite bound): asym (min, max), sym (-, absmax).
template <bool SYM>
__device__ __forceinline__ void lane_stats(const FloatLane& L, int nvalid, float& lo, float& hi) {
  if (nvalid == kLaneElems) {
    float a[16], b[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const float x = SYM ? fabsf(L.v[2 * k]) : L.v[2 * k];
      const float y = SYM ? fabsf(L.v[2 * k + 1]) : L.v[2 * k + 1];
      a[k] = fmin_nan(x, y);
      b[k] = fmax_nan(x, y);
    }
#pragma unroll
    for (int w = 8; w >= 1; w >>= 1)
#pragma unroll
      for (int k = 0; k < w; ++k) {
        a[k] = fmin_nan(a[k], a[k + w]);
        b[k] = fmax_nan(b[k], b[k + w]);
      }
    lo = a[0];
    hi = b[0];
  } else {
    lo = INFINITY;
    hi = -INFINITY;
#pragma unroll
    for (int k = 0; k < kLaneElems; ++k)
      if (k < nvalid) {
        const float x = SYM ? fabsf(L.v[k]) : L.v[k];
        lo = fmin_nan(lo, x);
        hi = fmax_nan(hi, x);
      }
  }
}

template <bool SYM, typename T>
__device__ __forceinline__ void lane_stats(const PackedLane<T>& L, int nvalid, float& lo, float& hi) {
  using V2 = typename std::conditional<std::is_same<T, __nv_bfloat16>::value, __nv_bfloat162, __half2>::type;
  if (nvalid == kLaneElems) {
    V2 a[8], b[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      V2 x = *reinterpret_cast<const V2*>(&L.w[2 * k]);
      V2 y = *reinterpret_cast<const V2*>(&L.w[2 * k + 1]);
      if (SYM) {
        x = __habs2(x);
        y = __habs2(y);
      }
      a[k] = __hmin2_nan(x, y);
      b[k] = __hmax2_nan(x, y);
    }
#pragma unroll
    for (int w = 4; w >= 1; w >>= 1)
#pragma unroll
      for (int k = 0; k < w; ++k) {
        a[k] = __hmin2_nan(a[k], a[k + w]);
        b[k] = __hmax2_nan(b[k], b[k + w]);
      }
    const float2 fa = std::is_same<T, __nv_bfloat16>::value ? __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&a[0]))
                                                             : __half22float2(*reinterpret_cast<__half2*>(&a[0]));
    const float2 fb = std::is_same<T, __nv_bfloat16>::value ? __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&b[0]))
                                                             : __half22float2(*reinterpret_cast<__half2*>(&b[0]));
    lo = fmin_nan(fa.x, fa.y);
    hi = fmax_nan(fb.x, fb.y);
  } else {
    lo = INFINITY;
    hi = -INFINITY;
#pragma unroll
    for (int k = 0; k < kLaneElems; ++k)
      if (k < nvalid) {
        const float x = SYM ? fabsf(L.get(k)) : L.get(k);
        lo = fmin_nan(lo, x);
        hi = fmax_nan(hi, x);
      }
  }
}

// codes of one lane chunk (see the derivation above)
template <int SB, bool CEIL, class Src>
__device__ __forceinline__ void lane_codes(const Src& L, float s, int z, int qmax, uint32_t* w) {
  const float r = __frcp_rn(s);
  const float C0 = 12582912.0f;  // 1.5 * 2^23
  const float lob = -(float)z, hib = (float)(qmax - z);
  const int zb = z - 0x4B400000;
#pragma unroll
  for (int k = 0; k < kLaneElems; ++k) {
    const float x = L.get(k);
    const float t = x * r;
    const float q1 = fmaf(fmaf(-t, s, x), r, t);
    const float qc = fminf(fmaxf(q1, lob), hib);
    const float y = CEIL ? __fadd_ru(qc, C0) : __fadd_rn(qc, C0);
    const uint32_t code = (uint32_t)(__float_as_int(y) + zb);
    if (SB == 4) {
      if ((k & 7) == 0) w[k >> 3] = 0;
      w[k >> 3] |= code << (4 * (k & 7));
    } else {
      if ((k & 3) == 0) w[k >> 2] = 0;
      w[k >> 2] |= code << (8 * (k & 3));
    }
  }
}

__device__ __forceinline__ float group_allreduce_min(float v, int lpg) {
  for (int o = 1; o < lpg; o <<= 1) v = fmin_nan(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float group_allreduce_max(float v, int lpg) {
  for (int o = 1; o < lpg; o <<= 1) v = fmax_nan(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// returns true if a valid element of the lane's group is NaN/inf (codec.py:230-231)
template <int CW, class Src>
__device__ __forceinline__ bool lane_quantize(const DevCodec& c, const Src& L, int nvalid, LaneQuant<CW>& q) {
  if constexpr (CW == 16) {
    if (c.kind == FC_KIND_FP16) {
      float lo, hi;
      lane_stats<true>(L, nvalid, lo, hi);
#pragma unroll
      for (int k = 0; k < kLaneElems; k += 2) {
        __half2 h = __floats2half2_rn(k < nvalid ? L.get(k) : 0.0f, k + 1 < nvalid ? L.get(k + 1) : 0.0f);
        q.w[k / 2] = *reinterpret_cast<uint32_t*>(&h);
      }
      q.s16 = __ushort_as_half(0);
      q.s = 1.0f;
      q.mz = 0.0f;
      q.xr = 0u;
      q.z8 = 0;
      return nvalid > 0 && !(hi <= 3.402823466e38f);
    }
  }
  float lo, hi;
  if (c.sym) {
    lane_stats<true>(L, nvalid, lo, hi);
    hi = group_allreduce_max(hi, c.lpg);
    lo = -hi;
  } else {
    lane_stats<false>(L, nvalid, lo, hi);
    lo = group_allreduce_min(lo, c.lpg);
    hi = group_allreduce_max(hi, c.lpg);
  }
  const bool bad = nvalid > 0 && !(fabsf(lo) <= 3.402823466e38f && fabsf(hi) <= 3.402823466e38f);
  int z;
  if (c.sym) {
    q.s16 = snap_scale((double)hi / c.qdiv, c.floor);
    z = 1 << (c.bits - 1);
    q.z8 = 0;
  } else {
    q.s16 = snap_scale(((double)hi - (double)lo) / c.qdiv, c.floor);
    double zd = ceil(-(double)lo / (double)__half2float(q.s16));
    zd = fmin(fmax(zd, 0.0), (double)c.qmax_f);
    z = bad ? 0 : (int)zd;
    q.z8 = (uint8_t)z;
  }
  q.s = __half2float(q.s16);
  q.mz = 8388608.0f + (float)z;
  q.xr = rep_xor(c);
  const int qmax = (1 << c.bits) - 1;
  if (c.sb == 4) {
    if (c.ceil_mode)
      lane_codes<4, true>(L, q.s, z, qmax, q.w);
    else
      lane_codes<4, false>(L, q.s, z, qmax, q.w);
  } else {
    if (c.ceil_mode)
      lane_codes<8, true>(L, q.s, z, qmax, q.w);
    else
      lane_codes<8, false>(L, q.s, z, qmax, q.w);
  }
  const int nw = c.sb == 4 ? 4 : 8;
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (i < nw) q.w[i] ^= q.xr;  // offset binary -> stored (two's complement for sym)
  if (nvalid < kLaneElems) {     // stored code 0 past the end of the range
    const int per = 32 / c.sb;   // codes per word
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int first = i * per;
      if (i < nw && first + per > nvalid) {
        const int keep = max(0, nvalid - first);
        const uint32_t m = keep >= per ? 0xFFFFFFFFu : ((1u << (keep * c.sb)) - 1u);
        q.w[i] &= m;
      }
    }
  }
  return bad;
}

template <typename T>
using LaneOf = typename std::conditional<sizeof(T) == 4, FloatLane, PackedLane<T>>::type;

// Direct (non-staged) load of a lane chunk into its source representation;
// elements past M read as 0 (collectives.py:145-149).
template <typename T>
__device__ __forceinline__ void load_lane_src(const T* __restrict__ base, int64_t idx0, int64_t M, int nvalid,
                                              LaneOf<T>& L) {
  if constexpr (sizeof(T) == 4) {
    load_chunk(base, idx0, M, nvalid, L.v);
  } else {
    if (nvalid == kLaneElems && idx0 + kLaneElems <= M) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 u = ld_nc_v4(base + idx0 + 8 * q);
        L.w[4 * q] = u.x;
        L.w[4 * q + 1] = u.y;
        L.w[4 * q + 2] = u.z;
        L.w[4 * q + 3] = u.w;
      }
    } else {
      const uint16_t* b16 = reinterpret_cast<const uint16_t*>(base);
#pragma unroll
      for (int k = 0; k < kLaneElems; k += 2) {
        const uint32_t lo = (k < nvalid && idx0 + k < M) ? b16[idx0 + k] : 0u;
        const uint32_t hi = (k + 1 < nvalid && idx0 + k + 1 < M) ? b16[idx0 + k + 1] : 0u;
        L.w[k / 2] = lo | (hi << 16);
      }
    }
  }
}

// bytes of packed codes per 32-element lane chunk
__device__ __forceinline__ int lane_code_bytes(const DevCodec& c) { return c.sb * 4; }

// Store a quantized lane chunk into a buffer (local or peer memory).
// p0: element offset of the chunk within the quantized range.
template <int CW>
__device__ __forceinline__ void store_lane(const DevCodec& c, uint8_t* buf, int64_t p0, int nvalid,
                                           const LaneQuant<CW>& q, int lane) {
  if (nvalid <= 0) return;  // chunk lies past the end of the range
  uint8_t* cp = buf + p0 * c.sb / 8;
  const int nq = c.sb / 4;  // number of 16-B vectors: 1 (int4), 2 (int8), 4 (fp16)
#pragma unroll
  for (int i = 0; i < CW / 4; ++i)
    if (i < nq) st_v4(cp + 16 * i, make_uint4(q.w[4 * i], q.w[4 * i + 1], q.w[4 * i + 2], q.w[4 * i + 3]));
  if (c.kind == FC_KIND_INT && (lane & (c.lpg - 1)) == 0) {
    const int64_t grp = p0 >> c.gshift;
    reinterpret_cast<__half*>(buf + c.scales_off)[grp] = q.s16;
    if (!c.sym) buf[c.zeros_off + grp] = q.z8;
  }
}

// Decode helpers ------------------------------------------------------------

// in-register codes of a freshly quantized lane, in offset binary
template <int CW>
__device__ __forceinline__ void lane_codes_from(const DevCodec& c, const LaneQuant<CW>& q, LaneCodes<CW>& L) {
#pragma unroll
  for (int i = 0; i < CW; ++i) L.w[i] = (c.kind == FC_KIND_INT && i < 8) ? (q.w[i] ^ q.xr) : q.w[i];
  L.s = q.s;
  L.mz = q.mz;
}

template <int CW>
__device__ __forceinline__ void load_lane(const DevCodec& c, const uint8_t* buf, int64_t p0, LaneCodes<CW>& L) {
  const uint8_t* cp = buf + p0 * c.sb / 8;
  const int nq = c.sb / 4;
#pragma unroll
  for (int i = 0; i < CW / 4; ++i) {
    if (i >= nq) break;
    uint4 u = ld_cg_v4(cp + 16 * i);
    L.w[4 * i] = u.x;
    L.w[4 * i + 1] = u.y;
    L.w[4 * i + 2] = u.z;
    L.w[4 * i + 3] = u.w;
  }
  if (c.kind == FC_KIND_INT) {
    const int64_t grp = p0 >> c.gshift;
    L.s = __half2float(__ldcg(reinterpret_cast<const __half*>(buf + c.scales_off) + grp));
    const uint32_t xr = rep_xor(c);
    L.mz = 8388608.0f + (c.sym ? (float)(1 << (c.bits - 1)) : (float)__ldcg(buf + c.zeros_off + grp));
#pragma unroll
    for (int i = 0; i < 8; ++i) L.w[i] ^= xr;
  } else {
    L.s = 1.0f;
    L.mz = 0.0f;
  }
}

// magic(c) = 2^23 + c as fp32 bits, from byte `b` of word `w`
__device__ __forceinline__ float magic_byte(uint32_t w, int b) {
  return __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7440u | (uint32_t)b));
}

// out[k] = (c_k - z) * s, exact in fp32 (codec.py:383-384); fp16 kind: value
// ACC: out[k] += that value with one rounding (fp32 sum, collectives.py:186)
template <bool ACC, int CW>
__device__ __forceinline__ void lane_decode(const DevCodec& c, const LaneCodes<CW>& L, float out[kLaneElems]) {
  if constexpr (CW == 16) {
   if (c.kind == FC_KIND_FP16) {
#pragma unroll
    for (int k = 0; k < kLaneElems; k += 2) {
      __half2 h = *reinterpret_cast<const __half2*>(&L.w[k / 2]);
      const float2 f = __half22float2(h);
      if (ACC) {
        out[k] += f.x;
        out[k + 1] += f.y;
      } else {
        out[k] = f.x;
        out[k + 1] = f.y;
      }
    }
    return;
   }
  }
  if (c.sb == 4) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t lo = L.w[i] & 0x0F0F0F0Fu, hi = (L.w[i] >> 4) & 0x0F0F0F0Fu;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const float d0 = magic_byte(lo, b) - L.mz, d1 = magic_byte(hi, b) - L.mz;
        const int k = 8 * i + 2 * b;
        if (ACC) {
          out[k] = fmaf(d0, L.s, out[k]);
          out[k + 1] = fmaf(d1, L.s, out[k + 1]);
        } else {
          out[k] = d0 * L.s;
          out[k + 1] = d1 * L.s;
        }
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const float d = magic_byte(L.w[i], b) - L.mz;
        const int k = 4 * i + b;
        out[k] = ACC ? fmaf(d, L.s, out[k]) : d * L.s;
      }
  }
}

// --------------------------------------------------------------------------
// memory-model helpers for cross-GPU flags

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
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
