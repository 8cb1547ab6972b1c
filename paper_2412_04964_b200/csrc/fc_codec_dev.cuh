// Generic (any group size) codec kernels. One thread per group computes the
// group parameters; one thread per packed byte writes codes, so INT4 bytes
// that straddle two groups (odd group sizes) are never written by two
// threads. Same numerics as the fast lane quantizer (fc_common.cuh).
#pragma once

#include "fc_common.cuh"

namespace fc {

// value sources ---------------------------------------------------------------

// element p of a zero-padded rank segment: base[off + p], 0 beyond M
// (collectives.py:145-149)
template <typename T>
struct SrcSeg {
  const T* base;
  int64_t off;
  int64_t M;
  __device__ __forceinline__ float operator()(int64_t p) const {
    const int64_t i = off + p;
    return i < M ? DT<T>::to_f(base[i]) : 0.0f;
  }
};

struct SrcF32 {
  const float* p;
  __device__ __forceinline__ float operator()(int64_t i) const { return p[i]; }
};

// ---- minifloat codes (minifloat.py:58-124, codec.py:332-351): grid value of
// RN64(x / s), ties to even, saturating; IEEE-style subnormals
__device__ __forceinline__ uint32_t mf_code(const DevCodec& c, float x, float s) {
  const double q = __ddiv_rn((double)x, (double)s);
  const double a = fabs(q);
  const double min_normal = ldexp(1.0, 1 - c.mf_bias), sub_q = ldexp(1.0, 1 - c.mf_bias - c.mf_mant);
  int e2;
  frexp(a, &e2);
  const double quantum = a < min_normal ? sub_q : ldexp(1.0, e2 - 1 - c.mf_mant);
  const double r = fmin(rint(a / quantum) * quantum, c.mf_max);
  const uint32_t sign = (q < 0.0 && r > 0.0) ? 1u : 0u;  // encode() tests v < 0 on the signed grid value
  uint32_t ec, mc;
  if (r < min_normal) {
    ec = 0;
    mc = (uint32_t)(r / sub_q);
  } else {
    int er;
    frexp(r, &er);
    ec = (uint32_t)(er - 1 + c.mf_bias);
    mc = (uint32_t)((ldexp(r, -(er - 1)) - 1.0) * (double)(1 << c.mf_mant));
  }
  return (sign << (c.mf_exp + c.mf_mant)) | (ec << c.mf_mant) | mc;
}
__device__ __forceinline__ float mf_value(const DevCodec& c, uint32_t code) {
  const uint32_t mc = code & ((1u << c.mf_mant) - 1u), ec = (code >> c.mf_mant) & ((1u << c.mf_exp) - 1u);
  const float mag = ec == 0 ? (float)mc * ldexpf(1.0f, 1 - c.mf_bias - c.mf_mant)
                            : (1.0f + (float)mc / (float)(1 << c.mf_mant)) * ldexpf(1.0f, (int)ec - c.mf_bias);
  return (code >> (c.mf_exp + c.mf_mant)) ? -mag : mag;
}

__device__ __forceinline__ uint32_t code_of(const DevCodec& c, float v, float s, float zf) {
  if (c.kind == FC_KIND_MINIFLOAT) return mf_code(c, v, s);
  float t = __fdiv_rn(v, s);
  t = c.ceil_mode ? ceilf(t) : rintf(t);
  t = fminf(fmaxf(t + zf, c.qmin_f), c.qmax_f);
  return (uint32_t)(int)t & ((1u << c.bits) - 1u);
}

__device__ __forceinline__ float value_of(const DevCodec& c, uint32_t code, float s, float zf) {
  float cf;
  if (c.sym) {
    const int sh = 32 - c.bits;
    cf = (float)(((int)(code << sh)) >> sh);
  } else {
    cf = (float)code;
  }
  return (cf - zf) * s;
}

// per-group parameters (codec.py:309-326), one thread per group
template <class Src>
__global__ void k_gen_params(Src src, int64_t n, DevCodec c, uint8_t* dst, uint32_t* err, uint32_t rank) {
  const int64_t groups = (n + c.g - 1) / c.g;
  for (int64_t gi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; gi < groups;
       gi += (int64_t)gridDim.x * blockDim.x) {
    const int64_t start = gi * c.g;
    const int64_t end = min(start + (int64_t)c.g, n);
    float lo = INFINITY, hi = -INFINITY, probe = 0.0f;
    const bool absmax = c.sym || c.kind == FC_KIND_MINIFLOAT;
    for (int64_t p = start; p < end; ++p) {
      const float v = src(p);
      probe = fmaf(v, 0.0f, probe);
      if (absmax) {
        hi = fmaxf(hi, fabsf(v));
      } else {
        lo = fminf(lo, v);
        hi = fmaxf(hi, v);
      }
    }
    if (probe != probe && err) atomicOr(err, make_err(kErrNonFinite, 0, 0, rank));
    __half s16;
    uint8_t z8 = 0;
    if (absmax) {  // sym: absmax / (2^(b-1)-1); minifloat: absmax / max_finite (codec.py:345)
      s16 = snap_scale((double)hi / c.qdiv, c.floor);
    } else {
      s16 = snap_scale(((double)hi - (double)lo) / c.qdiv, c.floor);
      double z = ceil(-(double)lo / (double)__half2float(s16));
      z = fmin(fmax(z, 0.0), (double)c.qmax_f);
      z8 = (uint8_t)(int)z;
    }
    reinterpret_cast<__half*>(dst + c.scales_off)[gi] = s16;
    if (!absmax) dst[c.zeros_off + gi] = z8;
  }
}

__host__ __device__ inline int64_t gen_code_units(const DevCodec& c, int64_t n) {
  return c.sb == 4 ? (n + 1) / 2 : n;
}

// codes: one thread per output byte (INT4: 2 elements; INT8: 1; fp16: 1 element -> 2 bytes)
template <class Src>
__global__ void k_gen_codes(Src src, int64_t n, DevCodec c, uint8_t* dst, uint32_t* err, uint32_t rank) {
  const int64_t units = gen_code_units(c, n);
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < units;
       u += (int64_t)gridDim.x * blockDim.x) {
    if (c.kind == FC_KIND_FP16) {
      const float v = src(u);
      if (fmaf(v, 0.0f, 0.0f) != 0.0f && err) atomicOr(err, make_err(kErrNonFinite, 0, 0, rank));
      reinterpret_cast<__half*>(dst)[u] = __float2half_rn(v);
      continue;
    }
    const __half* sc = reinterpret_cast<const __half*>(dst + c.scales_off);
    const int per = c.sb == 4 ? 2 : 1;
    uint32_t byte = 0;
    for (int k = 0; k < per; ++k) {
      const int64_t p = u * per + k;
      if (p >= n) break;
      const int64_t gi = p / c.g;
      const float s = __half2float(sc[gi]);
      const float zf = (c.sym || c.kind == FC_KIND_MINIFLOAT) ? 0.0f : (float)dst[c.zeros_off + gi];
      byte |= code_of(c, src(p), s, zf) << (4 * k);
    }
    dst[u] = (uint8_t)byte;
  }
}

__device__ __forceinline__ float gen_value_at(const DevCodec& c, const uint8_t* src, int64_t i) {
  if (c.kind == FC_KIND_FP16) return __half2float(reinterpret_cast<const __half*>(src)[i]);
  uint32_t code;
  if (c.sb == 4) {
    code = (src[i >> 1] >> (4 * (i & 1))) & 0xFu;
  } else {
    code = src[i];
  }
  const int64_t gi = i / c.g;
  const float s = __half2float(reinterpret_cast<const __half*>(src + c.scales_off)[gi]);
  if (c.kind == FC_KIND_MINIFLOAT) return mf_value(c, code) * s;  // exact (<= 4 x 11 significant bits)
  const float zf = c.sym ? 0.0f : (float)src[c.zeros_off + gi];
  return value_of(c, code, s, zf);
}

// out[out_off + i] = dequant(src)[i] for out_off + i < M (M <= 0: no limit)
template <typename To>
__global__ void k_gen_dequant(const uint8_t* src, int64_t n, DevCodec c, To* out, int64_t out_off,
                              int64_t M = 0) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (M > 0 && out_off + i >= M) continue;
    out[out_off + i] = DT<To>::from_f(gen_value_at(c, src, i));
  }
}

}  // namespace fc
