// Lane-8 Flash All-Reduce path: a thread owns 8 consecutive elements, a group
// of g elements (g = 8..256) spans g/8 consecutive lanes of one warp. It
// carries every codec the compile-time lanes do not: the group-scaled
// minifloats (codec.py:332-351; e4m3 / e5m2 / e2m1 through the native
// cvt.rn.satfinite conversions) and any integer scheme (runtime flags), and
// it fuses the blocked Hadamard rotation (rotation.py:38-83,
// collectives.py:350-351 / 390-391) into the scatter / reduce prologue
// (forward H(D x) of the input) and the reduce / gather epilogue (inverse
// D(H y) of the output): float64 butterflies in the reference's order, the
// cross-lane stages over warp shuffles, one rounding to float32.
//
// Numerics. Minifloat code of x in a group with fp16 scale s: the reference
// rounds RN64(x / s) to the format grid (minifloat.py:58-75). Here the
// quotient is RN32(x / s) (reciprocal + one FMA correction) and cvt.rn.satfinite rounds it to the
// grid: x has <= 24 and s <= 11 significant bits, so an exact quotient that
// is not a grid tie lies more than half an f32 ulp away from every tie, and
// RN32 cannot move it across one (same argument as the integer codes);
// saturation at the largest finite value and the subnormal range are the
// conversion's own. A zero magnitude is stored with the sign bit clear, as
// encode() does (it tests v < 0 on the signed grid value). Decoding converts
// the code to fp16 (exact) and multiplies by the scale (<= 4 x 11 significant
// bits: exact in fp32).
#pragma once

#include "fc_codec_dev.cuh"
#include "fc_flash.cuh"

namespace fc {

constexpr int kL8 = 8;            // elements per thread
constexpr int kL8Threads = 256;   // threads per CTA
constexpr int kL8MaxRot = 256;    // largest fused rotation block (32 lanes x 8)

// rotation state of a call (dim 0: none); signs: dim device floats of +-1 or null
struct L8Rot {
  int dim;
  int normalize;
  const float* signs;
};

// ------------------------------------------------------------------ lane-8 codec

// 8 codes packed in storage order (sb 4: one word, little nibble first; sb 8: two words)
struct L8Codes {
  uint32_t w0, w1;
};

// quantize 8 values (v[e] for e < nvalid; the rest are outside the piece) of one lane;
// every lane of the warp calls it together (group statistics over g/8 lanes by shuffles).
// Returns the codes, the group's fp16 scale / zero byte and the decoded values (QDQ).
// F: 0 = any codec (runtime flags), 1 + fc_minifloat_format = that minifloat (compile time)
template <int F>
struct L8F {
  static constexpr bool MF = F > 0;
  static constexpr int FMT = F - 1;
  static constexpr int SB = F == 3 ? 4 : 8;  // storage bits when MF
};
__host__ inline int l8_f_of(const fc_codec& c1, const fc_codec& c2) {
  return (c1.kind == FC_KIND_MINIFLOAT && c2.kind == FC_KIND_MINIFLOAT && c1.reserved == c2.reserved) ? 1 + c1.reserved
                                                                                                        : 0;
}

template <int F>
__device__ __forceinline__ bool l8_quant(const DevCodec& c, const float v[kL8], int nvalid, L8Codes& q,
                                         __half& s16, uint8_t& z8, float deq[kL8]) {
  const bool mf = L8F<F>::MF || c.kind == FC_KIND_MINIFLOAT;
  const int sb = L8F<F>::MF ? L8F<F>::SB : c.sb;
  const bool absmax = mf || c.sym;
  float lo = INFINITY, hi = -INFINITY, probe = 0.0f;
#pragma unroll
  for (int e = 0; e < kL8; ++e) {
    if (e < nvalid) {
      probe = fmaf(v[e], 0.0f, probe);
      if (absmax) {
        hi = fmaxf(hi, fabsf(v[e]));
      } else {
        lo = fminf(lo, v[e]);
        hi = fmaxf(hi, v[e]);
      }
    }
  }
  const int lpg = c.g / kL8;
  for (int o = 1; o < lpg; o <<= 1) {
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    if (!absmax) lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
  }
  const bool bad = probe != probe;
  float zf = 0.0f;
  if (absmax) {  // sym: absmax / (2^(b-1)-1); minifloat: absmax / max_finite (codec.py:309-316, 345)
    s16 = snap_scale((double)hi / c.qdiv, c.floor);
    z8 = 0;
  } else {
    s16 = snap_scale(((double)hi - (double)lo) / c.qdiv, c.floor);
    double zd = ceil(-(double)lo / (double)__half2float(s16));
    zd = fmin(fmax(zd, 0.0), (double)c.qmax_f);
    z8 = (uint8_t)(int)(bad ? 0.0 : zd);
    zf = (float)z8;
  }
  const float s = __half2float(s16);
  uint32_t code[kL8];
  if (mf) {
    const int fmt = L8F<F>::MF ? L8F<F>::FMT : c.mf_fmt;
    // RN32(x / s) without div.rn's slow-path checks: r = RN(1/s), t = RN(x r), one FMA
    // correction (Markstein: correctly rounded for normal quotients, which |x / s| <= 2^17 and
    // the tiny quotients that round to a zero code anyway are)
    const float rcp = __frcp_rn(s);
    auto quot = [&](float x) { const float t = x * rcp; return fmaf(fmaf(-t, s, x), rcp, t); };
#pragma unroll
    for (int e = 0; e < kL8; e += 2) {
      const float x0 = e < nvalid ? quot(v[e]) : 0.0f;
      const float x1 = e + 1 < nvalid ? quot(v[e + 1]) : 0.0f;
      const uint32_t two = mf_enc2(fmt, x0, x1);
      const int sh = sb == 4 ? 4 : 8;
      code[e] = two & ((1u << sh) - 1u);
      code[e + 1] = two >> sh;
      mf_dec2(fmt, two, deq[e], deq[e + 1]);
      deq[e] *= s;
      deq[e + 1] *= s;
    }
  } else {  // code_of (fc_codec_dev.cuh) with the reciprocal + FMA-corrected quotient
    const float rcp = __frcp_rn(s);
#pragma unroll
    for (int e = 0; e < kL8; ++e) {
      const float t0 = v[e] * rcp, t = fmaf(fmaf(-t0, s, v[e]), rcp, t0);
      const float tq = fminf(fmaxf((c.ceil_mode ? ceilf(t) : rintf(t)) + zf, c.qmin_f), c.qmax_f);
      code[e] = e < nvalid ? ((uint32_t)(int)tq & ((1u << c.bits) - 1u)) : 0u;
      deq[e] = value_of(c, code[e], s, zf);
    }
  }
  if (sb == 4) {
    q.w0 = 0;
#pragma unroll
    for (int e = 0; e < kL8; ++e) q.w0 |= (code[e] & 0xFu) << (4 * e);
    q.w1 = 0;
  } else {
    q.w0 = code[0] | (code[1] << 8) | (code[2] << 16) | (code[3] << 24);
    q.w1 = code[4] | (code[5] << 8) | (code[6] << 16) | (code[7] << 24);
  }
  return bad;
}

// the raw codes, scale and zero point of one lane of a stored tensor at element p0; the loads
// are issued here and consumed by l8_decode, so a caller can keep several in flight
struct L8Raw {
  uint32_t w0, w1;
  unsigned short s16;  // raw fp16 scale bits and zero byte: converted in l8_decode, so the loads
  uint32_t z8;         // of several fetches stay in flight together (no use right after the load)
};
template <int F>
__device__ __forceinline__ L8Raw l8_fetch(const DevCodec& c, const uint8_t* buf, int64_t p0) {
  const bool mf = L8F<F>::MF || c.kind == FC_KIND_MINIFLOAT;
  const int sb = L8F<F>::MF ? L8F<F>::SB : c.sb;
  L8Raw r;
  r.w1 = 0;
  if (sb == 4) {
    r.w0 = __ldcg(reinterpret_cast<const unsigned int*>(buf + p0 / 2));
  } else {
    const uint2 u = __ldcg(reinterpret_cast<const uint2*>(buf + p0));
    r.w0 = u.x;
    r.w1 = u.y;
  }
  const int64_t gi = p0 >> (31 - __clz(c.g));  // g is a power of two (no 64-bit division)
  r.s16 = __ldcg(reinterpret_cast<const unsigned short*>(buf + c.scales_off) + gi);
  r.z8 = (mf || c.sym) ? 0u : (uint32_t)__ldcg(buf + c.zeros_off + gi);
  return r;
}
template <int F>
__device__ __forceinline__ void l8_decode(const DevCodec& c, const L8Raw& r, float out[kL8]) {
  const bool mf = L8F<F>::MF || c.kind == FC_KIND_MINIFLOAT;
  const int sb = L8F<F>::MF ? L8F<F>::SB : c.sb;
  const float rs = __half2float(__ushort_as_half(r.s16)), rzf = (float)r.z8;
  if (mf) {
    const int fmt = L8F<F>::MF ? L8F<F>::FMT : c.mf_fmt;
#pragma unroll
    for (int e = 0; e < kL8; e += 2) {
      uint32_t two;
      if (sb == 4)
        two = (r.w0 >> (4 * e)) & 0xFFu;
      else
        two = ((e < 4 ? r.w0 : r.w1) >> (8 * (e & 3))) & 0xFFFFu;
      mf_dec2(fmt, two, out[e], out[e + 1]);
      out[e] *= rs;
      out[e + 1] *= rs;
    }
  } else {
#pragma unroll
    for (int e = 0; e < kL8; ++e) {
      const uint32_t code = c.sb == 4 ? (r.w0 >> (4 * e)) & 0xFu : ((e < 4 ? r.w0 : r.w1) >> (8 * (e & 3))) & 0xFFu;
      out[e] = value_of(c, code, rs, rzf);
    }
  }
}

// kernel sweep over the lanes [0, span) of a round (span a multiple of 32): U lanes per
// thread per step, all U loads issued before any is used (bytes in flight), whole warps in
// step (the codec's shuffles)
template <int U, class Load, class Work, class Regs>
__device__ __forceinline__ void l8_sweep(int64_t span, Load load, Work work, Regs* regs) {
  const int64_t G = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k0 < span; k0 += G * U) {
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (k0 + u * G < span) load(k0 + u * G, regs[u]);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (k0 + u * G < span) work(k0 + u * G, regs[u]);
  }
}
constexpr int kL8UQ = 4;  // lanes in flight per thread: quantize-type (16-32 B of input each)
constexpr int kL8UD = 4;  // dequantize-type (codes + scale + zero each)

// store 8 codes (+ the group's metadata from its first lane) at element p0 of a slot
template <int F>
__device__ __forceinline__ void l8_store(const DevCodec& c, uint8_t* buf, int64_t p0, int nvalid, const L8Codes& q,
                                         __half s16, uint8_t z8) {
  if (nvalid <= 0) return;
  const bool mf = L8F<F>::MF || c.kind == FC_KIND_MINIFLOAT;
  const int sb = L8F<F>::MF ? L8F<F>::SB : c.sb;
  if (sb == 4)
    *reinterpret_cast<unsigned int*>(buf + p0 / 2) = q.w0;
  else
    *reinterpret_cast<uint2*>(buf + p0) = make_uint2(q.w0, q.w1);
  if ((p0 & (c.g - 1)) == 0) {  // g is a power of two
    const int64_t gi = p0 >> (31 - __clz(c.g));
    reinterpret_cast<__half*>(buf + c.scales_off)[gi] = s16;
    if (!(mf || c.sym)) buf[c.zeros_off + gi] = z8;
  }
}

// ------------------------------------------------------------------ fused rotation

// in-place FWHT of the rotation block this lane belongs to (dim/8 consecutive lanes, 8
// elements each) in float64, stages h = 1, 2, 4, ... as rotation.py:38-49 (top = a + b,
// bottom = a - b); the lanes >= 8 apart exchange over shuffles
__device__ __forceinline__ void l8_fwht(double y[kL8], int dim) {
#pragma unroll
  for (int h = 1; h < kL8; h <<= 1) {
    if (h >= dim) break;
#pragma unroll
    for (int i = 0; i < kL8; ++i) {
      if (i & h) continue;
      const double a = y[i], b = y[i + h];
      y[i] = a + b;
      y[i + h] = a - b;
    }
  }
  const int lane = threadIdx.x & 31;
  for (int lh = 1; lh < dim / kL8; lh <<= 1) {
    const bool upper = (lane & lh) != 0;
#pragma unroll
    for (int i = 0; i < kL8; ++i) {
      const double o = __shfl_xor_sync(0xffffffffu, y[i], lh);
      y[i] = upper ? o - y[i] : y[i] + o;
    }
  }
}

// forward H(D x) / sqrt(dim) of the lane's 8 values (rotation.py:61-71), float32 result
__device__ __forceinline__ void l8_rotate(const L8Rot& rot, int64_t p, float v[kL8]) {
  double y[kL8];
  const int b = (int)(p & (rot.dim - 1));
#pragma unroll
  for (int e = 0; e < kL8; ++e) y[e] = rot.signs ? (double)v[e] * (double)rot.signs[b + e] : (double)v[e];
  l8_fwht(y, rot.dim);
  const double rs = sqrt((double)rot.dim);
#pragma unroll
  for (int e = 0; e < kL8; ++e) v[e] = (float)(rot.normalize ? y[e] / rs : y[e]);
}

// inverse D(H y) (rotation.py:74-83): / sqrt(dim) (normalize) or / dim, then the signs
__device__ __forceinline__ void l8_unrotate(const L8Rot& rot, int64_t p, float v[kL8]) {
  double y[kL8];
#pragma unroll
  for (int e = 0; e < kL8; ++e) y[e] = (double)v[e];
  l8_fwht(y, rot.dim);
  const double rs = sqrt((double)rot.dim);
  const int b = (int)(p & (rot.dim - 1));
#pragma unroll
  for (int e = 0; e < kL8; ++e) {
    double t = rot.normalize ? y[e] / rs : y[e] / (double)rot.dim;
    if (rot.signs) t *= (double)rot.signs[b + e];
    v[e] = (float)t;
  }
}

// ------------------------------------------------------------------ element access

// 8 elements of a lane: one 16-B access (two for float32) when all 8 are inside the piece and
// below M and the address is 16-B aligned (rank tensors are, segment and lane offsets are
// multiples of 8), else element by element. l8_fetch_in only issues the loads (raw words);
// l8_unpack converts them, so a thread keeps several lanes' loads in flight
template <typename T>
struct L8In {
  uint4 u[sizeof(T) == 4 ? 2 : 1];
  float v[kL8];  // the scalar (edge) path converts at once
  bool vec;
};
template <typename T>
__device__ __forceinline__ void l8_fetch_in(const T* base, int64_t off, int64_t M, int nvalid, L8In<T>& in) {
  const T* p = base + off;
  in.vec = nvalid == kL8 && off + kL8 <= M && ((uintptr_t)p & 15) == 0;
  if (in.vec) {
#pragma unroll
    for (int i = 0; i < (sizeof(T) == 4 ? 2 : 1); ++i) in.u[i] = __ldg(reinterpret_cast<const uint4*>(p) + i);
  } else {
#pragma unroll
    for (int e = 0; e < kL8; ++e) in.v[e] = (e < nvalid && off + e < M) ? DT<T>::to_f(base[off + e]) : 0.0f;
  }
}
template <typename T>
__device__ __forceinline__ void l8_unpack(const L8In<T>& in, float v[kL8]) {
  if (!in.vec) {
#pragma unroll
    for (int e = 0; e < kL8; ++e) v[e] = in.v[e];
    return;
  }
  if constexpr (sizeof(T) == 4) {
    const uint4 a = in.u[0], b = in.u[1];
    v[0] = __uint_as_float(a.x), v[1] = __uint_as_float(a.y), v[2] = __uint_as_float(a.z), v[3] = __uint_as_float(a.w);
    v[4] = __uint_as_float(b.x), v[5] = __uint_as_float(b.y), v[6] = __uint_as_float(b.z), v[7] = __uint_as_float(b.w);
  } else {
    const uint32_t w[4] = {in.u[0].x, in.u[0].y, in.u[0].z, in.u[0].w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const unsigned short lo = (unsigned short)(w[i] & 0xFFFFu), hi = (unsigned short)(w[i] >> 16);
      T a, b;
      memcpy(&a, &lo, 2);
      memcpy(&b, &hi, 2);
      v[2 * i] = DT<T>::to_f(a);
      v[2 * i + 1] = DT<T>::to_f(b);
    }
  }
}
template <typename T>
__device__ __forceinline__ void l8_load(const T* base, int64_t off, int64_t M, int nvalid, float v[kL8]) {
  L8In<T> in;
  l8_fetch_in(base, off, M, nvalid, in);
  l8_unpack(in, v);
}
template <typename T>
__device__ __forceinline__ void l8_write(T* base, int64_t off, int64_t M, int nvalid, const float v[kL8]) {
  T* p = base + off;
  if (nvalid == kL8 && off + kL8 <= M && ((uintptr_t)p & 15) == 0) {
    if constexpr (sizeof(T) == 4) {
      reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
      reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
    } else {
      uint32_t w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const T a = DT<T>::from_f(v[2 * i]), b = DT<T>::from_f(v[2 * i + 1]);
        unsigned short lo, hi;
        memcpy(&lo, &a, 2);
        memcpy(&hi, &b, 2);
        w[i] = (uint32_t)lo | ((uint32_t)hi << 16);
      }
      *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    return;
  }
#pragma unroll
  for (int e = 0; e < kL8; ++e)
    if (e < nvalid && off + e < M) base[off + e] = DT<T>::from_f(v[e]);
}

// lane k's elements [8k, 8k+8) of a round: count inside it
__device__ __forceinline__ int l8_valid(int64_t len, int64_t p0) {
  const int64_t d = len - p0;
  return d <= 0 ? 0 : (d >= kL8 ? kL8 : (int)d);
}

// ------------------------------------------------------------------ phase kernels

struct L8Vals {
  float v[kL8];
};

// scatter: rank r's piece j (blockIdx.y = job) -> recv_slot[j][r]; rotation applied first
template <typename Tin, int F>
__global__ void __launch_bounds__(kL8Threads) k_l8_scatter(FlashArgs a, L8Rot rot) {
  int r, j;
  pair_of(a, blockIdx.y, r, j);
  const int64_t off = (int64_t)j * a.seg + a.sub_off;
  const Tin* src = reinterpret_cast<const Tin*>(a.in[r]);
  uint8_t* dst = recv_slot(a, j, r);
  const int64_t span = ((a.sub_len + kL8 - 1) / kL8 + 31) / 32 * 32;  // whole warps (shuffles)
  bool bad = false;
  L8In<Tin> regs[kL8UQ];
  l8_sweep<kL8UQ>(
      span,
      [&](int64_t k, L8In<Tin>& R) { l8_fetch_in(src, off + k * kL8, a.M, l8_valid(a.sub_len, k * kL8), R); },
      [&](int64_t k, L8In<Tin>& R) {
        const int64_t p0 = k * kL8;
        const int nvalid = l8_valid(a.sub_len, p0);
        float v[kL8];
        l8_unpack(R, v);
        if (rot.dim) l8_rotate(rot, off + p0, v);
        L8Codes q;
        __half s16;
        uint8_t z8;
        float deq[kL8];
        bad |= l8_quant<F>(a.c1, v, nvalid, q, s16, z8, deq);
        l8_store<F>(a.c1, dst, p0, nvalid, q, s16, z8);
      },
      regs);
  if (bad) atomicOr(errw(a, r), make_err(kErrNonFinite, kPhScatter, j, r));
}

// reduce: owner j (blockIdx.y) -- own piece QDQ (rotated), the N pieces summed in ascending
// source rank, stage-2 quantize -> every peer's gather slot [j], own output (inverse rotation);
// the peers' codes of a lane (up to 8 sources) are fetched before any is decoded
template <typename Tin, typename Tout, int F>
__global__ void __launch_bounds__(kL8Threads) k_l8_reduce(FlashArgs a, L8Rot rot) {
  constexpr int B = 8;
  const int j = a.rank_lo + blockIdx.y;
  const int64_t off = (int64_t)j * a.seg + a.sub_off;
  const int64_t span = ((a.sub_len + kL8 - 1) / kL8 + 31) / 32 * 32;
  bool bad = false;
  const int64_t G = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < span; k += G) {
    const int64_t p0 = k * kL8;
    const int nvalid = l8_valid(a.sub_len, p0);
    float own[kL8];
    l8_load(reinterpret_cast<const Tin*>(a.in[j]), off + p0, a.M, nvalid, own);
    float acc[kL8];
#pragma unroll
    for (int e = 0; e < kL8; ++e) acc[e] = 0.0f;  // 0 + v is exact (v never -0)
    for (int b0 = 0; b0 < a.world; b0 += B) {
      L8Raw raw[B];
#pragma unroll
      for (int q = 0; q < B; ++q) {
        const int s = b0 + q;
        if (s < a.world && s != j && nvalid > 0) raw[q] = l8_fetch<F>(a.c1, recv_slot(a, j, s), p0);
      }
      if (j >= b0 && j < b0 + B) {  // own piece: QDQ while the peers' codes are in flight
        if (rot.dim) l8_rotate(rot, off + p0, own);
        L8Codes q;
        __half s16;
        uint8_t z8;
        float v[kL8];
#pragma unroll
        for (int e = 0; e < kL8; ++e) v[e] = own[e];
        bad |= l8_quant<F>(a.c1, v, nvalid, q, s16, z8, own);  // collectives.py:364-365
      }
#pragma unroll
      for (int q = 0; q < B; ++q) {  // collectives.py:182-187
        const int s = b0 + q;
        if (s >= a.world) break;
        float d[kL8];
        if (s == j) {
#pragma unroll
          for (int e = 0; e < kL8; ++e) d[e] = own[e];
        } else if (nvalid > 0) {
          l8_decode<F>(a.c1, raw[q], d);
        } else {
#pragma unroll
          for (int e = 0; e < kL8; ++e) d[e] = 0.0f;
        }
#pragma unroll
        for (int e = 0; e < kL8; ++e) acc[e] += d[e];
      }
    }
    L8Codes q2;
    __half s2;
    uint8_t z2;
    float o[kL8];
    bad |= l8_quant<F>(a.c2, acc, nvalid, q2, s2, z2, o);
    for (int pp = 1; pp < a.world; ++pp) {
      int p = j + pp;
      if (p >= a.world) p -= a.world;
      l8_store<F>(a.c2, gath_slot(a, p, j), p0, nvalid, q2, s2, z2);
    }
    if (rot.dim) l8_unrotate(rot, off + p0, o);
    l8_write(reinterpret_cast<Tout*>(a.out[j]), off + p0, a.M, nvalid, o);  // collectives.py:378
  }
  if (bad) atomicOr(errw(a, j), make_err(kErrNonFinite, kPhReduce, j, j));
}

// gather: rank r decodes owner j's stage-2 piece (blockIdx.y = job), inverse rotation
template <typename Tout, int F>
__global__ void __launch_bounds__(kL8Threads) k_l8_gather(FlashArgs a, L8Rot rot) {
  int r, j;
  pair_of(a, blockIdx.y, r, j);
  const int64_t off = (int64_t)j * a.seg + a.sub_off;
  const uint8_t* src = gath_slot(a, r, j);
  const int64_t span = ((a.sub_len + kL8 - 1) / kL8 + 31) / 32 * 32;
  L8Raw regs[kL8UD];
  l8_sweep<kL8UD>(
      span,
      [&](int64_t k, L8Raw& R) {
        if (l8_valid(a.sub_len, k * kL8) > 0) R = l8_fetch<F>(a.c2, src, k * kL8);
      },
      [&](int64_t k, L8Raw& R) {
        const int64_t p0 = k * kL8;
        const int nvalid = l8_valid(a.sub_len, p0);
        float o[kL8];
        if (nvalid > 0) {
          l8_decode<F>(a.c2, R, o);
        } else {
#pragma unroll
          for (int e = 0; e < kL8; ++e) o[e] = 0.0f;
        }
        if (rot.dim) l8_unrotate(rot, off + p0, o);
        l8_write(reinterpret_cast<Tout*>(a.out[r]), off + p0, a.M, nvalid, o);
      },
      regs);
}

// single-GPU codec (fc_quantize / fc_dequantize of a minifloat codec): whole tensor, group-
// aligned lanes
template <typename Tin, int F>
__global__ void __launch_bounds__(kL8Threads) k_l8_quant(const Tin* x, int64_t n, DevCodec c, uint8_t* dst,
                                                          uint32_t* err) {
  const int64_t span = ((n + kL8 - 1) / kL8 + 31) / 32 * 32;
  bool bad = false;
  L8In<Tin> regs[kL8UQ];
  l8_sweep<kL8UQ>(
      span, [&](int64_t k, L8In<Tin>& R) { l8_fetch_in(x, k * kL8, n, l8_valid(n, k * kL8), R); },
      [&](int64_t k, L8In<Tin>& R) {
        const int64_t p0 = k * kL8;
        const int nvalid = l8_valid(n, p0);
        float v[kL8];
        l8_unpack(R, v);
        L8Codes q;
        __half s16;
        uint8_t z8;
        float deq[kL8];
        bad |= l8_quant<F>(c, v, nvalid, q, s16, z8, deq);
        l8_store<F>(c, dst, p0, nvalid, q, s16, z8);
      },
      regs);
  if (bad && err) atomicOr(err, make_err(kErrNonFinite, 0, 0, 0));
}
template <typename Tout, int F>
__global__ void __launch_bounds__(kL8Threads) k_l8_dequant(const uint8_t* src, int64_t n, DevCodec c, Tout* out) {
  const int64_t span = ((n + kL8 - 1) / kL8 + 31) / 32 * 32;
  L8Raw regs[kL8UD];
  l8_sweep<kL8UD>(
      span,
      [&](int64_t k, L8Raw& R) {
        if (l8_valid(n, k * kL8) > 0) R = l8_fetch<F>(c, src, k * kL8);
      },
      [&](int64_t k, L8Raw& R) {
        const int64_t p0 = k * kL8;
        const int nvalid = l8_valid(n, p0);
        if (nvalid <= 0) return;
        float o[kL8];
        l8_decode<F>(c, R, o);
        l8_write(out, p0, n, nvalid, o);
      },
      regs);
}

}  // namespace fc
