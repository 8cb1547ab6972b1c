// Specialised lane codec for the common schemes (compile-time storage width,
// symmetry and rounding), same numerics as the generic lane codec of
// fc_common.cuh (reference codec.py:235-248,292-329,354-384), fewer
// instructions per element:
//
//  * group parameters once per lane: raw scale RN64(RN64(max-min)/(2^b-1))
//    with a Markstein division by the constant (DMUL + 2 DFMA; checked
//    against IEEE division on 9e8 random fp32 ranges, 0 mismatches), one
//    cvt.rn.f16.f64, inf -> 65504 and the floor bump folded into an integer
//    min/max on the fp16 bit pattern (codec.py:242-248); zero point
//    ceil(-min/s) from the correctly rounded fp32 quotient with an exact
//    residual test (equal to numpy's ceil of the float64 quotient);
//  * per element, in packed fp32x2 (FMUL2/FFMA2/FADD2 on sm_100a): the
//    correctly rounded quotient q = RN(t + r*RN(x - t*s)), t = RN(x*r), then
//    the magic add q + 1.5*2^23 (RN: ties-to-even, RP: ceil) leaves round(q)
//    in the low 16 bits. Two elements' rounded quotients are merged into one
//    register (PRMT) and "+ z, clamp to [0, 2^b-1]" is one VIADDMNMX plus one
//    VIMNMX3 on signed 16x2 lanes. Exact whenever |x/s| < 2^14 for the whole
//    lane (checked per lane; otherwise the generic float-clamp loop runs).
//  * nibble/byte packing by shifted adds of the 16x2 code pairs: INT4 pairs
//    elements (a, a+4) of each 8, INT8 pairs (a, a+2) of each 4, so the
//    packed word is P0 + P1<<4 + P2<<8 + P3<<12 (INT4) / P0 + P1<<8 (INT8),
//    canonical little-nibble-first (bitpack.py:48-62).
//  * decode: PRMT builds 2^23 + c as a float, FADD2 subtracts 2^23 + z
//    (exact), FMUL2 / FFMA2 scale and accumulate (one rounding per add, the
//    rank-ordered fp32 sum of collectives.py:182-187).
#pragma once

#include "fc_common.cuh"

namespace fc {

// ------------------------------------------------------------------ fp32x2

__device__ __forceinline__ uint64_t f2_pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2_unpack(uint64_t v, float& a, float& b) {
  asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ void f2_bits(uint64_t v, uint32_t& a, uint32_t& b) {
  asm("mov.b64 {%0,%1}, %2;" : "=r"(a), "=r"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t f2_mul(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t f2_add_rp(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rp.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t f2_splat(float a) { return f2_pack(a, a); }

// ------------------------------------------------------------------ specs

// Compile-time codec scheme. GenSpec = the generic runtime-flag lane codec.
struct GenSpec {
  static constexpr bool kFast = false;
  static constexpr bool kLegacy = true;  // the cp.async-staged kernels are compiled for this scheme
  static constexpr int SB = 0;
  static constexpr bool SYM = false, CEIL = false;
  static constexpr bool MF = false;
};
#ifndef FC_STAGED
#define FC_STAGED 0  // make STAGED=1: also compile the cp.async-staged kernels for the compile-time presets (A/B)
#endif
template <int SB_, bool SYM_, bool CEIL_>
struct IntSpec {
  static constexpr bool kFast = true;
  // the staged kernels of the compile-time presets are an A/B build option (FC_STAGED); the
  // streaming, fused and small-message kernels are the product path, the runtime-codec
  // (GenSpec) staged kernels serve every other scheme
  static constexpr bool kLegacy = FC_STAGED && !SYM_ && !CEIL_;
  static constexpr int SB = SB_;  // storage bits: 4 (bits 2..4) or 8 (bits 5..8)
  static constexpr bool SYM = SYM_;
  static constexpr bool CEIL = CEIL_;
  static constexpr bool MF = false;
};
// group-scaled minifloat codec (codec.py:332-351) on the streaming codec kernels
// (k_qstream_gpl / k_dstream): absmax groups (SYM), no zero point, codes by
// cvt.rn.satfinite (mf_enc2) and back by cvt.rn.f16x2 (mf_dec2)
template <int FMT_>
struct MfSpec {
  static constexpr bool kFast = true;
  static constexpr bool kLegacy = false;
  static constexpr int SB = FMT_ == FC_FMT_E2M1 ? 4 : 8;
  static constexpr bool SYM = true, CEIL = false;
  static constexpr bool MF = true;
  static constexpr int FMT = FMT_;
};
using SpecA4 = IntSpec<4, false, false>;  // INT4 asym nearest (FlashConfig.from_bits(4))
using SpecA8 = IntSpec<8, false, false>;  // INT8 asym nearest (from_bits(8), INT6 stage 2)
using SpecS4 = IntSpec<4, true, false>;   // symmetric, bits 2..4
using SpecS8 = IntSpec<8, true, false>;   // symmetric, bits 5..8
using SpecC4 = IntSpec<4, false, true>;   // asym, ceil rounding (codec.py:288-289)
using SpecC8 = IntSpec<8, false, true>;

// ------------------------------------------------------------------ element access

// elements a and b of a lane source as an fp32 pair
template <typename T>
__device__ __forceinline__ uint64_t lane_pair(const PackedLane<T>& L, int a, int b) {
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    const uint32_t wa = L.w[a >> 1], wb = L.w[b >> 1];
    const uint32_t xa = (a & 1) ? (wa & 0xFFFF0000u) : (wa << 16);
    const uint32_t xb = (b & 1) ? (wb & 0xFFFF0000u) : (wb << 16);
    uint64_t r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "r"(xa), "r"(xb));
    return r;
  } else {
    return f2_pack(L.get(a), L.get(b));
  }
}
__device__ __forceinline__ uint64_t lane_pair(const FloatLane& L, int a, int b) { return f2_pack(L.v[a], L.v[b]); }

// fp32 lane held as packed pairs in the canonical pairing of a storage
// width: SB=4 pairs elements (8i+a, 8i+a+4), SB=8 pairs (4i+a, 4i+a+2), so
// that decode, accumulate (FFMA2) and re-encode of the same width never move
// registers.
template <int SB>
struct PairLane {
  uint64_t p[16];
  __device__ static constexpr int pair_of(int k) {
    return SB == 4 ? (k >> 3) * 4 + (k & 3) : (k >> 2) * 2 + (k & 1);
  }
  __device__ static constexpr bool is_hi(int k) { return SB == 4 ? ((k & 4) != 0) : ((k & 2) != 0); }
  __device__ __forceinline__ float get(int k) const {
    float a, b;
    f2_unpack(p[pair_of(k)], a, b);
    return is_hi(k) ? b : a;
  }
};

template <int SB>
__device__ __forceinline__ uint64_t lane_pair(const PairLane<SB>& L, int a, int b) {
  if (PairLane<SB>::pair_of(a) == PairLane<SB>::pair_of(b) && !PairLane<SB>::is_hi(a) && PairLane<SB>::is_hi(b))
    return L.p[PairLane<SB>::pair_of(a)];
  return f2_pack(L.get(a), L.get(b));
}

template <int SB>
__device__ __forceinline__ void to_float_lane(const PairLane<SB>& L, FloatLane& F) {
#pragma unroll
  for (int k = 0; k < kLaneElems; ++k) F.v[k] = L.get(k);
}

template <bool SYM, int SB>
__device__ __forceinline__ void lane_stats(const PairLane<SB>& L, int nvalid, float& lo, float& hi) {
  FloatLane F;
  to_float_lane(L, F);
  lane_stats<SYM>(F, nvalid, lo, hi);
}

// ------------------------------------------------------------------ statistics

__device__ __forceinline__ float fmin3_nan(float a, float b, float c) {
  float r;
  asm("min.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float fmax3_nan(float a, float b, float c) {
  float r;
  asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// min/max (SYM: -, absmax) of a full 32-element fp32 lane with 3-input FMNMX3
template <bool SYM, class Src>
__device__ __forceinline__ void stats32_f32(const Src& L, float& lo, float& hi) {
  float v[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) v[k] = SYM ? fabsf(L.get(k)) : L.get(k);
  float a[11], b[11];
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    a[i] = fmin3_nan(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
    b[i] = fmax3_nan(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
  }
  a[10] = fmin_nan(v[30], v[31]);
  b[10] = fmax_nan(v[30], v[31]);
  const float a0 = fmin3_nan(a[0], a[1], a[2]), a1 = fmin3_nan(a[3], a[4], a[5]), a2 = fmin3_nan(a[6], a[7], a[8]);
  const float b0 = fmax3_nan(b[0], b[1], b[2]), b1 = fmax3_nan(b[3], b[4], b[5]), b2 = fmax3_nan(b[6], b[7], b[8]);
  lo = fmin3_nan(fmin3_nan(a0, a1, a2), a[9], a[10]);
  hi = fmax3_nan(fmax3_nan(b0, b1, b2), b[9], b[10]);
}

// group-wide min/max over lpg lanes (uniform), NaN-propagating
__device__ __forceinline__ void group_minmax(float& lo, float& hi, int lpg) {
#pragma unroll
  for (int o = 1; o < 8; o <<= 1) {
    if (o < lpg) {
      lo = fmin_nan(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmax_nan(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
  }
}
// bf16-exact bounds: (lo, -hi) travel as one bf16x2 word, one shuffle + one HMNMX2 per step
__device__ __forceinline__ void group_minmax_bf16(float& lo, float& hi, int lpg) {
  uint32_t w = (__float_as_uint(lo) >> 16) | (__float_as_uint(-hi) & 0xFFFF0000u);
#pragma unroll
  for (int o = 1; o < 8; o <<= 1) {
    if (o < lpg) {
      const uint32_t u = __shfl_xor_sync(0xffffffffu, w, o);
      asm("min.NaN.bf16x2 %0, %1, %2;" : "=r"(w) : "r"(w), "r"(u));
    }
  }
  lo = __uint_as_float(w << 16);
  hi = -__uint_as_float(w & 0xFFFF0000u);
}

// full-lane statistics + group reduction for each source kind
template <bool SYM, typename T>
__device__ __forceinline__ void group_stats(const DevCodec& c, const PackedLane<T>& L, float& lo, float& hi) {
  lane_stats<SYM>(L, kLaneElems, lo, hi);
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    if (SYM) lo = -hi;
    group_minmax_bf16(lo, hi, c.lpg);
  } else {
    group_minmax(lo, hi, c.lpg);
  }
}
template <bool SYM>
__device__ __forceinline__ void group_stats(const DevCodec& c, const FloatLane& L, float& lo, float& hi) {
  struct G {
    const FloatLane& l;
    __device__ float get(int k) const { return l.v[k]; }
  } g{L};
  stats32_f32<SYM>(g, lo, hi);
  group_minmax(lo, hi, c.lpg);
}
template <bool SYM, int SB>
__device__ __forceinline__ void group_stats(const DevCodec& c, const PairLane<SB>& L, float& lo, float& hi) {
  stats32_f32<SYM>(L, lo, hi);
  group_minmax(lo, hi, c.lpg);
}

// ------------------------------------------------------------------ group parameters

struct GroupQ {
  float s;          // scale (exact fp16 value)
  float r;          // RN(1/s)
  uint32_t z;       // zero point (asym) / 2^(b-1) (sym, offset binary)
  unsigned short s16;
  bool normal;      // every |x/s| of the group < 2^14: packed 16-bit rounding is exact
};

// lo/hi: group min/max (asym) or -, absmax (sym), already reduced over the group
template <class Spec>
__device__ __forceinline__ void group_params(const DevCodec& c, float lo, float hi, GroupQ& g) {
  const double d = Spec::SYM ? (double)hi : (double)hi - (double)lo;
  const double q0 = d * c.qinv;
  const double raw = fma(fma(-q0, c.qdiv, d), c.qinv, q0);  // RN64(d / qdiv), Markstein
  const double rf = fmax(raw, c.floor);
  uint32_t b = __half_as_ushort(__double2half(rf));        // one rounding (numpy astype(float16))
  b = max(min(b, 0x7BFFu), c.floor16);                     // inf -> 65504; below floor -> next fp16 up
  g.s16 = (unsigned short)b;
  g.s = __half2float(__ushort_as_half(g.s16));
  g.r = __frcp_rn(g.s);
  float amax;
  if constexpr (Spec::SYM) {
    g.z = 1u << (c.bits - 1);
    amax = hi;
  } else {
    const float a = -lo;
    const float t = a * g.r;
    const float q = fmaf(fmaf(-t, g.s, a), g.r, t);  // RN(-lo/s)
    float zc = ceilf(q);
    if (zc == q && fmaf(-q, g.s, a) > 0.0f) zc += 1.0f;  // exact residual: true quotient above q
    zc = fminf(fmaxf(zc, 0.0f), c.qmax_f);               // codec.py:321 (NaN -> 0)
    g.z = (uint32_t)zc;
    amax = fmaxf(fabsf(lo), fabsf(hi));
  }
  g.normal = amax * g.r < 16384.0f;  // false for NaN/inf
}

// ------------------------------------------------------------------ codes

// Offset-binary codes of a full 32-element lane chunk into w[0..SB-1]
// (INT4: 4 words, INT8: 8 words). Requires g.normal.
template <class Spec, class Src>
__device__ __forceinline__ void lane_codes_packed(const Src& L, const GroupQ& g, uint32_t qmax, uint32_t* w) {
  const uint64_t R2 = f2_splat(g.r), NS2 = f2_splat(-g.s), C2 = f2_splat(12582912.0f);
  const uint32_t Z2 = g.z * 0x00010001u, Q2 = qmax * 0x00010001u;
  auto code_pair = [&](int a, int b) -> uint32_t {
    const uint64_t X = lane_pair(L, a, b);
    const uint64_t T = f2_mul(X, R2);
    const uint64_t Q = f2_fma(f2_fma(T, NS2, X), R2, T);
    const uint64_t Y = Spec::CEIL ? f2_add_rp(Q, C2) : f2_add(Q, C2);
    uint32_t ya, yb;
    f2_bits(Y, ya, yb);
    const uint32_t p = __byte_perm(ya, yb, 0x5410);  // (round(q_a), round(q_b)) as s16x2
    const uint32_t c = __viaddmax_s16x2(p, Z2, 0u);   // max(k + z, 0)
    return __vimin3_s16x2(c, Q2, Q2);                  // min(., qmax)
  };
  if constexpr (Spec::SB == 4) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = 8 * i;
      const uint32_t p0 = code_pair(e + 0, e + 4), p1 = code_pair(e + 1, e + 5);
      const uint32_t p2 = code_pair(e + 2, e + 6), p3 = code_pair(e + 3, e + 7);
      w[i] = p0 + (p1 << 4) + (p2 << 8) + (p3 << 12);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int e = 4 * i;
      const uint32_t p0 = code_pair(e + 0, e + 2), p1 = code_pair(e + 1, e + 3);
      w[i] = p0 + (p1 << 8);
    }
  }
}

// Fast quantize of a full lane chunk; same contract as lane_quantize (the
// group's lanes call it together). Returns true on non-finite input.
template <class Spec, int CW, class Src>
__device__ __forceinline__ bool lane_quantize_fast(const DevCodec& c, const Src& L, LaneQuant<CW>& q) {
  float lo, hi;
  group_stats<Spec::SYM>(c, L, lo, hi);
  if constexpr (Spec::SYM) lo = -hi;
  const bool bad = !(fabsf(lo) <= 3.402823466e38f && fabsf(hi) <= 3.402823466e38f);
  GroupQ g;
  group_params<Spec>(c, lo, hi, g);
  if (bad) g.z = Spec::SYM ? g.z : 0u;
  const uint32_t qmax = (1u << c.bits) - 1u;
  if (g.normal) {
    lane_codes_packed<Spec>(L, g, qmax, q.w);
  } else {  // |x/s| may exceed the 16-bit lanes: float clamp before rounding
    lane_codes<Spec::SB, Spec::CEIL>(L, g.s, (int)g.z, (int)qmax, q.w);
  }
  q.s16 = __ushort_as_half(g.s16);
  q.s = g.s;
  q.z8 = Spec::SYM ? 0 : (uint8_t)g.z;
  q.mz = 8388608.0f + (float)g.z;
  q.xr = Spec::SYM ? (Spec::SB == 4 ? (1u << (c.bits - 1)) * 0x11111111u : (1u << (c.bits - 1)) * 0x01010101u) : 0u;
  if constexpr (Spec::SYM) {
#pragma unroll
    for (int i = 0; i < Spec::SB; ++i) q.w[i] ^= q.xr;
  }
  return bad;
}

// Dispatch: the fast path for full chunks of a compile-time scheme, the
// generic lane codec otherwise (tails, unusual schemes, fp16 passthrough).
// The fast/generic choice is warp-uniform (__all_sync): both codecs reduce the
// group bounds with full-warp shuffles, which every lane must execute at the
// same instruction.
template <class Spec, int CW, class Src>
__device__ __forceinline__ bool quantize_lane(const DevCodec& c, const Src& L, int nvalid, LaneQuant<CW>& q) {
  if constexpr (Spec::kFast) {
    if (__all_sync(0xffffffffu, nvalid == kLaneElems)) return lane_quantize_fast<Spec>(c, L, q);
  }
  return lane_quantize(c, L, nvalid, q);
}
template <class Spec, int CW, int SB>
__device__ __forceinline__ bool quantize_lane(const DevCodec& c, const PairLane<SB>& L, int nvalid, LaneQuant<CW>& q) {
  if constexpr (Spec::kFast) {
    if (__all_sync(0xffffffffu, nvalid == kLaneElems)) return lane_quantize_fast<Spec>(c, L, q);
  }
  FloatLane F;
  to_float_lane(L, F);
  return lane_quantize(c, F, nvalid, q);
}

// ------------------------------------------------------------------ decode

// out[k] (+)= (c_k - z) * s for offset-binary codes L.w (exact products,
// one rounding per accumulation)
template <class Spec, bool ACC, int CW>
__device__ __forceinline__ void decode_lane(const DevCodec& c, const LaneCodes<CW>& L, float out[kLaneElems]) {
  if constexpr (!Spec::kFast) {
    lane_decode<ACC>(c, L, out);
  } else {
    const uint64_t S2 = f2_splat(L.s), NMZ2 = f2_splat(-L.mz);
    auto emit = [&](int a, int b, uint32_t va, uint32_t vb) {  // va/vb: magic float bits 2^23 + c
      uint64_t M;
      asm("mov.b64 %0, {%1,%2};" : "=l"(M) : "r"(va), "r"(vb));
      const uint64_t D = f2_add(M, NMZ2);  // c - z, exact
      uint64_t R;
      if (ACC)
        R = f2_fma(D, S2, f2_pack(out[a], out[b]));
      else
        R = f2_mul(D, S2);
      f2_unpack(R, out[a], out[b]);
    };
    if constexpr (Spec::SB == 4) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t lo = L.w[i] & 0x0F0F0F0Fu, hi = (L.w[i] >> 4) & 0x0F0F0F0Fu;
        const int e = 8 * i;
        // lo bytes hold elements e, e+2, e+4, e+6; hi bytes e+1, e+3, e+5, e+7
        emit(e + 0, e + 4, __byte_perm(lo, 0x4B000000u, 0x7440u), __byte_perm(lo, 0x4B000000u, 0x7442u));
        emit(e + 2, e + 6, __byte_perm(lo, 0x4B000000u, 0x7441u), __byte_perm(lo, 0x4B000000u, 0x7443u));
        emit(e + 1, e + 5, __byte_perm(hi, 0x4B000000u, 0x7440u), __byte_perm(hi, 0x4B000000u, 0x7442u));
        emit(e + 3, e + 7, __byte_perm(hi, 0x4B000000u, 0x7441u), __byte_perm(hi, 0x4B000000u, 0x7443u));
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t v = L.w[i];
        const int e = 4 * i;
        emit(e + 0, e + 2, __byte_perm(v, 0x4B000000u, 0x7440u), __byte_perm(v, 0x4B000000u, 0x7442u));
        emit(e + 1, e + 3, __byte_perm(v, 0x4B000000u, 0x7441u), __byte_perm(v, 0x4B000000u, 0x7443u));
      }
    }
  }
}


// decode into packed pairs of the codec's own pairing: out (+)= (c - z) * s
template <class Spec, bool ACC, int CW>
__device__ __forceinline__ void decode_pairs(const LaneCodes<CW>& L, PairLane<Spec::SB>& out) {
  static_assert(Spec::kFast, "compile-time codec");
  const uint64_t S2 = f2_splat(L.s), NMZ2 = f2_splat(-L.mz);
  auto emit = [&](int idx, uint32_t va, uint32_t vb, uint64_t nmz, uint64_t sc) {
    uint64_t M;
    asm("mov.b64 %0, {%1,%2};" : "=l"(M) : "r"(va), "r"(vb));
    const uint64_t D = f2_add(M, nmz);  // (c - z) or 16 (c - z), exact
    out.p[idx] = ACC ? f2_fma(D, sc, out.p[idx]) : f2_mul(D, sc);
  };
  if constexpr (Spec::SB == 4) {
    // high nibbles stay in place (byte = 16 c): decode 16 (c - z) * (s / 16), the same exact
    // product, and save the shift that would isolate them
    const uint64_t S16 = f2_splat(L.s * 0.0625f), NMZ16 = f2_splat(-fmaf(L.mz, 16.0f, -125829120.0f));
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t lo = L.w[i] & 0x0F0F0F0Fu, hi = L.w[i] & 0xF0F0F0F0u;
      emit(4 * i + 0, __byte_perm(lo, 0x4B000000u, 0x7440u), __byte_perm(lo, 0x4B000000u, 0x7442u), NMZ2, S2);
      emit(4 * i + 2, __byte_perm(lo, 0x4B000000u, 0x7441u), __byte_perm(lo, 0x4B000000u, 0x7443u), NMZ2, S2);
      emit(4 * i + 1, __byte_perm(hi, 0x4B000000u, 0x7440u), __byte_perm(hi, 0x4B000000u, 0x7442u), NMZ16, S16);
      emit(4 * i + 3, __byte_perm(hi, 0x4B000000u, 0x7441u), __byte_perm(hi, 0x4B000000u, 0x7443u), NMZ16, S16);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t v = L.w[i];
      emit(2 * i + 0, __byte_perm(v, 0x4B000000u, 0x7440u), __byte_perm(v, 0x4B000000u, 0x7442u), NMZ2, S2);  // e, e+2
      emit(2 * i + 1, __byte_perm(v, 0x4B000000u, 0x7441u), __byte_perm(v, 0x4B000000u, 0x7443u), NMZ2, S2);  // e+1, e+3
    }
  }
}

// ------------------------------------------------------------------ minifloat codes (cvt)

// two f32 quotients -> two codes: byte codes (e4m3 / e5m2) in the low / high byte of the
// result, e2m1 nibbles in the low / high nibble; zero magnitude -> +0 pattern
__device__ __forceinline__ uint32_t mf_enc2(int fmt, float x0, float x1) {
  uint32_t r;
  if (fmt == FC_FMT_E4M3) {
    unsigned short h;
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(h) : "f"(x1), "f"(x0));
    r = h;
    if ((r & 0x007Fu) == 0) r &= 0xFF00u;
    if ((r & 0x7F00u) == 0) r &= 0x00FFu;
  } else if (fmt == FC_FMT_E5M2) {
    unsigned short h;
    asm("cvt.rn.satfinite.e5m2x2.f32 %0, %1, %2;" : "=h"(h) : "f"(x1), "f"(x0));
    r = h;
    if ((r & 0x007Fu) == 0) r &= 0xFF00u;
    if ((r & 0x7F00u) == 0) r &= 0x00FFu;
  } else {
    asm("{\n .reg .b8 t;\n cvt.rn.satfinite.e2m1x2.f32 t, %1, %2;\n cvt.u32.u8 %0, t;\n}" : "=r"(r) : "f"(x1), "f"(x0));
    if ((r & 0x07u) == 0) r &= 0xF0u;
    if ((r & 0x70u) == 0) r &= 0x0Fu;
  }
  return r;
}

// mf_enc2 without the +0 fix-up (cvt.rn.satfinite only): the streaming kernels pack the codes
// into words first and fix a whole word at once (mf_fix_zero)
__device__ __forceinline__ uint32_t mf_enc2_raw(int fmt, float x0, float x1) {
  uint32_t r;
  if (fmt == FC_FMT_E4M3) {
    unsigned short h;
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(h) : "f"(x1), "f"(x0));
    r = h;
  } else if (fmt == FC_FMT_E5M2) {
    unsigned short h;
    asm("cvt.rn.satfinite.e5m2x2.f32 %0, %1, %2;" : "=h"(h) : "f"(x1), "f"(x0));
    r = h;
  } else {
    asm("{\n .reg .b8 t;\n cvt.rn.satfinite.e2m1x2.f32 t, %1, %2;\n cvt.u32.u8 %0, t;\n}" : "=r"(r) : "f"(x1), "f"(x0));
  }
  return r;
}

// a word of minifloat codes (4 bytes e4m3 / e5m2, 8 nibbles e2m1): every code whose magnitude
// bits are zero becomes +0 (encode() stores zero magnitudes as +0). Per code, magnitude +
// all-ones-magnitude carries into the sign position iff the magnitude is non-zero (no carry
// crosses a code), so the sign survives exactly there
template <int FMT>
__device__ __forceinline__ uint32_t mf_fix_zero(uint32_t w) {
  constexpr uint32_t MAG = FMT == FC_FMT_E2M1 ? 0x77777777u : 0x7F7F7F7Fu;
  const uint32_t mag = w & MAG;
  return mag | (w & (mag + MAG) & ~MAG);
}

// two codes (as packed by mf_enc2) -> two exact fp32 grid values
__device__ __forceinline__ void mf_dec2(int fmt, uint32_t code2, float& v0, float& v1) {
  uint32_t h2;
  if (fmt == FC_FMT_E4M3) {
    asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h2) : "h"((unsigned short)code2));
  } else if (fmt == FC_FMT_E5M2) {
    asm("cvt.rn.f16x2.e5m2x2 %0, %1;" : "=r"(h2) : "h"((unsigned short)code2));
  } else {
    asm("{\n .reg .b8 t;\n cvt.u8.u32 t, %1;\n cvt.rn.f16x2.e2m1x2 %0, t;\n}" : "=r"(h2) : "r"(code2 & 0xFFu));
  }
  v0 = __half2float(__ushort_as_half((unsigned short)(h2 & 0xFFFFu)));
  v1 = __half2float(__ushort_as_half((unsigned short)(h2 >> 16)));
}

}  // namespace fc
