// Single-GPU group codec kernels: quantize (codec.py:292-329) and dequantize
// (codec.py:354-384), plus the generic (any group size) kernels that the
// flash path reuses for group sizes outside {32, 64, 128, 256}.
#include <cstring>
#include <algorithm>
#include <map>
#include <mutex>

#include "fc_codec_dev.cuh"
#include "fc_lane.cuh"
#include "fc_stream.cuh"
#include "fc_stage.cuh"
#include "fc_host.h"

namespace fc {

// --------------------------------------------------------------------------
// fast path: one 32-element chunk per thread, groups of g/32 lanes

template <typename T, int CW, class Spec>
__global__ void __launch_bounds__(kThreads) k_quant_fast(const T* __restrict__ x, int64_t n, DevCodec c,
                                                         uint8_t* __restrict__ dst, uint32_t* err, int S) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int CB = Chunk<T>::kBytes;
  const int lane = threadIdx.x & 31;
  const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(smem) + threadIdx.x * CB;
  const int64_t tiles = (n + kTileElems - 1) / kTileElems;
  auto issue = [&](int64_t t, int st) {
    if (t < tiles) {
      const int64_t p0 = t * kTileElems + (int64_t)threadIdx.x * kLaneElems;
      const int nvalid = (int)max((int64_t)0, min(n - p0, (int64_t)kLaneElems));
      chunk_issue<T>(s0 + st * kThreads * CB, x, p0, n, nvalid, lane);
    }
    cp_async_commit();
  };
  for (int k = 0; k < S - 1; ++k) issue(blockIdx.x + (int64_t)k * gridDim.x, k);
  int st = 0;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    issue(t + (int64_t)(S - 1) * gridDim.x, st == 0 ? S - 1 : st - 1);
    cp_async_wait_dyn(S - 1);
    const int64_t p0 = t * kTileElems + (int64_t)threadIdx.x * kLaneElems;
    const int nvalid = (int)max((int64_t)0, min(n - p0, (int64_t)kLaneElems));
    LaneOf<T> v;
    chunk_read_src<T>(s0 + st * kThreads * CB, lane, v);
    LaneQuant<CW> q;
    const bool bad = quantize_lane<Spec>(c, v, nvalid, q);
    store_lane(c, dst, p0, nvalid, q, lane);
    if (bad && err) atomicOr(err, make_err(kErrNonFinite, 0, 0, 0));
    st = (st + 1 == S) ? 0 : st + 1;
  }
}

template <typename To, int CW, class Spec>
__global__ void __launch_bounds__(kThreads) k_dequant_fast(const uint8_t* __restrict__ src, int64_t n, DevCodec c,
                                                           To* __restrict__ out, int S) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int CB = code_chunk_bytes(c);
  const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(smem) + threadIdx.x * CB;
  const int64_t tiles = (n + kTileElems - 1) / kTileElems;
  auto issue = [&](int64_t t, int st) {
    if (t < tiles) {
      const int64_t p0 = t * kTileElems + (int64_t)threadIdx.x * kLaneElems;
      if (p0 < n) code_issue(c, s0 + st * kThreads * CB, src, p0);
    }
    cp_async_commit();
  };
  for (int k = 0; k < S - 1; ++k) issue(blockIdx.x + (int64_t)k * gridDim.x, k);
  int st = 0;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    issue(t + (int64_t)(S - 1) * gridDim.x, st == 0 ? S - 1 : st - 1);
    cp_async_wait_dyn(S - 1);
    const int64_t p0 = t * kTileElems + (int64_t)threadIdx.x * kLaneElems;
    const int nvalid = (int)max((int64_t)0, min(n - p0, (int64_t)kLaneElems));
    if (nvalid > 0) {
      LaneCodes<CW> L;
      code_read(c, s0 + st * kThreads * CB, p0, L);
      float v[kLaneElems];
      decode_lane<Spec, false>(c, L, v);
      store_chunk(out, p0, n, nvalid, v);
    }
    st = (st + 1 == S) ? 0 : st + 1;
  }
}

static fc_status ensure_smem_attr(const void* kern, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  int& have = done[{kern, dev}];
  if (bytes > have) {
    FC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    have = bytes;
  }
  return FC_OK;
}

static unsigned resident_grid(const void* kern, int smem, int64_t items, int sms) {
  int dev = 0;
  cudaGetDevice(&dev);
  const int occ = std::max(1, occupancy(kern, kThreads, smem, dev));
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(items, (int64_t)occ * sms));
}

static int cur_sms();

// --------------------------------------------------------------------------
// blocked Hadamard rotation (rotation.py:38-83): one CTA per block of `dim`
// elements at a time, float64 butterflies in shared memory in the reference's
// order (top = a + b, bottom = a - b, h = 1, 2, 4, ...), one final rounding

template <typename Ti, typename To>
__global__ void __launch_bounds__(256) k_hadamard(const Ti* __restrict__ x, int64_t n, int64_t n_padded, int dim,
                                                  int normalize, const float* __restrict__ signs, int inverse,
                                                  To* __restrict__ out, int64_t n_out) {
  extern __shared__ __align__(16) double hs[];
  const double rs = sqrt((double)dim);
  for (int64_t base = (int64_t)blockIdx.x * dim; base < n_padded; base += (int64_t)gridDim.x * dim) {
    for (int i = threadIdx.x; i < dim; i += blockDim.x) {
      const int64_t gi = base + i;
      double v = gi < n ? (double)DT<Ti>::to_f(x[gi]) : 0.0;
      if (!inverse && signs) v *= (double)signs[i];  // H(D x)
      hs[i] = v;
    }
    __syncthreads();
    for (int h = 1; h < dim; h <<= 1) {
      for (int k = threadIdx.x; k < dim / 2; k += blockDim.x) {
        const int i = (k / h) * 2 * h + (k % h);
        const double a = hs[i], b = hs[i + h];
        hs[i] = a + b;
        hs[i + h] = a - b;
      }
      __syncthreads();
    }
    for (int i = threadIdx.x; i < dim; i += blockDim.x) {
      double y = hs[i];
      if (!inverse) {
        if (normalize) y = y / rs;
      } else {
        y = normalize ? y / rs : y / (double)dim;
        if (signs) y *= (double)signs[i];  // D(H x)
      }
      const int64_t gi = base + i;
      if (gi < n_out) out[gi] = DT<To>::from_f((float)y);  // float32 result (astype(float32)), then the output dtype
    }
    __syncthreads();
  }
}

fc_status launch_hadamard(const void* x, int in_dtype, int64_t n, int64_t n_padded, int dim, int normalize,
                          const float* signs, int inverse, void* out, int out_dtype, int64_t n_out, cudaStream_t st) {
  const int smem = dim * (int)sizeof(double);
  const int64_t blocks = n_padded / dim;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)cur_sms() * 8));
#define FC_HD(TI, TO)                                                                                        \
  do {                                                                                                       \
    const void* k = (const void*)k_hadamard<TI, TO>;                                                         \
    FC_TRY(ensure_smem_attr(k, smem));                                                                       \
    k_hadamard<TI, TO><<<grid, 256, smem, st>>>((const TI*)x, n, n_padded, dim, normalize, signs, inverse,    \
                                                (TO*)out, n_out);                                            \
  } while (0)
#define FC_HD_OUT(TI)                                            \
  switch (out_dtype) {                                           \
    case FC_DTYPE_F32: FC_HD(TI, float); break;                  \
    case FC_DTYPE_F16: FC_HD(TI, __half); break;                 \
    default: FC_HD(TI, __nv_bfloat16); break;                    \
  }
  switch (in_dtype) {
    case FC_DTYPE_F32: FC_HD_OUT(float); break;
    case FC_DTYPE_F16: FC_HD_OUT(__half); break;
    default: FC_HD_OUT(__nv_bfloat16); break;
  }
#undef FC_HD_OUT
#undef FC_HD
  FC_CUDA_TRY(cudaGetLastError());
  return FC_OK;
}

// --------------------------------------------------------------------------
// launchers

// 1: INT4 asym nearest, 2: INT8 asym nearest (compile-time lane codecs), 0: generic
static int codec_spec(const fc_codec& c) {
  if (c.kind != FC_KIND_INT || c.symmetric || c.rounding != FC_ROUND_NEAREST_EVEN) return 0;
  return storage_bits(c) == 4 ? 1 : 2;
}

int num_sms(int device) {
  static int cache[64] = {0};
  if (device < 0 || device >= 64) return 148;
  if (!cache[device]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || v <= 0) v = 148;
    cache[device] = v;
  }
  return cache[device];
}

static int cur_sms() {
  int d = 0;
  cudaGetDevice(&d);
  return num_sms(d);
}


// single-GPU codec through the streaming kernels (fc_stream.cuh, mode 1)
static FlashArgs codec_args(const void* in, void* out, int64_t n, const DevCodec& dc, uint32_t* err) {
  FlashArgs a{};
  a.mode = 1;
  a.world = 1;
  a.rank_lo = 0;
  a.rank_hi = 1;
  a.M = n;
  a.seg = n;
  a.sub_off = 0;
  a.sub_len = n;
  a.tiles = (int)((n + kTileElems - 1) / kTileElems);
  a.c1 = dc;
  a.c2 = dc;
  a.cerr = err;
  a.in[0] = in;
  a.out[0] = out;
  return a;
}

static unsigned stream_grid_cur(const void* kern, int threads, int smem, int64_t items) {
  int dev = 0;
  cudaGetDevice(&dev);
  const int occ = std::max(1, occupancy(kern, threads, smem, dev));
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(items, (int64_t)occ * cur_sms()));
}

// A/B selection of the codec quantize kernel (measurement only): FC_CODEC_QKERNEL=lane|gpl|gq
static int codec_qkernel() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FC_CODEC_QKERNEL");
    v = !e ? 0 : (!strcmp(e, "lane") ? 1 : !strcmp(e, "gpl") ? 2 : !strcmp(e, "gq") ? 3 : !strcmp(e, "l8") ? 4 : 0);
  }
  return v;
}

template <typename T, class Spec, int G>
static fc_status quant_gq(FlashArgs a, cudaStream_t st) {
  const void* k = (const void*)k_qstream_gq<T, Spec, G>;
  const int smem = a.stages * (kTileElems * 2 + 16);
  FC_TRY(ensure_smem_attr(k, smem));
  k_qstream_gq<T, Spec, G><<<stream_grid_cur(k, kGplThreads, smem, a.tiles), kGplThreads, smem, st>>>(a);
  return FC_OK;
}

template <typename T, class Spec>
static fc_status quant_stream(const T* x, int64_t n, const DevCodec& dc, uint8_t* dst, uint32_t* err, cudaStream_t st) {
  FlashArgs a = codec_args(x, dst, n, dc, err);
  a.stages = 4;
  const int smem = a.stages * (kTileElems * 2 + 16);
  const int sel = codec_qkernel();
  // group-lane slices (k_qstream_gq) for g in {64, 128, 256} (INT8) / {64, 256} (INT4); INT4
  // g = 128 keeps the register-resident-group kernel (k_qstream_gpl), g = 32 the 32-element
  // lanes (k_qstream: four float64 group tails per slice cost more than the shuffles;
  // profiles/r02_codec_ab.txt)
  const bool gq_ok = dc.g == 32 || dc.g == 64 || dc.g == 128 || dc.g == 256;
  // INT4 g in {64, 128, 256}: the register-resident group-per-lane kernel (k_qstream_gpl<G>)
  // (g = 32, four groups per slice, measured slower than the 32-element lanes: 40.8 vs 35.6 us)
  const bool gpl_ok = Spec::SB == 4 && (dc.g == 64 || dc.g == 128 || dc.g == 256);
  const bool gq_auto = dc.g != 32 && !gpl_ok;
  if (gq_ok && (sel == 3 || (sel == 0 && gq_auto))) {
    a.stages = 3;
    switch (dc.g) {
      case 32: return quant_gq<T, Spec, 32>(a, st);
      case 64: return quant_gq<T, Spec, 64>(a, st);
      case 128: return quant_gq<T, Spec, 128>(a, st);
      default: return quant_gq<T, Spec, 256>(a, st);
    }
  }
  if (sel != 1 && gpl_ok) {  // a lane per 128-element slice, the slice's groups in registers (INT4)
    auto launch = [&](const void* k, auto kern) -> fc_status {
      FC_TRY(ensure_smem_attr(k, smem));
      kern<<<stream_grid_cur(k, kGplThreads, smem, a.tiles), kGplThreads, smem, st>>>(a);
      return FC_OK;
    };
    switch (dc.g) {
      case 64: return launch((const void*)k_qstream_gpl<T, Spec, 64>, k_qstream_gpl<T, Spec, 64>);
      case 256: return launch((const void*)k_qstream_gpl<T, Spec, 256>, k_qstream_gpl<T, Spec, 256>);
      default: return launch((const void*)k_qstream_gpl<T, Spec, 128>, k_qstream_gpl<T, Spec, 128>);
    }
  }
  const void* k = (const void*)k_qstream<T, Spec>;
  FC_TRY(ensure_smem_attr(k, smem));
  k_qstream<T, Spec><<<stream_grid_cur(k, kStreamThreads, smem, a.tiles), kStreamThreads, smem, st>>>(a);
  return FC_OK;
}

template <typename T, class Spec>
static fc_status dequant_stream(const uint8_t* src, int64_t n, const DevCodec& dc, T* out, cudaStream_t st) {
  FlashArgs a = codec_args(src, out, n, dc, nullptr);
  a.stages = dstream_stages<Spec>();
  const int smem = a.stages * ((int)dstage_bytes(dc) + 16);
  const void* k = (const void*)k_dstream<T, Spec>;
  FC_TRY(ensure_smem_attr(k, smem));
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(a.tiles, (int64_t)kDCtasPerSm * cur_sms()));
  k_dstream<T, Spec><<<grid, kStreamThreads, smem, st>>>(a);
  return FC_OK;
}

template <typename T>
static void quant_generic(const T* x, int64_t n, const DevCodec& dc, uint8_t* dst, uint32_t* err, cudaStream_t st) {
  SrcSeg<T> src{x, 0, n};
  if (dc.kind != FC_KIND_FP16) {  // int and minifloat codes need per-group scales
    const int64_t groups = (n + dc.g - 1) / dc.g;
    k_gen_params<<<(unsigned)((groups + 255) / 256), 256, 0, st>>>(src, n, dc, dst, err, 0u);
  }
  const int64_t units = gen_code_units(dc, n);
  k_gen_codes<<<(unsigned)((units + 255) / 256), 256, 0, st>>>(src, n, dc, dst, err, 0u);
}

// group-scaled minifloat codecs: the lane-8 kernels (fc_l8.cuh, cvt.rn.satfinite), g = 8..256
static bool l8_codec_ok(const fc_codec& c) {
  return c.kind == FC_KIND_MINIFLOAT && c.group_size >= 8 && c.group_size <= 256 &&
         (c.group_size & (c.group_size - 1)) == 0;
}

// minifloat codec on the TMA-fed streaming kernels: 16-bit inputs, g in {64, 128, 256}, whole
// tiles (the ragged-tail path of q_role_gpl is the integer lane codec), 16-B aligned buffers
static bool mf_stream_ok(const fc_codec& c, int dtype, int64_t n, const void* a, const void* b, bool quant) {
  return c.kind == FC_KIND_MINIFLOAT && (c.group_size == 64 || c.group_size == 128 || c.group_size == 256) &&
         dtype != FC_DTYPE_F32 && (!quant || n % kTileElems == 0) && (uintptr_t)a % 16 == 0 &&
         (uintptr_t)b % 16 == 0 && codec_qkernel() != 4;  // FC_CODEC_QKERNEL=4: lane-8 kernels (A/B)
}
template <typename T, class Spec>
static fc_status mf_quant_stream(const T* x, int64_t n, const DevCodec& dc, uint8_t* dst, uint32_t* err, cudaStream_t st) {
  FlashArgs a = codec_args(x, dst, n, dc, err);
  a.stages = 4;
  const int smem = a.stages * (kTileElems * 2 + 16);
  auto launch = [&](const void* k, auto kern) -> fc_status {
    FC_TRY(ensure_smem_attr(k, smem));
    kern<<<stream_grid_cur(k, kGplThreads, smem, a.tiles), kGplThreads, smem, st>>>(a);
    return FC_OK;
  };
  switch (dc.g) {
    case 64: return launch((const void*)k_qstream_gpl<T, Spec, 64>, k_qstream_gpl<T, Spec, 64>);
    case 256: return launch((const void*)k_qstream_gpl<T, Spec, 256>, k_qstream_gpl<T, Spec, 256>);
    default: return launch((const void*)k_qstream_gpl<T, Spec, 128>, k_qstream_gpl<T, Spec, 128>);
  }
}
template <class Spec>
static fc_status mf_quant_any(const void* x, int in_dtype, int64_t n, const DevCodec& dc, void* dst, uint32_t* err,
                              cudaStream_t st) {
  if (in_dtype == FC_DTYPE_F16) return mf_quant_stream<__half, Spec>((const __half*)x, n, dc, (uint8_t*)dst, err, st);
  return mf_quant_stream<__nv_bfloat16, Spec>((const __nv_bfloat16*)x, n, dc, (uint8_t*)dst, err, st);
}
template <class Spec>
static fc_status mf_dequant_any(const void* src, int64_t n, const DevCodec& dc, void* out, int out_dtype,
                                cudaStream_t st);

fc_status launch_quantize(const void* x, int in_dtype, int64_t n, const fc_codec& c, void* dst, uint32_t* err,
                          cudaStream_t st, bool allow_fast) {
  const fc_layout L = layout_of(c, n);
  const DevCodec dc = dev_codec(c, L);
  if (allow_fast && mf_stream_ok(c, in_dtype, n, x, dst, true)) {
    fc_status r = c.reserved == FC_FMT_E4M3 ? mf_quant_any<MfSpec<FC_FMT_E4M3>>(x, in_dtype, n, dc, dst, err, st)
                  : c.reserved == FC_FMT_E5M2 ? mf_quant_any<MfSpec<FC_FMT_E5M2>>(x, in_dtype, n, dc, dst, err, st)
                                               : mf_quant_any<MfSpec<FC_FMT_E2M1>>(x, in_dtype, n, dc, dst, err, st);
    FC_TRY(r);
    FC_CUDA_TRY(cudaGetLastError());
    return FC_OK;
  }
  if (allow_fast && l8_codec_ok(c)) return l8_codec_quantize(x, in_dtype, n, dc, dst, err, st);
  const bool aligned = ((uintptr_t)x % 16 == 0) && ((uintptr_t)dst % 16 == 0);
  if (allow_fast && fast_group(c) && aligned) {
    const int64_t tiles = (n + kTileElems - 1) / kTileElems;
    uint8_t* d = (uint8_t*)dst;
    const bool pass = c.kind == FC_KIND_FP16;
    const int spec = codec_spec(c);
    if (spec && in_dtype != FC_DTYPE_F32 && allow_fast) {
      if (in_dtype == FC_DTYPE_F16) {
        FC_TRY((spec == 1 ? quant_stream<__half, SpecA4>((const __half*)x, n, dc, d, err, st)
                         : quant_stream<__half, SpecA8>((const __half*)x, n, dc, d, err, st)));
      } else {
        FC_TRY((spec == 1 ? quant_stream<__nv_bfloat16, SpecA4>((const __nv_bfloat16*)x, n, dc, d, err, st)
                         : quant_stream<__nv_bfloat16, SpecA8>((const __nv_bfloat16*)x, n, dc, d, err, st)));
      }
      FC_CUDA_TRY(cudaGetLastError());
      return FC_OK;
    }
#define FC_QF(T)                                                                                  \
  do {                                                                                            \
    const void* k = pass ? (const void*)k_quant_fast<T, 16, GenSpec>                              \
                         : spec == 1 ? (const void*)k_quant_fast<T, 8, SpecA4>                    \
                         : spec == 2 ? (const void*)k_quant_fast<T, 8, SpecA8>                    \
                                     : (const void*)k_quant_fast<T, 8, GenSpec>;                  \
    const int S = sizeof(T) == 4 ? 3 : 4;                                                         \
    const int smem = S * kThreads * Chunk<T>::kBytes;                                             \
    FC_TRY(ensure_smem_attr(k, smem));                                                            \
    const unsigned g = resident_grid(k, smem, tiles, cur_sms());                                  \
    if (pass)                                                                                     \
      k_quant_fast<T, 16, GenSpec><<<g, kThreads, smem, st>>>((const T*)x, n, dc, d, err, S);    \
    else if (spec == 1)                                                                           \
      k_quant_fast<T, 8, SpecA4><<<g, kThreads, smem, st>>>((const T*)x, n, dc, d, err, S);      \
    else if (spec == 2)                                                                           \
      k_quant_fast<T, 8, SpecA8><<<g, kThreads, smem, st>>>((const T*)x, n, dc, d, err, S);      \
    else                                                                                          \
      k_quant_fast<T, 8, GenSpec><<<g, kThreads, smem, st>>>((const T*)x, n, dc, d, err, S);     \
  } while (0)
    switch (in_dtype) {
      case FC_DTYPE_F32: FC_QF(float); break;
      case FC_DTYPE_F16: FC_QF(__half); break;
      default: FC_QF(__nv_bfloat16); break;
    }
#undef FC_QF
  } else {
    uint8_t* d = (uint8_t*)dst;
    switch (in_dtype) {
      case FC_DTYPE_F32: quant_generic((const float*)x, n, dc, d, err, st); break;
      case FC_DTYPE_F16: quant_generic((const __half*)x, n, dc, d, err, st); break;
      default: quant_generic((const __nv_bfloat16*)x, n, dc, d, err, st); break;
    }
  }
  FC_CUDA_TRY(cudaGetLastError());
  return FC_OK;
}

template <class Spec>
static fc_status mf_dequant_any(const void* src, int64_t n, const DevCodec& dc, void* out, int out_dtype,
                                cudaStream_t st) {
  const uint8_t* s = (const uint8_t*)src;
  switch (out_dtype) {
    case FC_DTYPE_F32: return dequant_stream<float, Spec>(s, n, dc, (float*)out, st);
    case FC_DTYPE_F16: return dequant_stream<__half, Spec>(s, n, dc, (__half*)out, st);
    default: return dequant_stream<__nv_bfloat16, Spec>(s, n, dc, (__nv_bfloat16*)out, st);
  }
}

fc_status launch_dequantize(const void* src, int64_t n, const fc_codec& c, void* out, int out_dtype,
                            cudaStream_t st, bool allow_fast) {
  const fc_layout L = layout_of(c, n);
  const DevCodec dc = dev_codec(c, L);
  if (allow_fast && mf_stream_ok(c, FC_DTYPE_BF16, n, src, out, false)) {
    fc_status r = c.reserved == FC_FMT_E4M3 ? mf_dequant_any<MfSpec<FC_FMT_E4M3>>(src, n, dc, out, out_dtype, st)
                  : c.reserved == FC_FMT_E5M2 ? mf_dequant_any<MfSpec<FC_FMT_E5M2>>(src, n, dc, out, out_dtype, st)
                                               : mf_dequant_any<MfSpec<FC_FMT_E2M1>>(src, n, dc, out, out_dtype, st);
    FC_TRY(r);
    FC_CUDA_TRY(cudaGetLastError());
    return FC_OK;
  }
  if (allow_fast && l8_codec_ok(c)) return l8_codec_dequantize(src, n, dc, out, out_dtype, st);
  const uint8_t* s = (const uint8_t*)src;
  const bool aligned = ((uintptr_t)src % 16 == 0) && ((uintptr_t)out % 16 == 0);
  if (allow_fast && fast_group(c) && aligned) {
    const int64_t tiles = (n + kTileElems - 1) / kTileElems;
    const bool pass = c.kind == FC_KIND_FP16;
    const int spec = codec_spec(c);
    if (spec) {
      switch (out_dtype) {
        case FC_DTYPE_F32:
          FC_TRY((spec == 1 ? dequant_stream<float, SpecA4>(s, n, dc, (float*)out, st)
                           : dequant_stream<float, SpecA8>(s, n, dc, (float*)out, st)));
          break;
        case FC_DTYPE_F16:
          FC_TRY((spec == 1 ? dequant_stream<__half, SpecA4>(s, n, dc, (__half*)out, st)
                           : dequant_stream<__half, SpecA8>(s, n, dc, (__half*)out, st)));
          break;
        default:
          FC_TRY((spec == 1 ? dequant_stream<__nv_bfloat16, SpecA4>(s, n, dc, (__nv_bfloat16*)out, st)
                           : dequant_stream<__nv_bfloat16, SpecA8>(s, n, dc, (__nv_bfloat16*)out, st)));
      }
      FC_CUDA_TRY(cudaGetLastError());
      return FC_OK;
    }
    const int S = 4;
    const int smem = S * kThreads * code_chunk_bytes(dc);
#define FC_DF(T)                                                                                      \
  do {                                                                                                \
    const void* k = pass ? (const void*)k_dequant_fast<T, 16, GenSpec>                                \
                         : spec == 1 ? (const void*)k_dequant_fast<T, 8, SpecA4>                      \
                         : spec == 2 ? (const void*)k_dequant_fast<T, 8, SpecA8>                      \
                                     : (const void*)k_dequant_fast<T, 8, GenSpec>;                    \
    FC_TRY(ensure_smem_attr(k, smem));                                                                \
    const unsigned g = resident_grid(k, smem, tiles, cur_sms());                                      \
    if (pass)                                                                                         \
      k_dequant_fast<T, 16, GenSpec><<<g, kThreads, smem, st>>>(s, n, dc, (T*)out, S);               \
    else if (spec == 1)                                                                               \
      k_dequant_fast<T, 8, SpecA4><<<g, kThreads, smem, st>>>(s, n, dc, (T*)out, S);                 \
    else if (spec == 2)                                                                               \
      k_dequant_fast<T, 8, SpecA8><<<g, kThreads, smem, st>>>(s, n, dc, (T*)out, S);                 \
    else                                                                                              \
      k_dequant_fast<T, 8, GenSpec><<<g, kThreads, smem, st>>>(s, n, dc, (T*)out, S);                \
  } while (0)
    switch (out_dtype) {
      case FC_DTYPE_F32: FC_DF(float); break;
      case FC_DTYPE_F16: FC_DF(__half); break;
      default: FC_DF(__nv_bfloat16); break;
    }
#undef FC_DF
  } else {
    const unsigned grid = (unsigned)((n + 255) / 256);
    switch (out_dtype) {
      case FC_DTYPE_F32: k_gen_dequant<float><<<grid, 256, 0, st>>>(s, n, dc, (float*)out, 0); break;
      case FC_DTYPE_F16: k_gen_dequant<__half><<<grid, 256, 0, st>>>(s, n, dc, (__half*)out, 0); break;
      default: k_gen_dequant<__nv_bfloat16><<<grid, 256, 0, st>>>(s, n, dc, (__nv_bfloat16*)out, 0); break;
    }
  }
  FC_CUDA_TRY(cudaGetLastError());
  return FC_OK;
}

}  // namespace fc
