// Per-thread cp.async staging rings (LDGSTS on sm_100a).
//
// Every thread copies exactly the bytes it will consume into its own
// shared-memory region, S items ahead, and waits only on its own copy groups
// (cp.async.wait_group). No CTA barrier is needed and no register is held
// while the bytes are in flight, so each thread keeps S x (its chunk) of
// HBM traffic outstanding — the memory-level parallelism an HBM-bound
// kernel needs at the occupancy its register budget allows.
//
// Layouts are swizzled at 16-B granularity so that a warp reading one 16-B
// vector per lane from contiguous per-lane regions hits distinct banks.
#pragma once

#include "fc_common.cuh"

namespace fc {

__device__ __forceinline__ void cp_async16(uint32_t sdst, const void* gsrc, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sdst), "l"(gsrc), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t sdst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sdst), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// runtime depth (uniform), N in [0, 3]
__device__ __forceinline__ void cp_async_wait_dyn(int n) {
  if (n <= 0)
    cp_async_wait<0>();
  else if (n == 1)
    cp_async_wait<1>();
  else if (n == 2)
    cp_async_wait<2>();
  else
    cp_async_wait<3>();
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a) : "memory");
  return r;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t r;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(a) : "memory");
  return r;
}

// ---------------------------------------------------------------- input chunks

template <typename T>
struct Chunk {
  static constexpr int kBytes = kLaneElems * (int)sizeof(T);  // 64 (16-bit) or 128 (fp32)
  static constexpr int kVecs = kBytes / 16;
  static constexpr int kPer = 16 / (int)sizeof(T);            // elements per 16-B vector
  __device__ static __forceinline__ int slot(int q, int lane) {
    return q ^ (kVecs == 4 ? ((lane >> 1) & 3) : (lane & 7));
  }
};

// Async copy of elements [idx0, idx0+32) of `base` into this thread's region
// `sdst`. Elements at or past M arrive as 0 (zero-fill = the segment padding
// of collectives.py:145-149); vectors entirely past nvalid are not read.
template <typename T>
__device__ __forceinline__ void chunk_issue(uint32_t sdst, const T* base, int64_t idx0, int64_t M, int nvalid,
                                            int lane) {
  if (nvalid == kLaneElems && idx0 + kLaneElems <= M) {  // common case: whole chunk in range
#pragma unroll
    for (int q = 0; q < Chunk<T>::kVecs; ++q)
      cp_async16(sdst + 16 * Chunk<T>::slot(q, lane), base + idx0 + q * Chunk<T>::kPer, 16);
    return;
  }
#pragma unroll
  for (int q = 0; q < Chunk<T>::kVecs; ++q) {
    const int64_t i = idx0 + q * Chunk<T>::kPer;
    int n = 0;
    if (q * Chunk<T>::kPer < nvalid) n = (int)max((int64_t)0, min(M - i, (int64_t)Chunk<T>::kPer));
    cp_async16(sdst + 16 * Chunk<T>::slot(q, lane), n > 0 ? (const void*)(base + i) : (const void*)base,
               n * (int)sizeof(T));
  }
}

template <typename T>
__device__ __forceinline__ void chunk_read(uint32_t ssrc, int lane, float v[kLaneElems]) {
#pragma unroll
  for (int q = 0; q < Chunk<T>::kVecs; ++q) {
    const uint4 u = lds128(ssrc + 16 * Chunk<T>::slot(q, lane));
    if constexpr (sizeof(T) == 4) {
      v[4 * q + 0] = __uint_as_float(u.x);
      v[4 * q + 1] = __uint_as_float(u.y);
      v[4 * q + 2] = __uint_as_float(u.z);
      v[4 * q + 3] = __uint_as_float(u.w);
    } else {
      unpack2(u.x, v[8 * q + 0], v[8 * q + 1], (T*)nullptr);
      unpack2(u.y, v[8 * q + 2], v[8 * q + 3], (T*)nullptr);
      unpack2(u.z, v[8 * q + 4], v[8 * q + 5], (T*)nullptr);
      unpack2(u.w, v[8 * q + 6], v[8 * q + 7], (T*)nullptr);
    }
  }
}


// staged read into the lane's source representation
template <typename T>
__device__ __forceinline__ void chunk_read_src(uint32_t ssrc, int lane, LaneOf<T>& L) {
  if constexpr (sizeof(T) == 4) {
    chunk_read<T>(ssrc, lane, L.v);
  } else {
#pragma unroll
    for (int q = 0; q < Chunk<T>::kVecs; ++q) {
      const uint4 u = lds128(ssrc + 16 * Chunk<T>::slot(q, lane));
      L.w[4 * q] = u.x;
      L.w[4 * q + 1] = u.y;
      L.w[4 * q + 2] = u.z;
      L.w[4 * q + 3] = u.w;
    }
  }
}

// ---------------------------------------------------------------- code lanes

// Region of one quantized lane chunk: CW/4 vectors of codes (only c.sb/4 are
// copied), then the 4-B words holding the group's fp16 scale and zero byte.
__host__ __device__ inline int code_chunk_bytes(const DevCodec& c) { return 16 * (c.sb / 4) + 16; }

__device__ __forceinline__ void code_issue(const DevCodec& c, uint32_t sdst, const uint8_t* buf, int64_t p0) {
  const uint8_t* cp = buf + p0 * c.sb / 8;
  const int nq = c.sb / 4;
  for (int i = 0; i < nq; ++i) cp_async16(sdst + 16 * i, cp + 16 * i, 16);
  if (c.kind == FC_KIND_INT) {
    const int64_t grp = p0 >> c.gshift;
    cp_async4(sdst + 16 * nq, buf + c.scales_off + ((grp * 2) & ~(int64_t)3));
    if (!c.sym) cp_async4(sdst + 16 * nq + 4, buf + c.zeros_off + (grp & ~(int64_t)3));
  }
}

template <int CW>
__device__ __forceinline__ void code_read(const DevCodec& c, uint32_t ssrc, int64_t p0, LaneCodes<CW>& L) {
  const int nq = c.sb / 4;
#pragma unroll
  for (int i = 0; i < CW / 4; ++i) {
    if (i >= nq) break;
    const uint4 u = lds128(ssrc + 16 * i);
    L.w[4 * i] = u.x;
    L.w[4 * i + 1] = u.y;
    L.w[4 * i + 2] = u.z;
    L.w[4 * i + 3] = u.w;
  }
  if (c.kind == FC_KIND_INT) {
    const int64_t grp = p0 >> c.gshift;
    const uint32_t sw = lds32(ssrc + 16 * nq);
    L.s = __half2float(__ushort_as_half((unsigned short)((grp & 1) ? (sw >> 16) : (sw & 0xFFFFu))));
    float zf;
    if (c.sym) {
      zf = (float)(1 << (c.bits - 1));
    } else {
      const uint32_t zw = lds32(ssrc + 16 * nq + 4);
      zf = (float)((zw >> (8 * (grp & 3))) & 0xFFu);
    }
    L.mz = 8388608.0f + zf;
    const uint32_t xr = rep_xor(c);
#pragma unroll
    for (int i = 0; i < 8 && i < CW; ++i) L.w[i] ^= xr;
  } else {
    L.s = 1.0f;
    L.mz = 0.0f;
  }
}

}  // namespace fc
