// Communicator state shared by the C-ABI translation units.
#pragma once

#include <vector>

#include <cuda_runtime.h>

#include <string>

#include "fc_host.h"

namespace fc {
extern thread_local int64_t g_launch_count;  // kernels launched by the current call
fc_status fail(fc_status s, const char* fmt, ...);
int64_t group_of(const fc_codec& c);
}  // namespace fc

using fc::kMaxRanks;

struct fc_comm {
  int world = 0;
  bool ipc = false;
  int my_rank = 0;  // ipc
  int devices[kMaxRanks] = {0};
  int64_t slot_bytes = 0;
  int64_t flags_cap = 0;
  int64_t block_bytes = 0;
  uint8_t* blk[kMaxRanks] = {nullptr};
  bool owned[kMaxRanks] = {false};
  bool opened[kMaxRanks] = {false};
  float* scratch[kMaxRanks] = {nullptr};
  int64_t scratch_elems[kMaxRanks] = {0};
  cudaEvent_t ev[kMaxRanks] = {nullptr};
  uint32_t epoch = 0;
  // options
  int64_t fused = -1, ctas = 0, timeout_ms = 5000, lag = 0, fast = 1;  // fused: -1 auto
  int64_t stream_mask = 0;
  int64_t phases = 0;
  int64_t oneshot = 1;  // decode-sized rounds: the one-launch k_small (1: across GPUs/processes, 2: also one GPU)
  int64_t role_profile = 0;  // record the fused kernel's per-CTA role timeline
  uint64_t* tprof[kMaxRanks] = {nullptr};
  int32_t tprof_ctas[kMaxRanks] = {0};
  int64_t fused_gather_ctas = 0;  // fused stream kernel: gather-role CTAs per SM (0 = auto)
  int64_t fused_chunk = 0;  // fused stream kernel: tiles per schedule chunk (0 = auto)  // measurement: phase mask of the one-GPU split path (0 = all)
  int64_t reduce_stages = 0, q_stages = 0, d_stages = 0, ctas_per_sm = 0;  // 0 = auto
  int64_t launches = 0, last_launches = 0;  // kernels launched by the last call
  // segment-relative element span [span_lo, span_hi) the next run processes (-1: whole segment);
  // set only by the host-buffer pipeline around each of its chunk runs
  int64_t span_lo = 0, span_hi = -1;
  // host-buffer pipeline (fc_flash_all_reduce_host): device staging per rank, copy/compute
  // streams per device (owned by the device's first rank), events per (chunk, rank)
  int64_t host_chunk_bytes = 0;  // H2D bytes per rank per chunk (0 = auto)
  void* hs_in[kMaxRanks] = {nullptr};
  void* hs_out[kMaxRanks] = {nullptr};
  int64_t hs_in_bytes[kMaxRanks] = {0}, hs_out_bytes[kMaxRanks] = {0};
  cudaStream_t hs_h2d[kMaxRanks] = {nullptr}, hs_comp[kMaxRanks] = {nullptr}, hs_d2h[kMaxRanks] = {nullptr};
  std::vector<cudaEvent_t> hs_ev;  // [chunk][rank][in, out]
  // fused Hadamard rotation of the next runs (fc_comm_set_rotation; dim 0: none): block size,
  // normalize flag, per-rank device pointer to the dim seeded signs (or null)
  int32_t rot_dim = 0, rot_normalize = 1;
  const float* rot_signs[kMaxRanks] = {nullptr};
  // last call (debug export)
  fc_codec last_c1{}, last_c2{};
  int64_t last_R = 0, last_sub_len = 0;
};

namespace fc {
inline uint8_t* h_recv_slot(const fc_comm* c, int owner, int src) { return c->blk[owner] + (int64_t)src * c->slot_bytes; }
inline uint8_t* h_gath_slot(const fc_comm* c, int owner, int src) {
  return c->blk[owner] + (int64_t)(c->world + src) * c->slot_bytes;
}
// run_typed<Tin, Tout>: instantiated in fc_run_{f32,f16,bf16}.cu
template <typename Tin, typename Tout>
fc_status run_typed(fc_comm* c, const void* const* ins, void* const* outs, int64_t n, const fc_flash_cfg* cfg,
                    cudaStream_t* st, int only_rank);
template <typename Tin, typename Tout>
fc_status identity_typed(const void* in, void* out, int64_t n, int device, cudaStream_t st);
}  // namespace fc
