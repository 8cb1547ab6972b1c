/*
 * flashcomm.h — C ABI of the B200-native Flash All-Reduce (arXiv 2412.04964).
 *
 * Drop-in boundary for the hot path of the reference package `qcollectives`
 * (/root/reference/pkg/src/qcollectives). Plain pointers and sizes only; no
 * torch types. Every entry point cites the reference interface it replaces.
 *
 * Conventions
 *   - Device pointers are CUDA device addresses; `stream` is a cudaStream_t
 *     (0 = legacy default stream). Calls are asynchronous and stream-ordered
 *     unless stated otherwise.
 *   - Status codes map 1:1 onto the reference exception taxonomy
 *     (errors.py:4-22). On failure, fc_last_error() returns a message.
 *   - Device-side faults (non-finite input, a peer that never arrives) are
 *     latched in a device error word and surface at fc_comm_check() /
 *     fc_error_word_check(), as FC_ERR_DOMAIN / FC_ERR_PROTOCOL.
 */
#ifndef FLASHCOMM_H_
#define FLASHCOMM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define FC_API __attribute__((visibility("default")))
#else
#define FC_API
#endif

#define FC_MAX_RANKS 16
#define FC_IPC_HANDLE_BYTES 64

/* errors.py:4-22 */
typedef enum {
  FC_OK = 0,
  FC_ERR_CONFIG = 1,    /* ConfigError    (errors.py:12-13)  */
  FC_ERR_DOMAIN = 2,    /* DomainError    (errors.py:8-9)    */
  FC_ERR_INTEGRITY = 3, /* IntegrityError (errors.py:16-17)  */
  FC_ERR_PROTOCOL = 4,  /* ProtocolError  (errors.py:20-22)  */
  FC_ERR_CUDA = 5       /* CUDA runtime failure (no reference analogue) */
} fc_status;

typedef enum { FC_DTYPE_F32 = 0, FC_DTYPE_F16 = 1, FC_DTYPE_BF16 = 2 } fc_dtype;
typedef enum { FC_KIND_INT = 0, FC_KIND_FP16 = 1, FC_KIND_MINIFLOAT = 2 } fc_codec_kind;
/* minifloat formats (minifloat.py:40-45), in fc_codec.reserved for FC_KIND_MINIFLOAT */
typedef enum { FC_FMT_E4M3 = 0, FC_FMT_E5M2 = 1, FC_FMT_E2M1 = 2 } fc_minifloat_format;
typedef enum { FC_ROUND_NEAREST_EVEN = 0, FC_ROUND_CEIL = 1 } fc_rounding;

/* CodecConfig (codec.py:45-73): integer codes (bits 2..8, group-wise
 * asym/sym, nearest-even/ceil), group-scaled minifloat codes (e4m3 / e5m2 /
 * e2m1: kind FC_KIND_MINIFLOAT, reserved = fc_minifloat_format, bits = code
 * bits; codec.py:332-351) or the fp16 passthrough (codec.py:162). */
typedef struct {
  int32_t kind;      /* fc_codec_kind */
  int32_t bits;      /* 2..8 for FC_KIND_INT */
  int32_t group_size;/* >= 1 */
  int32_t symmetric; /* 0/1 */
  int32_t rounding;  /* fc_rounding */
  int32_t reserved;
  double scale_floor;/* > 0, default 1e-8 */
} fc_codec;

/* FlashConfig (collectives.py:37-75). chunk_elems <= 0 means "None"
 * (default near 64 Ki elements); results never depend on it
 * (collectives.py:14-16), it is validated exactly like the reference. */
typedef struct {
  fc_codec stage1;
  fc_codec stage2;
  int64_t chunk_elems;
} fc_flash_cfg;

/* Device layout of one quantized tensor: codes at byte 0 (canonical
 * little-nibble-first packing, bitpack.py:48-62), fp16 scales at
 * scales_offset, uint8 zeros at zeros_offset (asym int only). Regions are
 * 16-byte aligned; `wire_bytes` is the reference's serialized size
 * (codec.py:128-133, codes||scales||zeros without padding). */
typedef struct {
  int64_t elements;
  int64_t groups;
  int64_t codes_bytes;
  int64_t scales_offset;
  int64_t zeros_offset;
  int64_t total_bytes;
  int64_t wire_bytes;
} fc_layout;

FC_API const char* fc_version(void);
FC_API const char* fc_last_error(void);

/* CodecConfig.__post_init__ validation (codec.py:61-73) + wire_byte_len. */
FC_API fc_status fc_codec_validate(const fc_codec* codec);
FC_API fc_status fc_codec_layout(const fc_codec* codec, int64_t n, fc_layout* out);
/* FlashConfig.resolve_chunk_size (collectives.py:65-75). */
FC_API fc_status fc_flash_resolve_chunk(const fc_flash_cfg* cfg, int32_t world, int64_t* chunk_out);

/* quantize(x, config) (codec.py:292-329) on one GPU. x: n elements of
 * `in_dtype`; dst: fc_codec_layout(codec, n).total_bytes bytes.
 * err_word (device, may be NULL): set non-zero if x holds NaN/inf
 * (codec.py:230-231 DomainError), checked by fc_error_word_check. */
FC_API fc_status fc_quantize(const void* x, int32_t in_dtype, int64_t n, const fc_codec* codec, void* dst,
                      uint32_t* err_word, void* stream);
/* dequantize(q) (codec.py:354-384): src laid out as fc_codec_layout. */
FC_API fc_status fc_dequantize(const void* src, int64_t n, const fc_codec* codec, void* out, int32_t out_dtype,
                        void* stream);
/* Synchronizes `stream` and maps a device error word to a status. */
FC_API fc_status fc_error_word_check(const uint32_t* err_word, void* stream);

/* Blocked Hadamard rotation (rotation.py:61-83): per block of `dim` (power of
 * two <= 8192) elements of the zero-padded length-n_padded vector x (n valid
 * elements), forward H(D x) or inverse D(H x), scaled by 1/sqrt(dim)
 * (normalize) or, for the inverse without normalize, 1/dim; float64
 * arithmetic, one rounding to out_dtype; the first n_out elements are
 * written. signs: NULL or `dim` device floats of +-1 (the seeded diagonal). */
FC_API fc_status fc_hadamard(const void* x, int32_t in_dtype, int64_t n, int64_t n_padded, int32_t dim,
                             int32_t normalize, const float* signs, int32_t inverse, void* out, int32_t out_dtype,
                             int64_t n_out, void* stream);

/* ---- communicator: replaces the simulated fabric (fabric.py:111-246) ----
 * Every rank owns one device block: N stage-1 receive slots, N stage-2
 * gather slots, per-tile arrival flags and an error word. Peers write into
 * it over NVLink (P2P / CUDA IPC mapping). */
typedef struct fc_comm fc_comm;

/* One process drives all `world` ranks (the reference's list-of-tensors
 * call, collectives.py:321). devices[r] is rank r's GPU; several ranks may
 * share one GPU. slot_bytes: capacity of one slot (larger calls run in
 * rounds; results do not change, collectives.py:14-16). */
FC_API fc_status fc_comm_create_local(int32_t world, const int32_t* devices, int64_t slot_bytes, fc_comm** out);
/* One process per rank (torch.distributed launch): allocate this rank's
 * block, export its IPC handle, open every peer's. */
FC_API fc_status fc_comm_create_ipc(int32_t world, int32_t rank, int32_t device, int64_t slot_bytes, fc_comm** out);
FC_API fc_status fc_comm_ipc_handle(fc_comm* comm, void* handle_out /* FC_IPC_HANDLE_BYTES */);
FC_API fc_status fc_comm_ipc_open(fc_comm* comm, const void* handles /* world * FC_IPC_HANDLE_BYTES */);
FC_API fc_status fc_comm_destroy(fc_comm* comm);

typedef enum {
  FC_OPT_FUSED = 0,        /* -1 (default): the fused kernel (one cooperative launch per rank, per-tile
                              flags, k_fstream) whenever ranks live on different GPUs or processes and the
                              round is eligible (g = 128, one storage width, 16-bit in/out, whole tiles),
                              else the phase-split streaming kernels (flag barriers between phases
                              across GPUs); 1: the fused kernel wherever eligible (also all ranks on one
                              GPU); 0: phase-split */
  FC_OPT_CTAS = 1,         /* CTA cap per rank of the fused kernels (0 = auto) */
  FC_OPT_TIMEOUT_MS = 2,   /* flag-wait timeout -> ProtocolError (fabric.py:158-178); default 5000 */
  FC_OPT_LAG = 3,          /* fused schedule: tiles between a tile's scatter and its reduce (0 = auto) */
  FC_OPT_FAST = 4,         /* 0: force the generic (any group size) kernels; for testing */
  FC_OPT_LAST_LAUNCHES = 5,/* read-only: kernels launched by the last all-reduce call */
  FC_OPT_REDUCE_STAGES = 6,/* ring depth of the phase-split reduce kernel (0 = auto) */
  FC_OPT_SCATTER_STAGES = 7,/* ring depth of the streaming scatter / quantize kernel (0 = auto) */
  FC_OPT_GATHER_STAGES = 8, /* ring depth of the streaming gather / dequantize kernel (0 = auto) */
  FC_OPT_CTAS_PER_SM = 9,   /* cap on resident CTAs per SM of the streaming kernels (0 = occupancy) */
  FC_OPT_STREAM_MASK = 10,  /* A/B testing: bit 0/1/2 runs scatter/reduce/gather on the cp.async-staged kernels; bit 4: INT8 g=128 scatter on the group-per-lane kernel; bit 5: its code stores direct (not staged); bits 6/7: g=128 scatter/reduce on the 32-element lane layout; bit 10: minifloat flash rounds on the lane-8 kernels instead of the streaming ones; bit 11: small-message kernel as a plain launch; bit 12: group-lane reduce consumers in lockstep; bit 13: phase kernels as plain launches (no programmatic dependent launch, A/B); measurement only (results invalid): bit 8 skips the fused kernel's flag waits, bit 9 its flag publications */
  FC_OPT_PHASES = 11,       /* measurement only: run just these phases (bit 0/1/2) of a one-GPU split call */
  FC_OPT_FUSED_CHUNK = 12,  /* fused kernel schedule: tiles per chunk (step s scatters chunk s, reduces s-1,
                               gathers s-2); 0 = auto: the whole round on one GPU, a quarter across GPUs */
  FC_OPT_ONESHOT = 13,      /* decode-sized rounds (<= 8 tiles per segment) as ONE flag-synchronised launch per rank
                               (k_small) across GPUs / processes: 1 (default), 0 off, 2 also on one GPU */
  FC_OPT_HOST_CHUNK_BYTES = 14, /* fc_flash_all_reduce_host: H2D bytes per rank per pipeline chunk (0 = auto) */
  FC_OPT_FUSED_GATHER_CTAS = 15, /* fused kernel: gather-role CTAs per SM (0 = auto) */
  FC_OPT_ROLE_PROFILE = 16  /* measurement: record the fused kernel's per-CTA role timeline (fc_comm_role_profile) */
} fc_option;
FC_API fc_status fc_comm_set_option(fc_comm* comm, int32_t option, int64_t value);
FC_API fc_status fc_comm_get_option(fc_comm* comm, int32_t option, int64_t* value);

/* flash_all_reduce (collectives.py:321-402), one-process form: ins[r]/outs[r]
 * are rank r's device buffers of n elements; streams[r] (may be NULL ->
 * default stream) orders rank r's work. in may alias out. */
FC_API fc_status fc_flash_all_reduce_local(fc_comm* comm, const void* const* ins, void* const* outs, int64_t n,
                                    int32_t in_dtype, int32_t out_dtype, const fc_flash_cfg* cfg,
                                    void* const* streams);
/* flash_all_reduce on HOST buffers (the reference's call shape: arrays in,
 * new arrays out, blocking; collectives.py:321-402) for a local communicator.
 * host_ins[r] / host_outs[r] are rank r's host buffers of n elements;
 * host_outs[r] may be NULL (rank r's result is not read back). The comm's
 * device staging is filled chunk by chunk: the H2D copy of chunk k+1, the
 * flash all-reduce of chunk k (groups keep their segment anchors, so results
 * equal one whole-tensor call bit for bit) and the D2H copy of chunk k-1 run
 * concurrently on per-device copy/compute streams. Pinned host memory
 * (cudaHostAlloc / cudaHostRegister) gives full PCIe bandwidth; pageable
 * memory works at the driver's staged-copy speed. Device faults are returned
 * like fc_comm_check. */
FC_API fc_status fc_flash_all_reduce_host(fc_comm* comm, const void* const* host_ins, void* const* host_outs, int64_t n,
                                          int32_t in_dtype, int32_t out_dtype, const fc_flash_cfg* cfg);
/* fc_flash_all_reduce_host, per-rank form (IPC world): this rank's host
 * buffers; every rank calls it with the same n / cfg / FC_OPT_HOST_CHUNK_BYTES
 * (the chunk sequence must match across ranks). host_out may be NULL. */
FC_API fc_status fc_flash_all_reduce_host_rank(fc_comm* comm, const void* host_in, void* host_out, int64_t n,
                                               int32_t in_dtype, int32_t out_dtype, const fc_flash_cfg* cfg);
/* flash_all_reduce, per-rank form (IPC world): every rank calls it with the
 * same n/cfg in the same order. in may alias out; both 16-byte aligned
 * (FC_ERR_DOMAIN otherwise: the kernel path, which every rank must share,
 * depends on it). */
FC_API fc_status fc_flash_all_reduce(fc_comm* comm, const void* in, void* out, int64_t n, int32_t in_dtype,
                              int32_t out_dtype, const fc_flash_cfg* cfg, void* stream);

/* ---- fused rotation (FlashConfig.rotation, collectives.py:350-351 / 390-391) ----
 * Sets the blocked Hadamard rotation (rotation.py:38-83) the next flash runs of
 * `comm` fuse into the scatter / reduce prologue (H(D x)) and the reduce /
 * gather epilogue (D(H y)): dim (power of two, 8..256; 0 clears), normalize,
 * signs = `dim` device floats of +-1 on the rank's device or NULL; rank -1 sets
 * every rank of a local communicator. fc_flash_rotation_fusable tells whether
 * a run of n elements per rank with `cfg` can fuse a rotation of `dim` (the
 * round and segment sizes must be multiples of dim, group sizes 8..256); runs
 * that cannot fail with FC_ERR_CONFIG while a rotation is set. */
FC_API fc_status fc_comm_set_rotation(fc_comm* comm, int32_t rank, int32_t dim, int32_t normalize,
                                      const float* signs);
FC_API int32_t fc_flash_rotation_fusable(fc_comm* comm, int64_t n, const fc_flash_cfg* cfg, int32_t dim);

/* Synchronize rank's device work and map its error word: a timed-out wait
 * -> FC_ERR_PROTOCOL "deadlock: rank r timed out waiting on rank p"
 * (fabric.py:171-175); non-finite input -> FC_ERR_DOMAIN (codec.py:230). */
FC_API fc_status fc_comm_check(fc_comm* comm, int32_t rank);
/* Teardown check of an IPC communicator (fabric.py:228-236): every rank has
 * completed the same number of rounds (device epoch counters, read over the
 * peer mappings); a rank that ran a round its peers never joined left
 * messages nobody consumed -> FC_ERR_PROTOCOL naming the ranks. Synchronises
 * the device; call after the ranks' last collective (e.g. behind a barrier). */
FC_API fc_status fc_comm_teardown_check(fc_comm* comm);

/* Debug/parity: layout of rank's stage-1 receive slot `src` (stage 1) or
 * stage-2 gather slot `src` (stage 2) as written by the last round of the
 * last call; if dst (device memory, layout->total_bytes) is not NULL the
 * slot is copied there (synchronous). Stage-1 slot [rank] (the rank's own
 * piece) is written only by the kernels that read it back (the group-lane
 * reduce and the fused kernel); the others keep the own piece in registers. */
FC_API fc_status fc_comm_slot(fc_comm* comm, int32_t rank, int32_t stage, int32_t src, void* dst,
                              fc_layout* layout);
/* Topology discovery: peer-access matrix (world*world ints) and NVLink
 * multicast support of rank's device. */
FC_API fc_status fc_comm_topology(fc_comm* comm, int32_t* can_access, int32_t* multicast);
/* Measurement: per-CTA role timeline of rank's last fused-kernel launch
 * (FC_OPT_ROLE_PROFILE = 1 first): FC_ROLE_PROFILE_U64 %globaltimer values
 * per CTA — first start / last end / busy ns of the scatter, reduce and
 * gather roles, kernel start, kernel end. Copies up to max_ctas CTAs into
 * host memory and stores the launch's CTA count (synchronous). */
#define FC_ROLE_PROFILE_U64 16
FC_API fc_status fc_comm_role_profile(fc_comm* comm, int32_t rank, uint64_t* host_dst, int32_t max_ctas,
                                      int32_t* ctas);

#ifdef __cplusplus
}
#endif
#endif /* FLASHCOMM_H_ */
