/*
 * fdmoe.h — C ABI of the B200-native FlashDMoE operator (libfdmoe.so).
 *
 * Drop-in boundary for the reference's operator API
 *   moefabric::forward(const MoeConfig&, const std::vector<TokenMatrix>& shards,
 *                      const ModelWeights&, const ForwardOptions&) -> ForwardResult
 *   (/root/reference/proj/include/moefabric/runtime.hpp:802-1002).
 * include/moefabric_b200.hpp restates that C++ API on top of these entry points; the
 * Python host mirror (paper_2506_04667_b200/) binds them with ctypes.
 *
 * Plain pointers and sizes only: no torch or CUDA runtime types in the signatures
 * (streams are passed as void*). Every entry point returns an fdmoe_status; the message
 * of the last failure on the calling thread is available from fdmoe_last_error().
 *
 * Status codes map 1:1 to the reference's exception types (config.hpp:16-30):
 *   FDMOE_ERR_CONFIG   <-> ConfigError   (shape / configuration errors)
 *   FDMOE_ERR_PROTOCOL <-> ProtocolError (invalid one-sided write, double signal)
 *   FDMOE_ERR_RUNTIME  <-> RuntimeFault  (device watchdog expired, accounting mismatch)
 *   FDMOE_ERR_CUDA     -- CUDA runtime/driver failure (no reference equivalent)
 *   FDMOE_ERR_UNSUPPORTED -- valid for the reference but outside this operator's envelope
 *
 * A handle owns one or more "ranks" (the reference's simulated devices, config.hpp:54-75).
 * Ranks may live on distinct GPUs of this process, on one GPU ("virtual ranks": CTAs of a
 * single persistent launch are partitioned by rank; the exchange protocol is unchanged),
 * or in other processes (one rank per process; peers attached with fdmoe_import_peers).
 * A handle is not re-entrant: one in-flight forward per handle.
 */
#ifndef FDMOE_H
#define FDMOE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FDMOE_ABI_VERSION 3

typedef enum fdmoe_status {
    FDMOE_OK = 0,
    FDMOE_ERR_CONFIG = 1,
    FDMOE_ERR_PROTOCOL = 2,
    FDMOE_ERR_RUNTIME = 3,
    FDMOE_ERR_CUDA = 4,
    FDMOE_ERR_UNSUPPORTED = 5
} fdmoe_status;

/* config.hpp:32 Activation */
typedef enum fdmoe_activation { FDMOE_RELU = 0, FDMOE_GELU = 1, FDMOE_IDENTITY = 2 } fdmoe_activation;

/* Arithmetic of the expert FFN. The gate/routing is FP32-exact in both modes. */
typedef enum fdmoe_precision {
    FDMOE_FP32 = 0, /* FP32-accurate: 3xTF32 split on tcgen05 (hi*hi + hi*lo + lo*hi) */
    FDMOE_BF16 = 1  /* bf16 operands, FP32 accumulation */
} fdmoe_precision;

typedef enum fdmoe_where { FDMOE_HOST = 0, FDMOE_DEVICE = 1 } fdmoe_where;

/* MoeConfig (config.hpp:53-87), field for field, plus the GPU precision mode. */
typedef struct fdmoe_config {
    int64_t tokens_per_device; /* S */
    int64_t embed_dim;         /* H */
    int64_t ffn_dim;           /* D */
    int64_t experts_total;     /* E_total */
    int64_t devices;           /* P */
    int64_t topk;              /* k */
    double capacity_factor;    /* cf */
    int64_t tile_rows;         /* bM (reference tile; sizes the padded capacity C' only) */
    int64_t tile_cols;         /* bN (reference tile; accounting only) */
    int32_t activation;        /* fdmoe_activation */
    int32_t precision;         /* fdmoe_precision */
    uint64_t seed;
} fdmoe_config;

/* StragglerSpec::Kind (runtime.hpp:78-84) */
typedef enum fdmoe_straggler_kind {
    FDMOE_STRAGGLER_NONE = 0,
    FDMOE_STRAGGLER_CONSTANT = 1,  /* a = delay ms per packet */
    FDMOE_STRAGGLER_UNIFORM = 2,   /* U(a, b) ms per packet */
    FDMOE_STRAGGLER_LOGNORMAL = 3  /* lognormal(log a, b) ms per packet */
} fdmoe_straggler_kind;

/* ForwardOptions (runtime.hpp:86-92). `processors` is accepted for source compatibility; on the
 * GPU the persistent launch uses every co-resident CTA. */
typedef struct fdmoe_options {
    int32_t processors;         /* reference processor threads per device (ignored) */
    int32_t sequential;         /* ScheduleMode::sequential: bulk-synchronous baseline inside the
                                 * same launch — gate+dispatch | group barrier | expert FFN |
                                 * group barrier | combine (runtime.hpp:885-908) */
    int64_t deadlock_budget_ms; /* in-kernel watchdog budget (runtime.hpp:90, default 5000) */
    int32_t exact_gate;         /* 1: reference-exact gate logits for every token (G_phi and
                                 * combine weights bit-identical to the reference); 0 (default):
                                 * certified gate — FFMA logits, routing (assignment, slots, drops)
                                 * proven identical per token, exact recompute where unproven */
    int32_t trace_events;       /* 1: record the device event log (fdmoe_read_events) */
    /* StragglerSpec (runtime.hpp:78-84): rank `straggler_device` holds back each of its dispatch
     * packet signals by a delay sampled per packet, in the reference's order and RNG stream
     * (runtime.hpp:312-326, 341-362); delays accumulate as the reference's sleeps do. */
    int32_t straggler_kind;     /* fdmoe_straggler_kind */
    int32_t straggler_device;
    double straggler_a;
    double straggler_b;
    uint64_t seed;              /* ForwardOptions::seed (straggler sampling) */
} fdmoe_options;

/* Per-rank routing surface (GateOutput, gate.hpp:24-37). All host pointers, nullable.
 * g_phi: S x E; table_token / table_weight: E x C (token -1 = empty slot);
 * slot_counts: E; dropped: 2 * S * k int64 (token, expert) pairs in the reference's
 * emission order (ascending token, pick order); n_dropped: 1.
 * picks_expert / picks_slot / picks_weight: S x k (slot -1 = capacity-dropped). */
typedef struct fdmoe_routing {
    float* g_phi;
    int64_t* table_token;
    float* table_weight;
    int64_t* slot_counts;
    int64_t* dropped;
    int64_t* n_dropped;
    int32_t* picks_expert;
    int32_t* picks_slot;
    float* picks_weight;
} fdmoe_routing;

/* TaskStats (runtime.hpp:94-106) with GPU meaning, per local rank:
 * gemm0/gemm1 = 128-row FFN tiles executed (counted by the signal warps), combine = combine tasks,
 * launches = kernel launches this forward (1).
 * Task accounting (runtime.hpp:122-165, 407-415 on the kernel's static tile grid):
 *   bound_initial   = El * MT * (NB0 + NB1) FFN tasks (+ ceil(S/16) combine tasks when the combine is a
 *                     separate phase) -- the initial_task_bound analogue;
 *   bound_final     = bound_initial self-corrected on the device: each row tile whose dispatch signals
 *                     resolve to zero rows removes its NB0 + NB1 tasks (self_correct_task_bound);
 *   scheduled_final = non-empty FFN tasks the device producers scheduled (+ combine tasks);
 *   enqueued        = scheduled_final; tiles_resolved = row tiles whose signals were resolved.
 * A correct forward has bound_final == scheduled_final == executed (the reference terminates on
 * scheduled == bound, runtime.hpp:633-647). */
typedef struct fdmoe_stats {
    int64_t gemm0, gemm1, combine, enqueued, executed;
    int64_t bound_initial, bound_final, scheduled_final, launches;
    double kernel_ms;     /* device time of the layer launch on this rank (CUDA events) */
    int64_t gate_exact_tokens; /* tokens whose logits were recomputed exactly for all experts
                                * (all S with exact_gate; ties / near-ties otherwise) */
    int64_t gate_pair_tokens;  /* tokens the certified gate decided from exact candidate logits */
    int64_t tiles_resolved;    /* row tiles whose dispatch signals the device producers resolved */
} fdmoe_stats;

typedef struct fdmoe_handle fdmoe_handle;

/* ---- pure functions (no GPU needed) --------------------------------------- */
int32_t fdmoe_abi_version(void);
const char* fdmoe_last_error(void);
/* MoeConfig::validate (config.hpp:68-86) plus this operator's envelope checks when
 * gpu_envelope != 0 (returns FDMOE_ERR_UNSUPPORTED with a message). */
fdmoe_status fdmoe_config_validate(const fdmoe_config* cfg, int32_t gpu_envelope);
int64_t fdmoe_expert_capacity(const fdmoe_config* cfg);               /* config.hpp:94 */
int64_t fdmoe_padded_capacity(int64_t capacity, int64_t tile_rows);   /* config.hpp:104 */
uint64_t fdmoe_size_L(const fdmoe_config* cfg);                       /* layout.hpp:106 */
/* layout.hpp:67-79: element offset of slot row (p*, round, buffer, expert, slot) in the
 * reference layout L (P x 2 x 2 x E_local x C' x H); -1 when out of bounds. */
int64_t fdmoe_flat_index(int64_t devices, int64_t local_experts, int64_t slot_capacity,
                         int64_t embed_dim, int64_t p_star, int64_t round, int64_t buffer,
                         int64_t expert, int64_t slot);
/* layout.hpp:91-100: 0 ok, 1 = rule 1 violated, 2 = rule 2 violated. */
int32_t fdmoe_validate_write(int64_t src, int64_t dst, int64_t p_star, int64_t buffer);
/* runtime.hpp:122-165 task-count arithmetic (reference tile grid bM x bN). */
int64_t fdmoe_gemm_tasks_for_rows(const fdmoe_config* cfg, int64_t rows);
int64_t fdmoe_combine_tiles_for_rows(const fdmoe_config* cfg, int64_t rows);
int64_t fdmoe_initial_task_bound(const fdmoe_config* cfg);

/* StragglerSpec sampling (runtime.hpp:312-326, 341-362): cum_ns[devices * local_experts] = running
 * sum of the per-packet delays the straggler device would sleep, in the reference's packet order and
 * RNG stream; packet e's dispatch signal is held back by cum_ns[e] after dispatch starts. */
fdmoe_status fdmoe_straggler_delays(const fdmoe_options* opts, int64_t devices, int64_t local_experts,
                                    uint64_t* cum_ns);

/* Seeded synthetic model / shards, restating harness.hpp:76-109 bit for bit
 * (std::mt19937_64 + std::normal_distribution<float>). Layouts: wg H x E; w1 E x H x D;
 * b1 E x D; w2 E x D x H; b2 E x H; shards P x S x H. */
fdmoe_status fdmoe_synth_model(const fdmoe_config* cfg, uint64_t seed, float* wg, float* w1,
                               float* b1, float* w2, float* b2);
fdmoe_status fdmoe_synth_shards(const fdmoe_config* cfg, uint64_t seed, float* shards);

/* ---- operator --------------------------------------------------------------- */
/* Create the ranks [first_rank, first_rank + n_local) of a cfg->devices-rank group.
 * device_ids[i] is the CUDA device of local rank i (repeats allowed: virtual ranks).
 * Allocates each rank's symmetric heap and scratch, one launch group per device. */
fdmoe_status fdmoe_create(const fdmoe_config* cfg, const int32_t* device_ids, int32_t n_local,
                          int32_t first_rank, fdmoe_handle** out);
fdmoe_status fdmoe_destroy(fdmoe_handle* h);

/* Multi-process attach: export this handle's (single) rank heap as an opaque blob of
 * fdmoe_ipc_size() bytes; import all ranks' blobs (rank-major, world x size). */
size_t fdmoe_ipc_size(void);
fdmoe_status fdmoe_export_heap(fdmoe_handle* h, void* blob);
fdmoe_status fdmoe_import_peers(fdmoe_handle* h, const void* blobs, int32_t world);

/* ModelWeights (config.hpp:130-147) for all E_total experts; each local rank uploads
 * its own E_local experts (device p owns [p*E_local, (p+1)*E_local), config.hpp:66) and
 * repacks them K-major once (FP32, split into tf32 hi/lo on chip per tile; or bf16).
 * Also precomputes |Wg[:, e]| and Wg^T for the certified gate. Layouts as fdmoe_synth_model. */
fdmoe_status fdmoe_set_weights(fdmoe_handle* h, const float* wg, const float* w1, const float* b1,
                               const float* w2, const float* b2, int32_t where);

/* One MoE-layer forward: exactly one persistent kernel launch per device.
 * in_shards / out_shards: n_local pointers to S x H FP32 (host or device per `where`).
 * routing / stats: arrays of n_local entries, nullable. Synchronous.
 * Aliasing: an output shard must not overlap its input shard (FDMOE_ERR_CONFIG) -- the kernel still
 * reads input rows (dispatch) while the fused combine zeroes and accumulates output rows.
 * Numerics: the fused FP32 combine (k <= 2) adds fl(w*y) terms with float RED atomics, which flush
 * subnormal results to zero; outputs equal the reference's pick-order sum except where that sum (or a
 * term) is subnormal (|x| < 2^-126), where the device returns 0.
 * Ordering: launches of one handle are serialised across streams (a launch on a different stream than
 * the previous one waits for it). */
fdmoe_status fdmoe_forward(fdmoe_handle* h, const float* const* in_shards, float* const* out_shards,
                           int32_t where, const fdmoe_options* opts, fdmoe_routing* routing,
                           fdmoe_stats* stats);
/* Asynchronous device-pointer variant: enqueue on streams[i] (cudaStream_t as void*,
 * one per local rank; NULL = the handle's own stream). Pair with fdmoe_sync. */
fdmoe_status fdmoe_forward_async(fdmoe_handle* h, const float* const* in_dev, float* const* out_dev,
                                 void* const* streams, const fdmoe_options* opts);
/* Serving loop over n_batches host batches (in_batches / out_batches: n_batches * n_local host
 * pointers, batch-major; pinned memory for overlap). Batch b's host->device copy, layer launch and
 * device->host copy run on three streams with double-buffered device shards, so the PCIe copies of
 * neighbouring batches overlap the launch of batch b. One kernel launch per device per batch;
 * synchronous (returns when every output has landed). */
fdmoe_status fdmoe_forward_stream(fdmoe_handle* h, int32_t n_batches, const float* const* in_batches,
                                  float* const* out_batches, const fdmoe_options* opts);
/* Wait for the last forward, check the device watchdog/error word. */
fdmoe_status fdmoe_sync(fdmoe_handle* h);

/* Introspection for tests/bench. */
typedef struct fdmoe_info {
    int64_t capacity;       /* C */
    int64_t packet_rows;    /* rows reserved per (source, expert) packet in the receive buffer */
    int64_t heap_bytes;     /* symmetric heap per rank */
    int64_t scratch_bytes;  /* private device scratch per rank */
    int64_t weight_bytes;   /* resident expert weights per rank */
    int32_t ctas_per_rank;
    int32_t smem_bytes;
    int32_t num_sms;
    int32_t ranks_per_launch;
    int32_t fused_combine;  /* 1: overlapped launches fold the combine into the GEMM1 epilogues (k <= 2, every
                             * rank of the group on one device; both precisions); sequential launches never do */
} fdmoe_info;
fdmoe_status fdmoe_get_info(fdmoe_handle* h, fdmoe_info* info);
/* Device time of the most recent forward's launch (CUDA events on the launching stream;
 * max over this handle's devices). Call after fdmoe_sync / fdmoe_forward. */
fdmoe_status fdmoe_last_kernel_ms(fdmoe_handle* h, double* ms);
/* Device trace of the most recent launch (the reference's TraceBuffer role, trace.hpp:17-118, at
 * phase granularity): per CTA of local rank `local_rank`, 28 u64 = %globaltimer ns at kernel start,
 * gate done, grid barrier passed, dispatch done, FFN tiles done, combine done, exit; the number of
 * FFN tiles that CTA executed; then SM cycles blocked per FFN pipeline edge: MMA<-tokens,
 * MMA<-weights, MMA<-accumulator, converter<-weight TMA, converter<-TMEM stage, producer<-weight
 * slot, producer<-token slot, epilogue<-accumulator, MMA<-task ring; producer cycles fetching and
 * resolving tiles; epilogue busy cycles; FFN tiles issued by the MMA warp.
 * Writes min(cap/20, ctas) rows, then clears. */
fdmoe_status fdmoe_read_trace(fdmoe_handle* h, int32_t local_rank, uint64_t* out, int32_t cap, int32_t* n_ctas);
/* Device event log of the most recent launch with opts->trace_events (the reference's TraceEvent
 * stream, trace.hpp:17-60, recorded by the kernel with %globaltimer ns). One record per event: */
typedef enum fdmoe_event_kind {
    FDMOE_EV_SPAWN = 0,          /* per CTA: t0 = kernel start, t1 = exit */
    FDMOE_EV_GATE_DONE = 1,      /* per CTA: t0 = start, t1 = its gate tokens routed */
    FDMOE_EV_DISPATCH_PUT = 2,   /* packet signal published: src = this rank, peer = owner,
                                  * expert = owner-local expert, value = rows (pgas put) */
    FDMOE_EV_EXEC = 3,           /* task executed [t0, t1]: type 1 gemm0 / 2 gemm1 (expert, rb = row
                                  * tile, cb = feature block, src = first source packet, peer =
                                  * packets in the tile, value = rows) or 3 combine (rb = token block) */
    FDMOE_EV_TILE_PUT = 4,       /* GEMM1 tile stored into origin `peer`'s combine buffer and
                                  * signalled: expert, rb = row tile, cb, value = rows */
    FDMOE_EV_BARRIER_ENTER = 5,  /* sequential mode group barrier (value = barrier id) */
    FDMOE_EV_BARRIER_EXIT = 6
} fdmoe_event_kind;
typedef struct fdmoe_event {
    uint64_t t0, t1;
    int32_t kind, cta, type, src, expert, rb, cb, peer;
    int64_t value;
} fdmoe_event;
/* Copies up to `cap` records of local rank `local_rank`; *n = events recorded (may exceed cap or
 * the device buffer; *dropped = records lost to the device buffer's capacity). */
fdmoe_status fdmoe_read_events(fdmoe_handle* h, int32_t local_rank, fdmoe_event* out, int64_t cap, int64_t* n,
                               int64_t* dropped);

#ifdef __cplusplus
}
#endif
#endif /* FDMOE_H */
