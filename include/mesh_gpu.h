/* mesh_gpu — B200 data plane of the co-located token step (C ABI).
 *
 * The reference LLM-Mesh artifact only PRICES these actions with latency
 * stand-ins; this library EXECUTES them on one GPU per handle. Each entry point
 * names the reference site it replaces (paths under the reference's proj/):
 *
 *   mesh_gpu_instance_create  <- ModelLoad ScaleOp, cluster.cpp:394-399 / cold_start_time perfmodel.cpp:116-119
 *   mesh_gpu_instance_destroy <- ModelUnload ScaleOp, cluster.cpp:865-871
 *   mesh_gpu_kv_resize        <- KvUp/KvDown ScaleOp (memory.hpp:69-81) priced by scale_latency perfmodel.cpp:107-114
 *   mesh_gpu_step             <- IterationPlan (compute.hpp:63-69) scheduled at cluster.cpp:556-572, whose
 *                                duration is iter_time perfmodel.cpp:97-100 and whose effect is
 *                                complete_iteration compute.cpp:155-201
 *   mesh_gpu_request_free     <- request completion / drop (compute.cpp:180-197)
 *   mesh_gpu_swap_out         <- eviction (cluster.cpp:419-428, 742-750); the reference drops the KV and
 *                                re-prefills, here the KV is parked in pinned host memory (async gather on a
 *                                side stream) and restored when the request's re-prefill step runs
 *   mesh_gpu_swap_in          <- the same re-prefill, started early: event-gated scatter on a side stream
 *   mesh_gpu_migrate          <- displaced-request placement (cluster.cpp:439-463) as a P2P KV copy over
 *                                NVLink instead of a re-prefill
 *
 * Conventions mirror llmmesh.h: every call returns mesh_status; on failure
 * mesh_gpu_last_error() holds a message owned by the handle (overwritten by
 * the next failure). Handles are not thread-safe; one host thread drives a
 * handle. Steps are asynchronous: mesh_gpu_step returns a ticket, completed
 * with mesh_gpu_step_wait. There is no CPU fallback: without a usable sm_100
 * device mesh_gpu_open fails with MESH_ERR_CUDA.
 */
#ifndef MESH_GPU_H
#define MESH_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mesh_gpu mesh_gpu;

typedef enum mesh_status {
    MESH_OK = 0,
    MESH_ERR_ARG = 1,      /* null handle / bad argument / unknown id */
    MESH_ERR_CONFIG = 2,   /* unsupported shape or configuration */
    MESH_ERR_RUNTIME = 3,  /* invariant violation in the data plane */
    MESH_ERR_CUDA = 4,     /* CUDA / driver failure (incl. no device) */
    MESH_ERR_NOMEM = 5     /* device KV pool or HBM exhausted */
} mesh_status;

typedef struct mesh_model_shape {
    int32_t n_layers, d_model, n_heads, n_kv_heads, d_head, d_ff, vocab;
    int32_t tied_embeddings; /* lm_head shares the embedding table */
    int32_t max_seq_len;     /* L_max of the instance (rope table rows) */
    float rope_theta;
    float rms_eps;
} mesh_model_shape;

typedef struct mesh_gpu_cfg {
    int32_t device;         /* CUDA ordinal */
    int32_t sm_quota;       /* CTAs of the persistent decode kernel; 0 = all SMs */
    int64_t kv_pool_bytes;  /* physical HBM of the KV arena (granule slots, backed on first use or at
                               open with MESH_GPU_KV_PREALLOC_GB) */
    uint64_t prompt_seed;   /* synthetic prompt ids: hash(seed, request, position) */
    int64_t kv_granule_bytes; /* arena slot (one cuMemCreate/cuMemMap), multiple of 2 MiB; 0 = 32 MiB */
    int32_t lanes;          /* concurrent execution lanes (stream + scratch + an even share of the SM
                               quota); instances bind to the lane with the fewest weight bytes and
                               co-located instances on different lanes step concurrently.
                               0 = MESH_GPU_LANES from the environment, else 1 */
    int32_t swap_pool_mb;   /* pinned host swap space to pin at open (shared by the process's handles;
                               0 = pin 256 MiB chunks on first use) */
} mesh_gpu_cfg;

typedef struct mesh_step_plan {
    int32_t is_prefill;
    int64_t prefill_request;
    int32_t prefill_len;        /* min(I + O, L_max) tokens (compute.cpp:112) */
    int32_t prefill_input_len;  /* I: prompt length for first admission */
    int32_t n_decode;           /* decode: requests in batch (admission) order, <= 8 */
    const int64_t* decode_requests;
} mesh_step_plan;

typedef struct mesh_gpu_stats {
    int64_t kv_mapped_bytes;      /* KV arena bytes assigned to instances (capacity + lazy slack) */
    int64_t kv_pool_bytes;        /* configured physical limit */
    int64_t blocks_moved;         /* compaction block copies */
    int64_t bytes_moved;          /* compaction bytes (read + write counted once) */
    int64_t swap_out_bytes, swap_in_bytes, migrate_bytes;
    int64_t steps, decode_tokens, prefill_tokens;
    double last_step_ms;          /* device time of the last waited step (CUDA events) */
    double last_kernel_ms;        /* device time of its kernels (descriptor copy excluded) */
    int64_t kernel_launches;      /* kernels launched by steps */
    int64_t h2d_bytes, d2h_bytes; /* per-step host<->device traffic (descriptors, prompts, tokens) */
    int64_t kv_granule_bytes;     /* physical chunk size of the KV pool */
    int64_t vmm_calls;            /* cuMemMap / cuMemUnmap / cuMemSetAccess calls */
    double vmm_ms;                /* host time inside them */
    int64_t kv_reclaims;          /* lazy-shrink slack reclaims (stream-ordered, no host wait) */
    double last_step_end_ms;      /* end of the last waited step on the device timeline of timer
                                     mark 0 (all lanes), -1 before the mark */
    int64_t weight_cache_hits;    /* instance creates that shared a live or cached weight set of the
                                     same model (no allocation, no init kernels) */
    int64_t peer_devices;         /* devices granted NVLink access to this device's KV (migration) */
    int64_t vmm_unmaps;           /* cuMemUnmap calls (subset of vmm_calls) */
    double host_ms_create, host_ms_destroy, host_ms_kv_resize, host_ms_step; /* host time inside those calls */
} mesh_gpu_stats;

/* mesh_gpu_swap_state values */
enum { MESH_SWAP_NONE = 0, MESH_SWAP_HISTORY = 1, MESH_SWAP_COPYING = 2, MESH_SWAP_PARKED = 3 };

const char* mesh_gpu_version(void);
int32_t mesh_gpu_device_count(void);

mesh_status mesh_gpu_open(const mesh_gpu_cfg* cfg, mesh_gpu** out);
void mesh_gpu_close(mesh_gpu* g);
const char* mesh_gpu_last_error(const mesh_gpu* g);

mesh_status mesh_gpu_instance_create(mesh_gpu* g, int64_t instance_id, const mesh_model_shape* shape,
                                     uint64_t weight_seed);
mesh_status mesh_gpu_instance_destroy(mesh_gpu* g, int64_t instance_id);
/* Optional, before serving: sizes the lanes' scratch for the largest of `n`
 * shapes and grows the weight allocator's pool by the weight sets of all `n`
 * (one entry per distinct model), so no later instance_create resizes scratch
 * (a device-wide sync) or maps allocator memory (a device drain). */
mesh_status mesh_gpu_reserve(mesh_gpu* g, const mesh_model_shape* shapes, int32_t n);

/* Physically applies a KV ScaleOp at issue time. Every instance's
 * KV lives in one device-wide arena of granule slots; a grow assigns extents of
 * free slots (>= 32 whole blocks each) to the instance, a shrink compacts live
 * blocks below the new high-water mark with a batched block-copy kernel and
 * keeps the extents above it (lazy) until another instance's grow finds no free
 * run and takes them back. Neither path calls the VMM driver or waits on the
 * host: a reassigned slot's new owner waits on an event of the previous owner's
 * queued work. Only a slot's first use maps memory (cuMemMap drains the whole
 * device), so MESH_GPU_KV_PREALLOC_GB backs the arena at open. Block ids
 * (request_info) are the instance's logical ids; the device sees arena ids.
 * `from` must equal the instance's current target. */
mesh_status mesh_gpu_kv_resize(mesh_gpu* g, int64_t instance_id, int64_t from_bytes, int64_t to_bytes);

mesh_status mesh_gpu_step(mesh_gpu* g, int64_t instance_id, const mesh_step_plan* plan, int64_t* ticket);
/* Blocks until the step finished. tokens_out receives one greedy token per
 * emitting request (prefill: 1; decode: n_decode, in plan order). logits_out
 * (nullable, needs logits capture on) receives [n][vocab] fp32. */
mesh_status mesh_gpu_step_wait(mesh_gpu* g, int64_t ticket, int32_t* tokens_out, int32_t cap, int32_t* n_out,
                               float* logits_out, int64_t logits_cap);
/* Non-blocking completion poll (wall-clock mode): *done = 1 once the step's
 * work finished on the device (its tokens are then collected by step_wait
 * without blocking). Replaces the IterationComplete the reference schedules
 * at now + iter_time (cluster.cpp:556-572). */
mesh_status mesh_gpu_step_done(mesh_gpu* g, int64_t ticket, int32_t* done);
mesh_status mesh_gpu_set_capture_logits(mesh_gpu* g, int32_t enable);

mesh_status mesh_gpu_request_free(mesh_gpu* g, int64_t instance_id, int64_t request_id);
/* Preemption swap (SURVEY 8a d-new). swap_out parks a resident request: one
 * copy kernel on the handle's swap stream gathers its KV blocks straight into
 * pinned host memory, ordered after the request's queued steps by an event;
 * the call never waits on the device, and the blocks return to the instance's
 * free list once the gather finished. The request's next prefill step with
 * prefill_len == ctx + 1 (the reference's re-prefill of I+O tokens) resumes
 * from the parked KV and feeds one token; swap_in starts that restore early
 * on a side stream (the instance's lane waits on it by event). Parked
 * requests are process-wide: any handle may resume them. */
mesh_status mesh_gpu_swap_out(mesh_gpu* g, int64_t instance_id, int64_t request_id);
mesh_status mesh_gpu_swap_in(mesh_gpu* g, int64_t instance_id, int64_t request_id);
/* Non-blocking: MESH_SWAP_NONE (not parked), _HISTORY (token history only),
 * _COPYING (gather in flight), _PARKED (KV in pinned host memory). */
mesh_status mesh_gpu_swap_state(mesh_gpu* g, int64_t request_id, int32_t* state);
/* Live KV migration (SURVEY 8a e-new): one copy kernel on dst's device loads
 * the request's blocks from src's VA range (peer access over NVLink when the
 * devices differ) into fresh blocks of dst_instance; both lanes are ordered
 * by events, the host waits only for src's in-flight steps of the instance
 * (token history). */
mesh_status mesh_gpu_migrate(mesh_gpu* src, int64_t src_instance, mesh_gpu* dst, int64_t dst_instance,
                             int64_t request_id);

/* Introspection for tests / the control plane. */
mesh_status mesh_gpu_request_info(mesh_gpu* g, int64_t instance_id, int64_t request_id, int32_t* ctx_len,
                                  int32_t* blocks, int32_t* block_ids, int32_t cap);
mesh_status mesh_gpu_request_tokens(mesh_gpu* g, int64_t instance_id, int64_t request_id, int32_t* tokens,
                                    int32_t cap, int32_t* n_out);
/* Execution lane an instance is bound to and that lane's SM quota (CTAs). Quotas
 * are re-split at every instance create / destroy in proportion to the weight
 * bytes bound to each lane (token-level SM quotas, summing to <= the SMs). */
mesh_status mesh_gpu_instance_lane(mesh_gpu* g, int64_t instance_id, int32_t* lane, int32_t* ctas);

mesh_status mesh_gpu_instance_kv(mesh_gpu* g, int64_t instance_id, int64_t* target_bytes, int64_t* mapped_bytes,
                                 int32_t* capacity_blocks, int32_t* live_blocks);
mesh_status mesh_gpu_read_weight(mesh_gpu* g, int64_t instance_id, int32_t tensor, int32_t layer, int32_t row,
                                 float* out, int32_t n);
mesh_status mesh_gpu_stats_get(mesh_gpu* g, mesh_gpu_stats* out);
mesh_status mesh_gpu_sync(mesh_gpu* g);
/* Device-side timing of a region of work on the compute stream: `mark` records
 * a CUDA event (slot 0..7) on the stream every step is launched on; `elapsed`
 * waits for slot b and returns the device time between slots a and b. */
mesh_status mesh_gpu_timer_mark(mesh_gpu* g, int32_t slot);
mesh_status mesh_gpu_timer_elapsed(mesh_gpu* g, int32_t a, int32_t b, double* ms);
/* Times `iters` back-to-back decode steps of the plan's batch on the device
 * (CUDA events around the launches only) without advancing request state. */
mesh_status mesh_gpu_bench_decode(mesh_gpu* g, int64_t instance_id, const mesh_step_plan* plan, int32_t iters,
                                  double* ms_per_step);

#ifdef __cplusplus
}
#endif

#endif /* MESH_GPU_H */
