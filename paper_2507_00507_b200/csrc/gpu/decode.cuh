// Persistent, SM-quota-bounded decode step (one token for every request of
// the planned instance; SURVEY 8a rows a-new-1 / a3 / a6).
#pragma once

#include "model.cuh"

namespace meshgpu {

constexpr int DEC_NCW = 8;                       // consumer (math) warps
constexpr int DEC_THREADS = (DEC_NCW + 1) * 32;  // + one TMA producer warp
constexpr int DEC_NSTAGE = 16;                   // weight ring depth
constexpr int DEC_STAGE_BYTES = 8192;            // 16 rows x 256 cols bf16
constexpr int DEC_CHUNK_COLS = 256;
constexpr int DEC_KSEG_MAX = 4096;  // activation columns resident in smem at once
constexpr int DEC_MAXT = 4;         // tiles accumulated per group
constexpr int DEC_MAXB = 8;         // batch columns of the mma (n = 8)
constexpr int DEC_BT_MAX = 256;     // block-table entries per request -> contexts up to 4096 tokens
constexpr int MAX_BT_UPDATES = 64;
constexpr int DEC_CLAIM_MAX = 256;  // claim counters per lane: n_layers * 4 + 1 <= 256
constexpr int DEC_KV_HEADS_MAX = 64;

constexpr int DEC_SMEM_RING = DEC_NSTAGE * DEC_STAGE_BYTES;
constexpr int DEC_SMEM_ACT = DEC_MAXB * (DEC_KSEG_MAX + 8) * 2;
constexpr int DEC_SMEM_ACC = DEC_NCW * DEC_MAXT * 128 * 4;  // per-warp tile partials
constexpr int DEC_SMEM_BARS = 2 * DEC_NSTAGE * 8;
constexpr int DEC_SMEM_MISC = 1024;
constexpr int DEC_SMEM_BT = DEC_MAXB * DEC_BT_MAX * 4;
constexpr int DEC_TACC_TILES = 12;  // multi-segment phases: per-tile sums kept across activation segments
constexpr int DEC_SMEM_TACC = DEC_TACC_TILES * 128 * 4;
constexpr int DEC_SMEM_TOTAL =
    DEC_SMEM_RING + DEC_SMEM_ACT + DEC_SMEM_ACC + DEC_SMEM_BARS + DEC_SMEM_MISC + DEC_SMEM_BT + DEC_SMEM_TACC;

// Per-step input written by the host (one H2D copy) before the launch.
struct StepDesc {
    int B;                    // requests decoded this step (<= 8)
    int slot[DEC_MAXB];       // request slots in the instance's request table
    int pos[DEC_MAXB];        // position of the token being fed (= context length before the step)
    int n_upd;                // block-table entries to install before attention reads them
    int upd[MAX_BT_UPDATES][3];  // (slot, block index, block id)
};

struct DecodeArgs {
    Shape s;
    Weights w;
    uint8_t* kv_base;      // instance KV region (block b at kv_base + b * block_bytes)
    long long block_bytes;
    int* block_table;      // [slots][bt_stride]
    int bt_stride;
    int* last_tok;         // [slots] token fed at the next step (written by this step)
    const StepDesc* desc;
    // scratch owned by the device context
    float* h;          // [8][d] residual stream
    uint16_t* act;     // [8][d] bf16(h * gamma) for the next normed GEMV
    uint16_t* attn;    // [8][d] attention output
    uint16_t* abuf;    // [8][ff] silu(gate) * up
    float* q;          // [8][n_heads][dh] roped queries
    float* ssA;        // [d/16][8] sum-of-squares partials feeding QKV / lm_head
    float* ssB;        // [d/16][8] ... feeding gate/up
    float* apart;      // attention partials: [stage slot][gq][m, l, acc[dh]]
    int* acnt;         // [8][n_kv] partial arrival counters (self-resetting)
    float* arg_val;    // [grid][8]
    int* arg_idx;      // [grid][8]
    int* arg_cnt;      // [1] (self-resetting)
    int* claim;        // [n_layers * 4 + 1] tile-claim counters of the dynamic GEMV phases (reset at step end)
    int* qkv_done;     // [n_kv] QKV tiles finished per KV-head group, monotonic over the step's layers (reset at step end)
    float* logits;     // optional [8][vocab]
    int* tok_out;      // [8]
    unsigned int* bar_count;
    unsigned int* bar_gen;
    volatile int* progress;  // optional host-mapped [grid][2]: consumer phase, producer stage
    unsigned long long* trace;  // optional [4096]: %globaltimer at CTA 0's phase boundaries
    unsigned long long* arrive; // optional [barriers][grid]: %globaltimer of every CTA's barrier arrival
    int nstage;    // weight-ring stages in use (<= DEC_NSTAGE): bounds bytes in flight per SM
    int w_lanes;   // weight stages of dynamic claims / static single-segment and segment-outer phases by decoupled lanes
    int kv_lanes;  // attention KV stages issued by decoupled producer lanes (1) or the batched push/flush (0)
    int l2pf;      // weight stages: also prefetch the bytes this many 8 KB stages ahead into L2 (0: off)
    int skip;      // debug: 1 skips attention, 2 the GEMV phases, 8 / 16 the attention / GEMV math (ring only); results are garbage
};

cudaError_t launch_decode(const DecodeArgs& a, int grid, cudaStream_t stream);
size_t decode_apart_floats(const Shape& s);

}  // namespace meshgpu
