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
constexpr int DEC_MAXT = 16;        // tiles accumulated per group
constexpr int DEC_MAXB = 8;         // batch columns of the mma (n = 8)
constexpr int ATT_SPLIT = 256;      // context tokens per attention work unit
constexpr int ATT_MAX_SPLITS = 32;  // supports contexts up to 8192
constexpr int MAX_BT_UPDATES = 64;

constexpr int DEC_SMEM_RING = DEC_NSTAGE * DEC_STAGE_BYTES;
constexpr int DEC_SMEM_ACT = DEC_MAXB * (DEC_KSEG_MAX + 8) * 2;
constexpr int DEC_SMEM_ACC = 2 * DEC_MAXT * 128 * 4;
constexpr int DEC_SMEM_BARS = 2 * DEC_NSTAGE * 8;
constexpr int DEC_SMEM_MISC = 1024;
constexpr int DEC_SMEM_TOTAL = DEC_SMEM_RING + DEC_SMEM_ACT + DEC_SMEM_ACC + DEC_SMEM_BARS + DEC_SMEM_MISC;

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
    float* apart;      // attention split partials
    int* acnt;         // [8][n_kv] split arrival counters (self-resetting)
    float* arg_val;    // [grid][8]
    int* arg_idx;      // [grid][8]
    int* arg_cnt;      // [1] (self-resetting)
    float* logits;     // optional [8][vocab]
    int* tok_out;      // [8]
    unsigned int* bar_count;
    unsigned int* bar_gen;
};

cudaError_t launch_decode(const DecodeArgs& a, int grid, cudaStream_t stream);
size_t decode_apart_floats(const Shape& s);

}  // namespace meshgpu
