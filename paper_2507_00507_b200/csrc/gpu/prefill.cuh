// Prefill step: one request, L tokens (SURVEY 8a row a-new-2, plan_for
// prefill branch compute.cpp:104-115).
#pragma once

#include "model.cuh"

namespace meshgpu {

struct PrefillArgs {
    Shape s;
    Weights w;
    uint8_t* kv_base;
    long long block_bytes;
    long long kv_blocks;  // blocks the instance's KV VA range can address (tensor-map extent)
    const int* bt_row;  // block table row of the request (device)
    int slot;
    int L;              // tokens in this pass
    int p0;             // absolute position of the first token
    const int* tokens;  // [L] device
    // scratch sized for max_seq tokens
    float* h;           // [L][d]
    uint16_t* act;      // [L][d]
    float* rs;          // [L]
    uint16_t* q;        // [L][H][dh] bf16 (RoPE applied; the attention MMA operand)
    uint16_t* attn;     // [L][d]
    uint16_t* abuf;     // [L][ff]
    float* logits;      // [vocab] (last token)
    int* last_tok;      // instance request table
    int* tok_out;       // [1]
    int max_ctas;       // SM quota of the lane (persistent GEMM grid); 0 = all SMs
    int pair_ok;        // CTA-pair GEMMs allowed: no other lane holds an instance (co-located
                        // decode grids leave few free SM pairs; measured slower there)
    int* tile_ctr;      // lane's dynamic tile counter (zero between launches; self-resetting)
    float* sk_ws;       // split-K partial tiles [units][128][256] fp32 (units <= 2 x SMs)
    int* sk_cnt;        // split-K arrivals per output tile (self-resetting), >= SK_TILES_MAX
};

constexpr int SK_TILES_MAX = 1024;
cudaError_t launch_prefill(const PrefillArgs& a, cudaStream_t stream);
// kernels one launch_prefill issues (embed, per layer 2 norms + 4 GEMMs + attention, final norm/lm_head/argmax)
inline int prefill_launch_count(const Shape& s) { return 1 + 7 * s.n_layers + 3; }

}  // namespace meshgpu
