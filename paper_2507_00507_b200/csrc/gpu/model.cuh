// Model description shared by the decode/prefill kernels and the host-side
// data plane: Llama-family shapes, the deterministic weight generator, the
// physical row permutations applied when weights are tiled, and the paged KV
// block layout. The CPU oracle (oracle/llama_ref.c) restates the generator.
#pragma once

#include <stddef.h>
#include <stdint.h>

#include "common.cuh"

namespace meshgpu {

struct Shape {
    int n_layers, d, n_heads, n_kv, dh, ff, vocab;
    int tied;          // lm_head == embedding (Llama-3.2-3B)
    float rope_theta;  // rotate-half RoPE base
    float eps;         // RMSNorm epsilon
    int max_seq;       // longest context the instance serves (rope table rows)
    __host__ __device__ int gq() const { return n_heads / n_kv; }
    __host__ __device__ int qkv_rows() const { return (n_heads + 2 * n_kv) * dh; }
    __host__ __device__ long long kv_bytes_per_token() const { return 2LL * n_layers * n_kv * dh * 2; }
};

// Tensor ids of the generator (part of the weight contract with the oracle).
enum TensorId : uint32_t {
    T_EMB = 0, T_WQ = 1, T_WK = 2, T_WV = 3, T_WO = 4, T_WGATE = 5, T_WUP = 6, T_WDOWN = 7,
    T_LM = 8, T_GATTN = 9, T_GMLP = 10, T_GFINAL = 11,
};

__host__ __device__ inline uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
__host__ __device__ inline uint64_t tensor_key(uint64_t seed, uint32_t tensor, uint32_t layer) {
    return splitmix64(seed ^ (uint64_t(tensor) << 56) ^ (uint64_t(layer) << 40) ^ 0x5eedull);
}
// Signed 24-bit integer drawn from the element's hash.
__host__ __device__ inline int32_t elem_i24(uint64_t tkey, uint64_t index) {
    return int32_t(splitmix64(tkey + index) >> 40) - (1 << 23);
}
// Weights: uniform on [-2^-5, 2^-5) (std 0.018), exact in fp32 before the bf16 rounding.
__host__ __device__ inline float weight_value(uint64_t tkey, uint64_t index) {
    return float(elem_i24(tkey, index)) * (1.0f / 268435456.0f);  // 2^-28
}
// RMSNorm gains: 1 + uniform on [-2^-4, 2^-4).
__host__ __device__ inline float gain_value(uint64_t tkey, uint64_t index) {
    return 1.0f + float(elem_i24(tkey, index)) * (1.0f / 134217728.0f);  // 2^-27
}
// Synthetic prompt ids, keyed (seed, request id, position).
__host__ __device__ inline int prompt_token(uint64_t seed, int64_t request, int pos, int vocab) {
    uint64_t h = splitmix64(splitmix64(seed ^ 0x70726f6d7074ull) + uint64_t(request) * 0x100000001b3ull +
                            uint64_t(pos));
    return int(h % uint64_t(vocab));
}

// ---- physical row maps of the fused/permuted matrices (tile = 16 rows) ----
// QKV: sections q (n_heads), k (n_kv), v (n_kv); within a head, tile j holds
// dims [8j, 8j+8) in rows 0-7 and [8j+dh/2, 8j+dh/2+8) in rows 8-15 so every
// rotate-half RoPE pair lands in one thread's mma accumulator (rows g, g+8).
struct QkvRow {
    int section;  // 0 q, 1 k, 2 v
    int head;
    int dim;
};
__host__ __device__ inline QkvRow qkv_row(const Shape& s, int prow) {
    // Rows are grouped by KV head: group g = the GQA group's q heads, then k head
    // g, then v head g (dh rows each), so the tiles of one group are contiguous
    // and the decode attention of (request, kv head g) can start as soon as the
    // group's tiles are done, without a grid-wide barrier after the QKV phase.
    int tiles_per_head = s.dh / 16;
    int tile = prow >> 4, r = prow & 15;
    int head_global = tile / tiles_per_head, j = tile % tiles_per_head;
    const int gq = s.n_heads / s.n_kv, per_group = gq + 2;
    const int grp = head_global / per_group, idx = head_global % per_group;
    QkvRow out;
    if (idx < gq) {
        out.section = 0;
        out.head = grp * gq + idx;
    } else if (idx == gq) {
        out.section = 1;
        out.head = grp;
    } else {
        out.section = 2;
        out.head = grp;
    }
    out.dim = (r < 8) ? (8 * j + r) : (8 * j + (r - 8) + s.dh / 2);
    return out;
}
// QKV tiles of KV-head group g: [g * qkv_group_tiles, (g + 1) * qkv_group_tiles)
__host__ __device__ inline int qkv_group_tiles(const Shape& s) { return (s.n_heads / s.n_kv + 2) * (s.dh / 16); }
// Gate/up: tile j holds gate rows [8j, 8j+8) in rows 0-7 and the matching up
// rows in rows 8-15, so silu(gate) * up is formed in registers.
__host__ __device__ inline void gu_row(int prow, int* is_up, int* row) {
    int tile = prow >> 4, r = prow & 15;
    *is_up = r >= 8;
    *row = 8 * tile + (r & 7);
}

// ---- paged KV block layout ----
// A block holds KV_BLOCK_TOKENS tokens of every layer: [layer][kv_head][k|v][slot][dh] bf16.
// The K and V rows of one (layer, kv head) are adjacent, so the decode ring moves
// a block's K+V in ONE bulk copy (4 KB at dh = 64, 8 KB at dh = 128): scattered
// 2 KB copies cap a TMA ring at ~30 GB/s per SM, 4 KB at ~56, 8 KB at ~91
// (profiles/readbw_grid_r01.json). Within a token row the 16-byte chunks are
// XOR-swizzled by (slot & 7) so that ldmatrix over 8 consecutive token rows
// hits 8 distinct bank groups.
constexpr int KV_BLOCK_TOKENS = 16;
__host__ __device__ inline size_t kv_offset(const Shape& s, int layer, int kv, int head, int slot) {
    return ((((size_t(layer) * s.n_kv + head) * 2 + kv) * KV_BLOCK_TOKENS + slot) * s.dh) * 2;
}
// byte offset of element `dim` inside a token row of block-slot `slot`
__host__ __device__ inline uint32_t kv_dim_off(int slot, int dim) {
    return uint32_t((((dim >> 3) ^ (slot & 7)) << 4) + (dim & 7) * 2);
}

// ---- device view of one instance's weights ----
struct Weights {
    const uint8_t* qkv;    // [L] tiled [qkv_rows][d]
    const uint8_t* o;      // [L] tiled [d][H*dh]
    const uint8_t* gu;     // [L] tiled [2ff][d]
    const uint8_t* down;   // [L] tiled [d][ff]
    const uint8_t* lm;     // tiled [V][d]
    const uint16_t* emb;   // row-major [V][d] bf16
    const float* g_attn;   // [L][d]
    const float* g_mlp;    // [L][d]
    const float* g_final;  // [d]
    const float2* rope;    // [max_seq][dh/2] (cos, sin)
    size_t qkv_layer, o_layer, gu_layer, down_layer;  // bytes per layer
};

}  // namespace meshgpu
