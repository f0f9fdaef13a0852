// Decode step as ONE persistent kernel per instance step.
//
// Grid = the instance's SM quota (one CTA per SM). Every CTA runs a TMA
// producer warp that streams its share of ALL weight tiles of the step (every
// layer's QKV, O, gate/up, down, then lm_head) through a 16-stage shared-memory
// ring with 1-D bulk copies, never waiting on activations: weights do not
// depend on them, so the stream runs ahead across the grid barriers that
// separate the phases. Eight consumer warps wait for the ring, multiply the
// 16-row weight tiles with the (<= 8) activation columns on the tensor cores
// (mma.m16n8k16, bf16 in / fp32 accumulate) and apply fused epilogues:
//   QKV   : RMSNorm scale, rotate-half RoPE, q -> scratch, k/v -> paged KV cache
//   ATTN  : paged GQA attention, split over context, deterministic combine
//   O     : residual add, next RMSNorm numerator and sum-of-squares partials
//   GU    : RMSNorm scale, silu(gate) * up
//   DOWN  : residual add, next RMSNorm numerator and sum-of-squares partials
//   LM    : final RMSNorm scale, optional logits, greedy argmax
// Tiles are dealt round-robin across CTAs continuing from phase to phase, so
// every CTA streams (within one tile) the same number of bytes per step.
#include "decode.cuh"

#include <math.h>

namespace meshgpu {

namespace {

enum PhaseKind { PH_QKV = 0, PH_O = 1, PH_GU = 2, PH_DOWN = 3, PH_LM = 4 };

struct GemvPhase {
    int kind, layer;
    int tiles;   // 16-row tiles
    int K;       // columns
    const uint8_t* base;
};

__device__ __forceinline__ GemvPhase gemv_phase(const DecodeArgs& a, int kind, int layer) {
    const Shape& s = a.s;
    GemvPhase p;
    p.kind = kind;
    p.layer = layer;
    switch (kind) {
        case PH_QKV: p.tiles = s.qkv_rows() / 16; p.K = s.d; p.base = a.w.qkv + layer * a.w.qkv_layer; break;
        case PH_O: p.tiles = s.d / 16; p.K = s.n_heads * s.dh; p.base = a.w.o + layer * a.w.o_layer; break;
        case PH_GU: p.tiles = 2 * s.ff / 16; p.K = s.d; p.base = a.w.gu + layer * a.w.gu_layer; break;
        case PH_DOWN: p.tiles = s.d / 16; p.K = s.ff; p.base = a.w.down + layer * a.w.down_layer; break;
        default: p.tiles = s.vocab / 16; p.K = s.d; p.base = a.w.lm; break;
    }
    return p;
}

// This CTA's tiles of a phase: t0, t0 + G, ... (round-robin offset `off`).
struct MyTiles {
    int t0, n;
};
__device__ __forceinline__ MyTiles my_tiles(int tiles, int off, int cta, int G) {
    int t0 = (cta - off) % G;
    if (t0 < 0) t0 += G;
    MyTiles m;
    m.t0 = t0;
    m.n = t0 < tiles ? (tiles - 1 - t0) / G + 1 : 0;
    return m;
}
__device__ __forceinline__ int n_segments(int K) {
    int chunks = K / DEC_CHUNK_COLS;
    int per = DEC_KSEG_MAX / DEC_CHUNK_COLS;
    return (chunks + per - 1) / per;
}
__device__ __forceinline__ void seg_range(int K, int nseg, int s, int& c0, int& c1) {
    int chunks = K / DEC_CHUNK_COLS;
    c0 = (chunks * s) / nseg;
    c1 = (chunks * (s + 1)) / nseg;
}

struct Smem {
    uint8_t* ring;
    uint16_t* act;
    float* acc;
    uint64_t* full;
    uint64_t* empty;
    float* misc;
};

__device__ __forceinline__ Smem carve(uint8_t* base) {
    Smem m;
    m.ring = base;
    m.act = reinterpret_cast<uint16_t*>(base + DEC_SMEM_RING);
    m.acc = reinterpret_cast<float*>(base + DEC_SMEM_RING + DEC_SMEM_ACT);
    m.full = reinterpret_cast<uint64_t*>(base + DEC_SMEM_RING + DEC_SMEM_ACT + DEC_SMEM_ACC);
    m.empty = m.full + DEC_NSTAGE;
    m.misc = reinterpret_cast<float*>(base + DEC_SMEM_RING + DEC_SMEM_ACT + DEC_SMEM_ACC + DEC_SMEM_BARS);
    return m;
}

constexpr int CONSUMER_THREADS = DEC_NCW * 32;
__device__ __forceinline__ void csync() { named_bar_sync(1, CONSUMER_THREADS); }

// ----------------------------------------------------------------- producer
__device__ void producer_loop(const DecodeArgs& a, Smem& sm, int cta, int G) {
    const uint64_t pol = l2_evict_first_policy();
    uint32_t q = 0;
    int off = 0;
    auto produce = [&](int kind, int layer) {
        GemvPhase p = gemv_phase(a, kind, layer);
        MyTiles mt = my_tiles(p.tiles, off, cta, G);
        off = (off + p.tiles) % G;
        if (mt.n == 0) return;
        const size_t tile_bytes = size_t(p.K) * 32;
        int nseg = n_segments(p.K);
        for (int g0 = 0; g0 < mt.n; g0 += DEC_MAXT) {
            int gn = min(DEC_MAXT, mt.n - g0);
            for (int sg = 0; sg < nseg; ++sg) {
                int c0, c1;
                seg_range(p.K, nseg, sg, c0, c1);
                for (int ti = 0; ti < gn; ++ti) {
                    int tile = mt.t0 + (g0 + ti) * G;
                    const uint8_t* tsrc = p.base + size_t(tile) * tile_bytes;
                    for (int c = c0; c < c1; ++c) {
                        uint32_t slot = q % DEC_NSTAGE;
                        uint32_t par = (q / DEC_NSTAGE) & 1u;
                        mbar_wait(&sm.empty[slot], par ^ 1u);
                        mbar_arrive_expect_tx(&sm.full[slot], DEC_STAGE_BYTES);
                        bulk_g2s_evict_first(sm.ring + size_t(slot) * DEC_STAGE_BYTES,
                                             tsrc + size_t(c) * DEC_STAGE_BYTES, DEC_STAGE_BYTES,
                                             &sm.full[slot], pol);
                        ++q;
                    }
                }
            }
        }
    };
    for (int l = 0; l < a.s.n_layers; ++l) {
        produce(PH_QKV, l);
        produce(PH_O, l);
        produce(PH_GU, l);
        produce(PH_DOWN, l);
    }
    produce(PH_LM, 0);
}

// ----------------------------------------------------------------- consumer
struct Ctx {
    const DecodeArgs* a;
    Smem sm;
    int cta, G, warp, lane, tid;  // tid in [0, 256)
    int B;
    int slot[DEC_MAXB];
    int pos[DEC_MAXB];
    uint32_t q;     // stage counter (mirrors the producer)
    int off;        // round-robin offset (mirrors the producer)
    int accbuf;     // acc double-buffer parity
};

__device__ void grid_sync(Ctx& c) {
    csync();
    if (c.tid == 0) grid_barrier(c.a->bar_count, c.a->bar_gen, unsigned(c.G));
    csync();
}

// rs[b] = 1/sqrt(mean(h_b^2) + eps) from per-tile partials, summed in a fixed order.
__device__ void compute_rs(Ctx& c, const float* ss, float* rs_out) {
    const DecodeArgs& a = *c.a;
    int nt = a.s.d / 16;
    int b = c.warp;  // 8 warps <-> 8 batch columns
    float acc = 0.f;
    for (int t = c.lane; t < nt; t += 32) acc += ldcg_f32(ss + t * 8 + b);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (c.lane == 0) rs_out[b] = rsqrtf(acc / float(a.s.d) + a.s.eps);
}

// Load activation columns [k0, k1) of the 8 batch rows (bf16, global) into smem.
__device__ void load_act(Ctx& c, const uint16_t* src, int ld, int k0, int k1) {
    int n = k1 - k0;  // multiple of 256
    int stride = n + 8;
    int vec_per_row = n / 8;
    for (int i = c.tid; i < DEC_MAXB * vec_per_row; i += CONSUMER_THREADS) {
        int b = i / vec_per_row, v = i % vec_per_row;
        uint4 val = make_uint4(0, 0, 0, 0);
        if (b < c.B) val = ldcg_u4(src + size_t(b) * ld + k0 + v * 8);
        *reinterpret_cast<uint4*>(c.sm.act + b * stride + v * 8) = val;
    }
}

// One 8 KB stage: 16 rows x 256 columns against the 8 activation columns.
__device__ __forceinline__ void consume_stage(Ctx& c, uint32_t qi, int act_col, int act_stride,
                                              float* acc_slot) {
    uint32_t slot = qi % DEC_NSTAGE;
    uint32_t par = (qi / DEC_NSTAGE) & 1u;
    mbar_wait(&c.sm.full[slot], par);
    const uint32_t stage_addr = smem_u32(c.sm.ring + size_t(slot) * DEC_STAGE_BYTES);
    const int lane = c.lane;
    const int r = lane & 15;
    const int g = lane >> 2, t = lane & 3;
    const uint16_t* actrow = c.sm.act + g * act_stride + act_col + 2 * t;
    float d0[4] = {0.f, 0.f, 0.f, 0.f}, d1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        int kb = j >> 2;
        int chunk = ((j & 3) << 1) + (lane >> 4);
        uint32_t addr = stage_addr + kb * 2048 + r * 128 + (uint32_t((chunk ^ (r & 7))) << 4);
        uint32_t a0, a1, a2, a3;
        ldmatrix_x4(addr, a0, a1, a2, a3);
        uint32_t b0 = *reinterpret_cast<const uint32_t*>(actrow + j * 16);
        uint32_t b1 = *reinterpret_cast<const uint32_t*>(actrow + j * 16 + 8);
        if (j & 1)
            mma_bf16_16816(d1, a0, a1, a2, a3, b0, b1);
        else
            mma_bf16_16816(d0, a0, a1, a2, a3, b0, b1);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&c.sm.empty[slot]);
    float* dst = acc_slot + lane * 4;
    atomicAdd(dst + 0, d0[0] + d1[0]);
    atomicAdd(dst + 1, d0[1] + d1[1]);
    atomicAdd(dst + 2, d0[2] + d1[2]);
    atomicAdd(dst + 3, d0[3] + d1[3]);
}

// ---- epilogues: lane holds rows (g, g+8) x batch columns (2t, 2t+1) of tile `tile`.
__device__ void epi_qkv(Ctx& c, int layer, int tile, const float v[4], const float* rs) {
    const DecodeArgs& a = *c.a;
    const Shape& s = a.s;
    int g = c.lane >> 2, t = c.lane & 3;
    QkvRow r1 = qkv_row(s, tile * 16 + g);  // dim in [0, dh/2); row g+8 is dim + dh/2
    const int half = s.dh / 2;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        int b = 2 * t + j;
        if (b >= c.B) continue;
        float x1 = v[j] * rs[b], x2 = v[2 + j] * rs[b];
        int pos = c.pos[b];
        float o1 = x1, o2 = x2;
        if (r1.section < 2) {
            float2 cs = a.w.rope[size_t(pos) * half + r1.dim];
            o1 = x1 * cs.x - x2 * cs.y;
            o2 = x2 * cs.x + x1 * cs.y;
        }
        if (r1.section == 0) {
            float* qd = a.q + (size_t(b) * s.n_heads + r1.head) * s.dh;
            qd[r1.dim] = o1;
            qd[r1.dim + half] = o2;
        } else {
            int blk = ldcg_i32(a.block_table + size_t(c.slot[b]) * a.bt_stride + pos / KV_BLOCK_TOKENS);
            uint8_t* p = a.kv_base + size_t(blk) * a.block_bytes +
                         kv_offset(s, layer, r1.section - 1, r1.head, pos % KV_BLOCK_TOKENS);
            uint16_t* e = reinterpret_cast<uint16_t*>(p);
            e[r1.dim] = f_to_bf16(o1);
            e[r1.dim + half] = f_to_bf16(o2);
        }
    }
}

__device__ void epi_gu(Ctx& c, int tile, const float v[4], const float* rs) {
    const DecodeArgs& a = *c.a;
    int g = c.lane >> 2, t = c.lane & 3;
    int row = tile * 8 + g;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        int b = 2 * t + j;
        if (b >= c.B) continue;
        float gt = v[j] * rs[b], up = v[2 + j] * rs[b];
        float act = gt / (1.f + __expf(-gt)) * up;
        a.abuf[size_t(b) * a.s.ff + row] = f_to_bf16(act);
    }
}

// Residual add for rows owned by this tile + the next RMSNorm's numerator and
// the per-tile sum of squares.
__device__ void epi_residual(Ctx& c, int tile, const float v[4], const float* gamma_next, float* ss_out) {
    const DecodeArgs& a = *c.a;
    const int d = a.s.d;
    int g = c.lane >> 2, t = c.lane & 3;
    float sq[2] = {0.f, 0.f};
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
        int row = tile * 16 + g + 8 * rr;
        float gm = gamma_next[row];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            int b = 2 * t + j;
            if (b >= c.B) continue;
            float* hp = a.h + size_t(b) * d + row;
            float hv = ldcg_f32(hp) + v[2 * rr + j];
            *hp = hv;
            a.act[size_t(b) * d + row] = f_to_bf16(hv * gm);
            sq[j] += hv * hv;
        }
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) sq[j] += __shfl_xor_sync(0xffffffffu, sq[j], o);
    }
    if (g == 0) {
        ss_out[tile * 8 + 2 * t] = sq[0];
        ss_out[tile * 8 + 2 * t + 1] = sq[1];
    }
}

__device__ __forceinline__ void better(float& bv, int& bi, float v, int i) {
    if (v > bv || (v == bv && i < bi)) {
        bv = v;
        bi = i;
    }
}

// ------------------------------------------------------------ GEMV phase
__device__ void run_gemv(Ctx& c, int kind, int layer, float* best_v, int* best_i) {
    const DecodeArgs& a = *c.a;
    GemvPhase p = gemv_phase(a, kind, layer);
    MyTiles mt = my_tiles(p.tiles, c.off, c.cta, c.G);
    c.off = (c.off + p.tiles) % c.G;

    float* rs = c.sm.misc;  // [8]
    if (kind == PH_QKV || kind == PH_LM) compute_rs(c, a.ssA, rs);
    if (kind == PH_GU) compute_rs(c, a.ssB, rs);
    if (mt.n == 0) {
        csync();
        return;
    }
    const uint16_t* src;
    int ld;
    switch (kind) {
        case PH_O: src = a.attn; ld = a.s.d; break;
        case PH_DOWN: src = a.abuf; ld = a.s.ff; break;
        default: src = a.act; ld = a.s.d; break;
    }
    int nseg = n_segments(p.K);
    for (int g0 = 0; g0 < mt.n; g0 += DEC_MAXT) {
        int gn = min(DEC_MAXT, mt.n - g0);
        float* accb = c.sm.acc + c.accbuf * DEC_MAXT * 128;
        for (int sg = 0; sg < nseg; ++sg) {
            int c0, c1;
            seg_range(p.K, nseg, sg, c0, c1);
            int nch = c1 - c0;
            if (nseg > 1 || g0 == 0) {
                csync();
                load_act(c, src, ld, c0 * DEC_CHUNK_COLS, c1 * DEC_CHUNK_COLS);
                csync();
            }
            int act_stride = nch * DEC_CHUNK_COLS + 8;
            int n = gn * nch;
            for (int i = c.warp; i < n; i += DEC_NCW) {
                int ti = i / nch, ch = i % nch;
                consume_stage(c, c.q + i, ch * DEC_CHUNK_COLS, act_stride, accb + ti * 128);
            }
            c.q += n;
        }
        csync();
        // epilogue: one warp per tile slot
        for (int ti = c.warp; ti < gn; ti += DEC_NCW) {
            int tile = mt.t0 + (g0 + ti) * c.G;
            float4 v4 = *reinterpret_cast<float4*>(accb + ti * 128 + c.lane * 4);
            *reinterpret_cast<float4*>(accb + ti * 128 + c.lane * 4) = make_float4(0.f, 0.f, 0.f, 0.f);
            float v[4] = {v4.x, v4.y, v4.z, v4.w};
            switch (kind) {
                case PH_QKV: epi_qkv(c, layer, tile, v, rs); break;
                case PH_GU: epi_gu(c, tile, v, rs); break;
                case PH_O:
                    epi_residual(c, tile, v, a.w.g_mlp + size_t(layer) * a.s.d, a.ssB);
                    break;
                case PH_DOWN: {
                    const float* gn_next = (layer + 1 < a.s.n_layers)
                                               ? a.w.g_attn + size_t(layer + 1) * a.s.d
                                               : a.w.g_final;
                    epi_residual(c, tile, v, gn_next, a.ssA);
                    break;
                }
                default: {  // lm_head
                    int g = c.lane >> 2, t = c.lane & 3;
#pragma unroll
                    for (int rr = 0; rr < 2; ++rr) {
                        int row = tile * 16 + g + 8 * rr;
#pragma unroll
                        for (int j = 0; j < 2; ++j) {
                            int b = 2 * t + j;
                            if (b >= c.B) continue;
                            float logit = v[2 * rr + j] * rs[b];
                            if (a.logits) a.logits[size_t(b) * a.s.vocab + row] = logit;
                            better(best_v[j], best_i[j], logit, row);
                        }
                    }
                    break;
                }
            }
        }
        c.accbuf ^= 1;
    }
    csync();
}

// ------------------------------------------------------------ attention
template <int DH>
__device__ void attn_unit(Ctx& c, int layer, int b, int kvh, int split) {
    const DecodeArgs& a = *c.a;
    const Shape& s = a.s;
    const int GQ = s.n_heads / s.n_kv;
    const int len = c.pos[b] + 1;
    const int nsplit = (len + ATT_SPLIT - 1) / ATT_SPLIT;
    const float scale = rsqrtf(float(DH));
    constexpr int DPL = DH / 32;

    float* q_s = reinterpret_cast<float*>(c.sm.act);          // [GQ][DH]
    float* p_s = q_s + 8 * DH;                                  // [8 warps][32][9]
    float* mw = p_s + DEC_NCW * 32 * 9;                         // [8][8]
    float* lw = mw + 64;                                        // [8][8]
    float* accw = lw + 64;                                      // [8][GQ*DH]
    int* flag = reinterpret_cast<int*>(c.sm.misc + 16);

    const float* qsrc = a.q + (size_t(b) * s.n_heads + size_t(kvh) * GQ) * DH;
    for (int i = c.tid; i < GQ * DH; i += CONSUMER_THREADS) q_s[i] = ldcg_f32(qsrc + i);
    csync();

    const int* bt = a.block_table + size_t(c.slot[b]) * a.bt_stride;
    const int t0 = split * ATT_SPLIT + c.warp * 32;
    const int tok = t0 + c.lane;
    const bool valid = tok < len;
    float sc[8];
#pragma unroll
    for (int h = 0; h < 8; ++h) sc[h] = 0.f;
    if (valid) {
        int blk = ldcg_i32(bt + tok / KV_BLOCK_TOKENS);
        const uint8_t* kp = a.kv_base + size_t(blk) * a.block_bytes +
                            kv_offset(s, layer, 0, kvh, tok % KV_BLOCK_TOKENS);
#pragma unroll
        for (int cix = 0; cix < DH / 8; ++cix) {
            uint4 kv = ldcg_u4(kp + cix * 16);
            float kf[8] = {bf16_lo(kv.x), bf16_hi(kv.x), bf16_lo(kv.y), bf16_hi(kv.y),
                           bf16_lo(kv.z), bf16_hi(kv.z), bf16_lo(kv.w), bf16_hi(kv.w)};
#pragma unroll
            for (int h = 0; h < 8; ++h) {
                if (h < GQ) {
                    const float4* qv = reinterpret_cast<const float4*>(q_s + h * DH + cix * 8);
                    float4 qa = qv[0], qb = qv[1];
                    sc[h] += qa.x * kf[0] + qa.y * kf[1] + qa.z * kf[2] + qa.w * kf[3] + qb.x * kf[4] +
                             qb.y * kf[5] + qb.z * kf[6] + qb.w * kf[7];
                }
            }
        }
    }
    float m[8], l[8];
#pragma unroll
    for (int h = 0; h < 8; ++h) {
        float x = valid ? sc[h] * scale : -INFINITY;
        float mx = x;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        float p = (valid && mx != -INFINITY) ? __expf(x - mx) : 0.f;
        float ls = p;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, o);
        m[h] = mx;
        l[h] = ls;
        if (h < GQ) p_s[(c.warp * 32 + c.lane) * 9 + h] = p;
    }
    __syncwarp();
    float acc[8][DPL];
#pragma unroll
    for (int h = 0; h < 8; ++h)
#pragma unroll
        for (int e = 0; e < DPL; ++e) acc[h][e] = 0.f;
    int nvalid = min(32, len - t0);
    const int d0 = c.lane * DPL;
    for (int j = 0; j < nvalid; ++j) {
        int tk = t0 + j;
        int blk = ldcg_i32(bt + tk / KV_BLOCK_TOKENS);
        const uint8_t* vp = a.kv_base + size_t(blk) * a.block_bytes +
                            kv_offset(s, layer, 1, kvh, tk % KV_BLOCK_TOKENS) + d0 * 2;
        float vf[DPL];
        if constexpr (DPL == 2) {
            uint32_t vv = ldcg_u32(vp);
            vf[0] = bf16_lo(vv);
            vf[1] = bf16_hi(vv);
        } else {
            uint2 vv = ldcg_u2(vp);
            vf[0] = bf16_lo(vv.x);
            vf[1] = bf16_hi(vv.x);
            vf[2] = bf16_lo(vv.y);
            vf[3] = bf16_hi(vv.y);
        }
        const float* pj = p_s + (c.warp * 32 + j) * 9;
#pragma unroll
        for (int h = 0; h < 8; ++h) {
            if (h < GQ) {
                float pv = pj[h];
#pragma unroll
                for (int e = 0; e < DPL; ++e) acc[h][e] += pv * vf[e];
            }
        }
    }
#pragma unroll
    for (int h = 0; h < 8; ++h) {
        if (h < GQ) {
            if (c.lane == 0) {
                mw[c.warp * 8 + h] = m[h];
                lw[c.warp * 8 + h] = l[h];
            }
#pragma unroll
            for (int e = 0; e < DPL; ++e) accw[(c.warp * GQ + h) * DH + d0 + e] = acc[h][e];
        }
    }
    csync();
    // combine the 8 warps -> this split's partial
    float* part = a.apart + ((size_t(b) * s.n_kv + kvh) * ATT_MAX_SPLITS + split) * GQ * (DH + 2);
    for (int i = c.tid; i < GQ * DH; i += CONSUMER_THREADS) {
        int h = i / DH, dd = i % DH;
        float M = -INFINITY;
        for (int w = 0; w < DEC_NCW; ++w) M = fmaxf(M, mw[w * 8 + h]);
        float L = 0.f, A = 0.f;
        for (int w = 0; w < DEC_NCW; ++w) {
            float mwv = mw[w * 8 + h];
            if (mwv == -INFINITY) continue;
            float f = __expf(mwv - M);
            L += lw[w * 8 + h] * f;
            A += accw[(w * GQ + h) * DH + dd] * f;
        }
        float* ph = part + h * (DH + 2);
        ph[2 + dd] = A;
        if (dd == 0) {
            ph[0] = M;
            ph[1] = L;
        }
    }
    __threadfence();
    csync();
    if (c.tid == 0) {
        int old = atomicAdd(a.acnt + b * s.n_kv + kvh, 1);
        *flag = (old == nsplit - 1);
    }
    csync();
    if (*flag) {
        __threadfence();
        const float* base = a.apart + (size_t(b) * s.n_kv + kvh) * ATT_MAX_SPLITS * GQ * (DH + 2);
        for (int i = c.tid; i < GQ * DH; i += CONSUMER_THREADS) {
            int h = i / DH, dd = i % DH;
            float M = -INFINITY;
            for (int sp = 0; sp < nsplit; ++sp) M = fmaxf(M, ldcg_f32(base + (sp * GQ + h) * (DH + 2)));
            float L = 0.f, A = 0.f;
            for (int sp = 0; sp < nsplit; ++sp) {
                const float* ph = base + (sp * GQ + h) * (DH + 2);
                float f = __expf(ldcg_f32(ph) - M);
                L += ldcg_f32(ph + 1) * f;
                A += ldcg_f32(ph + 2 + dd) * f;
            }
            a.attn[size_t(b) * s.d + (size_t(kvh) * GQ + h) * DH + dd] = f_to_bf16(A / L);
        }
        if (c.tid == 0) atomicExch(a.acnt + b * s.n_kv + kvh, 0);
    }
    csync();
}

__device__ void run_attention(Ctx& c, int layer) {
    const Shape& s = c.a->s;
    int total = 0;
    int per_b[DEC_MAXB];
    for (int b = 0; b < c.B; ++b) {
        per_b[b] = s.n_kv * ((c.pos[b] + ATT_SPLIT) / ATT_SPLIT);  // ceil((pos+1)/SPLIT)
        total += per_b[b];
    }
    for (int u = c.cta; u < total; u += c.G) {
        int b = 0, r = u;
        while (r >= per_b[b]) {
            r -= per_b[b];
            ++b;
        }
        int nsplit = per_b[b] / s.n_kv;
        int kvh = r / nsplit, split = r % nsplit;
        if (s.dh == 64)
            attn_unit<64>(c, layer, b, kvh, split);
        else
            attn_unit<128>(c, layer, b, kvh, split);
    }
}

// ------------------------------------------------------------ embedding
__device__ void run_embed(Ctx& c) {
    const DecodeArgs& a = *c.a;
    const Shape& s = a.s;
    if (c.cta == 0) {
        const StepDesc* dsc = a.desc;
        for (int i = c.tid; i < dsc->n_upd; i += CONSUMER_THREADS)
            a.block_table[size_t(dsc->upd[i][0]) * a.bt_stride + dsc->upd[i][1]] = dsc->upd[i][2];
    }
    int nt = s.d / 16;
    int items = DEC_MAXB * nt;
    for (int it = c.cta * DEC_NCW + c.warp; it < items; it += c.G * DEC_NCW) {
        int b = it / nt, tile = it % nt;
        float sq = 0.f;
        if (b < c.B && c.lane < 16) {
            int tok = ldcg_i32(a.last_tok + c.slot[b]);
            int row = tile * 16 + c.lane;
            float hv = bf16_to_f(a.w.emb[size_t(tok) * s.d + row]);
            a.h[size_t(b) * s.d + row] = hv;
            a.act[size_t(b) * s.d + row] = f_to_bf16(hv * a.w.g_attn[row]);
            sq = hv * hv;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        if (c.lane == 0) a.ssA[tile * 8 + b] = sq;
    }
}

__device__ void run_argmax_combine(Ctx& c, float best_v[2], int best_i[2]) {
    const DecodeArgs& a = *c.a;
    // reduce over the 8 lanes sharing t, then across warps through smem
#pragma unroll
    for (int j = 0; j < 2; ++j) {
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
            float ov = __shfl_xor_sync(0xffffffffu, best_v[j], o);
            int oi = __shfl_xor_sync(0xffffffffu, best_i[j], o);
            better(best_v[j], best_i[j], ov, oi);
        }
    }
    float* wv = c.sm.misc + 32;                              // [8 warps][8]
    int* wi = reinterpret_cast<int*>(c.sm.misc + 96);        // [8 warps][8]
    int* flag = reinterpret_cast<int*>(c.sm.misc + 16);
    if (c.lane < 4) {
        wv[c.warp * 8 + 2 * c.lane] = best_v[0];
        wi[c.warp * 8 + 2 * c.lane] = best_i[0];
        wv[c.warp * 8 + 2 * c.lane + 1] = best_v[1];
        wi[c.warp * 8 + 2 * c.lane + 1] = best_i[1];
    }
    csync();
    if (c.tid < DEC_MAXB) {
        float bv = -INFINITY;
        int bi = 0x7fffffff;
        for (int w = 0; w < DEC_NCW; ++w) better(bv, bi, wv[w * 8 + c.tid], wi[w * 8 + c.tid]);
        a.arg_val[c.cta * 8 + c.tid] = bv;
        a.arg_idx[c.cta * 8 + c.tid] = bi;
    }
    __threadfence();
    csync();
    if (c.tid == 0) {
        int old = atomicAdd(a.arg_cnt, 1);
        *flag = (old == c.G - 1);
    }
    csync();
    if (*flag) {
        __threadfence();
        if (c.tid < c.B) {
            float bv = -INFINITY;
            int bi = 0x7fffffff;
            for (int k = 0; k < c.G; ++k)
                better(bv, bi, ldcg_f32(a.arg_val + k * 8 + c.tid), ldcg_i32(a.arg_idx + k * 8 + c.tid));
            a.tok_out[c.tid] = bi;
            a.last_tok[c.slot[c.tid]] = bi;
        }
        if (c.tid == 0) atomicExch(a.arg_cnt, 0);
    }
}

__global__ void __launch_bounds__(DEC_THREADS, 1) decode_kernel(const __grid_constant__ DecodeArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    Smem sm = carve(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < DEC_NSTAGE; ++i) {
            mbar_init(&sm.full[i], 1);
            mbar_init(&sm.empty[i], 1);
        }
        fence_mbar_init();
    }
    // zero the accumulation buffers
    for (int i = threadIdx.x; i < 2 * DEC_MAXT * 128; i += DEC_THREADS) sm.acc[i] = 0.f;
    __syncthreads();

    if (warp == DEC_NCW) {
        if (lane == 0) producer_loop(a, sm, blockIdx.x, gridDim.x);
        return;
    }
    Ctx c;
    c.a = &a;
    c.sm = sm;
    c.cta = blockIdx.x;
    c.G = gridDim.x;
    c.warp = warp;
    c.lane = lane;
    c.tid = threadIdx.x;
    c.B = a.desc->B;
    for (int b = 0; b < DEC_MAXB; ++b) {
        c.slot[b] = b < c.B ? a.desc->slot[b] : 0;
        c.pos[b] = b < c.B ? a.desc->pos[b] : 0;
    }
    c.q = 0;
    c.off = 0;
    c.accbuf = 0;

    float best_v[2] = {-INFINITY, -INFINITY};
    int best_i[2] = {0x7fffffff, 0x7fffffff};

    run_embed(c);
    grid_sync(c);
    for (int l = 0; l < a.s.n_layers; ++l) {
        run_gemv(c, PH_QKV, l, best_v, best_i);
        grid_sync(c);
        run_attention(c, l);
        grid_sync(c);
        run_gemv(c, PH_O, l, best_v, best_i);
        grid_sync(c);
        run_gemv(c, PH_GU, l, best_v, best_i);
        grid_sync(c);
        run_gemv(c, PH_DOWN, l, best_v, best_i);
        grid_sync(c);
    }
    run_gemv(c, PH_LM, 0, best_v, best_i);
    run_argmax_combine(c, best_v, best_i);
}

}  // namespace

size_t decode_apart_floats(const Shape& s) {
    return size_t(DEC_MAXB) * s.n_kv * ATT_MAX_SPLITS * s.gq() * (s.dh + 2);
}

cudaError_t launch_decode(const DecodeArgs& a, int grid, cudaStream_t stream) {
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             DEC_SMEM_TOTAL);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    decode_kernel<<<grid, DEC_THREADS, DEC_SMEM_TOTAL, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace meshgpu
