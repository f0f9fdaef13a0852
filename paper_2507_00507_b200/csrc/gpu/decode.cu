// Decode step as ONE persistent kernel per instance step.
//
// Grid = the instance's SM quota (one CTA per SM). Every CTA runs a TMA
// producer warp that streams its share of ALL bytes of the step through a
// shared-memory ring with 1-D bulk copies (cp.async.bulk + mbarrier
// complete_tx): every layer's QKV, attention KV, O, gate/up and down, then
// lm_head. Neither the weights nor the KV of earlier tokens depend on this
// step's activations, so the stream runs ahead across the grid barriers that
// separate the phases; only the current token's K/V (written by this step's
// QKV phase) is read directly. Eight consumer warps wait for the ring and:
//   QKV   : 16-row weight tiles x (<= 8) activation columns on the tensor cores
//           (mma.m16n8k16, bf16 in / fp32 acc); RMSNorm scale, rotate-half RoPE,
//           q -> scratch, k/v -> paged KV cache
//   ATTN  : per-warp online softmax over 8 KB KV stages; partials combined in a
//           fixed order by the last contributor of each (request, kv head)
//   O     : residual add, next RMSNorm numerator, sum-of-squares partials
//   GU    : RMSNorm scale, silu(gate) * up
//   DOWN  : residual add, next RMSNorm numerator, sum-of-squares partials
//   LM    : final RMSNorm scale, optional logits, greedy argmax
// Weight tiles of single-segment phases with >= 4 tiles per CTA are claimed
// dynamically (per-phase counter, groups of up to 4 tiles, in tile order);
// the others are dealt round-robin across CTAs continuing from phase to phase,
// multi-segment ones segment-outer. Attention stages are dealt in contiguous
// ranges.
#include "decode.cuh"

#include <math.h>

namespace meshgpu {

namespace {

enum PhaseKind { PH_QKV = 0, PH_O = 1, PH_GU = 2, PH_DOWN = 3, PH_LM = 4 };

constexpr int CONSUMER_THREADS = DEC_NCW * 32;
__device__ __forceinline__ void csync() { named_bar_sync(1, CONSUMER_THREADS); }

struct GemvPhase {
    int kind, layer;
    int tiles;  // 16-row tiles
    int K;      // columns
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
    return {t0, t0 < tiles ? (tiles - 1 - t0) / G + 1 : 0};
}
__device__ __forceinline__ int n_segments(int K) {
    const int chunks = K / DEC_CHUNK_COLS, per = DEC_KSEG_MAX / DEC_CHUNK_COLS;
    return (chunks + per - 1) / per;
}
// Single-segment GEMV phases (the activation fits in shared memory: QKV, O,
// gate/up, lm_head) are scheduled dynamically: the producer claims groups of
// `claim_tiles` consecutive tiles from a per-phase counter and hands each
// claim to the consumers through a 4-deep descriptor ring. A CTA that streams
// slower (HBM channel contention varies from layer to layer: the static
// round-robin deal showed up to 18 us of barrier skew in a 68 us gate/up
// phase) simply claims fewer groups. Claims advance in tile order, so the CTAs
// still stream neighbouring tiles (DRAM row locality). Multi-segment phases
// (down: d_ff columns exceed the activation buffer) and phases with fewer than
// 4 tiles per CTA (where a claim round trip on the phase's critical path costs
// more than the imbalance it removes) keep the static round-robin deal.
__device__ __forceinline__ bool dynamic_phase(int K, int tiles, int G) { return K <= DEC_KSEG_MAX && tiles >= 4 * G; }
__device__ __forceinline__ int claim_tiles(int tiles, int G) { return max(1, min(DEC_MAXT, tiles / (2 * G))); }
__device__ __forceinline__ int claim_index(const Shape& s, int kind, int layer) {
    return kind == PH_LM ? s.n_layers * 4 : layer * 4 + kind;
}
__device__ __forceinline__ void seg_range(int K, int nseg, int s, int& c0, int& c1) {
    const int chunks = K / DEC_CHUNK_COLS;
    c0 = (chunks * s) / nseg;
    c1 = (chunks * (s + 1)) / nseg;
}

// Stages of the first `upto` activation segments of a segment-outer static phase.
__device__ __forceinline__ int seg_stages(int K, int nseg, int upto, int ntiles) {
    int c0, c1;
    seg_range(K, nseg, upto, c0, c1);  // c0 of segment `upto` = chunks before it
    (void)c1;
    return c0 * ntiles;
}

// ---- attention work plan (identical on producer and consumers) ----
// Stages enumerate (kv head, request b, chunk s of RT = 2048/dh tokens) in
// HEAD-major order; stage = the K and V rows of those tokens for one layer,
// 8 KB. Head-major puts each CTA's contiguous range on one or a few KV heads,
// so a CTA starts as soon as ITS heads' QKV tiles are done (the QKV tiles are
// claimed in group order): the tail of the QKV phase overlaps attention. Pair
// id of (b, kv head) = kvh * nb + b (consecutive in stage order).
struct AttnPlan {
    int rt;             // tokens per stage
    int nst[DEC_MAXB];  // stages per (b, kv head)
    int nb;             // requests
    int hst;            // stages per kv head (all requests)
    int total;          // stages per layer
    int a0, a1;         // this CTA's contiguous range
};
// c * total < 2^31 for every plan (<= 148 CTAs x 8 x 64 heads x 256 stages): 32-bit math
__device__ __forceinline__ int range_lo(int c, int total, int G) { return int(unsigned(c) * unsigned(total) / unsigned(G)); }
__device__ __forceinline__ AttnPlan attn_plan(const Shape& s, int B, const int* pos, int cta, int G) {
    AttnPlan p;
    p.rt = 2048 / s.dh;
    p.nb = B;
    p.hst = 0;
    for (int b = 0; b < DEC_MAXB; ++b) {
        p.nst[b] = b < B ? (pos[b] + p.rt) / p.rt : 0;  // ceil((pos + 1) / rt)
        p.hst += p.nst[b];
    }
    p.total = s.n_kv * p.hst;
    p.a0 = int(range_lo(cta, p.total, G));
    p.a1 = int(range_lo(cta + 1, p.total, G));
    return p;
}
struct AttnStage {
    int b, kvh, s, pair, pair_lo;  // pair_lo: global index of the pair's first stage
};
__device__ __forceinline__ AttnStage attn_stage_of(const AttnPlan& p, int n_kv, int i) {
    (void)n_kv;
    AttnStage st;
    st.kvh = i / p.hst;
    const int r = i - st.kvh * p.hst;
    int base = 0;
    for (int b = 0; b < p.nb; ++b) {
        if (r < base + p.nst[b]) {
            st.b = b;
            st.s = r - base;
            st.pair = st.kvh * p.nb + b;
            st.pair_lo = st.kvh * p.hst + base;
            return st;
        }
        base += p.nst[b];
    }
    st.b = st.kvh = st.s = st.pair = st.pair_lo = 0;
    return st;
}
__device__ __forceinline__ int cta_of_stage(int i, int total, int G) {
    return int((unsigned(i + 1) * unsigned(G) - 1u) / unsigned(total));
}
// Where a warp's partial for a (request, kv head) pair goes. Within a CTA the
// pair's stages [lo, hi) go to warps (i - a0) mod 8, i.e. n = min(8, hi - lo)
// consecutive warps. When n >= 2 (and the CTA's pair-local index k fits the
// shared staging area) the CTA pre-combines its n warp partials in shared
// memory and contributes ONE global partial; otherwise each warp contributes
// its own. rank/count index the pair's global partial slots deterministically.
constexpr int ATT_PT_MAX = 32;  // pairs per CTA with precomputed slot metadata
struct PairSlot {
    int pre;    // this CTA pre-combines the pair
    int k;      // pair-local index within this CTA's stage range
    int r, n;   // warp rank within the CTA's contributors, their number
    int rank;   // global slot of this contributor (the CTA when pre)
    int count;  // global partials of the pair
};
__device__ __forceinline__ PairSlot pair_slot(const AttnPlan& ap, int n_kv, int pair, int lo_p, int hi_p, int G,
                                              int cta, int warp, int cap_pairs) {
    PairSlot ps;
    ps.pre = 0;
    ps.k = ps.r = ps.n = 0;
    ps.rank = -1;
    ps.count = 0;
    const int c0 = cta_of_stage(lo_p, ap.total, G), c1 = cta_of_stage(hi_p - 1, ap.total, G);
    for (int c = c0; c <= c1; ++c) {
        const int a0 = int(range_lo(c, ap.total, G)), a1 = int(range_lo(c + 1, ap.total, G));
        const int lo = max(lo_p, a0), hi = min(hi_p, a1);
        if (hi <= lo) continue;
        const int n = min(8, hi - lo);
        const int k = pair - attn_stage_of(ap, n_kv, a0).pair;
        const int pre = n >= 2 && k < cap_pairs && k < ATT_PT_MAX;
        if (c == cta) {
            ps.pre = pre;
            ps.k = k;
            ps.n = n;
            ps.r = ((warp - (lo - a0)) % 8 + 8) % 8;
            ps.rank = pre ? ps.count : ps.count + ps.r;
        }
        ps.count += pre ? 1 : n;
    }
    return ps;
}

// Per-step slot metadata of the pairs this CTA's stage range touches (the
// attention plan is the same for every layer, so it is computed once).
struct AttnPair {
    int lo_p;          // pair's first global stage
    int pre, n, r0;    // CTA pre-combines; contributing warps; warp of the CTA's first stage of the pair
    int rank0, count;  // CTA's first global partial slot; the pair's global partial count
};

struct Smem {
    uint8_t* ring;
    uint16_t* act;
    float* acc;
    uint64_t* full;
    uint64_t* empty;
    float* misc;
    int* bt;  // [8][DEC_BT_MAX] block-table rows of the step's requests
    float* tacc;  // [DEC_TACC_TILES][128] per-tile sums across activation segments (down projection)
    // claim descriptors of dynamic GEMV phases (producer -> consumers)
    int* dt0;         // [4] first tile of the claim
    int* dgn;         // [4] tiles in the claim (0: phase exhausted)
    uint64_t* dfull;  // [4]
    uint64_t* dempty; // [4]
};

__device__ __forceinline__ Smem carve(uint8_t* base) {
    Smem m;
    m.ring = base;
    m.act = reinterpret_cast<uint16_t*>(base + DEC_SMEM_RING);
    m.acc = reinterpret_cast<float*>(base + DEC_SMEM_RING + DEC_SMEM_ACT);
    m.full = reinterpret_cast<uint64_t*>(base + DEC_SMEM_RING + DEC_SMEM_ACT + DEC_SMEM_ACC);
    m.empty = m.full + DEC_NSTAGE;
    m.misc = reinterpret_cast<float*>(base + DEC_SMEM_RING + DEC_SMEM_ACT + DEC_SMEM_ACC + DEC_SMEM_BARS);
    m.bt = reinterpret_cast<int*>(base + DEC_SMEM_RING + DEC_SMEM_ACT + DEC_SMEM_ACC + DEC_SMEM_BARS + DEC_SMEM_MISC);
    m.tacc = reinterpret_cast<float*>(base + DEC_SMEM_RING + DEC_SMEM_ACT + DEC_SMEM_ACC + DEC_SMEM_BARS +
                                      DEC_SMEM_MISC + DEC_SMEM_BT);
    return m;
}

// ----------------------------------------------------------------- producer
// The producer warp runs the stage enumeration uniformly on DEC_PLANES lanes;
// lane j captures the descriptor of stage qb + j, and every DEC_PLANES stages
// all lanes claim their ring slots and issue their bulk copies concurrently.
// One issuing thread serialises wait -> expect_tx -> copy at ~210 ns per stage
// (measured: tools/readbw.cu, 8 KB stages cap at 5.2 TB/s); 8 lanes reach
// 7.3 TB/s, above plain LDG streaming.
#ifndef DEC_PLANES_N
#define DEC_PLANES_N 8
#endif
constexpr int DEC_PLANES = DEC_PLANES_N;
// Lanes of the producer warp that run the stage enumeration: the first
// DEC_PLANES issue the batched GEMV stages; all of them issue the decoupled
// attention KV stages. Measured: 16 lanes made the batched GEMV path slower
// (the idle lanes ride along the enumeration) and faulted at 3B / 148 SMs; 32
// lanes would share ring slots (parity aliasing). 8 it is.
#ifndef DEC_PRODUCER_LANES_N
#define DEC_PRODUCER_LANES_N 8
#endif
constexpr int DEC_PRODUCER_LANES = DEC_PRODUCER_LANES_N;
constexpr unsigned DEC_PRODUCER_MASK = DEC_PRODUCER_LANES == 32 ? 0xffffffffu : (1u << DEC_PRODUCER_LANES) - 1u;

struct StageSrc {
    const uint8_t* p0;  // weight tile chunk, or the K row block of the first KV block
    const uint8_t* p1;  // K row block of the second KV block (dh = 64); weight stage: end of its matrix
    int nblk;           // -1: weight stage; else KV blocks in the stage (0..2)
};

struct Producer {
    const DecodeArgs& a;
    Smem& sm;
    const int lane;
    uint32_t q = 0;    // stages enumerated
    uint32_t qb = 0;   // first stage of the pending batch
    uint32_t nsh, nmask;
    uint64_t pol;
    uint32_t kv_blk;   // bytes of one (layer, head, k|v) block; its K and V are adjacent
    StageSrc mine;     // this lane's pending stage
    const uint8_t* wend = nullptr;  // end of the current GEMV phase's weight matrix (prefetch bound)
    uint32_t dk = 0;   // claim descriptors written
    __device__ __forceinline__ Producer(const DecodeArgs& args, Smem& s, int ln) : a(args), sm(s), lane(ln) {
        nsh = uint32_t(__ffs(a.nstage) - 1);
        nmask = uint32_t(a.nstage) - 1u;
        pol = l2_evict_first_policy();
        kv_blk = uint32_t(KV_BLOCK_TOKENS * a.s.dh * 2);
        mine.p0 = mine.p1 = nullptr;
        mine.nblk = -1;
    }
    __device__ __forceinline__ void flush() {
        const uint32_t n = q - qb;
        if (uint32_t(lane) < n) {
            const uint32_t qi = qb + uint32_t(lane);
            const uint32_t slot = qi & nmask, par = (qi >> nsh) & 1u;
            mbar_wait(&sm.empty[slot], par ^ 1u);
            uint8_t* dst = sm.ring + size_t(slot) * DEC_STAGE_BYTES;
            if (mine.nblk < 0) {
                mbar_arrive_expect_tx(&sm.full[slot], DEC_STAGE_BYTES);
                bulk_g2s_evict_first(dst, mine.p0, DEC_STAGE_BYTES, &sm.full[slot], pol);
                // Weight tiles are contiguous and claimed in address order: pulling the
                // bytes a few stages ahead into L2 now lets the ring's copy of them hit
                // L2 later, so more bytes are in flight per SM than the ring holds.
                const uint8_t* ahead = mine.p0 + size_t(a.l2pf) * DEC_STAGE_BYTES;
                if (a.l2pf && ahead < mine.p1) bulk_prefetch_l2(ahead, DEC_STAGE_BYTES);
            } else {
                // one copy per KV block: [K rows | V rows] of the (layer, head)
                mbar_arrive_expect_tx(&sm.full[slot], 2u * uint32_t(mine.nblk) * kv_blk);
                if (mine.nblk > 0) bulk_g2s(dst, mine.p0, 2u * kv_blk, &sm.full[slot]);
                if (mine.nblk > 1) bulk_g2s(dst + 2u * kv_blk, mine.p1, 2u * kv_blk, &sm.full[slot]);
            }
        }
        qb = q;
    }
    __device__ __forceinline__ void push(const uint8_t* p0, const uint8_t* p1, int nblk) {
        if (uint32_t(lane) == q - qb) {
            mine.p0 = p0;
            mine.p1 = p1;
            mine.nblk = nblk;
        }
        if (++q - qb == DEC_PLANES) flush();
    }
    // Weight stages [q, q + n) issued by decoupled lanes (lane j: stages j, j + P,
    // ...), each waiting only for its own ring slot; addr_of(i) = source of stage i.
    template <typename AddrOf>
    __device__ __forceinline__ void issue_lanes(int n, AddrOf addr_of) {
        flush();
        const uint32_t q0 = q;
        for (int i = lane; i < n; i += DEC_PLANES) {
            const uint32_t qi = q0 + uint32_t(i);
            const uint32_t slot = qi & nmask, par = (qi >> nsh) & 1u;
            const uint8_t* src = addr_of(i);
            mbar_wait(&sm.empty[slot], par ^ 1u);
            mbar_arrive_expect_tx(&sm.full[slot], DEC_STAGE_BYTES);
            bulk_g2s_evict_first(sm.ring + size_t(slot) * DEC_STAGE_BYTES, src, DEC_STAGE_BYTES, &sm.full[slot], pol);
        }
        __syncwarp(DEC_PRODUCER_MASK);
        q = qb = q0 + uint32_t(n);
    }
    __device__ __forceinline__ void gemv_dynamic(int kind, int layer, int G) {
        const GemvPhase p = gemv_phase(a, kind, layer);
        wend = p.base + size_t(p.tiles) * p.K * 32;
        const int cl_big = claim_tiles(p.tiles, G), nch = p.K / DEC_CHUNK_COLS;
        int* ctr = a.claim + claim_index(a.s, kind, layer);
        const size_t tile_bytes = size_t(p.K) * 32;
        int cl = cl_big, next = 0;
        if (lane == 0) next = atomicAdd(ctr, cl);
        for (;;) {
            const int t0 = __shfl_sync(DEC_PRODUCER_MASK, next, 0);
            const int gn = max(0, min(cl, p.tiles - t0));
            // issue every pending stage first: the consumers may need them to
            // get to the descriptor slot this claim waits for
            flush();
            const uint32_t ds = dk & 3u, dpar = (dk >> 2) & 1u;
            if (lane == 0) {
                mbar_wait(&sm.dempty[ds], dpar ^ 1u);
                sm.dt0[ds] = t0;
                sm.dgn[ds] = gn;
                mbar_arrive(&sm.dfull[ds]);
            }
            ++dk;
            if (gn == 0) return;
            if (a.w_lanes) {
                const uint8_t* g0 = p.base + size_t(t0) * tile_bytes;  // the group's tiles are contiguous
                issue_lanes(gn * nch, [&](int i) { return g0 + size_t(i) * DEC_STAGE_BYTES; });
            } else {
                for (int ti = 0; ti < gn; ++ti) {
                    const uint8_t* t = p.base + size_t(t0 + ti) * tile_bytes;
                    for (int ch = 0; ch < nch; ++ch) push(t + size_t(ch) * DEC_STAGE_BYTES, wend, -1);
                }
            }
            // Next claim once this group's stages are issued: a ring's depth of them is
            // still to be consumed, which hides the round trip, and a CTA that streams
            // slowly claims late. Guided sizes (remaining / 2G, at most cl_big, at
            // least 1) end the phase on single tiles, so the tail imbalance across
            // CTAs is about one tile.
            cl = max(1, min(cl_big, (p.tiles - (t0 + gn)) / (2 * G)));
            if (lane == 0) next = atomicAdd(ctr, cl);
        }
    }
    __device__ __forceinline__ void gemv(int kind, int layer, int& off, int cta, int G) {
        const GemvPhase p = gemv_phase(a, kind, layer);
        if (dynamic_phase(p.K, p.tiles, G)) {
            gemv_dynamic(kind, layer, G);
            return;
        }
        const MyTiles mt = my_tiles(p.tiles, off, cta, G);
        off = (off + p.tiles) % G;
        if (mt.n == 0) return;
        wend = p.base + size_t(p.tiles) * p.K * 32;
        const size_t tile_bytes = size_t(p.K) * 32;
        const int nseg = n_segments(p.K);
        if (a.w_lanes && nseg == 1) {
            const int nch = p.K / DEC_CHUNK_COLS;
            issue_lanes(mt.n * nch, [&](int i) {
                const int ti = i / nch, ch = i - ti * nch;
                return p.base + size_t(mt.t0 + ti * G) * tile_bytes + size_t(ch) * DEC_STAGE_BYTES;
            });
            return;
        }
        if (nseg > 1 && mt.n <= DEC_TACC_TILES) {
            // segment-outer, as the consumers run it (run_gemv): every tile's
            // chunks of segment 0, then of segment 1, ...
            if (a.w_lanes) {
                issue_lanes(seg_stages(p.K, nseg, nseg, mt.n), [&](int i) {
                    int sg = 0;
                    while (i >= seg_stages(p.K, nseg, sg + 1, mt.n)) ++sg;
                    int c0, c1;
                    seg_range(p.K, nseg, sg, c0, c1);
                    const int r = i - seg_stages(p.K, nseg, sg, mt.n), w = c1 - c0;
                    const int ti = r / w, ch = c0 + (r - ti * w);
                    return p.base + size_t(mt.t0 + ti * G) * tile_bytes + size_t(ch) * DEC_STAGE_BYTES;
                });
                return;
            }
            for (int sg = 0; sg < nseg; ++sg) {
                int c0, c1;
                seg_range(p.K, nseg, sg, c0, c1);
                for (int ti = 0; ti < mt.n; ++ti) {
                    const uint8_t* t = p.base + size_t(mt.t0 + ti * G) * tile_bytes;
                    for (int ch = c0; ch < c1; ++ch) push(t + size_t(ch) * DEC_STAGE_BYTES, wend, -1);
                }
            }
            return;
        }
        for (int g0 = 0; g0 < mt.n; g0 += DEC_MAXT) {
            const int gn = min(DEC_MAXT, mt.n - g0);
            for (int sg = 0; sg < nseg; ++sg) {
                int c0, c1;
                seg_range(p.K, nseg, sg, c0, c1);
                for (int ti = 0; ti < gn; ++ti) {
                    const uint8_t* t = p.base + size_t(mt.t0 + (g0 + ti) * G) * tile_bytes;
                    for (int ch = c0; ch < c1; ++ch) push(t + size_t(ch) * DEC_STAGE_BYTES, wend, -1);
                }
            }
        }
    }
    // KV stages of this CTA's attention range: only blocks that were complete
    // before this step (every position < pos) are streamed; the current token
    // is read directly by the consumer.
    int ntr = 0;
    __device__ __forceinline__ void ptrace(int cta, int tag) {  // producer timeline (CTA 0) at trace[2048..]
        if (a.trace && cta == 0 && lane == 0 && ntr < 2000) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            a.trace[2048 + ntr++] = (t << 4) | unsigned(tag);
        }
    }
    // KV stages with the issuing lanes decoupled: lane j walks stages a0 + j,
    // a0 + j + P, ... on its own, waiting only for its own ring slots. A KV stage
    // (one (layer, head) run of a paged block, its own 2 MB page at 3B/7B) has a
    // long and variable latency; in the batched push/flush a batch of P copies
    // waits for its slowest slot, which kept the attention stream at ~30 GB/s per
    // SM at the lanes' quotas (weights: ~50).
    __device__ __forceinline__ void attention_lanes(int layer, const AttnPlan& ap, const int* pos) {
        flush();  // the previous phase's pending stages go first (q == qb)
        if (ap.a1 <= ap.a0) return;
        const Shape& s = a.s;
        const int bps = ap.rt / KV_BLOCK_TOKENS;
        const size_t head_stride = size_t(2) * KV_BLOCK_TOKENS * s.dh * 2;
        const uint8_t* layer_base = a.kv_base + kv_offset(s, layer, 0, 0, 0);
        const uint32_t q0 = q;
        // lane's first stage decoded once, then walked DEC_PRODUCER_LANES stages at a time
        AttnStage st = attn_stage_of(ap, s.n_kv, min(ap.a0 + lane, ap.a1 - 1));
        for (int i = ap.a0 + lane; i < ap.a1; i += DEC_PRODUCER_LANES) {
            const int k0 = st.s * bps, p = pos[st.b];
            int nblk = 0;
            if (k0 * KV_BLOCK_TOKENS < p) nblk = (bps == 2 && (k0 + 1) * KV_BLOCK_TOKENS < p) ? 2 : 1;
            if (a.skip & 4) nblk = 0;
            const int* btrow = sm.bt + st.b * DEC_BT_MAX;
            const size_t hoff = size_t(st.kvh) * head_stride;
            const uint32_t qi = q0 + uint32_t(i - ap.a0);
            const uint32_t slot = qi & nmask, par = (qi >> nsh) & 1u;
            mbar_wait(&sm.empty[slot], par ^ 1u);
            uint8_t* dst = sm.ring + size_t(slot) * DEC_STAGE_BYTES;
            mbar_arrive_expect_tx(&sm.full[slot], 2u * uint32_t(nblk) * kv_blk);
            if (nblk > 0) bulk_g2s(dst, layer_base + size_t(btrow[k0]) * a.block_bytes + hoff, 2u * kv_blk, &sm.full[slot]);
            if (nblk > 1)
                bulk_g2s(dst + 2u * kv_blk, layer_base + size_t(btrow[k0 + 1]) * a.block_bytes + hoff, 2u * kv_blk,
                         &sm.full[slot]);
            st.s += DEC_PRODUCER_LANES;  // next stage of this lane: requests inner, kv heads outer
            while (st.s >= ap.nst[st.b]) {
                st.s -= ap.nst[st.b];
                if (++st.b == ap.nb) {
                    st.b = 0;
                    ++st.kvh;
                }
                if (st.kvh >= s.n_kv) break;  // past the last stage (the loop ends)
            }
        }
        __syncwarp(DEC_PRODUCER_MASK);
        q = qb = q0 + uint32_t(ap.a1 - ap.a0);
    }
    // KV stages of this CTA's attention range: only blocks that were complete
    // before this step (every position < pos) are streamed; the current token
    // is read directly by the consumer. The (b, kv head, chunk) walk is
    // incremental and all per-layer offsets are hoisted: the single producer
    // thread must issue a stage every ~100 cycles to keep up with HBM.
    __device__ __forceinline__ void attention(int layer, const AttnPlan& ap, const int* pos) {
        if (ap.a1 <= ap.a0) return;
        const Shape& s = a.s;
        const int bps = ap.rt / KV_BLOCK_TOKENS;  // blocks per stage
        const size_t head_stride = size_t(2) * KV_BLOCK_TOKENS * s.dh * 2;  // K + V of one head
        const uint8_t* layer_base = a.kv_base + kv_offset(s, layer, 0, 0, 0);
        // decode the first stage once, then walk
        AttnStage st = attn_stage_of(ap, s.n_kv, ap.a0);
        int b = st.b, kvh = st.kvh, sc = st.s;
        int nst_b = ap.nst[b];
        int p = pos[b];
        const int* btrow = sm.bt + b * DEC_BT_MAX;
        for (int i = ap.a0; i < ap.a1; ++i) {
            const int k0 = sc * bps;
            int nblk = 0;
            if (k0 * KV_BLOCK_TOKENS < p) nblk = (bps == 2 && (k0 + 1) * KV_BLOCK_TOKENS < p) ? 2 : 1;
            if (a.skip & 4) nblk = 0;  // debug: no KV traffic
            const size_t hoff = size_t(kvh) * head_stride;
            const uint8_t* kb0 = nblk > 0 ? layer_base + size_t(btrow[k0]) * a.block_bytes + hoff : nullptr;
            const uint8_t* kb1 = nblk > 1 ? layer_base + size_t(btrow[k0 + 1]) * a.block_bytes + hoff : nullptr;
            push(kb0, kb1, nblk);
            if (++sc == nst_b) {  // next (kv head, b): requests inner
                sc = 0;
                if (++b == ap.nb) {
                    b = 0;
                    ++kvh;
                }
                nst_b = ap.nst[b];
                p = pos[b];
                btrow = sm.bt + b * DEC_BT_MAX;
            }
        }
    }
};

__device__ __forceinline__ void producer_loop(const DecodeArgs& a, Smem& sm, int cta, int G, int B, const int* pos,
                                              int lane) {
    if (a.skip & 2) return;
    Producer pr(a, sm, lane);
    const AttnPlan ap = attn_plan(a.s, B, pos, cta, G);
    int off = 0;
    // one call site per phase body (see the consumer loop)
    const int L = a.s.n_layers;
#pragma unroll 1
    for (int it = 0; it <= 4 * L; ++it) {
        const int kind = it == 4 * L ? int(PH_LM) : (it & 3), l = it == 4 * L ? 0 : (it >> 2);
        if (kind == PH_QKV) pr.ptrace(cta, 8);
        pr.gemv(kind, l, off, cta, G);
        if (kind == PH_QKV && !(a.skip & 1)) {
            if (a.kv_lanes)
                pr.attention_lanes(l, ap, pos);
            else
                pr.attention(l, ap, pos);
        }
        if (kind == PH_DOWN && a.progress && lane == 0) a.progress[cta * 2 + 1] = int(pr.q);
    }
    pr.flush();
}

// ----------------------------------------------------------------- consumer
struct Ctx {
    int ntrace;           // trace cursor (CTA 0, thread 0)
    int nbar;             // grid barriers passed
    const DecodeArgs* a;  // shared-memory copy of the launch arguments
    Smem sm;
    int cta, G, warp, lane, tid;  // tid in [0, 256)
    int B;
    const int* slot;  // [8] in shared memory
    const int* pos;   // [8] in shared memory
    const int* cur_blk;  // [8] in shared memory: block holding each request's current token (-1: read the table)
    const AttnPair* pt;  // [ATT_PT_MAX] in shared memory
    int p0, np;          // first pair of this CTA's attention range, pairs touched
    uint32_t q;       // stage counter (mirrors the producer)
    uint32_t nsh, nmask;  // ring depth = 1 << nsh (8 or 16)
    int off;          // round-robin offset of static phases (mirrors the producer)
    uint32_t dk;      // claim descriptors read (mirrors the producer)
    uint64_t* actbar; // activation bulk-load mbarrier
    uint32_t actph;   // its phase
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// tag: 1 phase begin, 2 operands ready, 3 stages consumed, 4 epilogue done, 5 barrier passed,
//      6 attention begin, 7 attention end
__device__ __forceinline__ void trace(Ctx& c, int tag) {
    if (c.a->trace && c.cta == 0 && c.tid == 0 && c.ntrace < 4000)
        c.a->trace[c.ntrace++] = (gtimer() << 4) | unsigned(tag);
}
__device__ __forceinline__ void grid_sync(Ctx& c) {
    csync();
    if (c.a->arrive && c.tid == 0 && c.nbar < 256) c.a->arrive[size_t(c.nbar) * c.G + c.cta] = gtimer();
    ++c.nbar;
    if (c.a->progress && c.tid == 0) c.a->progress[c.cta * 2] += 1;
    if (c.tid == 0) grid_barrier_mono(c.a->bar_count, unsigned(c.nbar) * unsigned(c.G));
    csync();
    trace(c, 5);
}

__device__ __forceinline__ void wait_stage(Ctx& c, uint32_t qi, uint32_t& slot) {
    slot = qi & c.nmask;
    mbar_wait(&c.sm.full[slot], (qi >> c.nsh) & 1u);
}
__device__ __forceinline__ void release_stage(Ctx& c, uint32_t slot) {
    __syncwarp();
    if (c.lane == 0) mbar_arrive(&c.sm.empty[slot]);
}

// Activation columns [k0, k1) of the B batch rows (bf16, global) into smem
// (row stride k1 - k0 + 8) with one bulk copy per row, all issued at once by
// one thread on the activation mbarrier: the whole operand is one L2 round trip
// plus its transfer (the per-thread 16-byte loads it replaces took ~5 us for a
// 64 KB 7B operand under the phase's HBM load). Rows >= B are left as they are:
// they only feed mma columns whose results are discarded. Called by every
// consumer thread between csync()s.
__device__ __forceinline__ void load_act(Ctx& c, const uint16_t* src, int ld, int k0, int k1) {
    const int n = k1 - k0, stride = n + 8;
    if (c.tid == 0) {
        // the rows were written by other CTAs' generic stores (visible through the
        // grid barrier's acquire) and the destination was read by generic loads:
        // order both before the async-proxy copies
        asm volatile("fence.proxy.async.global;\n" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_arrive_expect_tx(c.actbar, uint32_t(c.B * n * 2));
        for (int b = 0; b < c.B; ++b)
            bulk_g2s(c.sm.act + b * stride, src + size_t(b) * ld + k0, uint32_t(n * 2), c.actbar);
    }
    mbar_wait(c.actbar, c.actph & 1u);
    ++c.actph;
}

// load_act + the RMSNorm scale rs[b] = 1/sqrt(mean(h_b^2) + eps) from the
// per-tile sum-of-squares partials (summed in a fixed order; warp b <-> batch
// column b). The partial loads are issued first, so the two L2 round trips of
// a normed phase's prologue overlap.
__device__ __forceinline__ void load_act_rs(Ctx& c, const uint16_t* src, int ld, int k0, int k1, const float* ss,
                                            float* rs_out) {
    const DecodeArgs& a = *c.a;
    const int nt = a.s.d / 16;
    const int b = c.warp;
    float pv[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const int t = c.lane + 32 * k;
        pv[k] = t < nt ? ldcg_f32(ss + t * 8 + b) : 0.f;
    }
    load_act(c, src, ld, k0, k1);
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k) acc += pv[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (c.lane == 0) rs_out[b] = rsqrtf(acc / float(a.s.d) + a.s.eps);
}

// One 8 KB weight stage: 16 rows x 256 columns against the 8 activation
// columns, accumulated into the warp's registers (two chains for ILP).
__device__ __forceinline__ void consume_stage(Ctx& c, uint32_t qi, int act_col, int act_stride, float (&d0)[4],
                                              float (&d1)[4]) {
    uint32_t slot;
    wait_stage(c, qi, slot);
    if (c.a->skip & 16) {  // debug: ring handshake only (results are garbage)
        release_stage(c, slot);
        return;
    }
    const uint32_t stage_addr = smem_u32(c.sm.ring + size_t(slot) * DEC_STAGE_BYTES);
    const int lane = c.lane, r = lane & 15, g = lane >> 2, t = lane & 3;
    const uint16_t* actrow = c.sm.act + g * act_stride + act_col + 2 * t;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const int kb = j >> 2, chunk = ((j & 3) << 1) + (lane >> 4);
        uint32_t a0, a1, a2, a3;
        ldmatrix_x4(stage_addr + kb * 2048 + r * 128 + (uint32_t((chunk ^ (r & 7))) << 4), a0, a1, a2, a3);
        const uint32_t b0 = *reinterpret_cast<const uint32_t*>(actrow + j * 16);
        const uint32_t b1 = *reinterpret_cast<const uint32_t*>(actrow + j * 16 + 8);
        if (j & 1)
            mma_bf16_16816(d1, a0, a1, a2, a3, b0, b1);
        else
            mma_bf16_16816(d0, a0, a1, a2, a3, b0, b1);
    }
    release_stage(c, slot);
}

// Epilogue operands that do not depend on the tile's sums (the residual rows
// and the next norm's gamma for O / down, the RoPE (cos, sin) for QKV), loaded
// by the warp that will run the tile's epilogue BEFORE it consumes the stages:
// the loads' L2 round trip overlaps the stage loop instead of sitting on the
// phase's critical path (the epilogue of a single tile took ~2 us at 148 SMs).
struct EpiPre {
    int tile;     // -1: nothing prefetched
    float x[6];   // O / down: h[4] = x[0..3], gamma[2] = x[4..5]; QKV: (cos, sin)[2] = x[0..3]
};
__device__ __forceinline__ const float* gamma_after(const DecodeArgs& a, int kind, int layer) {
    if (kind == PH_O) return a.w.g_mlp + size_t(layer) * a.s.d;
    return (layer + 1 < a.s.n_layers) ? a.w.g_attn + size_t(layer + 1) * a.s.d : a.w.g_final;
}
__device__ __forceinline__ EpiPre epi_prefetch(const Ctx& c, int kind, int layer, int tile) {
    const DecodeArgs& a = *c.a;
    const Shape& s = a.s;
    EpiPre e;
    e.tile = tile;
    const int g = c.lane >> 2, t = c.lane & 3;
#pragma unroll
    for (int k = 0; k < 6; ++k) e.x[k] = 0.f;
    if (tile < 0) return e;
    if (kind == PH_O || kind == PH_DOWN) {
        const float* gam = gamma_after(a, kind, layer);
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
            const int row = tile * 16 + g + 8 * rr;
            e.x[4 + rr] = gam[row];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int b = 2 * t + j;
                if (b < c.B) e.x[2 * rr + j] = ldcg_f32(a.h + size_t(b) * s.d + row);
            }
        }
    } else if (kind == PH_QKV) {
        const QkvRow r1 = qkv_row(s, tile * 16 + g);
        if (r1.section < 2) {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int b = 2 * t + j;
                if (b < c.B) {
                    const float2 cs = a.w.rope[size_t(c.pos[b]) * (s.dh / 2) + r1.dim];
                    e.x[2 * j] = cs.x;
                    e.x[2 * j + 1] = cs.y;
                }
            }
        }
    }
    return e;
}

// ---- GEMV epilogues: lane holds rows (g, g+8) x batch columns (2t, 2t+1) of `tile`.
__device__ __forceinline__ void epi_qkv(Ctx& c, int layer, int tile, const float v[4], const float* rs,
                                        const EpiPre& pre) {
    const DecodeArgs& a = *c.a;
    const Shape& s = a.s;
    const int g = c.lane >> 2, t = c.lane & 3;
    const QkvRow r1 = qkv_row(s, tile * 16 + g);  // dim in [0, dh/2); row g+8 is dim + dh/2
    const int half = s.dh / 2;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int b = 2 * t + j;
        if (b >= c.B) continue;
        const float x1 = v[j] * rs[b], x2 = v[2 + j] * rs[b];
        const int pos = c.pos[b];
        float o1 = x1, o2 = x2;
        if (r1.section < 2) {
            const float2 cs = pre.tile == tile ? make_float2(pre.x[2 * j], pre.x[2 * j + 1])
                                               : a.w.rope[size_t(pos) * half + r1.dim];
            o1 = x1 * cs.x - x2 * cs.y;
            o2 = x2 * cs.x + x1 * cs.y;
        }
        if (r1.section == 0) {
            float* qd = a.q + (size_t(b) * s.n_heads + r1.head) * s.dh;
            qd[r1.dim] = o1;
            qd[r1.dim + half] = o2;
        } else {
            const int blk = c.cur_blk[b] >= 0 ? c.cur_blk[b]
                                              : ldcg_i32(a.block_table + size_t(c.slot[b]) * a.bt_stride + pos / KV_BLOCK_TOKENS);
            const int slot = pos % KV_BLOCK_TOKENS;
            uint8_t* e = a.kv_base + size_t(blk) * a.block_bytes + kv_offset(s, layer, r1.section - 1, r1.head, slot);
            *reinterpret_cast<uint16_t*>(e + kv_dim_off(slot, r1.dim)) = f_to_bf16(o1);
            *reinterpret_cast<uint16_t*>(e + kv_dim_off(slot, r1.dim + half)) = f_to_bf16(o2);
        }
    }
}

__device__ __forceinline__ void epi_gu(Ctx& c, int tile, const float v[4], const float* rs) {
    const DecodeArgs& a = *c.a;
    const int g = c.lane >> 2, t = c.lane & 3;
    const int row = tile * 8 + g;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int b = 2 * t + j;
        if (b >= c.B) continue;
        const float gt = v[j] * rs[b], up = v[2 + j] * rs[b];
        a.abuf[size_t(b) * a.s.ff + row] = f_to_bf16(gt / (1.f + __expf(-gt)) * up);
    }
}

// Residual add for the rows this tile owns, the next RMSNorm's numerator and
// the per-tile sum of squares.
__device__ __forceinline__ void epi_residual(Ctx& c, int tile, const float v[4], const float* gamma_next,
                                             float* ss_out, const EpiPre& pre) {
    const bool have = pre.tile == tile;
    const DecodeArgs& a = *c.a;
    const int d = a.s.d;
    const int g = c.lane >> 2, t = c.lane & 3;
    float sq[2] = {0.f, 0.f};
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
        const int row = tile * 16 + g + 8 * rr;
        const float gm = have ? pre.x[4 + rr] : gamma_next[row];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int b = 2 * t + j;
            if (b >= c.B) continue;
            float* hp = a.h + size_t(b) * d + row;
            const float hv = (have ? pre.x[2 * rr + j] : ldcg_f32(hp)) + v[2 * rr + j];
            *hp = hv;
            a.act[size_t(b) * d + row] = f_to_bf16(hv * gm);
            sq[j] += hv * hv;
        }
    }
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) sq[j] += __shfl_xor_sync(0xffffffffu, sq[j], o);
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
// Stages of a group of gn tiles (one activation segment [c0, c1) of chunks),
// tile-major. Warp w consumes stages c.q + w + 8k: a warp's consecutive stages
// are exactly DEC_NCW apart, so it never waits on a ring slot a full cycle
// ahead (mbarrier parity would alias). Partial sums stay in registers while
// the warp's stages belong to one tile and are flushed to its part[] slot.
__device__ __forceinline__ void consume_group(Ctx& c, int gn, int sg, int nch) {
    float* part = c.sm.acc;  // per-warp partial sums: part[warp][tile][lane * 4 + e]
    const int n = gn * nch, act_stride = nch * DEC_CHUNK_COLS + 8;
    if (sg == 0)
        for (int ti = 0; ti < gn; ++ti)
            reinterpret_cast<float4*>(part + (c.warp * DEC_MAXT + ti) * 128)[c.lane] = make_float4(0.f, 0.f, 0.f, 0.f);
    float d0[4] = {0.f, 0.f, 0.f, 0.f}, d1[4] = {0.f, 0.f, 0.f, 0.f};
    int cur = -1;
    auto flush = [&](int ti) {
        float4* dst = reinterpret_cast<float4*>(part + (c.warp * DEC_MAXT + ti) * 128) + c.lane;
        const float4 o = *dst;
        *dst = make_float4(o.x + d0[0] + d1[0], o.y + d0[1] + d1[1], o.z + d0[2] + d1[2], o.w + d0[3] + d1[3]);
#pragma unroll
        for (int e = 0; e < 4; ++e) d0[e] = d1[e] = 0.f;
    };
    // (tile, chunk) of stage i walked incrementally (no per-stage integer division)
    int ti = c.warp / nch, ch = c.warp - (c.warp / nch) * nch;
    for (int i = c.warp; i < n; i += DEC_NCW) {
        if (ti != cur) {
            if (cur >= 0) flush(cur);
            cur = ti;
        }
        consume_stage(c, c.q + i, ch * DEC_CHUNK_COLS, act_stride, d0, d1);
        ch += DEC_NCW;
        while (ch >= nch) {
            ch -= nch;
            ++ti;
        }
    }
    if (cur >= 0) flush(cur);
    c.q += n;
}

// Epilogue of a group: one warp per tile, summing the eight warps' partials.
// Sum of the eight warps' partials of group tile ti (lane's 4 values).
__device__ __forceinline__ float4 warp_sum(const Ctx& c, int ti) {
    const float* part = c.sm.acc;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int w = 0; w < DEC_NCW; ++w) {
        const float4 pv = reinterpret_cast<const float4*>(part + (w * DEC_MAXT + ti) * 128)[c.lane];
        v.x += pv.x;
        v.y += pv.y;
        v.z += pv.z;
        v.w += pv.w;
    }
    return v;
}

// tacc_base >= 0: the tile sums were accumulated across segments in tacc[tacc_base + ti]
template <typename TileOf>
__device__ __forceinline__ void epilogue_group(Ctx& c, int kind, int layer, int gn, TileOf tile_of, const float* rs,
                                               float* best_v, int* best_i, const EpiPre& pre, int tacc_base = -1) {
    const DecodeArgs& a = *c.a;
    for (int ti = c.warp; ti < gn; ti += DEC_NCW) {
        const int tile = tile_of(ti);
        const float4 sv = tacc_base >= 0 ? reinterpret_cast<const float4*>(c.sm.tacc + (tacc_base + ti) * 128)[c.lane]
                                         : warp_sum(c, ti);
        float v[4] = {sv.x, sv.y, sv.z, sv.w};
        switch (kind) {
            case PH_QKV:
                epi_qkv(c, layer, tile, v, rs, pre);
                // publish the tile to the attention of its KV-head group (no grid barrier
                // between QKV and attention): one count per tile. The lanes' stores are
                // ordered before lane 0's release by the warp barrier and the release's
                // cumulativity (the attention partials use the same pattern); a
                // __threadfence here made every lane wait for its stores to reach L2.
                __syncwarp();
                if (c.lane == 0)
                    asm volatile("red.release.gpu.global.add.s32 [%0], 1;\n" ::"l"(a.qkv_done + tile / qkv_group_tiles(a.s))
                                 : "memory");
                break;
            case PH_GU: epi_gu(c, tile, v, rs); break;
            case PH_O: epi_residual(c, tile, v, gamma_after(a, PH_O, layer), a.ssB, pre); break;
            case PH_DOWN: epi_residual(c, tile, v, gamma_after(a, PH_DOWN, layer), a.ssA, pre); break;
            default: {  // lm_head
                const int g = c.lane >> 2, t = c.lane & 3;
#pragma unroll
                for (int rr = 0; rr < 2; ++rr) {
                    const int row = tile * 16 + g + 8 * rr;
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const int b = 2 * t + j;
                        if (b >= c.B) continue;
                        const float logit = v[2 * rr + j] * rs[b];
                        if (a.logits) a.logits[size_t(b) * a.s.vocab + row] = logit;
                        better(best_v[j], best_i[j], logit, row);
                    }
                }
                break;
            }
        }
    }
}

__device__ __forceinline__ void run_gemv(Ctx& c, int kind, int layer, float* best_v, int* best_i) {
    const DecodeArgs& a = *c.a;
    const GemvPhase p = gemv_phase(a, kind, layer);
    trace(c, 1);
    if (a.skip & 2) return;
    float* rs = c.sm.misc;  // [8]
    // the RMSNorm scale is folded into the first activation load (both L2 round trips overlap)
    const float* ss = (kind == PH_QKV || kind == PH_LM) ? a.ssA : (kind == PH_GU ? a.ssB : nullptr);
    const uint16_t* src;
    int ld;
    switch (kind) {
        case PH_O: src = a.attn; ld = a.s.d; break;
        case PH_DOWN: src = a.abuf; ld = a.s.ff; break;
        default: src = a.act; ld = a.s.d; break;
    }
    if (dynamic_phase(p.K, p.tiles, c.G)) {
        // the whole activation fits: load it once (overlaps the producer's first claim)
        csync();
        if (ss)
            load_act_rs(c, src, ld, 0, p.K, ss, rs);
        else
            load_act(c, src, ld, 0, p.K);
        csync();
        trace(c, 2);
        const int nch = p.K / DEC_CHUNK_COLS;
        for (;;) {
            const uint32_t ds = c.dk & 3u;
            mbar_wait(&c.sm.dfull[ds], (c.dk >> 2) & 1u);
            const int t0 = c.sm.dt0[ds], gn = c.sm.dgn[ds];
            ++c.dk;
            if (gn == 0) {
                csync();  // every consumer read the terminal descriptor
                if (c.tid == 0) mbar_arrive(&c.sm.dempty[ds]);
                return;
            }
            const EpiPre pre = epi_prefetch(c, kind, layer, c.warp < gn ? t0 + c.warp : -1);
            consume_group(c, gn, 0, nch);
            csync();
            if (c.tid == 0) mbar_arrive(&c.sm.dempty[ds]);  // every consumer read it before the csync
            trace(c, 3);
            epilogue_group(c, kind, layer, gn, [&](int ti) { return t0 + ti; }, rs, best_v, best_i, pre);
            csync();  // partials are rewritten by the next group
            trace(c, 4);
        }
    }
    const MyTiles mt = my_tiles(p.tiles, c.off, c.cta, c.G);
    c.off = (c.off + p.tiles) % c.G;
    if (mt.n == 0) {
        csync();
        return;
    }
    const int nseg = n_segments(p.K);
    if (nseg > 1 && mt.n <= DEC_TACC_TILES) {
        // Segment-outer: each activation segment is loaded once for all of the
        // CTA's tiles (group-outer reloads it per group of 4 tiles); per-tile
        // sums carry across segments in tacc.
        const EpiPre pre = epi_prefetch(c, kind, layer, c.warp < mt.n ? mt.t0 + c.warp * c.G : -1);
        for (int sg = 0; sg < nseg; ++sg) {
            int c0, c1;
            seg_range(p.K, nseg, sg, c0, c1);
            csync();
            if (sg == 0 && ss)  // d_model > 4096: normed phases are multi-segment too
                load_act_rs(c, src, ld, c0 * DEC_CHUNK_COLS, c1 * DEC_CHUNK_COLS, ss, rs);
            else
                load_act(c, src, ld, c0 * DEC_CHUNK_COLS, c1 * DEC_CHUNK_COLS);
            csync();
            trace(c, 2);
            for (int g0 = 0; g0 < mt.n; g0 += DEC_MAXT) {
                const int gn = min(DEC_MAXT, mt.n - g0);
                consume_group(c, gn, 0, c1 - c0);
                csync();
                for (int ti = c.warp; ti < gn; ti += DEC_NCW) {
                    float4* t = reinterpret_cast<float4*>(c.sm.tacc + (g0 + ti) * 128) + c.lane;
                    const float4 v = warp_sum(c, ti);
                    if (sg == 0) {
                        *t = v;
                    } else {
                        const float4 o = *t;
                        *t = make_float4(o.x + v.x, o.y + v.y, o.z + v.z, o.w + v.w);
                    }
                }
                csync();  // partials are rewritten by the next group
            }
        }
        trace(c, 3);
        epilogue_group(c, kind, layer, mt.n, [&](int ti) { return mt.t0 + ti * c.G; }, rs, best_v, best_i, pre, 0);
        csync();
        trace(c, 4);
        return;
    }
    for (int g0 = 0; g0 < mt.n; g0 += DEC_MAXT) {
        const int gn = min(DEC_MAXT, mt.n - g0);
        const EpiPre pre = epi_prefetch(c, kind, layer, c.warp < gn ? mt.t0 + (g0 + c.warp) * c.G : -1);
        for (int sg = 0; sg < nseg; ++sg) {
            int c0, c1;
            seg_range(p.K, nseg, sg, c0, c1);
            if (nseg > 1 || g0 == 0) {
                csync();
                if (g0 == 0 && sg == 0 && ss)
                    load_act_rs(c, src, ld, c0 * DEC_CHUNK_COLS, c1 * DEC_CHUNK_COLS, ss, rs);
                else
                    load_act(c, src, ld, c0 * DEC_CHUNK_COLS, c1 * DEC_CHUNK_COLS);
                csync();
                trace(c, 2);
            }
            consume_group(c, gn, sg, c1 - c0);
        }
        csync();
        trace(c, 3);
        epilogue_group(c, kind, layer, gn, [&](int ti) { return mt.t0 + (g0 + ti) * c.G; }, rs, best_v, best_i, pre);
        csync();  // partials are rewritten by the next group
        trace(c, 4);
    }
}

// ------------------------------------------------------------ attention
// Tensor-core decode attention, per warp and 8 KB ring stage of RT tokens, in
// transposed form so the GQA group (<= 8 query heads) is the mma N dimension:
//   S^T = K Q^T   mma.m16n8k16: A = 16 K rows (ldmatrix), B = Q^T (bf16 regs)
//   online softmax per head column (a column lives in 8 lanes x 2 regs)
//   O^T += V^T P^T  A = V^T (ldmatrix.trans), B = P^T (movmatrix.trans of S^T)
// Stage layout in the ring slot: one [K rows | V rows] run per KV block (its
// single bulk copy), blocks back to back: token r's K row at kv_row(r), its V
// row KVB bytes later, with the KV block's chunk swizzle (r & 7).
template <int DH>
struct AttnCfg {
    static constexpr int RT = 2048 / DH;  // tokens per 8 KB stage (K + V)
    static constexpr int KVB = KV_BLOCK_TOKENS * DH * 2;  // K (or V) rows of one block
    static __device__ __forceinline__ uint32_t kv_row(int r) {
        return uint32_t((r / KV_BLOCK_TOKENS) * 2 * KVB + (r % KV_BLOCK_TOKENS) * DH * 2);
    }
    static constexpr int KS = DH / 16;    // k-steps of S^T (head dims)
    static constexpr int MT = RT / 16;    // token m-tiles of S^T == k-steps of O^T
    static constexpr int MD = DH / 16;    // dim m-tiles of O^T
};

template <int DH>
struct AttnState {
    uint32_t qb[AttnCfg<DH>::KS][2];  // Q^T as mma B fragments (head g, dims 2t..)
    float o[AttnCfg<DH>::MD][4];      // O^T: rows dims 16md + g (+8), cols heads 2t, 2t+1
    float m[2], l[2];                 // running max / this lane's partial sum, heads 2t, 2t+1
};

// Attention partials: per slot, per head of the GQA group, [m, l, -, -, acc[DH]]
// (head stride DH + 4 keeps acc 16-byte aligned).
template <int DH>
__host__ __device__ constexpr int attn_hs() { return DH + 4; }

// Combine `count` partials (slot stride W floats) per head in slot order.
// Lane-parallel over (head, 4 dims). FINAL writes bf16(acc / l) to `out`,
// else one partial to `dst` (global).
template <int DH, bool FINAL, bool GLOBAL_SRC = false>
__device__ __forceinline__ void attn_combine(const float* src, int W, int count, int GQ, int lane, float* dst,
                                             uint16_t* out) {
    constexpr int D4 = DH / 4, HS = attn_hs<DH>();
    for (int item = lane; item < GQ * D4; item += 32) {
        const int h = item / D4, d0 = (item % D4) * 4;
        const float* hs = src + h * HS;
        float mx = -INFINITY;
        for (int i = 0; i < count; ++i) mx = fmaxf(mx, GLOBAL_SRC ? ldcg_f32(hs + size_t(i) * W) : hs[size_t(i) * W]);
        float L = 0.f;
        float4 A = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
        for (int i = 0; i < count; ++i) {
            const float* ph = hs + size_t(i) * W;
            float2 ml;
            float4 v;
            if constexpr (GLOBAL_SRC) {  // other SMs wrote these: bypass L1
                ml = __ldcg(reinterpret_cast<const float2*>(ph));
                v = __ldcg(reinterpret_cast<const float4*>(ph + 4 + d0));
            } else {
                ml = *reinterpret_cast<const float2*>(ph);
                v = *reinterpret_cast<const float4*>(ph + 4 + d0);
            }
            const float f = ml.x == -INFINITY ? 0.f : __expf(ml.x - mx);
            L += ml.y * f;
            A.x += v.x * f;
            A.y += v.y * f;
            A.z += v.z * f;
            A.w += v.w * f;
        }
        if constexpr (FINAL) {
            uint2 pk;
            pk.x = pack_bf16x2(A.x / L, A.y / L);
            pk.y = pack_bf16x2(A.z / L, A.w / L);
            *reinterpret_cast<uint2*>(out + h * DH + d0) = pk;
        } else {
            float* ph = dst + h * HS;
            if (d0 == 0) *reinterpret_cast<float2*>(ph) = make_float2(mx, L);
            *reinterpret_cast<float4*>(ph + 4 + d0) = A;
        }
    }
}

// Publish one global partial of `pair` (already written) and, if it is the
// pair's last, combine all of them into the attention output. `scratch` (or
// null) is shared memory for 8 slots: the partials are pulled in with one
// batch of cp.async (a single L2 round trip) and combined from there.
template <int DH>
__device__ __forceinline__ void attn_arrive(Ctx& c, int b, int kvh, int pair_lo, int count, float* scratch) {
    // pair id = kvh * B + b (head-major stage order)
    const DecodeArgs& a = *c.a;
    const Shape& s = a.s;
    const int GQ = s.n_heads / s.n_kv;
    const int W = GQ * attn_hs<DH>();
    const int pair = kvh * c.B + b;
    __syncwarp();
    int last = 0;
    if (c.lane == 0) last = atom_add_acq_rel_gpu(a.acnt + pair, 1) == count - 1;
    last = __shfl_sync(0xffffffffu, last, 0);
    if (!last) return;
    const float* src = a.apart + size_t(pair_lo) * W;
    uint16_t* out = a.attn + size_t(b) * s.d + size_t(kvh) * GQ * DH;
    if (scratch && count <= 8) {
        const int n16 = count * W / 4;
        const uint32_t sb = smem_u32(scratch);
        for (int i = c.lane; i < n16; i += 32) cp_async_16(sb + i * 16, src + i * 4);
        cp_async_wait_all();
        __syncwarp();
        attn_combine<DH, true>(scratch, W, count, GQ, c.lane, nullptr, out);
    } else {
        attn_combine<DH, true, true>(src, W, count, GQ, c.lane, nullptr, out);
    }
    if (c.lane == 0) atomicExch(a.acnt + pair, 0);
}

template <int DH>
__device__ __forceinline__ int attn_cap_pairs(const Shape& s) {
    const int W = (s.n_heads / s.n_kv) * attn_hs<DH>();
    return DEC_SMEM_ACT / (8 * W * 4);
}

template <int DH>
__device__ __forceinline__ void attn_flush(Ctx& c, const AttnPlan& ap, int b, int kvh, int pair_lo, int pair_n,
                                           AttnState<DH>& stt) {
    constexpr int MD = AttnCfg<DH>::MD;
    const DecodeArgs& a = *c.a;
    const Shape& s = a.s;
    const int GQ = s.n_heads / s.n_kv;
    constexpr int HS = attn_hs<DH>();
    const int W = GQ * HS;
    const unsigned FULL = 0xffffffffu;
    const int g = c.lane >> 2, t = c.lane & 3;
    const int pair = kvh * c.B + b, k = pair - c.p0;
    int pre, r, rank, count;
    if (k < ATT_PT_MAX) {
        const AttnPair& e = c.pt[k];
        pre = e.pre;
        r = (c.warp - e.r0 + 8) % 8;
        rank = pre ? e.rank0 : e.rank0 + r;
        count = e.count;
    } else {  // beyond the table: never pre-combined
        const PairSlot ps = pair_slot(ap, s.n_kv, pair, pair_lo, pair_lo + pair_n, c.G, c.cta, c.warp,
                                      attn_cap_pairs<DH>(s));
        pre = 0;
        r = ps.r;
        rank = ps.rank;
        count = ps.count;
    }
    float l0 = stt.l[0], l1 = stt.l[1];
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
        l0 += __shfl_xor_sync(FULL, l0, o);
        l1 += __shfl_xor_sync(FULL, l1, o);
    }
    float* pp = pre ? reinterpret_cast<float*>(c.sm.act) + size_t(k * 8 + r) * W : a.apart + size_t(pair_lo + rank) * W;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int h = 2 * t + j;
        if (h < GQ) {
            float* ph = pp + h * HS;
            if (g == 0) *reinterpret_cast<float2*>(ph) = make_float2(stt.m[j], j ? l1 : l0);
#pragma unroll
            for (int md = 0; md < MD; ++md) {
                ph[4 + 16 * md + g] = stt.o[md][j];
                ph[4 + 16 * md + 8 + g] = stt.o[md][2 + j];
            }
        }
    }
    // a direct pair's shared slots [8k, 8k + 8) are unused by this CTA: final-combine scratch
    if (!pre)
        attn_arrive<DH>(c, b, kvh, pair_lo, count,
                        k < min(attn_cap_pairs<DH>(s), ATT_PT_MAX) ? reinterpret_cast<float*>(c.sm.act) + size_t(k * 8) * W
                                                                   : nullptr);
}

// After every warp flushed: combine the pairs this CTA pre-combines (pair-local
// index k handled by warp k % 8), publish them, and finish complete pairs.
template <int DH>
__device__ __forceinline__ void attn_cta_combine(Ctx& c) {
    const DecodeArgs& a = *c.a;
    const Shape& s = a.s;
    const int GQ = s.n_heads / s.n_kv;
    const int W = GQ * attn_hs<DH>();
    for (int k = c.warp; k < min(c.np, ATT_PT_MAX); k += DEC_NCW) {
        const AttnPair& e = c.pt[k];
        if (!e.pre) continue;
        const int pair = c.p0 + k;
        trace(c, 16);
        float* slots = reinterpret_cast<float*>(c.sm.act) + size_t(k * 8) * W;
        attn_combine<DH, false>(slots, W, e.n, GQ, c.lane, a.apart + size_t(e.lo_p + e.rank0) * W, nullptr);
        trace(c, 17);
        __syncwarp();  // the slots become the final-combine scratch
        attn_arrive<DH>(c, pair % c.B, pair / c.B, e.lo_p, e.count, slots);
        trace(c, 18);
    }
}

template <int DH>
__device__ __forceinline__ void attn_consume(Ctx& c, int layer, const AttnStage& st, uint32_t qi, AttnState<DH>& stt) {
    using CFG = AttnCfg<DH>;
    constexpr int RT = CFG::RT, KS = CFG::KS, MT = CFG::MT, MD = CFG::MD;
    const DecodeArgs& a = *c.a;
    const Shape& s = a.s;
    const unsigned FULL = 0xffffffffu;
    const int cur = c.pos[st.b], len = cur + 1;
    const int t0 = st.s * RT;
    const int lane = c.lane, g = lane >> 2, t = lane & 3;
    const float scale = rsqrtf(float(DH));
    // the current token's K/V rows were written by this step's QKV phase: fetch
    // them from the paged cache (before the stage wait, to overlap the latency)
    // into their stage rows (same swizzle: row & 7 == slot & 7)
    constexpr int CH = DH / 8;  // 16-byte chunks per row; 2 * CH <= 32
    const bool patch = cur >= t0 && cur < t0 + RT;
    uint4 pv = make_uint4(0, 0, 0, 0);
    if (patch && lane < 2 * CH) {
        const int blk = c.cur_blk[st.b] >= 0
                            ? c.cur_blk[st.b]
                            : ldcg_i32(a.block_table + size_t(c.slot[st.b]) * a.bt_stride + cur / KV_BLOCK_TOKENS);
        pv = ldcg_u4(a.kv_base + size_t(blk) * a.block_bytes +
                     kv_offset(s, layer, lane / CH, st.kvh, cur % KV_BLOCK_TOKENS) + (lane % CH) * 16);
    }
    uint32_t slot;
    wait_stage(c, qi, slot);
    uint8_t* stage = c.sm.ring + size_t(slot) * DEC_STAGE_BYTES;
    if (patch) {
        if (lane < 2 * CH)
            *reinterpret_cast<uint4*>(stage + CFG::kv_row(cur - t0) + (lane / CH) * CFG::KVB + (lane % CH) * 16) = pv;
        // V rows past the current token hold stale memory (the unwritten tail of the
        // block, or a previous stage): their softmax weight is 0, but 0 x NaN would
        // still reach O through the PV mma, so clear them
        for (int i = lane; i < (RT - 1 - (cur - t0)) * CH; i += 32)
            *reinterpret_cast<uint4*>(stage + CFG::kv_row(cur - t0 + 1 + i / CH) + CFG::KVB + (i % CH) * 16) =
                make_uint4(0, 0, 0, 0);
        __syncwarp();
    }
    const uint32_t kbase = smem_u32(stage), vbase = kbase + CFG::KVB;
    // ldmatrix.x4 lane address: matrix j = lane >> 3 covers rows +8*(j&1), chunk +(j>>1)
    const int lrow = (lane & 7) + ((lane >> 3) & 1) * 8, lch = lane >> 4;
    // ---- S^T = K Q^T
    float sc[MT][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
        sc[mt][0] = sc[mt][1] = sc[mt][2] = sc[mt][3] = 0.f;
        const int row = mt * 16 + lrow;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            uint32_t k0, k1, k2, k3;
            ldmatrix_x4(kbase + CFG::kv_row(row) + (((2 * ks + lch) ^ (row & 7)) << 4), k0, k1, k2, k3);
            mma_bf16_16816(sc[mt], k0, k1, k2, k3, stt.qb[ks][0], stt.qb[ks][1]);
        }
    }
    // ---- online softmax per head column (tokens g, g+8 of each m-tile; heads 2t, 2t+1)
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int tok = t0 + mt * 16 + g + (e >> 1) * 8;
            sc[mt][e] = tok < len ? sc[mt][e] * scale : -INFINITY;
            mx[e & 1] = fmaxf(mx[e & 1], sc[mt][e]);
        }
    }
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
        mx[0] = fmaxf(mx[0], __shfl_xor_sync(FULL, mx[0], o));
        mx[1] = fmaxf(mx[1], __shfl_xor_sync(FULL, mx[1], o));
    }
    float corr[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const float mnew = fmaxf(stt.m[j], mx[j]);  // finite: token t0 is always valid
        corr[j] = __expf(stt.m[j] - mnew);
        stt.m[j] = mnew;
        stt.l[j] *= corr[j];
    }
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            sc[mt][e] = __expf(sc[mt][e] - stt.m[e & 1]);
            stt.l[e & 1] += sc[mt][e];
        }
    }
#pragma unroll
    for (int md = 0; md < MD; ++md) {
        stt.o[md][0] *= corr[0];
        stt.o[md][1] *= corr[1];
        stt.o[md][2] *= corr[0];
        stt.o[md][3] *= corr[1];
    }
    // ---- O^T += V^T P^T
#pragma unroll
    for (int kk = 0; kk < MT; ++kk) {
        const uint32_t pb0 = movmatrix_trans(pack_bf16x2(sc[kk][0], sc[kk][1]));
        const uint32_t pb1 = movmatrix_trans(pack_bf16x2(sc[kk][2], sc[kk][3]));
        // x4.trans: matrix j = (dims +8*(j&1)) x (tokens +8*(j>>1))
        const int row = kk * 16 + (lane & 7) + (lane >> 4) * 8;
        const int dsel = (lane >> 3) & 1;
#pragma unroll
        for (int md = 0; md < MD; ++md) {
            uint32_t v0, v1, v2, v3;
            ldmatrix_x4_trans(vbase + CFG::kv_row(row) + (((2 * md + dsel) ^ (row & 7)) << 4), v0, v1, v2, v3);
            mma_bf16_16816(stt.o[md], v0, v1, v2, v3, pb0, pb1);
        }
    }
    release_stage(c, slot);
}

template <int DH>
__device__ __forceinline__ void run_attention_t(Ctx& c, int layer, const AttnPlan& ap) {
    using CFG = AttnCfg<DH>;
    constexpr int KS = CFG::KS, MD = CFG::MD;
    const DecodeArgs& a = *c.a;
    const Shape& s = a.s;
    const int GQ = s.n_heads / s.n_kv;
    const int g = c.lane >> 2, t = c.lane & 3;
    const int n = ap.a1 - ap.a0;
    AttnState<DH> stt;
    int cur_pair = -1, cur_b = 0, cur_kvh = 0, cur_lo = 0, cur_n = 0;
    if (a.skip & 32) {  // debug: bare ring handshake (no pair bookkeeping, no combine; results are garbage)
        for (int i = c.warp; i < n; i += DEC_NCW) {
            uint32_t slot;
            wait_stage(c, c.q + i, slot);
            release_stage(c, slot);
        }
        c.q += n;
        csync();
        return;
    }
    // The warp's stages walked incrementally (DEC_NCW at a time), and ONE flush
    // site (the pass after the last stage flushes the open pair): attn_flush
    // inlines two partial-combine variants, so a second call site doubled them.
    AttnStage st = attn_stage_of(ap, s.n_kv, ap.a0 + min(c.warp, max(n - 1, 0)));
    for (int i = c.warp;; i += DEC_NCW) {
        const bool end = i >= n;
        if (end || st.pair != cur_pair) {
            if (cur_pair >= 0) attn_flush<DH>(c, ap, cur_b, cur_kvh, cur_lo, cur_n, stt);
            if (end) break;
            // this layer's q / current K,V of the group are written by the QKV phase's
            // tiles of group kvh (any CTA): wait for the group's count, not for the grid
            if (c.lane == 0) {
                const int need = (layer + 1) * qkv_group_tiles(s);
                while (int(ld_acquire_gpu(reinterpret_cast<const unsigned int*>(a.qkv_done + st.kvh))) < need) {
                }
            }
            __syncwarp();
            cur_pair = st.pair;
            cur_b = st.b;
            cur_kvh = st.kvh;
            cur_lo = st.pair_lo;
            cur_n = ap.nst[st.b];
            // Q^T of the GQA group as B fragments (columns >= GQ are zero)
            const float* qrow = a.q + (size_t(st.b) * s.n_heads + size_t(st.kvh) * GQ + g) * DH;
            float2 qv[KS][2];
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                qv[ks][0] = g < GQ ? __ldcg(reinterpret_cast<const float2*>(qrow + ks * 16 + 2 * t)) : make_float2(0.f, 0.f);
                qv[ks][1] = g < GQ ? __ldcg(reinterpret_cast<const float2*>(qrow + ks * 16 + 8 + 2 * t))
                                   : make_float2(0.f, 0.f);
            }
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                stt.qb[ks][0] = pack_bf16x2(qv[ks][0].x, qv[ks][0].y);
                stt.qb[ks][1] = pack_bf16x2(qv[ks][1].x, qv[ks][1].y);
            }
#pragma unroll
            for (int md = 0; md < MD; ++md) stt.o[md][0] = stt.o[md][1] = stt.o[md][2] = stt.o[md][3] = 0.f;
            stt.m[0] = stt.m[1] = -INFINITY;
            stt.l[0] = stt.l[1] = 0.f;
        }
        if (a.skip & 8) {  // debug: ring handshake only
            uint32_t slot;
            wait_stage(c, c.q + i, slot);
            release_stage(c, slot);
        } else {
            attn_consume<DH>(c, layer, st, c.q + i, stt);
        }
        if (i == c.warp) trace(c, 12);
        st.s += DEC_NCW;  // next stage of this warp: requests inner, kv heads outer
        while (st.s >= ap.nst[st.b]) {
            st.s -= ap.nst[st.b];
            st.pair_lo += ap.nst[st.b];
            if (++st.b == ap.nb) {
                st.b = 0;
                ++st.kvh;
            }
            st.pair = st.kvh * ap.nb + st.b;
            if (st.kvh >= s.n_kv) break;  // past the range (the loop ends)
        }
    }
    trace(c, 13);
    c.q += n;
    trace(c, 14);
    csync();  // warp partials of pre-combined pairs are in shared memory
    trace(c, 15);
    attn_cta_combine<DH>(c);
}

// ------------------------------------------------------------ embedding
__device__ __forceinline__ void run_embed(Ctx& c) {
    const DecodeArgs& a = *c.a;
    const Shape& s = a.s;
    if (c.cta == 0) {
        const StepDesc* dsc = a.desc;
        for (int i = c.tid; i < dsc->n_upd; i += CONSUMER_THREADS)
            a.block_table[size_t(dsc->upd[i][0]) * a.bt_stride + dsc->upd[i][1]] = dsc->upd[i][2];
    }
    const int nt = s.d / 16, items = DEC_MAXB * nt;
    for (int it = c.cta * DEC_NCW + c.warp; it < items; it += c.G * DEC_NCW) {
        const int b = it / nt, tile = it % nt;
        float sq = 0.f;
        if (b < c.B && c.lane < 16) {
            const int tok = ldcg_i32(a.last_tok + c.slot[b]);
            const int row = tile * 16 + c.lane;
            const float hv = bf16_to_f(a.w.emb[size_t(tok) * s.d + row]);
            a.h[size_t(b) * s.d + row] = hv;
            a.act[size_t(b) * s.d + row] = f_to_bf16(hv * a.w.g_attn[row]);
            sq = hv * hv;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        if (c.lane == 0) a.ssA[tile * 8 + b] = sq;
    }
}

__device__ __forceinline__ void run_argmax_combine(Ctx& c, float best_v[2], int best_i[2]) {
    const DecodeArgs& a = *c.a;
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, best_v[j], o);
            const int oi = __shfl_xor_sync(0xffffffffu, best_i[j], o);
            better(best_v[j], best_i[j], ov, oi);
        }
    float* wv = c.sm.misc + 32;                        // [8 warps][8]
    int* wi = reinterpret_cast<int*>(c.sm.misc + 96);  // [8 warps][8]
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
    csync();
    if (c.tid == 0) *flag = atom_add_acq_rel_gpu(a.arg_cnt, 1) == c.G - 1;
    csync();
    if (*flag) {
        const int b = c.warp;  // warp b reduces CTA partials lane, lane + 32, ...
        if (b < c.B) {
            float bv = -INFINITY, vv[8];
            int bi = 0x7fffffff, ii[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int cta = c.lane + 32 * k;
                vv[k] = cta < c.G ? ldcg_f32(a.arg_val + cta * 8 + b) : -INFINITY;
                ii[k] = cta < c.G ? ldcg_i32(a.arg_idx + cta * 8 + b) : 0x7fffffff;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) better(bv, bi, vv[k], ii[k]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                better(bv, bi, ov, oi);
            }
            if (c.lane == 0) {
                a.tok_out[b] = bi;
                a.last_tok[c.slot[b]] = bi;
            }
        }
        if (c.tid == 0) {
            atomicExch(a.arg_cnt, 0);
            atomicExch(a.bar_count, 0u);  // every CTA is past its last grid barrier
        }
        // every CTA is past its last claim: rearm the dynamic phases' counters for the next step
        for (int i = c.tid; i < a.s.n_layers * 4 + 1; i += CONSUMER_THREADS) a.claim[i] = 0;
        for (int i = c.tid; i < a.s.n_kv; i += CONSUMER_THREADS) a.qkv_done[i] = 0;
    }
}

__global__ void __launch_bounds__(DEC_THREADS, 1) decode_kernel(const __grid_constant__ DecodeArgs args) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ DecodeArgs a_s;  // launch arguments, read with LDS instead of generic param loads
    __shared__ int slot_s[DEC_MAXB], pos_s[DEC_MAXB], cur_blk_s[DEC_MAXB];
    __shared__ int dt0_s[4], dgn_s[4];
    __shared__ __align__(8) uint64_t dfull_s[4], dempty_s[4];
    __shared__ __align__(8) uint64_t actbar_s;
    Smem sm = carve(smem_raw);
    sm.dt0 = dt0_s;
    sm.dgn = dgn_s;
    sm.dfull = dfull_s;
    sm.dempty = dempty_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int B = args.desc->B;
    if (threadIdx.x == 0) {
        a_s = args;
        for (int i = 0; i < DEC_NSTAGE; ++i) {
            mbar_init(&sm.full[i], 1);
            mbar_init(&sm.empty[i], 1);
        }
        for (int i = 0; i < 4; ++i) {
            mbar_init(&sm.dfull[i], 1);
            mbar_init(&sm.dempty[i], 1);
        }
        mbar_init(&actbar_s, 1);
        fence_mbar_init();
    }
    if (threadIdx.x < DEC_MAXB) {
        slot_s[threadIdx.x] = int(threadIdx.x) < B ? args.desc->slot[threadIdx.x] : 0;
        pos_s[threadIdx.x] = int(threadIdx.x) < B ? args.desc->pos[threadIdx.x] : 0;
    }
    // block-table rows of the step's requests (entries that predate this step)
    for (int i = threadIdx.x; i < DEC_MAXB * DEC_BT_MAX; i += DEC_THREADS) {
        const int b = i / DEC_BT_MAX, k = i % DEC_BT_MAX;
        sm.bt[i] = (b < B && k < args.bt_stride) ? args.block_table[size_t(args.desc->slot[b]) * args.bt_stride + k] : 0;
    }
    // The block of each request's current token, as this step leaves the table (an
    // entry installed by this step's update list wins): the QKV epilogue's K/V
    // stores and attention's current-row patch then skip a dependent global load.
    if (threadIdx.x < DEC_MAXB) {
        const int b = threadIdx.x;
        int blk = -1;
        if (b < B) {
            const int k = args.desc->pos[b] / KV_BLOCK_TOKENS, sl = args.desc->slot[b];
            if (k < args.bt_stride) blk = args.block_table[size_t(sl) * args.bt_stride + k];
            for (int i = 0; i < args.desc->n_upd; ++i)
                if (args.desc->upd[i][0] == sl && args.desc->upd[i][1] == k) blk = args.desc->upd[i][2];
        }
        cur_blk_s[b] = blk;
    }
    __syncthreads();
    const DecodeArgs& a = a_s;

    if (warp == DEC_NCW) {
        if (lane < DEC_PRODUCER_LANES) producer_loop(a, sm, blockIdx.x, gridDim.x, B, pos_s, lane);
        return;
    }
    Ctx c;
    c.ntrace = 0;
    c.nbar = 0;
    c.a = &a_s;
    c.sm = sm;
    c.cta = blockIdx.x;
    c.G = gridDim.x;
    c.warp = warp;
    c.lane = lane;
    c.tid = threadIdx.x;
    c.B = B;
    c.slot = slot_s;
    c.pos = pos_s;
    c.cur_blk = cur_blk_s;
    c.q = 0;
    c.off = 0;
    c.dk = 0;
    c.actbar = &actbar_s;
    c.actph = 0;
    c.nsh = uint32_t(__ffs(a.nstage) - 1);
    c.nmask = uint32_t(a.nstage) - 1u;
    // attention plan + this CTA's pair table: identical for every layer of the step
    __shared__ AttnPlan ap_s;
    __shared__ AttnPair pt_s[ATT_PT_MAX];
    if (threadIdx.x == 0) ap_s = attn_plan(a.s, B, pos_s, c.cta, c.G);
    csync();
    const AttnPlan& ap = ap_s;
    c.pt = pt_s;
    c.p0 = c.np = 0;
    if (ap.a1 > ap.a0) {
        c.p0 = attn_stage_of(ap, a.s.n_kv, ap.a0).pair;
        c.np = attn_stage_of(ap, a.s.n_kv, ap.a1 - 1).pair - c.p0 + 1;
    }
    if (warp == 0 && lane < min(c.np, ATT_PT_MAX)) {
        const int pair = c.p0 + lane, b = pair % B, kvh = pair / B;
        int lo_p = kvh * ap.hst;
        for (int bb = 0; bb < b; ++bb) lo_p += ap.nst[bb];
        const int cap = a.s.dh == 64 ? attn_cap_pairs<64>(a.s) : attn_cap_pairs<128>(a.s);
        const PairSlot ps = pair_slot(ap, a.s.n_kv, pair, lo_p, lo_p + ap.nst[b], c.G, c.cta, 0, cap);
        AttnPair e;
        e.lo_p = lo_p;
        e.pre = ps.pre;
        e.n = ps.n;
        e.r0 = (8 - ps.r) % 8;  // warp 0 has rank r  =>  the first stage's warp is -r mod 8
        e.rank0 = ps.pre ? ps.rank : ps.rank - ps.r;
        e.count = ps.count;
        pt_s[lane] = e;
    }
    csync();

    float best_v[2] = {-INFINITY, -INFINITY};
    int best_i[2] = {0x7fffffff, 0x7fffffff};

    run_embed(c);
    grid_sync(c);
    // One call site per phase body: the phase kind is a runtime value, so the
    // GEMV code (schedules + epilogues) exists once instead of once per kind.
    // The kernel shrank from 33.9k to 21.3k SASS instructions and every phase's
    // fixed cost with it: code that runs once per layer (epilogues, combines)
    // was missing the instruction cache under the weight stream (same-box A/B:
    // 1.1B at 148 SMs 1.162 -> 1.068 ms, 7B 4.32 -> 3.92-3.98, 7B at 36 SMs
    // 9.43 -> 8.69-8.84). An out-of-line attn_combine (17.8k) measured slower.
    const int L = a.s.n_layers;
#pragma unroll 1
    for (int it = 0; it <= 4 * L; ++it) {
        const int kind = it == 4 * L ? int(PH_LM) : (it & 3), l = it == 4 * L ? 0 : (it >> 2);
        run_gemv(c, kind, l, best_v, best_i);
        if (kind == PH_LM) break;
        if (kind == PH_QKV) {
            trace(c, 6);
            if (!(a.skip & 1)) {
                if (a.s.dh == 64)
                    run_attention_t<64>(c, l, ap);
                else
                    run_attention_t<128>(c, l, ap);
            }
            trace(c, 7);
        }
        grid_sync(c);
    }
    run_argmax_combine(c, best_v, best_i);
}

}  // namespace

size_t decode_apart_floats(const Shape& s) {
    const int rt = 2048 / s.dh;
    return size_t(DEC_MAXB) * s.n_kv * ((s.max_seq + rt - 1) / rt) * s.gq() * (s.dh + 4);
}

cudaError_t launch_decode(const DecodeArgs& a, int grid, cudaStream_t stream) {
    static bool configured[MAX_DEVICES] = {};
    const int dev = cur_device();
    if (!configured[dev]) {
        cudaError_t e = cudaFuncSetAttribute(decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, DEC_SMEM_TOTAL);
        if (e != cudaSuccess) return e;
        configured[dev] = true;
    }
    decode_kernel<<<grid, DEC_THREADS, DEC_SMEM_TOTAL, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace meshgpu
