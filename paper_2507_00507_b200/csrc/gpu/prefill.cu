// Prefill step for one request (L tokens starting at absolute position p0).
//
// GEMMs are C^T = W . X^T on tcgen05 with the weight rows as the M operand, so
// the decode kernel's row permutations (RoPE pairs, gate/up interleave) put both
// members of a pair in lanes l and l^8 of one epilogue warp. The weights are
// streamed straight from their T16xSW128 tiled layout: each 16x64 block is a
// contiguous, pre-swizzled 2 KB run, which is exactly the canonical SW128
// K-major UMMA operand layout, so they need no tensor map. The token rows come
// in through a TMA tensor map with the hardware 128-byte swizzle. The epilogues
// are the decode ones applied per token: RoPE + paged KV write, the residual
// add, silu(gate)*up. Attention is causal over the paged cache.
#include "prefill.cuh"

#include <string>
#include <vector>
#include <cstring>
#include <cstdio>
#include <chrono>
#include <thread>

#include <cuda.h>
#include <math.h>
#include <stdlib.h>

#include <algorithm>

namespace meshgpu {

namespace {

enum PfKind { PF_QKV = 0, PF_O = 1, PF_GU = 2, PF_DOWN = 3 };

constexpr int PF_BM = 128, PF_BN = 64, PF_BK = 64, PF_STAGES = 4, PF_THREADS = 256;
constexpr int PF_A_STAGE = PF_BM * PF_BK * 2;  // 16 KB
constexpr int PF_B_STAGE = PF_BN * PF_BK * 2;  // 8 KB
constexpr int PF_SMEM = PF_STAGES * (PF_A_STAGE + PF_B_STAGE);

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// lm_head of the last prefill position: logits[V] = W_lm . act (one token), an
// mma.sync tile kernel (a single-column GEMM has no use for the tcgen05 path).
__global__ void __launch_bounds__(PF_THREADS) pf_lm_gemm(const __grid_constant__ PrefillArgs a,
                                                         const uint8_t* __restrict__ W, int K,
                                                         const uint16_t* __restrict__ X, int ldx, int Lrows) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* As = smem;
    uint8_t* Bs = smem + PF_STAGES * PF_A_STAGE;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int warp_m = warp & 3, warp_n = warp >> 2;
    const int row_tile0 = blockIdx.x * (PF_BM / 16);
    const int tok0 = blockIdx.y * PF_BN;
    const int nk = K / PF_BK;
    const size_t tile_bytes = size_t(K) * 32;

    auto load_stage = [&](int kt, int slot) {
        uint32_t a_dst = smem_u32(As + slot * PF_A_STAGE);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            int ch = tid + i * PF_THREADS;  // 1024 chunks of 16 B
            int t = ch >> 7, off = (ch & 127) << 4;
            const uint8_t* src = W + size_t(row_tile0 + t) * tile_bytes + size_t(kt) * 2048 + off;
            cp_async16(a_dst + t * 2048 + off, src, 16);
        }
        uint32_t b_dst = smem_u32(Bs + slot * PF_B_STAGE);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            int ch = tid + i * PF_THREADS;  // 512 chunks
            int r = ch >> 3, cc = ch & 7;
            int l = tok0 + r;
            const uint16_t* src = X + size_t(min(l, Lrows - 1)) * ldx + kt * PF_BK + cc * 8;
            cp_async16(b_dst + r * 128 + ((cc ^ (r & 7)) << 4), src, l < Lrows ? 16 : 0);
        }
    };

    float acc[2][4][4];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.f;

#pragma unroll
    for (int s = 0; s < PF_STAGES - 1; ++s) {
        if (s < nk) load_stage(s, s);
        cp_async_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<PF_STAGES - 2>();
        __syncthreads();
        int nxt = kt + PF_STAGES - 1;
        if (nxt < nk) load_stage(nxt, nxt % PF_STAGES);
        cp_async_commit();
        const int slot = kt % PF_STAGES;
        const uint32_t a_base = smem_u32(As + slot * PF_A_STAGE);
        const uint32_t b_base = smem_u32(Bs + slot * PF_B_STAGE);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
            uint32_t af[2][4];
#pragma unroll
            for (int mi = 0; mi < 2; ++mi) {
                int t = 2 * warp_m + mi;
                int r = lane & 15;
                int chunk = ks * 2 + (lane >> 4);
                ldmatrix_x4(a_base + t * 2048 + r * 128 + ((chunk ^ (r & 7)) << 4), af[mi][0], af[mi][1],
                            af[mi][2], af[mi][3]);
            }
            uint32_t bfr[4][2];
#pragma unroll
            for (int np = 0; np < 2; ++np) {
                int n0 = warp_n * 32 + np * 16;
                int r = n0 + (lane & 7) + ((lane >> 4) << 3);
                int chunk = ks * 2 + ((lane >> 3) & 1);
                ldmatrix_x4(b_base + r * 128 + ((chunk ^ (r & 7)) << 4), bfr[2 * np][0], bfr[2 * np][1],
                            bfr[2 * np + 1][0], bfr[2 * np + 1][1]);
            }
#pragma unroll
            for (int mi = 0; mi < 2; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni)
                    mma_bf16_16816(acc[mi][ni], af[mi][0], af[mi][1], af[mi][2], af[mi][3], bfr[ni][0],
                                   bfr[ni][1]);
        }
    }
    cp_async_wait<0>();

    // ---- epilogue: rms-scaled logits of the single token
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
        const int row = (row_tile0 + 2 * warp_m + mi) * 16 + g;  // rows row and row + 8
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int l = tok0 + warp_n * 32 + ni * 8 + 2 * t + j;
                if (l >= Lrows) continue;
                const float r = a.rs[0];
                a.logits[row] = acc[mi][ni][j] * r;
                a.logits[row + 8] = acc[mi][ni][2 + j] * r;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// tcgen05 GEMM: C^T[N x L] = W[N x K] . X[L x K]^T on the 5th-gen tensor cores.
//
// Persistent, one CTA per SM. Tiles are 128 weight rows x BN tokens, ordered
// token-block fastest so the CTAs that share a weight tile run together and the
// tile is fetched from HBM once. Warp roles (192 threads):
//   warp 0  producer: per 64-deep K block, 8 bulk copies of the pre-swizzled
//           16x64 weight blocks (A, 16 KB) + one TMA tensor load of the token
//           rows with the 128-byte swizzle (B, BN x 128 B)
//   warp 1  TMEM owner + single-thread tcgen05.mma issuer (M=128, N=BN, K=16)
//   warps 2-5 epilogue: tcgen05.ld 32x32b (thread = weight row) -> the fused
//           decode epilogues per token, double-buffered TMEM accumulators so
//           the epilogue of tile i overlaps the main loop of tile i+1.
// ---------------------------------------------------------------------------
constexpr int TC_BM = 128, TC_BK = 64, TC_THREADS = 192;
constexpr int TC_A_STAGE = TC_BM * TC_BK * 2;  // 16 KB

template <int BN>
struct TcCfg {
    static constexpr int B_STAGE = BN * TC_BK * 2;
    static constexpr int STAGES = (196608) / (TC_A_STAGE + B_STAGE);
    static constexpr int TMEM_COLS = 2 * BN;  // two accumulator buffers
    static constexpr int SMEM = 1024 + STAGES * (TC_A_STAGE + B_STAGE) + 512;  // + barriers, tile queue
    static_assert(TMEM_COLS == 128 || TMEM_COLS == 256 || TMEM_COLS == 512, "TMEM allocation must be 2^k");
};

// Epilogue for one weight row `row` and 32 consecutive tokens [l0, l0 + 32).
// Every global load of a chunk (per-token rms scale, RoPE table, block-table
// entries, the residual) is issued before the first store: the loads are
// independent, so they overlap instead of paying one memory round trip per
// token behind a possibly-aliasing store. Per-token scalars are loaded once by
// lane j and broadcast with shuffles.
template <int KIND>
__device__ __forceinline__ void tc_epilogue(const PrefillArgs& a, int row, int l0, const uint32_t (&v)[32],
                                            int Lrows, int layer, int lane) {
    const Shape& s = a.s;
    const int nvalid = min(32, Lrows - l0);
    if constexpr (KIND == PF_QKV || KIND == PF_GU) {
        const float rs_l = lane < nvalid ? a.rs[l0 + lane] : 0.f;
        if constexpr (KIND == PF_QKV) {
            // a warp's 32 rows lie inside one section (q / k / v sizes are multiples of 32 rows)
            const QkvRow qr = qkv_row(s, row);
            const bool hi = (row & 8) != 0;  // partner row (row ^ 8) sits in lane ^ 8
            const int half = s.dh / 2;
            const int d0 = hi ? qr.dim - half : qr.dim;
            const int p0 = a.p0 + l0;
            // RoPE (cos, sin) per token; v rows rotate by (1, 0), which is exact
            float2 cs[32];
            if (qr.section < 2) {
#pragma unroll
                for (int j = 0; j < 32; ++j) cs[j] = a.w.rope[size_t(p0 + min(j, nvalid - 1)) * half + d0];
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) cs[j] = make_float2(1.f, 0.f);
            }
            float o[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const float r = __shfl_sync(0xffffffffu, rs_l, j);
                const float xs = __uint_as_float(v[j]) * r;
                const float ps = __shfl_xor_sync(0xffffffffu, xs, 8);
                o[j] = hi ? (xs * cs[j].x + ps * cs[j].y) : (xs * cs[j].x - ps * cs[j].y);
            }
            if (qr.section == 0) {  // q: bf16 [l][head][dh]
                uint16_t* qd = a.q + (size_t(l0) * s.n_heads + qr.head) * s.dh + qr.dim;
                const size_t qstride = size_t(s.n_heads) * s.dh;
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (j < nvalid) qd[j * qstride] = f_to_bf16(o[j]);
            } else {  // k / v: bf16 into the paged cache
                // lane j: byte offset of token l0 + j's slot row inside the head's block run
                const int pos_l = p0 + min(lane, nvalid - 1);
                const long long off_l = (long long)a.bt_row[pos_l / KV_BLOCK_TOKENS] * a.block_bytes +
                                        (pos_l % KV_BLOCK_TOKENS) * s.dh * 2;
                uint8_t* kvh = a.kv_base + kv_offset(s, layer, qr.section - 1, qr.head, 0);
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const long long off = __shfl_sync(0xffffffffu, off_l, j);
                    if (j < nvalid)
                        *reinterpret_cast<uint16_t*>(kvh + off + kv_dim_off(p0 + j, qr.dim)) = f_to_bf16(o[j]);
                }
            }
        } else {
            // gate rows sit in lanes 0-7 / 16-23, up rows in lanes 8-15 / 24-31. Lane
            // pairs (l, l^8) split the chunk: the gate lane finishes tokens 0-15, the up
            // lane tokens 16-31, so every lane stores and no lane idles.
            const bool hi = (row & 8) != 0;
            const int grow = (row >> 4) * 8 + (row & 7);  // output column of the pair
            uint16_t* out = a.abuf + size_t(l0) * s.ff + grow;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const float mine = __uint_as_float(hi ? v[16 + j] : v[j]);
                const float give = __uint_as_float(hi ? v[j] : v[16 + j]);
                const float peer = __shfl_xor_sync(0xffffffffu, give, 8);
                const int tok = hi ? 16 + j : j;
                const float r = __shfl_sync(0xffffffffu, rs_l, tok);
                const float gt = (hi ? peer : mine) * r, up = (hi ? mine : peer) * r;
                const float act = __fdividef(gt, 1.f + __expf(-gt)) * up;
                if (tok < nvalid) out[size_t(tok) * s.ff] = f_to_bf16(act);
            }
        }
    } else {  // PF_O / PF_DOWN: residual add, one coalesced 128-B row segment per token
        float* hp = a.h + size_t(l0) * s.d + row;
        float hv[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) hv[j] = j < nvalid ? hp[size_t(j) * s.d] : 0.f;
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (j < nvalid) hp[size_t(j) * s.d] = hv[j] + __uint_as_float(v[j]);
    }
}

template <int KIND, int BN, int CS>
__global__ void __launch_bounds__(TC_THREADS, 1)
    pf_gemm_tc(const __grid_constant__ PrefillArgs a, const __grid_constant__ CUtensorMap wmap,
               const __grid_constant__ CUtensorMap xmap, int N, int K, int Lrows, int layer, int splits) {
    using C = TcCfg<BN>;
    constexpr int B_PART = C::B_STAGE / CS;      // token rows this CTA fetches for the whole cluster
    constexpr uint16_t MASK = (1u << CS) - 1u;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t* As = smem;
    uint8_t* Bs = smem + C::STAGES * TC_A_STAGE;
    uint64_t* full = reinterpret_cast<uint64_t*>(Bs + C::STAGES * C::B_STAGE);
    uint64_t* empty = full + C::STAGES;
    uint64_t* tfull = empty + C::STAGES;  // [2] accumulator ready
    uint64_t* tempty = tfull + 2;         // [2] accumulator drained
    uint64_t* qfull = tempty + 2;         // [4] tile-queue slot written (dynamic schedule)
    uint64_t* qempty = qfull + 4;         // [4] tile-queue slot read by the MMA thread + 4 epilogue warps
    int* qid = reinterpret_cast<int*>(qempty + 4);  // [4]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(qid + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rank = CS > 1 ? int(cluster_ctarank()) : 0;
    const int cluster = blockIdx.x / CS, nclusters = gridDim.x / CS;
    // a cluster owns CS consecutive weight tiles and one token tile
    const int nN = (Lrows + BN - 1) / BN, ntiles = (N / TC_BM / CS) * nN, nk = K / TC_BK;
    // Split-K (CS == 1, tiles < SMs): work unit u = (tile u / splits, K range u % splits).
    // Every unit of a split tile writes its fp32 partial to the lane's workspace; the
    // last to arrive sums the partials in split order (deterministic) and runs the
    // fused epilogue. No unit waits for another (no co-residency assumption).
    const int nunits = ntiles * splits;
    auto krange = [&](int u, int& k0, int& k1) {
        const int sp = u % splits;
        k0 = (nk * sp) / splits;
        k1 = (nk * (sp + 1)) / splits;
    };
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, CS);  // a B stage is free once every CTA of the cluster consumed it
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(tfull + i, 1);
            mbar_init(tempty + i, 4);
        }
        for (int i = 0; i < 4; ++i) {
            mbar_init(qfull + i, 1);
            mbar_init(qempty + i, 5);
        }
        fence_mbar_init();
        prefetch_tmap(&wmap);
        prefetch_tmap(&xmap);
    }
    if (warp == 1) tmem_alloc(smem_u32(tmem_slot), C::TMEM_COLS);
    tc_fence_before();
    if constexpr (CS > 1) cluster_sync_all(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // Tile sequence. CS == 1: dynamic - the producer draws tiles from a
    // self-resetting global counter (late CTAs, e.g. ones queued behind another
    // lane's decode grid, simply find less work) and hands each tile to the MMA
    // thread and the epilogue warps through a 4-slot shared-memory queue.
    // CS > 1: static round-robin over clusters.
    auto draw = [&](int i, int t_static) -> int {  // producer
        if constexpr (CS > 1) {
            return t_static < ntiles ? t_static : -1;
        } else {
            const int sl = i & 3;
            mbar_wait(qempty + sl, ((i >> 2) & 1) ^ 1);
            const int t = atomicAdd(a.tile_ctr, 1);
            // nunits + gridDim.x draws in all; the last one resets the counter for the next launch
            if (t == nunits + int(gridDim.x) - 1) *reinterpret_cast<volatile int*>(a.tile_ctr) = 0;
            qid[sl] = t < nunits ? t : -1;
            mbar_arrive(qfull + sl);
            return t < nunits ? t : -1;
        }
    };
    // whole_warp: every lane reads the slot, then lane 0 releases it; else one thread does both
    auto take = [&](int i, int t_static, bool whole_warp) -> int {  // MMA thread / epilogue warps
        if constexpr (CS > 1) {
            return t_static < ntiles ? t_static : -1;
        } else {
            const int sl = i & 3;
            mbar_wait(qfull + sl, (i >> 2) & 1);
            const int t = *reinterpret_cast<volatile int*>(qid + sl);
            if (whole_warp) __syncwarp();
            if (!whole_warp || lane == 0) mbar_arrive(qempty + sl);
            return t;
        }
    };

    if (warp == 0) {
        if (lane == 0) {  // ---- producer
            int stage = 0;
            uint32_t phase = 0;
            for (int i = 0;; ++i) {
                const int u = draw(i, cluster + i * nclusters);
                if (u < 0) break;
                const int t = u / splits;
                const int mt = (t / nN) * CS + rank, nt = t % nN;
                int k0, k1;
                krange(u, k0, k1);
                for (int kb = k0; kb < k1; ++kb) {
                    mbar_wait(empty + stage, phase ^ 1);
                    mbar_arrive_expect_tx(full + stage, TC_A_STAGE + C::B_STAGE);
                    // eight pre-swizzled 16x64 blocks, one TMA instruction
                    tma_load_4d(As + stage * TC_A_STAGE, &wmap, 0, 0, kb, mt * (TC_BM / 16), full + stage);
                    uint8_t* bd = Bs + stage * C::B_STAGE + rank * B_PART;
                    const int row0 = nt * BN + rank * (BN / CS);
                    if constexpr (CS > 1)
                        tma_load_2d_mc(bd, &xmap, kb * TC_BK, row0, full + stage, MASK);
                    else
                        tma_load_2d(bd, &xmap, kb * TC_BK, row0, full + stage);
                    if (++stage == C::STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer
            constexpr uint32_t idesc = umma_idesc_bf16(TC_BM, BN);
            int stage = 0, acc = 0;
            uint32_t phase = 0, aphase = 0;
            for (int i = 0;; ++i) {
                const int u = take(i, cluster + i * nclusters, false);
                if (u < 0) break;
                int k0, k1;
                krange(u, k0, k1);
                mbar_wait(tempty + acc, aphase ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + uint32_t(acc * BN);
                for (int kb = k0; kb < k1; ++kb) {
                    mbar_wait(full + stage, phase);
                    tc_fence_after();
                    const uint64_t ad = umma_desc_sw128(smem_u32(As + stage * TC_A_STAGE));
                    const uint64_t bd = umma_desc_sw128(smem_u32(Bs + stage * C::B_STAGE));
#pragma unroll
                    for (int k = 0; k < TC_BK / 16; ++k)  // +32 B along the swizzled row per K=16
                        umma_bf16(d, ad + 2 * k, bd + 2 * k, idesc, (kb != k0) || k != 0);
                    if constexpr (CS > 1)
                        umma_commit_mc(empty + stage, MASK);
                    else
                        umma_commit(empty + stage);
                    if (++stage == C::STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                umma_commit(tfull + acc);
                if (++acc == 2) {
                    acc = 0;
                    aphase ^= 1;
                }
            }
        }
    } else {  // ---- epilogue warps 2..5: warp w reads TMEM lanes [32(w%4), 32(w%4)+32)
        const int sub = warp & 3;
        int acc = 0;
        uint32_t aphase = 0;
        int* last_flag = qid + 4 + 2;  // smem word past the tile queue and the TMEM slot
        for (int i = 0;; ++i) {
            const int u = take(i, cluster + i * nclusters, true);
            if (u < 0) break;
            const int t = u / splits;
            const int mt = (t / nN) * CS + rank, nt = t % nN;
            mbar_wait(tfull + acc, aphase);
            tc_fence_after();
            const int row = mt * TC_BM + sub * 32 + lane;
            if (splits == 1) {
#pragma unroll 1
                for (int c = 0; c < BN / 32; ++c) {
                    const int l0 = nt * BN + c * 32;
                    if (l0 >= Lrows) break;
                    uint32_t v[32];
                    tmem_ld32(tmem + (uint32_t(sub * 32) << 16) + uint32_t(acc * BN + c * 32), v);
                    tc_epilogue<KIND>(a, row, l0, v, Lrows, layer, lane);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(tempty + acc);
            } else {
                // partial -> workspace [unit][chunk][j4][row] float4: consecutive rows (threads)
                // write consecutive 16 B, so every warp store is one 512 B run
                float4* mine = reinterpret_cast<float4*>(a.sk_ws) + size_t(u) * (BN / 4) * TC_BM + sub * 32 + lane;
#pragma unroll 1
                for (int c = 0; c < BN / 32; ++c) {
                    if (nt * BN + c * 32 >= Lrows) break;
                    uint32_t v[32];
                    tmem_ld32(tmem + (uint32_t(sub * 32) << 16) + uint32_t(acc * BN + c * 32), v);
#pragma unroll
                    for (int j = 0; j < 32; j += 4)
                        __stcg(mine + size_t(c * 8 + j / 4) * TC_BM,
                               make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]),
                                           __uint_as_float(v[j + 2]), __uint_as_float(v[j + 3])));
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(tempty + acc);  // the accumulator is free again
                __threadfence();
                named_bar_sync(2, 128);  // the 4 epilogue warps wrote their rows
                if (sub == 2 && lane == 0) {
                    const int prev = atomicAdd(a.sk_cnt + t, 1);
                    const int last = prev == splits - 1;
                    if (last) a.sk_cnt[t] = 0;  // every unit of the tile arrived: reset for the next launch
                    *reinterpret_cast<volatile int*>(last_flag) = last;
                }
                named_bar_sync(2, 128);
                if (*reinterpret_cast<volatile int*>(last_flag)) {
                    __threadfence();
                    const float4* base =
                        reinterpret_cast<const float4*>(a.sk_ws) + size_t(t) * splits * (BN / 4) * TC_BM + sub * 32 + lane;
                    const size_t ustride = size_t(BN / 4) * TC_BM;
#pragma unroll 1
                    for (int c = 0; c < BN / 32; ++c) {
                        const int l0 = nt * BN + c * 32;
                        if (l0 >= Lrows) break;
                        // all splits' loads of the chunk in flight at once, then summed in split order
                        float4 q[4][8];
#pragma unroll
                        for (int sp = 0; sp < 4; ++sp)
#pragma unroll
                            for (int j4 = 0; j4 < 8; ++j4)
                                q[sp][j4] = sp < splits ? __ldcg(base + sp * ustride + size_t(c * 8 + j4) * TC_BM)
                                                        : make_float4(0.f, 0.f, 0.f, 0.f);
                        uint32_t v[32];
#pragma unroll
                        for (int j4 = 0; j4 < 8; ++j4) {
                            float4 acc4 = q[0][j4];
#pragma unroll
                            for (int sp = 1; sp < 4; ++sp)
                                if (sp < splits) {
                                    acc4.x += q[sp][j4].x;
                                    acc4.y += q[sp][j4].y;
                                    acc4.z += q[sp][j4].z;
                                    acc4.w += q[sp][j4].w;
                                }
                            v[4 * j4] = __float_as_uint(acc4.x);
                            v[4 * j4 + 1] = __float_as_uint(acc4.y);
                            v[4 * j4 + 2] = __float_as_uint(acc4.z);
                            v[4 * j4 + 3] = __float_as_uint(acc4.w);
                        }
                        tc_epilogue<KIND>(a, row, l0, v, Lrows, layer, lane);
                    }
                }
                named_bar_sync(2, 128);  // last_flag is rewritten by the next unit
            }
            if (++acc == 2) {
                acc = 0;
                aphase ^= 1;
            }
        }
    }
    tc_fence_before();
    // no CTA may leave while a peer can still multicast into its smem / barriers
    if constexpr (CS > 1) cluster_sync_all(); else __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, C::TMEM_COLS);
    }
}

// ---------------------------------------------------------------------------
// CTA-pair tcgen05 GEMM (cta_group::2): a 2-CTA cluster computes a 256-row x BN
// tile with one M = 256 MMA per K = 16 step. Rank r holds weight rows
// [128 r, 128 r + 128) and token rows [BN/2 r, BN/2 r + BN/2) of every stage, so
// each SM fills 32 KB of shared memory per 64-deep K block for a 128 x 256
// output (the single-CTA 128 x 256 tile needs 48 KB, and its operand stream,
// not the tensor pipe, set its pace). Rank 0 issues the MMAs; its commits
// arrive on both CTAs' barriers; each CTA's epilogue warps drain their own TMEM
// half (128 rows x BN) with the same fused epilogues. Tiles are dealt
// round-robin over clusters (both CTAs walk the same sequence).
// ---------------------------------------------------------------------------
template <int BN>
struct Tc2Cfg {
    static constexpr int A_STAGE = TC_A_STAGE;           // 128 rows x 64 K
    static constexpr int B_STAGE = (BN / 2) * TC_BK * 2;  // this CTA's half of the tokens
    static constexpr int STAGES = 196608 / (A_STAGE + B_STAGE);
    static constexpr int TMEM_COLS = 2 * BN;
    static constexpr int SMEM = 1024 + STAGES * (A_STAGE + B_STAGE) + 512;
};

template <int KIND, int BN>
__global__ void __launch_bounds__(TC_THREADS, 1)
    pf_gemm_2sm(const __grid_constant__ PrefillArgs a, const __grid_constant__ CUtensorMap wmap,
                const __grid_constant__ CUtensorMap xmap, int N, int K, int Lrows, int layer) {
    using C = Tc2Cfg<BN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t* As = smem;
    uint8_t* Bs = smem + C::STAGES * C::A_STAGE;
    uint64_t* full = reinterpret_cast<uint64_t*>(Bs + C::STAGES * C::B_STAGE);  // rank 0's count both halves
    uint64_t* empty = full + C::STAGES;
    uint64_t* tfull = empty + C::STAGES;  // [2]
    uint64_t* tempty = tfull + 2;         // [2] rank 0: both CTAs' epilogue warps (8)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const int cluster = blockIdx.x / 2, nclusters = gridDim.x / 2;
    const int nN = (Lrows + BN - 1) / BN, ntiles = (N / 256) * nN, nk = K / TC_BK;
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(tfull + i, 1);
            mbar_init(tempty + i, 8);
        }
        fence_mbar_init();
        prefetch_tmap(&wmap);
        prefetch_tmap(&xmap);
    }
    if (warp == 1) tmem_alloc_2sm(smem_u32(tmem_slot), C::TMEM_COLS);
    tc_fence_before();
    cluster_sync_all();  // barriers initialised and TMEM allocated in both CTAs
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---- producer (both CTAs): this CTA's halves of A and B
            int stage = 0;
            uint32_t phase = 0;
            for (int t = cluster; t < ntiles; t += nclusters) {
                const int mt = t / nN, nt = t % nN;
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(empty + stage, phase ^ 1);
                    if (rank == 0) mbar_arrive_expect_tx(full + stage, 2 * (C::A_STAGE + C::B_STAGE));
                    tma_load_4d_2sm(As + stage * C::A_STAGE, &wmap, 0, 0, kb, mt * 16 + int(rank) * 8, full + stage);
                    tma_load_2d_2sm(Bs + stage * C::B_STAGE, &xmap, kb * TC_BK, nt * BN + int(rank) * (BN / 2),
                                    full + stage);
                    if (++stage == C::STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {  // ---- MMA issuer (rank 0 only)
            constexpr uint32_t idesc = umma_idesc_bf16(256, BN);
            int stage = 0, acc = 0;
            uint32_t phase = 0, aphase = 0;
            for (int t = cluster; t < ntiles; t += nclusters) {
                mbar_wait_cluster(tempty + acc, aphase ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + uint32_t(acc * BN);
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(full + stage, phase);
                    tc_fence_after();
                    const uint64_t ad = umma_desc_sw128(smem_u32(As + stage * C::A_STAGE));
                    const uint64_t bd = umma_desc_sw128(smem_u32(Bs + stage * C::B_STAGE));
#pragma unroll
                    for (int k = 0; k < TC_BK / 16; ++k)
                        umma_bf16_2sm(d, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
                    umma_commit_2sm_mc(empty + stage, 3);
                    if (++stage == C::STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                umma_commit_2sm_mc(tfull + acc, 3);
                if (++acc == 2) {
                    acc = 0;
                    aphase ^= 1;
                }
            }
        }
    } else {  // ---- epilogue warps 2..5 (both CTAs): this CTA's 128 rows of the tile
        const int sub = warp & 3;
        int acc = 0;
        uint32_t aphase = 0;
        for (int t = cluster; t < ntiles; t += nclusters) {
            const int mt = t / nN, nt = t % nN;
            mbar_wait_cluster(tfull + acc, aphase);
            tc_fence_after();
            const int row = mt * 256 + int(rank) * 128 + sub * 32 + lane;
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
                const int l0 = nt * BN + c * 32;
                if (l0 >= Lrows) break;
                uint32_t v[32];
                tmem_ld32(tmem + (uint32_t(sub * 32) << 16) + uint32_t(acc * BN + c * 32), v);
                tc_epilogue<KIND>(a, row, l0, v, Lrows, layer, lane);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (rank == 0)
                    mbar_arrive(tempty + acc);
                else
                    mbar_arrive_remote(tempty + acc, 0);
            }
            if (++acc == 2) {
                acc = 0;
                aphase ^= 1;
            }
        }
    }
    tc_fence_before();
    cluster_sync_all();  // no CTA leaves while its peer's MMAs or arrives may still target it
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_2sm(tmem, C::TMEM_COLS);
    }
}

__global__ void pf_embed(const __grid_constant__ PrefillArgs a) {
    const int l = blockIdx.x;
    const int tok = a.tokens[l];
    for (int i = threadIdx.x; i < a.s.d; i += blockDim.x)
        a.h[size_t(l) * a.s.d + i] = bf16_to_f(a.w.emb[size_t(tok) * a.s.d + i]);
}

// act[l] = bf16(h[l] * gamma), rs[l] = rsqrt(mean(h[l]^2) + eps); one warp per row.
// The row is read once into registers with 16-byte loads (d <= 32 * 4 * RN_MAXV),
// so the pass is one HBM read of h and one write of act (it was 19 us per 7B
// layer at L = 1024 with strided scalar loads read twice).
constexpr int RN_MAXV = 40;  // float4 per lane: d <= 5120
__global__ void __launch_bounds__(128) pf_rownorm(const float* __restrict__ h, const float* __restrict__ gamma,
                                                 uint16_t* act, float* rs, int rows, int d, float eps) {
    const int row = blockIdx.x * 4 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const float4* hr = reinterpret_cast<const float4*>(h + size_t(row) * d);
    const int nv = d / 128;  // float4 per lane
    float4 v[RN_MAXV];
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < RN_MAXV; ++i)
        if (i < nv) {
            v[i] = hr[i * 32 + lane];
            ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
        }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const float4* gr = reinterpret_cast<const float4*>(gamma);
    uint2* ar = reinterpret_cast<uint2*>(act + size_t(row) * d);
#pragma unroll
    for (int i = 0; i < RN_MAXV; ++i)
        if (i < nv) {
            const float4 g = gr[i * 32 + lane];
            ar[i * 32 + lane] = make_uint2(pack_bf16x2(v[i].x * g.x, v[i].y * g.y), pack_bf16x2(v[i].z * g.z, v[i].w * g.w));
        }
    if (lane == 0) rs[row] = rsqrtf(ss / float(d) + eps);
}

// Causal attention over the paged cache on the tensor cores (mma.sync
// m16n8k16, flash-attention style). Block = 64 queries of one head, 4 warps x
// 16 query rows. Keys stream in 64-token chunks: every 16-token KV block of a
// (layer, k|v, kv-head) is a contiguous run whose 16-byte chunks are already
// XOR-swizzled by (slot & 7), so the chunk is copied raw with cp.async (double
// buffered) and read conflict-free by ldmatrix (K) / ldmatrix.trans (V).
// S = Q.K^T, online softmax in fp32 (exp2 with the scale folded), O += P.V
// with P re-packed from the S accumulators as the A operand.
constexpr int PA_QT = 64, PA_KC = 64, PA_THREADS = 128;
template <int DH>
constexpr int pa_smem() { return 2 * 2 * PA_KC * DH * 2; }  // 2 stages x (K, V)

template <int DH>
__global__ void __launch_bounds__(PA_THREADS) pf_attn(const __grid_constant__ PrefillArgs a, int layer) {
    constexpr int ROWB = DH * 2, TILE = PA_KC * ROWB, NT = PA_KC / 8, DT = DH / 8;
    extern __shared__ __align__(128) uint8_t sm[];
    const Shape& s = a.s;
    const int nqt = (a.L + PA_QT - 1) / PA_QT;
    const int qt = nqt - 1 - int(blockIdx.x);  // longest rows first
    const int head = blockIdx.y, kvh = head / s.gq();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int q0 = qt * PA_QT;
    const int kmax = a.p0 + min(q0 + PA_QT, a.L) - 1;  // last key any query of the block sees
    const int nchunks = kmax / PA_KC + 1;
    const size_t koff = kv_offset(s, layer, 0, kvh, 0), voff = kv_offset(s, layer, 1, kvh, 0);
    const uint8_t* blk0 = a.kv_base + size_t(a.bt_row[0]) * a.block_bytes;  // mapped; zero-fill source

    auto load_chunk = [&](int c, int stage) {
        const uint32_t ks = smem_u32(sm + stage * 2 * TILE), vs = ks + TILE;
#pragma unroll
        for (int i = threadIdx.x; i < TILE / 16; i += PA_THREADS) {
            const int r = i / (ROWB / 16), cc = i % (ROWB / 16);
            const int pos = c * PA_KC + r;
            const bool ok = pos <= kmax;  // rows past the last key are zero-filled (no stale NaN)
            const uint8_t* base =
                ok ? a.kv_base + size_t(a.bt_row[pos / KV_BLOCK_TOKENS]) * a.block_bytes +
                         size_t(pos % KV_BLOCK_TOKENS) * ROWB + cc * 16
                   : blk0;
            cp_async16(ks + r * ROWB + cc * 16, ok ? base + koff : blk0, ok ? 16 : 0);
            cp_async16(vs + r * ROWB + cc * 16, ok ? base + voff : blk0, ok ? 16 : 0);
        }
    };

    // Q fragments (bf16) for this warp's 16 rows, straight from the fp32 q buffer
    const int r0 = q0 + warp * 16 + g, r1 = r0 + 8;
    uint32_t qa[DH / 16][4];
    {
        const uint16_t* qp0 = a.q + (size_t(r0) * s.n_heads + head) * DH;
        const uint16_t* qp1 = a.q + (size_t(r1) * s.n_heads + head) * DH;
        const bool v0 = r0 < a.L, v1 = r1 < a.L;
#pragma unroll
        for (int kc = 0; kc < DH / 16; ++kc) {
            const int c0 = kc * 16 + 2 * t;
            qa[kc][0] = v0 ? *reinterpret_cast<const uint32_t*>(qp0 + c0) : 0u;
            qa[kc][1] = v1 ? *reinterpret_cast<const uint32_t*>(qp1 + c0) : 0u;
            qa[kc][2] = v0 ? *reinterpret_cast<const uint32_t*>(qp0 + c0 + 8) : 0u;
            qa[kc][3] = v1 ? *reinterpret_cast<const uint32_t*>(qp1 + c0 + 8) : 0u;
        }
    }
    const int qpos0 = a.p0 + r0, qpos1 = a.p0 + r1;
    const int warp_last = a.p0 + q0 + warp * 16 + 15;
    const float sl2 = rsqrtf(float(DH)) * 1.4426950408889634f;

    float o[DT][4];
#pragma unroll
    for (int i = 0; i < DT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

    load_chunk(0, 0);
    cp_async_commit();
    for (int c = 0; c < nchunks; ++c) {
        if (c + 1 < nchunks) load_chunk(c + 1, (c + 1) & 1);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        const int kbase = c * PA_KC;
        if (kbase <= warp_last) {  // warp-uniform: some key of the chunk is visible to some row
            const uint32_t ks = smem_u32(sm + (c & 1) * 2 * TILE), vs = ks + TILE;
            float sc[NT][4];
#pragma unroll
            for (int i = 0; i < NT; ++i) sc[i][0] = sc[i][1] = sc[i][2] = sc[i][3] = 0.f;
#pragma unroll
            for (int kc = 0; kc < DH / 16; ++kc) {
#pragma unroll
                for (int np = 0; np < NT / 2; ++np) {
                    const int r = np * 16 + (lane & 7) + ((lane >> 4) << 3);
                    const int ch = kc * 2 + ((lane >> 3) & 1);
                    uint32_t b0, b1, b2, b3;
                    ldmatrix_x4(ks + r * ROWB + ((ch ^ (r & 7)) << 4), b0, b1, b2, b3);
                    mma_bf16_16816(sc[2 * np], qa[kc][0], qa[kc][1], qa[kc][2], qa[kc][3], b0, b1);
                    mma_bf16_16816(sc[2 * np + 1], qa[kc][0], qa[kc][1], qa[kc][2], qa[kc][3], b2, b3);
                }
            }
            // causal mask + scale (log2 domain), row maxima over the quad
            float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int key = kbase + nt * 8 + 2 * t + (e & 1);
                    const int qp = e < 2 ? qpos0 : qpos1;
                    const float v = key <= qp ? sc[nt][e] * sl2 : -INFINITY;
                    sc[nt][e] = v;
                    if (e < 2) mx0 = fmaxf(mx0, v); else mx1 = fmaxf(mx1, v);
                }
            }
#pragma unroll
            for (int off = 1; off < 4; off <<= 1) {
                mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
                mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
            }
            const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
            // a row with nothing visible yet keeps m = -inf: use 0 as the reference so exp2 gives 0
            const float b0r = mn0 == -INFINITY ? 0.f : mn0, b1r = mn1 == -INFINITY ? 0.f : mn1;
            const float cr0 = exp2f(m0 - b0r), cr1 = exp2f(m1 - b1r);
            m0 = mn0;
            m1 = mn1;
            l0 *= cr0;
            l1 *= cr1;
#pragma unroll
            for (int i = 0; i < DT; ++i) {
                o[i][0] *= cr0;
                o[i][1] *= cr0;
                o[i][2] *= cr1;
                o[i][3] *= cr1;
            }
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                sc[nt][0] = exp2f(sc[nt][0] - b0r);
                sc[nt][1] = exp2f(sc[nt][1] - b0r);
                sc[nt][2] = exp2f(sc[nt][2] - b1r);
                sc[nt][3] = exp2f(sc[nt][3] - b1r);
                l0 += sc[nt][0] + sc[nt][1];
                l1 += sc[nt][2] + sc[nt][3];
            }
            // O += P.V
#pragma unroll
            for (int kk = 0; kk < PA_KC / 16; ++kk) {
                const uint32_t p0 = pack_bf16x2(sc[2 * kk][0], sc[2 * kk][1]);
                const uint32_t p1 = pack_bf16x2(sc[2 * kk][2], sc[2 * kk][3]);
                const uint32_t p2 = pack_bf16x2(sc[2 * kk + 1][0], sc[2 * kk + 1][1]);
                const uint32_t p3 = pack_bf16x2(sc[2 * kk + 1][2], sc[2 * kk + 1][3]);
                const int key = kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
#pragma unroll
                for (int dp = 0; dp < DT / 2; ++dp) {
                    const int ch = dp * 2 + (lane >> 4);
                    uint32_t v0, v1, v2, v3;
                    ldmatrix_x4_trans(vs + key * ROWB + ((ch ^ (key & 7)) << 4), v0, v1, v2, v3);
                    mma_bf16_16816(o[2 * dp], p0, p1, p2, p3, v0, v1);
                    mma_bf16_16816(o[2 * dp + 1], p0, p1, p2, p3, v2, v3);
                }
            }
        }
        __syncthreads();  // the stage is refilled next iteration
    }
#pragma unroll
    for (int off = 1; off < 4; off <<= 1) {
        l0 += __shfl_xor_sync(0xffffffffu, l0, off);
        l1 += __shfl_xor_sync(0xffffffffu, l1, off);
    }
    const float i0 = 1.f / l0, i1 = 1.f / l1;
#pragma unroll
    for (int dt = 0; dt < DT; ++dt) {
        const int col = head * DH + dt * 8 + 2 * t;
        if (r0 < a.L)
            *reinterpret_cast<uint32_t*>(a.attn + size_t(r0) * s.d + col) = pack_bf16x2(o[dt][0] * i0, o[dt][1] * i0);
        if (r1 < a.L)
            *reinterpret_cast<uint32_t*>(a.attn + size_t(r1) * s.d + col) = pack_bf16x2(o[dt][2] * i1, o[dt][3] * i1);
    }
}

// ---------------------------------------------------------------------------
// Causal attention on the 5th-gen tensor cores (tcgen05, TMEM accumulators).
// Block = 128 queries of one head (the UMMA M); keys in 64-token chunks.
//   warp 0      TMA producer: every 16-token KV block of the chunk is two (dh 64:
//               one) 2 KB boxes per K and V, copied from the paged cache into the
//               canonical SW128 layout (the cache's chunk swizzle by slot & 7 IS
//               the 128-byte swizzle of an 8-row atom: the bytes land verbatim)
//   warp 1      TMEM owner + single-thread MMA issuer:
//                 S[j & 1] = Q . K_j^T   (M 128, N 64, K = dh; both K-major)
//                 O       += P_j . V_j   (M 128, N dh, K 64; V read MN-major)
//               S of chunk j+1 is issued before P_j is ready, so it overlaps the
//               softmax of chunk j
//   warps 2-5   softmax, one query row per thread straight from TMEM: causal
//               mask, running max in the log2 domain with a lazy O rescale (only
//               when the max grows by more than 2^8; numerator and denominator
//               share the reference, so the result is exact), P -> shared memory
//               as bf16 in the SW128 K-major layout, final O / l -> bf16
// TMEM: O in columns [0, dh), the two S buffers at 128 and 192.
constexpr int TA_QT = 128, TA_KC = 64, TA_THREADS = 192, TA_STAGES = 3;
// MESH_PF_ATTN_DEBUG: bounded mbarrier waits that record (block, thread, barrier, chunk) in
// host-mapped memory on a timeout and give up (results are then garbage), to locate a hang.
__device__ int* g_ta_dbg = nullptr;
__device__ __forceinline__ float ex2_approx(float x) {  // MUFU.EX2 without the denormal range fix-up
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ unsigned long long* g_ta_trace = nullptr;  // MESH_PF_ATTN_TRACE: CTA (0, 0) event timeline
__device__ __forceinline__ void ta_trace(int id, int j) {
    // plain stores into device memory at [id][j] (no atomics, no host round trips)
    if (!g_ta_trace || blockIdx.x != 0 || blockIdx.y != 0 || j >= 1024) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_ta_trace[id * 1024 + j] = t;
}
__device__ __forceinline__ void ta_wait(uint64_t* bar, uint32_t parity, int id, int j) {
    if (!g_ta_dbg) {
        mbar_wait(bar, parity);
        return;
    }
    if ((threadIdx.x & 31) == 0) {  // heartbeat: (barrier, chunk) each warp is about to wait on
        const int cta = blockIdx.y * gridDim.x + blockIdx.x;
        if (cta < 150) reinterpret_cast<volatile int*>(g_ta_dbg)[512 + cta * 6 + (threadIdx.x >> 5)] = (id << 16) | j;
    }
    for (long long spin = 0; !mbar_try_wait(bar, parity); ++spin)
        if (spin > (1ll << 40)) {
            volatile int* d = g_ta_dbg;
            const int slot = atomicAdd(const_cast<int*>(g_ta_dbg), 1) % 60;
            d[1 + slot * 6 + 0] = blockIdx.x;
            d[1 + slot * 6 + 1] = blockIdx.y;
            d[1 + slot * 6 + 2] = threadIdx.x;
            d[1 + slot * 6 + 3] = id;
            d[1 + slot * 6 + 4] = j;
            d[1 + slot * 6 + 5] = int(parity);
            __threadfence_system();
            return;
        }
}
template <int DH>
struct TaCfg {
    static constexpr int HALVES = DH / 64;                // 128-byte K atoms per row
    static constexpr int Q_HALF = TA_QT * 128;            // Q: [half][128 rows][128 B]
    static constexpr int KV_HALF = TA_KC * 128;           // K or V: [half][64 keys][128 B]
    static constexpr int K_BYTES = HALVES * KV_HALF;
    static constexpr int STAGE = 2 * K_BYTES;             // K, then V
    static constexpr int P_BYTES = TA_QT * 128;           // P: [128 queries][64 keys bf16]
    static constexpr int Q_OFF = 0, ST_OFF = HALVES * Q_HALF, P_OFF = ST_OFF + TA_STAGES * STAGE;
    static constexpr int BAR_OFF = P_OFF + P_BYTES;
    static constexpr int SMEM = 1024 + BAR_OFF + 256;
    static constexpr uint32_t TMEM_COLS = 256;
};

template <int DH>
__global__ void __launch_bounds__(TA_THREADS, 1)
    pf_attn_tc(const __grid_constant__ PrefillArgs a, const __grid_constant__ CUtensorMap kvmap, int layer) {
    using C = TaCfg<DH>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    uint64_t* kv_full = reinterpret_cast<uint64_t*>(sm + C::BAR_OFF);
    uint64_t* kv_empty = kv_full + TA_STAGES;
    uint64_t* s_full = kv_empty + TA_STAGES;  // [2]
    uint64_t* s_empty = s_full + 2;           // [2]
    uint64_t* p_full = s_empty + 2;
    uint64_t* pv_done = p_full + 1;
    uint64_t* q_ready = pv_done + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_ready + 1);

    const Shape& s = a.s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nqt = (a.L + TA_QT - 1) / TA_QT;
    const int qt = nqt - 1 - int(blockIdx.x);  // longest rows first
    const int head = blockIdx.y, kvh = head / s.gq();
    const int q0 = qt * TA_QT;
    const int kmax = a.p0 + min(q0 + TA_QT, a.L) - 1;  // last key any query of the block sees
    const int nchunks = kmax / TA_KC + 1;
    if (threadIdx.x == 0) {
        for (int i = 0; i < TA_STAGES; ++i) {
            mbar_init(kv_full + i, 1);
            mbar_init(kv_empty + i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(s_full + i, 1);
            mbar_init(s_empty + i, 128);
        }
        mbar_init(p_full, 128);
        mbar_init(pv_done, 1);
        mbar_init(q_ready, 128);
        fence_mbar_init();
        prefetch_tmap(&kvmap);
    }
    if (warp == 1) tmem_alloc(smem_u32(tmem_slot), C::TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer
            const int rK = ((layer * s.n_kv + kvh) * 2 + 0) * KV_BLOCK_TOKENS;
            const int rV = ((layer * s.n_kv + kvh) * 2 + 1) * KV_BLOCK_TOKENS;
            for (int j = 0; j < nchunks; ++j) {
                const int st = j % TA_STAGES;
                ta_wait(kv_empty + st, ((j / TA_STAGES) & 1) ^ 1, 1, j);
                uint8_t* kb = sm + C::ST_OFF + st * C::STAGE;
                mbar_arrive_expect_tx(kv_full + st, C::STAGE);
#pragma unroll
                for (int bi = 0; bi < TA_KC / KV_BLOCK_TOKENS; ++bi) {
                    const int pos = j * TA_KC + bi * KV_BLOCK_TOKENS;
                    // blocks past the last key: any mapped block (their rows are masked / zeroed)
                    const int blk = a.bt_row[(pos <= kmax ? pos : 0) / KV_BLOCK_TOKENS];
#pragma unroll
                    for (int hh = 0; hh < C::HALVES; ++hh) {
                        const int off = hh * C::KV_HALF + bi * KV_BLOCK_TOKENS * 128;
                        tma_load_4d(kb + off, &kvmap, 0, hh, rK, blk, kv_full + st);
                        tma_load_4d(kb + C::K_BYTES + off, &kvmap, 0, hh, rV, blk, kv_full + st);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer
            constexpr uint32_t idesc_s = umma_idesc_bf16(TA_QT, TA_KC);
            constexpr uint32_t idesc_o = umma_idesc_bf16(TA_QT, DH) | (1u << 16);  // B (V) MN-major
            const uint32_t q_addr = smem_u32(sm + C::Q_OFF), p_addr = smem_u32(sm + C::P_OFF);
            ta_wait(q_ready, 0, 2, 0);
            tc_fence_after();
            auto issue_s = [&](int j) {
                const int st = j % TA_STAGES, sb = j & 1;
                ta_wait(kv_full + st, (j / TA_STAGES) & 1, 3, j);
                ta_wait(s_empty + sb, ((j >> 1) & 1) ^ 1, 4, j);
                tc_fence_after();
                const uint32_t k_addr = smem_u32(sm + C::ST_OFF + st * C::STAGE);
#pragma unroll
                for (int hh = 0; hh < C::HALVES; ++hh) {
                    const uint64_t qd = umma_desc_sw128(q_addr + hh * C::Q_HALF);
                    const uint64_t kd = umma_desc_sw128(k_addr + hh * C::KV_HALF);
#pragma unroll
                    for (int k = 0; k < 4; ++k)  // +32 B along the swizzled row per K = 16
                        umma_bf16(tmem + 128u + uint32_t(sb * TA_KC), qd + 2 * k, kd + 2 * k, idesc_s, (hh | k) != 0);
                }
                umma_commit(s_full + sb);
            };
            issue_s(0);
            for (int j = 0; j < nchunks; ++j) {
                if (j + 1 < nchunks) issue_s(j + 1);
                const int st = j % TA_STAGES;
                ta_wait(p_full, j & 1, 5, j);
                tc_fence_after();
                const uint32_t v_addr = smem_u32(sm + C::ST_OFF + st * C::STAGE + C::K_BYTES);
                const uint64_t pd = umma_desc_sw128(p_addr);
#pragma unroll
                for (int k = 0; k < TA_KC / 16; ++k)  // 16 keys = two 8-row groups = 2048 B of V
                    umma_bf16(tmem, pd + 2 * k, umma_desc_sw128_mn(v_addr + k * 2048, C::KV_HALF), idesc_o,
                              (j | k) != 0);
                umma_commit(kv_empty + st);
                umma_commit(pv_done);
            }
        }
    } else {  // ---- softmax warps 2..5: thread = one query row (TMEM lane)
        const int sub = warp & 3, row = sub * 32 + lane;
        const uint32_t lane_addr = tmem + (uint32_t(sub * 32) << 16);
        const int r = q0 + row;
        {  // Q row -> canonical SW128 K-major (bf16, RoPE already applied)
            const uint4* src = reinterpret_cast<const uint4*>(a.q + (size_t(r) * s.n_heads + head) * DH);
#pragma unroll
            for (int c = 0; c < DH / 8; ++c) {
                const uint4 v = r < a.L ? src[c] : make_uint4(0, 0, 0, 0);
                const int hh = c >> 3, cc = c & 7;
                *reinterpret_cast<uint4*>(sm + C::Q_OFF + hh * C::Q_HALF + row * 128 + ((cc ^ (row & 7)) << 4)) = v;
            }
        }
        fence_proxy_async_smem();
        mbar_arrive(q_ready);
        const int qpos = a.p0 + r;
        const float sl2 = rsqrtf(float(DH)) * 1.4426950408889634f;
        float mref = -INFINITY, l = 0.f;
        for (int j = 0; j < nchunks; ++j) {
            const int sb = j & 1, kbase = j * TA_KC;
            ta_wait(s_full + sb, (j >> 1) & 1, 6, j);
            tc_fence_after();
            uint32_t sv[2][32];
            tmem_ld32(lane_addr + 128u + uint32_t(sb * TA_KC), sv[0]);
            tmem_ld32(lane_addr + 128u + uint32_t(sb * TA_KC + 32), sv[1]);
            tc_fence_before();
            mbar_arrive(s_empty + sb);
            float p[64];
            float mx = -INFINITY;
#pragma unroll
            for (int k = 0; k < 64; ++k) {
                const float v = __uint_as_float(sv[k >> 5][k & 31]);
                p[k] = kbase + k <= qpos ? v * sl2 : -INFINITY;
                mx = fmaxf(mx, p[k]);
            }
            if (j > 0) ta_wait(pv_done, (j - 1) & 1, 7, j);  // O stable, P buffer free
            tc_fence_after();
            // lazy rescale: only when a row's max grows by more than 2^8. tcgen05.ld / st are
            // warp-collective, so the warp rescales if any of its rows must (others by 1)
            const bool grow = mx > mref + 8.f;
            const float corr = (grow && mref != -INFINITY) ? exp2f(mref - mx) : 1.f;
            if (__any_sync(0xffffffffu, corr != 1.f)) {
#pragma unroll 1
                for (int c = 0; c < DH / 32; ++c) {
                    uint32_t o[32];
                    tmem_ld32(lane_addr + uint32_t(c * 32), o);
#pragma unroll
                    for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * corr);
                    tmem_st32(lane_addr + uint32_t(c * 32), o);
                }
            }
            l *= corr;
            if (grow) mref = mx;
            uint8_t* prow = sm + C::P_OFF + row * 128;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                float e[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    e[i] = mref == -INFINITY ? 0.f : exp2f(p[c * 8 + i] - mref);
                    l += e[i];
                }
                uint4 pk;
                pk.x = pack_bf16x2(e[0], e[1]);
                pk.y = pack_bf16x2(e[2], e[3]);
                pk.z = pack_bf16x2(e[4], e[5]);
                pk.w = pack_bf16x2(e[6], e[7]);
                *reinterpret_cast<uint4*>(prow + ((c ^ (row & 7)) << 4)) = pk;
            }
            if (j == nchunks - 1 && kmax < kbase + TA_KC - 1) {
                // keys past the last one: P is 0 there, but 0 x NaN (unwritten cache rows)
                // would still reach O through the MMA, so zero those V rows
                uint8_t* vb = sm + C::ST_OFF + (j % TA_STAGES) * C::STAGE + C::K_BYTES;
                const int k0 = kmax + 1 - kbase, n16 = (TA_KC - k0) * 8 * C::HALVES;
                for (int i = row; i < n16; i += 128) {
                    const int hh = i / ((TA_KC - k0) * 8), rem = i % ((TA_KC - k0) * 8);
                    *reinterpret_cast<uint4*>(vb + hh * C::KV_HALF + (k0 + rem / 8) * 128 + (rem % 8) * 16) =
                        make_uint4(0, 0, 0, 0);
                }
            }
            fence_proxy_async_smem();
            tc_fence_before();
            mbar_arrive(p_full);
        }
        ta_wait(pv_done, (nchunks - 1) & 1, 8, nchunks);
        tc_fence_after();
        const float inv = 1.f / l;
#pragma unroll 1
        for (int c = 0; c < DH / 32; ++c) {
            uint32_t o[32];
            tmem_ld32(lane_addr + uint32_t(c * 32), o);
            if (r < a.L) {
                uint16_t* dst = a.attn + size_t(r) * s.d + head * DH + c * 32;
#pragma unroll
                for (int i = 0; i < 32; i += 8) {
                    uint4 pk;
                    pk.x = pack_bf16x2(__uint_as_float(o[i]) * inv, __uint_as_float(o[i + 1]) * inv);
                    pk.y = pack_bf16x2(__uint_as_float(o[i + 2]) * inv, __uint_as_float(o[i + 3]) * inv);
                    pk.z = pack_bf16x2(__uint_as_float(o[i + 4]) * inv, __uint_as_float(o[i + 5]) * inv);
                    pk.w = pack_bf16x2(__uint_as_float(o[i + 6]) * inv, __uint_as_float(o[i + 7]) * inv);
                    *reinterpret_cast<uint4*>(dst + i) = pk;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, C::TMEM_COLS);
    }
}

// Two query tiles per CTA, ping-ponged on the tensor core (FA4-style): query
// tiles 2i and 2i+1 of one head share every K/V chunk (loaded once), and two
// softmax warpgroups alternate with the MMA pipe -- while warpgroup A turns S_A
// into P_A, the tensor core computes S_B / PV_B, and vice versa.
//   warp 0: TMA producer; warp 1: MMA issuer (+ TMEM owner);
//   warps 2-5: softmax of tile A, warps 6-9: softmax of tile B.
// S is double-buffered per tile so the issuer runs S_t(j+1) ahead of PV_t(j): a
// warpgroup's next scores are ready the moment it finishes P_t(j).
// TMEM (512 columns): O_A [0, dh), O_B [128, 128 + dh), S_t buffer b at 256 + 128 t + 64 b.
constexpr int T2_THREADS = 320;
template <int DH>
struct Ta2Cfg {
    static constexpr int HALVES = DH / 64;
    static constexpr int Q_HALF = TA_QT * 128;
    static constexpr int Q_TILE = HALVES * Q_HALF;        // one tile's Q
    static constexpr int KV_HALF = TA_KC * 128;
    static constexpr int K_BYTES = HALVES * KV_HALF;
    static constexpr int STAGE = 2 * K_BYTES;
    static constexpr int P_TILE = TA_QT * 128;
    static constexpr int Q_OFF = 0, ST_OFF = 2 * Q_TILE, P_OFF = ST_OFF + TA_STAGES * STAGE;
    static constexpr int BAR_OFF = P_OFF + 2 * P_TILE;
    static constexpr int SMEM = 1024 + BAR_OFF + 256;
    static constexpr uint32_t TMEM_COLS = 512;
};

template <int DH>
__global__ void __launch_bounds__(T2_THREADS, 1)
    pf_attn_tc2(const __grid_constant__ PrefillArgs a, const __grid_constant__ CUtensorMap kvmap, int layer) {
    using C = Ta2Cfg<DH>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    uint64_t* kv_full = reinterpret_cast<uint64_t*>(sm + C::BAR_OFF);
    uint64_t* kv_empty = kv_full + TA_STAGES;
    uint64_t* s_full = kv_empty + TA_STAGES;  // [tile][buffer]
    uint64_t* s_empty = s_full + 4;           // [tile][buffer]
    uint64_t* p_full = s_empty + 4;           // [tile]
    uint64_t* pv_done = p_full + 2;           // [tile]
    uint64_t* q_ready = pv_done + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_ready + 1);

    const Shape& s = a.s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nqt = (a.L + TA_QT - 1) / TA_QT, npair = (nqt + 1) / 2;
    const int qp = npair - 1 - int(blockIdx.x);  // longest rows first
    const int head = blockIdx.y, kvh = head / s.gq();
    // tile t covers queries [q0[t], q0[t] + 128); tile B may not exist (odd tile count)
    int q0[2], nch[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        q0[t] = (2 * qp + t) * TA_QT;
        nch[t] = q0[t] < a.L ? (a.p0 + min(q0[t] + TA_QT, a.L) - 1) / TA_KC + 1 : 0;
    }
    const int nchunks = max(nch[0], nch[1]);
    const int kmax = a.p0 + min(q0[nch[1] ? 1 : 0] + TA_QT, a.L) - 1;  // last key any query of the CTA sees
    if (threadIdx.x == 0) {
        for (int i = 0; i < TA_STAGES; ++i) {
            mbar_init(kv_full + i, 1);
            mbar_init(kv_empty + i, 1);
        }
        for (int t = 0; t < 4; ++t) {
            mbar_init(s_full + t, 1);
            mbar_init(s_empty + t, 128);
        }
        for (int t = 0; t < 2; ++t) {
            mbar_init(p_full + t, 128);
            mbar_init(pv_done + t, 1);
        }
        mbar_init(q_ready, 256);
        fence_mbar_init();
        prefetch_tmap(&kvmap);
    }
    if (warp == 1) tmem_alloc(smem_u32(tmem_slot), C::TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer (one K/V stream for both tiles)
            const int rK = ((layer * s.n_kv + kvh) * 2 + 0) * KV_BLOCK_TOKENS;
            const int rV = ((layer * s.n_kv + kvh) * 2 + 1) * KV_BLOCK_TOKENS;
            for (int j = 0; j < nchunks; ++j) {
                const int st = j % TA_STAGES;
                ta_wait(kv_empty + st, ((j / TA_STAGES) & 1) ^ 1, 1, j);
                uint8_t* kb = sm + C::ST_OFF + st * C::STAGE;
                ta_trace(10, j);
                mbar_arrive_expect_tx(kv_full + st, C::STAGE);
#pragma unroll
                for (int bi = 0; bi < TA_KC / KV_BLOCK_TOKENS; ++bi) {
                    const int pos = j * TA_KC + bi * KV_BLOCK_TOKENS;
                    const int blk = a.bt_row[(pos <= kmax ? pos : 0) / KV_BLOCK_TOKENS];
#pragma unroll
                    for (int hh = 0; hh < C::HALVES; ++hh) {
                        const int off = hh * C::KV_HALF + bi * KV_BLOCK_TOKENS * 128;
                        tma_load_4d(kb + off, &kvmap, 0, hh, rK, blk, kv_full + st);
                        tma_load_4d(kb + C::K_BYTES + off, &kvmap, 0, hh, rV, blk, kv_full + st);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer: S_A(0), S_B(0), then per chunk S_A(j+1), PV_A(j), S_B(j+1), PV_B(j)
            constexpr uint32_t idesc_s = umma_idesc_bf16(TA_QT, TA_KC);
            constexpr uint32_t idesc_o = umma_idesc_bf16(TA_QT, DH) | (1u << 16);  // B (V) MN-major
            ta_wait(q_ready, 0, 2, 0);
            tc_fence_after();
            auto issue_s = [&](int t, int j) {
                const int st = j % TA_STAGES;
                ta_wait(kv_full + st, (j / TA_STAGES) & 1, 3, j);
                ta_wait(s_empty + 2 * t + (j & 1), ((j >> 1) & 1) ^ 1, 4, j);
                tc_fence_after();
                const uint32_t k_addr = smem_u32(sm + C::ST_OFF + st * C::STAGE);
                const uint32_t q_addr = smem_u32(sm + C::Q_OFF + t * C::Q_TILE);
#pragma unroll
                for (int hh = 0; hh < C::HALVES; ++hh) {
                    const uint64_t qd = umma_desc_sw128(q_addr + hh * C::Q_HALF);
                    const uint64_t kd = umma_desc_sw128(k_addr + hh * C::KV_HALF);
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        umma_bf16(tmem + 256u + uint32_t(t * 128 + (j & 1) * 64), qd + 2 * k, kd + 2 * k, idesc_s,
                                  (hh | k) != 0);
                }
                umma_commit(s_full + 2 * t + (j & 1));
                ta_trace(30 + t, j);
            };
            auto issue_pv = [&](int t, int j) {
                const int st = j % TA_STAGES;
                ta_wait(p_full + t, j & 1, 5, j);
                ta_trace(20 + t, j);
                tc_fence_after();
                const uint32_t v_addr = smem_u32(sm + C::ST_OFF + st * C::STAGE + C::K_BYTES);
                const uint64_t pd = umma_desc_sw128(smem_u32(sm + C::P_OFF + t * C::P_TILE));
#pragma unroll
                for (int k = 0; k < TA_KC / 16; ++k)
                    umma_bf16(tmem + uint32_t(t * 128), pd + 2 * k, umma_desc_sw128_mn(v_addr + k * 2048, C::KV_HALF),
                              idesc_o, (j | k) != 0);
                umma_commit(pv_done + t);
            };
            for (int t = 0; t < 2; ++t)
                if (nch[t] > 0) issue_s(t, 0);
            for (int j = 0; j < nchunks; ++j) {
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    if (j >= nch[t]) continue;
                    if (j + 1 < nch[t]) issue_s(t, j + 1);
                    issue_pv(t, j);
                }
                umma_commit(kv_empty + (j % TA_STAGES));  // both tiles' MMAs of chunk j read the stage
            }
        }
    } else {  // ---- softmax warpgroups: tile t = (warp - 2) / 4, one query row per thread
        const int t = (warp - 2) >> 2, sub = warp & 3, row = sub * 32 + lane;
        const uint32_t lane_addr = tmem + (uint32_t(sub * 32) << 16);
        const uint32_t o_col = uint32_t(t * 128), s_col = 256u + uint32_t(t * 128);
        const int r = q0[t] + row;
        {
            const uint4* src = reinterpret_cast<const uint4*>(a.q + (size_t(r) * s.n_heads + head) * DH);
#pragma unroll
            for (int c = 0; c < DH / 8; ++c) {
                const uint4 v = r < a.L ? src[c] : make_uint4(0, 0, 0, 0);
                const int hh = c >> 3, cc = c & 7;
                *reinterpret_cast<uint4*>(sm + C::Q_OFF + t * C::Q_TILE + hh * C::Q_HALF + row * 128 +
                                          ((cc ^ (row & 7)) << 4)) = v;
            }
        }
        fence_proxy_async_smem();
        mbar_arrive(q_ready);
        const int qpos = a.p0 + r, n_t = nch[t];
        const float sl2 = rsqrtf(float(DH)) * 1.4426950408889634f;
        float mref = -INFINITY, l = 0.f;
        for (int j = 0; j < n_t; ++j) {
            const int kbase = j * TA_KC;
            ta_wait(s_full + 2 * t + (j & 1), (j >> 1) & 1, 6, j);
            if (lane == 0 && sub == 2) ta_trace(40 + t, j);
            tc_fence_after();
            uint32_t sv[2][32];
            tmem_ld32(lane_addr + s_col + uint32_t((j & 1) * 64), sv[0]);
            tmem_ld32(lane_addr + s_col + uint32_t((j & 1) * 64) + 32u, sv[1]);
            tc_fence_before();
            mbar_arrive(s_empty + 2 * t + (j & 1));
            // raw scores; the causal mask only in chunks that cross some row's diagonal
            float p[64];
            float mx = -INFINITY;
            if (__any_sync(0xffffffffu, kbase + TA_KC - 1 > qpos)) {
#pragma unroll
                for (int k = 0; k < 64; ++k) {
                    p[k] = kbase + k <= qpos ? __uint_as_float(sv[k >> 5][k & 31]) : -INFINITY;
                    mx = fmaxf(mx, p[k]);
                }
            } else {
#pragma unroll
                for (int k = 0; k < 64; ++k) {
                    p[k] = __uint_as_float(sv[k >> 5][k & 31]);
                    mx = fmaxf(mx, p[k]);
                }
            }
            mx *= sl2;  // log2 domain
            if (j > 0) ta_wait(pv_done + t, (j - 1) & 1, 7, j);  // O_t stable, P_t free
            if (lane == 0 && sub == 2) ta_trace(60 + t, j);
            tc_fence_after();
            const bool grow = mx > mref + 8.f;
            const float corr = (grow && mref != -INFINITY) ? exp2f(mref - mx) : 1.f;
            if (__any_sync(0xffffffffu, corr != 1.f)) {
#pragma unroll 1
                for (int c = 0; c < DH / 32; ++c) {
                    uint32_t o[32];
                    tmem_ld32(lane_addr + o_col + uint32_t(c * 32), o);
#pragma unroll
                    for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * corr);
                    tmem_st32(lane_addr + o_col + uint32_t(c * 32), o);
                }
            }
            l *= corr;
            if (grow) mref = mx;
            if (lane == 0 && sub == 2) ta_trace(70 + t, j);
            uint8_t* prow = sm + C::P_OFF + t * C::P_TILE + row * 128;
            const float moff = mref == -INFINITY ? 0.f : -mref;  // fully masked rows: ex2(-inf) = 0
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                float e[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    e[i] = ex2_approx(fmaf(p[c * 8 + i], sl2, moff));
                    l += e[i];
                }
                uint4 pk;
                pk.x = pack_bf16x2(e[0], e[1]);
                pk.y = pack_bf16x2(e[2], e[3]);
                pk.z = pack_bf16x2(e[4], e[5]);
                pk.w = pack_bf16x2(e[6], e[7]);
                *reinterpret_cast<uint4*>(prow + ((c ^ (row & 7)) << 4)) = pk;
            }
            // keys past the CTA's last key in its last chunk: zero those V rows (0 x NaN of
            // unwritten cache rows would reach O). Only the tile that alone processes the
            // last chunk does it: with two full tiles, tile A's range ends a chunk earlier.
            if (j == nchunks - 1 && kmax < kbase + TA_KC - 1 && (t == 1 || nch[1] < nchunks)) {
                uint8_t* vb = sm + C::ST_OFF + (j % TA_STAGES) * C::STAGE + C::K_BYTES;
                const int k0 = kmax + 1 - kbase, n16 = (TA_KC - k0) * 8 * C::HALVES;
                for (int i = row; i < n16; i += 128) {
                    const int hh = i / ((TA_KC - k0) * 8), rem = i % ((TA_KC - k0) * 8);
                    *reinterpret_cast<uint4*>(vb + hh * C::KV_HALF + (k0 + rem / 8) * 128 + (rem % 8) * 16) =
                        make_uint4(0, 0, 0, 0);
                }
            }
            if (lane == 0 && sub == 2) ta_trace(80 + t, j);
            fence_proxy_async_smem();
            tc_fence_before();
            if (lane == 0 && sub == 2) ta_trace(50 + t, j);
            mbar_arrive(p_full + t);
        }
        if (n_t > 0) {
            ta_wait(pv_done + t, (n_t - 1) & 1, 8, n_t);
            tc_fence_after();
            const float inv = 1.f / l;
#pragma unroll 1
            for (int c = 0; c < DH / 32; ++c) {
                uint32_t o[32];
                tmem_ld32(lane_addr + o_col + uint32_t(c * 32), o);
                if (r < a.L) {
                    uint16_t* dst = a.attn + size_t(r) * s.d + head * DH + c * 32;
#pragma unroll
                    for (int i = 0; i < 32; i += 8) {
                        uint4 pk;
                        pk.x = pack_bf16x2(__uint_as_float(o[i]) * inv, __uint_as_float(o[i + 1]) * inv);
                        pk.y = pack_bf16x2(__uint_as_float(o[i + 2]) * inv, __uint_as_float(o[i + 3]) * inv);
                        pk.z = pack_bf16x2(__uint_as_float(o[i + 4]) * inv, __uint_as_float(o[i + 5]) * inv);
                        pk.w = pack_bf16x2(__uint_as_float(o[i + 6]) * inv, __uint_as_float(o[i + 7]) * inv);
                        *reinterpret_cast<uint4*>(dst + i) = pk;
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, C::TMEM_COLS);
    }
}

bool make_kvmap(CUtensorMap* m, const PrefillArgs& a);

// MESH_PF_ATTN=mma selects the mma.sync kernel (kept as the A/B reference); default tcgen05.
template <int DH>
cudaError_t attn_tc_launch(const PrefillArgs& a, int layer, cudaStream_t st) {
    static bool cfg[MAX_DEVICES] = {};
    const int dev = cur_device();
    if (!cfg[dev]) {
        cudaError_t e = cudaFuncSetAttribute(pf_attn_tc<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             TaCfg<DH>::SMEM);
        if (e != cudaSuccess) return e;
        cfg[dev] = true;
    }
    CUtensorMap km;
    if (!make_kvmap(&km, a)) return cudaErrorInvalidValue;
    static int* dbg_host = nullptr;
    if (getenv("MESH_PF_ATTN_DEBUG") && !dbg_host) {
        int* dev = nullptr;
        if (cudaHostAlloc((void**)&dbg_host, 16384, cudaHostAllocMapped) != cudaSuccess) return cudaErrorMemoryAllocation;
        memset(dbg_host, 0, 16384);
        cudaHostGetDevicePointer((void**)&dev, dbg_host, 0);
        cudaMemcpyToSymbol(g_ta_dbg, &dev, sizeof(dev));
        std::thread([] {  // watchdog: dump the heartbeats if the process is still here after 10 s
            std::this_thread::sleep_for(std::chrono::seconds(10));
            fprintf(stderr, "pf_attn_tc heartbeats (cta: warp0..5 = barrier<<16|chunk):\n");
            for (int c = 0; c < 150; ++c) {
                bool any = false;
                for (int w = 0; w < 6; ++w) any |= dbg_host[512 + c * 6 + w] != 0;
                if (!any) continue;
                fprintf(stderr, "  cta %d:", c);
                for (int w = 0; w < 6; ++w) fprintf(stderr, " %x", dbg_host[512 + c * 6 + w]);
                fprintf(stderr, "\n");
            }
            fflush(stderr);
        }).detach();
        atexit([] {
            const int n = dbg_host[0];
            if (n) fprintf(stderr, "pf_attn_tc wait timeouts: %d\n", n);
            for (int i = 0; i < n && i < 60; ++i)
                fprintf(stderr, "  block (%d,%d) thread %d barrier %d chunk %d parity %d\n", dbg_host[1 + i * 6],
                        dbg_host[2 + i * 6], dbg_host[3 + i * 6], dbg_host[4 + i * 6], dbg_host[5 + i * 6],
                        dbg_host[6 + i * 6]);
        });
    }
    dim3 grid((a.L + TA_QT - 1) / TA_QT, a.s.n_heads);
    pf_attn_tc<DH><<<grid, TA_THREADS, TaCfg<DH>::SMEM, st>>>(a, km, layer);
    return cudaGetLastError();
}

template <int DH>
cudaError_t attn_tc2_launch(const PrefillArgs& a, int layer, cudaStream_t st) {
    static bool cfg[MAX_DEVICES] = {};
    const int dev = cur_device();
    if (!cfg[dev]) {
        cudaError_t e = cudaFuncSetAttribute(pf_attn_tc2<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             Ta2Cfg<DH>::SMEM);
        if (e != cudaSuccess) return e;
        cfg[dev] = true;
    }
    CUtensorMap km;
    if (!make_kvmap(&km, a)) return cudaErrorInvalidValue;
    static int trace_state = getenv("MESH_PF_ATTN_TRACE") ? 1 : 0;  // 1: trace the next launch
    unsigned long long* tr_dev = nullptr;
    if (trace_state == 1) {
        if (cudaMalloc((void**)&tr_dev, 8 * 96 * 1024) != cudaSuccess) return cudaErrorMemoryAllocation;
        cudaMemsetAsync(tr_dev, 0, 8 * 96 * 1024, st);
        cudaMemcpyToSymbolAsync(g_ta_trace, &tr_dev, sizeof(tr_dev), 0, cudaMemcpyHostToDevice, st);
    }
    const int nqt = (a.L + TA_QT - 1) / TA_QT;
    dim3 grid((nqt + 1) / 2, a.s.n_heads);
    pf_attn_tc2<DH><<<grid, T2_THREADS, Ta2Cfg<DH>::SMEM, st>>>(a, km, layer);
    if (trace_state == 1) {  // dump CTA (0, 0)'s timeline of this launch, then stop tracing
        trace_state = 2;
        std::vector<unsigned long long> h(96 * 1024);
        cudaStreamSynchronize(st);
        cudaMemcpy(h.data(), tr_dev, 8 * 96 * 1024, cudaMemcpyDeviceToHost);
        unsigned long long* null_ptr = nullptr;
        cudaMemcpyToSymbol(g_ta_trace, &null_ptr, sizeof(null_ptr));
        cudaFree(tr_dev);
        if (FILE* f = fopen(getenv("MESH_PF_ATTN_TRACE"), "w")) {
            for (int id = 0; id < 96; ++id)
                for (int j = 0; j < 1024; ++j)
                    if (h[id * 1024 + j]) fprintf(f, "%llu %d %d\n", h[id * 1024 + j], id, j);
            fclose(f);
        }
    }
    return cudaGetLastError();
}

// MESH_PF_ATTN: "tc2" (default) two query tiles per CTA ping-ponged, "tc" one tile per CTA,
// "mma" the mma.sync kernel. tc2 needs p0 == 0 whenever L > 128 (a fresh prefill; a resume
// feeds one token), which is how the data plane issues prefills.
template <int DH>
cudaError_t attn_launch(const PrefillArgs& a, int layer, cudaStream_t st) {
    static const int mode = [] {
        const char* e = getenv("MESH_PF_ATTN");
        if (e && std::string(e) == "mma") return 0;
        if (e && std::string(e) == "tc") return 1;
        return 2;
    }();
    if (mode == 2 && (a.p0 == 0 || a.L <= TA_QT)) return attn_tc2_launch<DH>(a, layer, st);
    if (mode >= 1) return attn_tc_launch<DH>(a, layer, st);
    static bool cfg[MAX_DEVICES] = {};
    const int dev = cur_device();
    if (!cfg[dev]) {
        cudaError_t e = cudaFuncSetAttribute(pf_attn<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, pa_smem<DH>());
        if (e != cudaSuccess) return e;
        cfg[dev] = true;
    }
    dim3 grid((a.L + PA_QT - 1) / PA_QT, a.s.n_heads);
    pf_attn<DH><<<grid, PA_THREADS, pa_smem<DH>(), st>>>(a, layer);
    return cudaGetLastError();
}

__global__ void pf_argmax(const __grid_constant__ PrefillArgs a) {
    __shared__ float sv[32];
    __shared__ int si[32];
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    for (int i = threadIdx.x; i < a.s.vocab; i += blockDim.x) {
        float v = a.logits[i];
        if (v > bv || (v == bv && i < bi)) {
            bv = v;
            bi = i;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
            bv = ov;
            bi = oi;
        }
    }
    if ((threadIdx.x & 31) == 0) {
        sv[threadIdx.x >> 5] = bv;
        si[threadIdx.x >> 5] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int best = si[0];
        float bestv = sv[0];
        for (int w = 1; w < int(blockDim.x >> 5); ++w)
            if (sv[w] > bestv || (sv[w] == bestv && si[w] < best)) {
                bestv = sv[w];
                best = si[w];
            }
        a.tok_out[0] = best;
        a.last_tok[a.slot] = best;
    }
}

// Single-token lm_head (the last position only): the mma.sync tile kernel.
cudaError_t lm_gemm(const PrefillArgs& a, cudaStream_t st) {
    static bool cfg[MAX_DEVICES] = {};
    const int dev = cur_device();
    if (!cfg[dev]) {
        cudaError_t e = cudaFuncSetAttribute(pf_lm_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, PF_SMEM);
        if (e != cudaSuccess) return e;
        cfg[dev] = true;
    }
    pf_lm_gemm<<<dim3(a.s.vocab / PF_BM, 1), PF_THREADS, PF_SMEM, st>>>(a, a.w.lm, a.s.d, a.act, a.s.d, 1);
    return cudaGetLastError();
}

// ---- host side of the tcgen05 GEMM
using EncodeTiledFn = decltype(&cuTensorMapEncodeTiled);
EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

// Token rows X[rows][ld] bf16, box = 64 columns (128 B, swizzled) x BN rows;
// rows past the end are zero-filled by the TMA unit.
bool make_xmap(CUtensorMap* m, const uint16_t* X, int K, int ld, int rows, int BN) {
    EncodeTiledFn enc = encode_tiled();
    if (!enc) return false;
    cuuint64_t dims[2] = {cuuint64_t(K), cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(ld) * 2};
    cuuint32_t box[2] = {cuuint32_t(TC_BK), cuuint32_t(BN)};
    cuuint32_t es[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t*>(X), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Tiled weights [N][K] (T16 x SW128) as a 4-D tensor {64 cols, 16 rows, K/64
// blocks, N/16 tiles}; the box {64, 16, 1, 8} is one 128-row x 64-column
// A stage, copied verbatim (the bytes are already in the SW128 UMMA layout).
bool make_wmap(CUtensorMap* m, const uint8_t* W, int N, int K) {
    EncodeTiledFn enc = encode_tiled();
    if (!enc) return false;
    cuuint64_t dims[4] = {64, 16, cuuint64_t(K / 64), cuuint64_t(N / 16)};
    cuuint64_t strides[3] = {128, 2048, cuuint64_t(K) * 32};
    cuuint32_t box[4] = {64, 16, 1, TC_BM / 16};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<uint8_t*>(W), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// The instance's KV region as a 4-D tensor {64 elements (128 B), halves of a row,
// rows R = ((layer * n_kv + head) * 2 + k|v) * 16 + slot, blocks}: box {64, 1,
// 16, 1} is one (block, layer, head, k|v) half: 16 rows x 128 B, the bytes of
// an SW128 atom pair as the cache stores them.
bool make_kvmap(CUtensorMap* m, const PrefillArgs& a) {
    EncodeTiledFn enc = encode_tiled();
    if (!enc) return false;
    const Shape& s = a.s;
    cuuint64_t dims[4] = {64, cuuint64_t(s.dh / 64), cuuint64_t(s.n_layers) * s.n_kv * 2 * KV_BLOCK_TOKENS,
                          cuuint64_t(a.kv_blocks)};
    cuuint64_t strides[3] = {128, cuuint64_t(s.dh) * 2, cuuint64_t(a.block_bytes)};
    cuuint32_t box[4] = {64, 1, KV_BLOCK_TOKENS, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, a.kv_base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int num_sms() {
    static int n[MAX_DEVICES] = {};
    const int dev = cur_device();
    if (!n[dev]) {
        int v = 148;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        n[dev] = v;
    }
    return n[dev];
}

// Token-tile width: minimise waves x per-K-block time, where a K block costs
// max(MMA = 2*BN cycles, shared-memory operand reads = 128 + BN cycles).
// MESH_PREFILL_BN=64|128|256 pins the width (parity tests cover every variant).
int pick_bn(int N, int rows) {
    if (const char* f = getenv("MESH_PREFILL_BN")) {
        const int v = atoi(f);
        if (v == 64 || v == 128 || v == 256) return v;
    }
    const int cand[3] = {256, 128, 64};
    int best = 256;
    long long best_cost = -1;
    for (int bn : cand) {
        long long tiles = (long long)(N / TC_BM) * ((rows + bn - 1) / bn);
        long long waves = (tiles + num_sms() - 1) / num_sms();
        long long cost = waves * std::max(2 * bn, 128 + bn);
        if (best_cost < 0 || cost < best_cost) {
            best_cost = cost;
            best = bn;
        }
    }
    return best;
}

// Split-K factor for a grid of G CTAs and T output tiles of nk K blocks: fewest
// waves x (1/S of a tile) + the partial write/read (~8 % of a tile), units <= 2G
// (the workspace), >= 8 K blocks per unit. MESH_PREFILL_SPLITK=0 disables it,
// =2..4 forces that factor wherever the workspace and K allow (tests).
int pick_splits(int T, int G, int nk) {
    const char* env = getenv("MESH_PREFILL_SPLITK");  // read per launch: tests flip it in-process
    const int force = env ? atoi(env) : -1;
    if (force == 0 || T > SK_TILES_MAX || nk < 16) return 1;
    if (force >= 2 && force <= 4 && T * force <= 2 * G && nk / force >= 8) return force;
    if (T >= G) return 1;
    int best = 1;
    double best_cost = double((T + G - 1) / G);
    for (int S = 2; S <= 4; ++S) {
        if (T * S > 2 * G || nk / S < 8) break;
        const double cost = double((T * S + G - 1) / G) / S + 0.08;
        if (cost < best_cost - 1e-9) {
            best_cost = cost;
            best = S;
        }
    }
    return best;
}

template <int KIND, int BN, int CS>
cudaError_t gemm_tc_launch(const PrefillArgs& a, const uint8_t* W, int N, int K, const uint16_t* X, int ldx,
                           int rows, int layer, cudaStream_t st) {
    using C = TcCfg<BN>;
    static int max_clusters_dev[MAX_DEVICES] = {};
    int& max_clusters = max_clusters_dev[cur_device()];
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(TC_THREADS);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (!max_clusters) {
        cudaError_t e = cudaFuncSetAttribute(pf_gemm_tc<KIND, BN, CS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             C::SMEM);
        if (e != cudaSuccess) return e;
        cfg.gridDim = dim3(CS * (num_sms() / CS));
        e = cudaOccupancyMaxActiveClusters(&max_clusters, pf_gemm_tc<KIND, BN, CS>, &cfg);
        if (e != cudaSuccess) return e;
        if (max_clusters < 1) return cudaErrorInvalidConfiguration;
    }
    CUtensorMap wm, xm;
    if (!make_wmap(&wm, W, N, K) || !make_xmap(&xm, X, K, ldx, rows, BN / CS)) return cudaErrorInvalidValue;
    const int ctiles = (N / TC_BM / CS) * ((rows + BN - 1) / BN);
    const int quota = a.max_ctas > 0 ? std::max(1, a.max_ctas / CS) : max_clusters;
    const int G = std::min(max_clusters, quota);
    // split-K only for the down projection (long K, residual-add epilogue): measured 3B L = 462
    // down 47.4 -> 41.5 us, while QKV (RoPE + paged-KV epilogue) and O got slower (41 -> 70, 24 -> 32)
    const int splits = (CS == 1 && KIND == PF_DOWN) ? pick_splits(ctiles, G, K / TC_BK) : 1;
    cfg.gridDim = dim3(CS * std::min(ctiles * splits, G));
    return cudaLaunchKernelEx(&cfg, pf_gemm_tc<KIND, BN, CS>, a, wm, xm, N, K, rows, layer, splits);
}

// Cluster size along the weight rows: the CTAs of a cluster share (multicast)
// the token tile, cutting the L2->SM operand traffic from 48 KB to 16 + 32/CS
// KB per 64-deep K block; the L2 read bandwidth, not the tensor pipe, bounds
// the single-CTA 128x256 tile.
template <int KIND, int BN>
cudaError_t gemm_tc_bn(const PrefillArgs& a, const uint8_t* W, int N, int K, const uint16_t* X, int ldx, int rows,
                       int layer, cudaStream_t st) {
    const int nM = N / TC_BM;
    int cs = 1;
    if (const char* f = getenv("MESH_PREFILL_CLUSTER")) {
        const int v = atoi(f);
        if ((v == 1 || v == 2 || v == 4) && nM % v == 0) cs = v;
    }
    switch (cs) {
        case 4: return gemm_tc_launch<KIND, BN, 4>(a, W, N, K, X, ldx, rows, layer, st);
        case 2: return gemm_tc_launch<KIND, BN, 2>(a, W, N, K, X, ldx, rows, layer, st);
        default: return gemm_tc_launch<KIND, BN, 1>(a, W, N, K, X, ldx, rows, layer, st);
    }
}

template <int KIND, int BN>
cudaError_t gemm_2sm_launch(const PrefillArgs& a, const uint8_t* W, int N, int K, const uint16_t* X, int ldx, int rows,
                            int layer, cudaStream_t st) {
    using C = Tc2Cfg<BN>;
    static int max_clusters_dev[MAX_DEVICES] = {};
    int& max_clusters = max_clusters_dev[cur_device()];
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(TC_THREADS);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (!max_clusters) {
        cudaError_t e = cudaFuncSetAttribute(pf_gemm_2sm<KIND, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        cfg.gridDim = dim3(2 * (num_sms() / 2));
        e = cudaOccupancyMaxActiveClusters(&max_clusters, pf_gemm_2sm<KIND, BN>, &cfg);
        if (e != cudaSuccess) return e;
        if (max_clusters < 1) return cudaErrorInvalidConfiguration;
    }
    CUtensorMap wm, xm;
    if (!make_wmap(&wm, W, N, K) || !make_xmap(&xm, X, K, ldx, rows, BN / 2)) return cudaErrorInvalidValue;
    const int tiles = (N / 256) * ((rows + BN - 1) / BN);
    const int quota = a.max_ctas > 0 ? std::max(1, a.max_ctas / 2) : max_clusters;
    cfg.gridDim = dim3(2 * std::min(tiles, std::min(max_clusters, quota)));
    return cudaLaunchKernelEx(&cfg, pf_gemm_2sm<KIND, BN>, a, wm, xm, N, K, rows, layer);
}

// CTA-pair GEMMs for N a multiple of 256 when the 256-row tiles fill every
// cluster at least once (else the single-CTA kernel's finer, dynamically claimed
// tiles fill the SMs better). BN 256 unless the token count makes 128 cheaper
// (waves x max(2 BN, 256 + BN) over the cluster count). MESH_PREFILL_2SM=0|1
// forces the choice off / on.
template <int KIND>
bool gemm_2sm(const PrefillArgs& a, const uint8_t* W, int N, int K, const uint16_t* X, int ldx, int rows, int layer,
              cudaStream_t st, cudaError_t* err) {
    const char* env = getenv("MESH_PREFILL_2SM");  // read per launch: tests flip it in-process
    const int mode = env ? atoi(env) : -1;
    if (mode == 0 || N % 256 || (mode < 0 && !a.pair_ok)) return false;
    const long long clusters = std::max(1, (a.max_ctas > 0 ? a.max_ctas : num_sms()) / 2);
    auto tiles = [&](int bn) { return (long long)(N / 256) * ((rows + bn - 1) / bn); };
    auto cost = [&](int bn) { return ((tiles(bn) + clusters - 1) / clusters) * std::max(2 * bn, 256 + bn); };
    const int bn = cost(128) < cost(256) ? 128 : 256;
    if (mode < 0 && tiles(bn) < clusters) return false;
    *err = bn == 128 ? gemm_2sm_launch<KIND, 128>(a, W, N, K, X, ldx, rows, layer, st)
                     : gemm_2sm_launch<KIND, 256>(a, W, N, K, X, ldx, rows, layer, st);
    return true;
}

template <int KIND>
cudaError_t gemm(const PrefillArgs& a, const uint8_t* W, int N, int K, const uint16_t* X, int ldx, int rows,
                 int layer, cudaStream_t st) {
    if (N % TC_BM || K % TC_BK) return cudaErrorInvalidValue;
    cudaError_t e2;
    if (gemm_2sm<KIND>(a, W, N, K, X, ldx, rows, layer, st, &e2)) return e2;
    switch (pick_bn(N, rows)) {
        case 256: return gemm_tc_bn<KIND, 256>(a, W, N, K, X, ldx, rows, layer, st);
        case 128: return gemm_tc_bn<KIND, 128>(a, W, N, K, X, ldx, rows, layer, st);
        default: return gemm_tc_bn<KIND, 64>(a, W, N, K, X, ldx, rows, layer, st);
    }
}

}  // namespace

cudaError_t launch_prefill(const PrefillArgs& a, cudaStream_t st) {
    const Shape& s = a.s;
    const int L = a.L;
    // the QKV epilogue branches on q / k / v per warp (32 weight rows; the k/v store shuffles)
    if ((s.n_heads * s.dh) % 32 || (s.n_kv * s.dh) % 32) return cudaErrorInvalidValue;
    pf_embed<<<L, 256, 0, st>>>(a);
    if (s.d % 128 || s.d > 128 * RN_MAXV) return cudaErrorInvalidValue;
    const int norm_blocks = (L + 3) / 4;
    cudaError_t e;
    for (int layer = 0; layer < s.n_layers; ++layer) {
        pf_rownorm<<<norm_blocks, 128, 0, st>>>(a.h, a.w.g_attn + size_t(layer) * s.d, a.act, a.rs, L, s.d, s.eps);
        if ((e = gemm<PF_QKV>(a, a.w.qkv + layer * a.w.qkv_layer, s.qkv_rows(), s.d, a.act, s.d, L, layer, st)))
            return e;
        if ((e = s.dh == 64 ? attn_launch<64>(a, layer, st) : attn_launch<128>(a, layer, st))) return e;
        if ((e = gemm<PF_O>(a, a.w.o + layer * a.w.o_layer, s.d, s.n_heads * s.dh, a.attn, s.d, L, layer, st)))
            return e;
        pf_rownorm<<<norm_blocks, 128, 0, st>>>(a.h, a.w.g_mlp + size_t(layer) * s.d, a.act, a.rs, L, s.d, s.eps);
        if ((e = gemm<PF_GU>(a, a.w.gu + layer * a.w.gu_layer, 2 * s.ff, s.d, a.act, s.d, L, layer, st))) return e;
        if ((e = gemm<PF_DOWN>(a, a.w.down + layer * a.w.down_layer, s.d, s.ff, a.abuf, s.ff, L, layer, st)))
            return e;
    }
    // final norm of the last token -> lm_head -> greedy token
    pf_rownorm<<<1, 128, 0, st>>>(a.h + size_t(L - 1) * s.d, a.w.g_final, a.act, a.rs, 1, s.d, s.eps);
    if ((e = lm_gemm(a, st))) return e;
    pf_argmax<<<1, 1024, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace meshgpu
