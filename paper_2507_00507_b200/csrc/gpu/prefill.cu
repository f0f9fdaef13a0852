// Prefill step for one request (L tokens starting at absolute position p0).
//
// GEMMs are C^T = W . X^T with the weight rows as the M operand so that the
// decode kernel's row permutations (RoPE pairs, gate/up interleave) put both
// members of a pair in one thread's accumulator here too; the weights are
// streamed straight from their T16xSW128 tiled layout (each 16x64 block is a
// contiguous, pre-swizzled 2 KB run) and the activation tile is staged with a
// matching software swizzle, so every ldmatrix is bank-conflict free. The
// epilogues are the decode ones applied per token: RoPE + paged KV write, the
// residual add, silu(gate)*up. Attention is causal over the paged cache.
#include "prefill.cuh"

#include <math.h>

namespace meshgpu {

namespace {

enum PfKind { PF_QKV = 0, PF_O = 1, PF_GU = 2, PF_DOWN = 3, PF_LM = 4 };

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

template <int KIND>
__global__ void __launch_bounds__(PF_THREADS) pf_gemm(const __grid_constant__ PrefillArgs a,
                                                      const uint8_t* __restrict__ W, int K,
                                                      const uint16_t* __restrict__ X, int ldx, int Lrows,
                                                      int layer) {
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

    // ---- fused epilogue
    const Shape& s = a.s;
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
        const int row = (row_tile0 + 2 * warp_m + mi) * 16 + g;  // rows row and row + 8
        const int tile = row >> 4;
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int l = tok0 + warp_n * 32 + ni * 8 + 2 * t + j;
                if (l >= Lrows) continue;
                const float v1 = acc[mi][ni][j], v2 = acc[mi][ni][2 + j];
                if constexpr (KIND == PF_QKV) {
                    const float r = a.rs[l];
                    QkvRow qr = qkv_row(s, row);
                    const int half = s.dh / 2;
                    const int pos = a.p0 + l;
                    float x1 = v1 * r, x2 = v2 * r, o1 = x1, o2 = x2;
                    if (qr.section < 2) {
                        float2 cs = a.w.rope[size_t(pos) * half + qr.dim];
                        o1 = x1 * cs.x - x2 * cs.y;
                        o2 = x2 * cs.x + x1 * cs.y;
                    }
                    if (qr.section == 0) {
                        float* qd = a.q + (size_t(l) * s.n_heads + qr.head) * s.dh;
                        qd[qr.dim] = o1;
                        qd[qr.dim + half] = o2;
                    } else {
                        const int blk = a.bt_row[pos / KV_BLOCK_TOKENS], slot = pos % KV_BLOCK_TOKENS;
                        uint8_t* e = a.kv_base + size_t(blk) * a.block_bytes +
                                     kv_offset(s, layer, qr.section - 1, qr.head, slot);
                        *reinterpret_cast<uint16_t*>(e + kv_dim_off(slot, qr.dim)) = f_to_bf16(o1);
                        *reinterpret_cast<uint16_t*>(e + kv_dim_off(slot, qr.dim + half)) = f_to_bf16(o2);
                    }
                } else if constexpr (KIND == PF_GU) {
                    const float r = a.rs[l];
                    float gt = v1 * r, up = v2 * r;
                    float act = gt / (1.f + __expf(-gt)) * up;
                    a.abuf[size_t(l) * s.ff + tile * 8 + g] = f_to_bf16(act);
                } else if constexpr (KIND == PF_O || KIND == PF_DOWN) {
                    a.h[size_t(l) * s.d + row] += v1;
                    a.h[size_t(l) * s.d + row + 8] += v2;
                } else {  // PF_LM, single row
                    const float r = a.rs[0];
                    a.logits[row] = v1 * r;
                    a.logits[row + 8] = v2 * r;
                }
            }
        }
    }
}

__global__ void pf_embed(const __grid_constant__ PrefillArgs a) {
    const int l = blockIdx.x;
    const int tok = a.tokens[l];
    for (int i = threadIdx.x; i < a.s.d; i += blockDim.x)
        a.h[size_t(l) * a.s.d + i] = bf16_to_f(a.w.emb[size_t(tok) * a.s.d + i]);
}

// act[l] = bf16(h[l] * gamma), rs[l] = rsqrt(mean(h[l]^2) + eps); one warp per row.
__global__ void pf_rownorm(const float* __restrict__ h, const float* __restrict__ gamma, uint16_t* act,
                           float* rs, int rows, int d, float eps) {
    int row = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const float* hr = h + size_t(row) * d;
    float ss = 0.f;
    for (int i = lane; i < d; i += 32) ss += hr[i] * hr[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    for (int i = lane; i < d; i += 32) act[size_t(row) * d + i] = f_to_bf16(hr[i] * gamma[i]);
    if (lane == 0) rs[row] = rsqrtf(ss / float(d) + eps);
}

// Causal attention over the paged cache. Block = (16 queries, one head).
constexpr int PA_Q = 16, PA_KC = 64;
template <int DH>
__global__ void __launch_bounds__(256) pf_attn(const __grid_constant__ PrefillArgs a, int layer) {
    const Shape& s = a.s;
    __shared__ float q_s[PA_Q][DH];
    __shared__ uint32_t k_s[PA_KC][DH / 2 + 1];
    __shared__ uint16_t v_s[PA_KC][DH];
    __shared__ float p_s[8][PA_KC];
    const int head = blockIdx.y, kvh = head / s.gq();
    const int i0 = blockIdx.x * PA_Q;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < PA_Q * DH; i += 256) {
        int qi = i / DH, dd = i % DH;
        int l = i0 + qi;
        q_s[qi][dd] = l < a.L ? a.q[(size_t(l) * s.n_heads + head) * DH + dd] : 0.f;
    }
    const int last_q = min(i0 + PA_Q, a.L) - 1;
    const int kmax = a.p0 + last_q;  // inclusive key position
    constexpr int DPL = DH / 32;
    float m_[2], l_[2], acc[2][DPL];
#pragma unroll
    for (int qq = 0; qq < 2; ++qq) {
        m_[qq] = -INFINITY;
        l_[qq] = 0.f;
#pragma unroll
        for (int e = 0; e < DPL; ++e) acc[qq][e] = 0.f;
    }
    const float scale = rsqrtf(float(DH));
    for (int k0 = 0; k0 <= kmax; k0 += PA_KC) {
        __syncthreads();
        // stage K (padded u32 rows) and V
        for (int i = tid; i < PA_KC * (DH / 8); i += 256) {
            int kr = i / (DH / 8), c8 = i % (DH / 8);
            int pos = k0 + kr;
            uint4 kv = make_uint4(0, 0, 0, 0), vv = make_uint4(0, 0, 0, 0);
            if (pos <= kmax) {
                const int blk = a.bt_row[pos / KV_BLOCK_TOKENS], slot = pos % KV_BLOCK_TOKENS;
                const uint8_t* base = a.kv_base + size_t(blk) * a.block_bytes;
                const uint32_t sw = kv_dim_off(slot, c8 * 8);  // swizzled 16-byte chunk
                kv = *reinterpret_cast<const uint4*>(base + kv_offset(s, layer, 0, kvh, slot) + sw);
                vv = *reinterpret_cast<const uint4*>(base + kv_offset(s, layer, 1, kvh, slot) + sw);
            }
            k_s[kr][c8 * 4 + 0] = kv.x;
            k_s[kr][c8 * 4 + 1] = kv.y;
            k_s[kr][c8 * 4 + 2] = kv.z;
            k_s[kr][c8 * 4 + 3] = kv.w;
            *reinterpret_cast<uint4*>(&v_s[kr][c8 * 8]) = vv;
        }
        __syncthreads();
#pragma unroll
        for (int qq = 0; qq < 2; ++qq) {
            const int qi = warp * 2 + qq;
            const int l = i0 + qi;
            if (l >= a.L) continue;
            const int qpos = a.p0 + l;
            float sc[2];
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
                int kr = lane + 32 * h2;
                float d = 0.f;
#pragma unroll 8
                for (int c2 = 0; c2 < DH / 2; ++c2) {
                    uint32_t kk = k_s[kr][c2];
                    d += q_s[qi][2 * c2] * bf16_lo(kk) + q_s[qi][2 * c2 + 1] * bf16_hi(kk);
                }
                sc[h2] = (k0 + kr <= qpos) ? d * scale : -INFINITY;
            }
            float mx = fmaxf(sc[0], sc[1]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            float mnew = fmaxf(m_[qq], mx);
            if (mnew == -INFINITY) continue;  // no visible key in this chunk yet
            float corr = __expf(m_[qq] - mnew);
            float p0v = __expf(sc[0] - mnew), p1v = __expf(sc[1] - mnew);
            float ps = p0v + p1v;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
            l_[qq] = l_[qq] * corr + ps;
            m_[qq] = mnew;
            p_s[warp][lane] = p0v;
            p_s[warp][lane + 32] = p1v;
            __syncwarp();
#pragma unroll
            for (int e = 0; e < DPL; ++e) acc[qq][e] *= corr;
            int nk = min(PA_KC, qpos - k0 + 1);
            for (int j = 0; j < nk; ++j) {
                float pj = p_s[warp][j];
#pragma unroll
                for (int e = 0; e < DPL; ++e) acc[qq][e] += pj * bf16_to_f(v_s[j][lane * DPL + e]);
            }
            __syncwarp();
        }
    }
#pragma unroll
    for (int qq = 0; qq < 2; ++qq) {
        const int l = i0 + warp * 2 + qq;
        if (l >= a.L) continue;
#pragma unroll
        for (int e = 0; e < DPL; ++e)
            a.attn[size_t(l) * s.d + size_t(head) * DH + lane * DPL + e] = f_to_bf16(acc[qq][e] / l_[qq]);
    }
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

template <int KIND>
cudaError_t gemm(const PrefillArgs& a, const uint8_t* W, int N, int K, const uint16_t* X, int ldx, int rows,
                 int layer, cudaStream_t st) {
    static bool cfg = false;
    if (!cfg) {
        cudaError_t e = cudaFuncSetAttribute(pf_gemm<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, PF_SMEM);
        if (e != cudaSuccess) return e;
        cfg = true;
    }
    dim3 grid(N / PF_BM, (rows + PF_BN - 1) / PF_BN);
    pf_gemm<KIND><<<grid, PF_THREADS, PF_SMEM, st>>>(a, W, K, X, ldx, rows, layer);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_prefill(const PrefillArgs& a, cudaStream_t st) {
    const Shape& s = a.s;
    const int L = a.L;
    pf_embed<<<L, 256, 0, st>>>(a);
    const int norm_blocks = (L + 7) / 8;
    cudaError_t e;
    for (int layer = 0; layer < s.n_layers; ++layer) {
        pf_rownorm<<<norm_blocks, 256, 0, st>>>(a.h, a.w.g_attn + size_t(layer) * s.d, a.act, a.rs, L, s.d, s.eps);
        if ((e = gemm<PF_QKV>(a, a.w.qkv + layer * a.w.qkv_layer, s.qkv_rows(), s.d, a.act, s.d, L, layer, st)))
            return e;
        dim3 ag((L + PA_Q - 1) / PA_Q, s.n_heads);
        if (s.dh == 64)
            pf_attn<64><<<ag, 256, 0, st>>>(a, layer);
        else
            pf_attn<128><<<ag, 256, 0, st>>>(a, layer);
        if ((e = gemm<PF_O>(a, a.w.o + layer * a.w.o_layer, s.d, s.n_heads * s.dh, a.attn, s.d, L, layer, st)))
            return e;
        pf_rownorm<<<norm_blocks, 256, 0, st>>>(a.h, a.w.g_mlp + size_t(layer) * s.d, a.act, a.rs, L, s.d, s.eps);
        if ((e = gemm<PF_GU>(a, a.w.gu + layer * a.w.gu_layer, 2 * s.ff, s.d, a.act, s.d, L, layer, st))) return e;
        if ((e = gemm<PF_DOWN>(a, a.w.down + layer * a.w.down_layer, s.d, s.ff, a.abuf, s.ff, L, layer, st)))
            return e;
    }
    // final norm of the last token -> lm_head -> greedy token
    pf_rownorm<<<1, 32, 0, st>>>(a.h + size_t(L - 1) * s.d, a.w.g_final, a.act, a.rs, 1, s.d, s.eps);
    if ((e = gemm<PF_LM>(a, a.w.lm, s.vocab, s.d, a.act, s.d, 1, 0, st))) return e;
    pf_argmax<<<1, 1024, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace meshgpu
