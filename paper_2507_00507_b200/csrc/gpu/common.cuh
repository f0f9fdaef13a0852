// Device-side building blocks for the sm_100a data plane: bf16 packing,
// mbarrier + 1-D bulk-copy (TMA engine) ring primitives, ldmatrix/mma.sync
// fragments, cache-global loads for data produced by other CTAs in the same
// launch, and a self-resetting grid barrier for persistent kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define MESH_DEV __device__ __forceinline__

namespace meshgpu {

// ---------------------------------------------------------------- bf16 utils
MESH_DEV float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }
MESH_DEV float bf16_hi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }
MESH_DEV float bf16_to_f(uint16_t v) { return __uint_as_float(uint32_t(v) << 16); }
// Round-to-nearest-even fp32 -> bf16 (matches the CPU oracle's rounding).
MESH_DEV uint16_t f_to_bf16(float f) {
    return __bfloat16_as_ushort(__float2bfloat16_rn(f));
}
MESH_DEV uint32_t pack_bf16x2(float lo, float hi) {
    return uint32_t(f_to_bf16(lo)) | (uint32_t(f_to_bf16(hi)) << 16);
}

// ------------------------------------------------------- cache-global loads
// Data written by other CTAs during the same launch must bypass L1.
MESH_DEV float ldcg_f32(const float* p) { return __ldcg(p); }
MESH_DEV int ldcg_i32(const int* p) { return __ldcg(p); }
MESH_DEV uint4 ldcg_u4(const void* p) { return __ldcg(reinterpret_cast<const uint4*>(p)); }
MESH_DEV uint2 ldcg_u2(const void* p) { return __ldcg(reinterpret_cast<const uint2*>(p)); }
MESH_DEV uint32_t ldcg_u32(const void* p) { return __ldcg(reinterpret_cast<const unsigned int*>(p)); }

// ------------------------------------------------------------------ mbarrier
MESH_DEV uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
MESH_DEV void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
MESH_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
MESH_DEV void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
MESH_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
MESH_DEV bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
MESH_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

// Wait with cluster-scope acquire (the phase may complete by another CTA's arrive).
MESH_DEV void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.b32 %0, 1, 0, p;\n\t}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}

// 1-D bulk copy global -> shared through the TMA engine, completing on `bar`.
MESH_DEV void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(smem_dst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// Same, with an L2 evict-first policy for streamed-once weights.
MESH_DEV void bulk_g2s_evict_first(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar,
                                   uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
            smem_u32(smem_dst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
MESH_DEV uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
    return pol;
}

// 16-byte global -> shared copy that bypasses L1 (LDGSTS); no registers held
MESH_DEV void cp_async_16(uint32_t smem_addr, const void* gptr) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_addr), "l"(gptr) : "memory");
}
MESH_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// ------------------------------------------------------------ tensor cores
MESH_DEV void ldmatrix_x4(uint32_t smem_addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                          uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(smem_addr));
}
MESH_DEV void ldmatrix_x2(uint32_t smem_addr, uint32_t& r0, uint32_t& r1) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];\n"
                 : "=r"(r0), "=r"(r1)
                 : "r"(smem_addr));
}
MESH_DEV void ldmatrix_x2_trans(uint32_t smem_addr, uint32_t& r0, uint32_t& r1) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];\n"
                 : "=r"(r0), "=r"(r1)
                 : "r"(smem_addr));
}
MESH_DEV void ldmatrix_x4_trans(uint32_t smem_addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(smem_addr));
}
// transpose an 8x8 b16 matrix held in ldmatrix fragment layout
MESH_DEV uint32_t movmatrix_trans(uint32_t x) {
    uint32_t y;
    asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;\n" : "=r"(y) : "r"(x));
    return y;
}
// D = A(16x16, row) * B(16x8, col) + D ; bf16 inputs, fp32 accumulate.
MESH_DEV void mma_bf16_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                             uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// ------------------------------------------------ tcgen05 (5th-gen tensor cores)
// TMEM is allocated by one whole warp; the base address lands in shared memory.
MESH_DEV void tmem_alloc(uint32_t smem_dst, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_dst), "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
MESH_DEV void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(ncols) : "memory");
}
MESH_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
MESH_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
// Shared-memory matrix descriptor: K-major operand in the canonical 128-byte
// swizzle layout (8-row x 128-byte atoms, 1024 B apart), Blackwell version 1.
MESH_DEV uint64_t umma_desc_sw128(uint32_t smem_addr) {
    return uint64_t((smem_addr >> 4) & 0x3fffu) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) |
           (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
// Instruction descriptor: bf16 x bf16 -> fp32, both operands K-major, M x N.
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}
// D[tmem] (+)= A[smem] . B[smem]^T, issued by one thread for the whole CTA.
MESH_DEV void umma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Arrive on `bar` once every previously issued tcgen05.mma of this thread completed.
MESH_DEV void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     smem_u32(bar))
                 : "memory");
}
// 32 lanes x 32 columns of fp32 from TMEM: thread i gets lane (base lane + i).
MESH_DEV void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}
// 32 lanes x 32 columns of fp32 into TMEM (thread i writes lane base + i).
MESH_DEV void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
}
// Shared-memory matrix descriptor of an MN-major operand in the canonical
// 128-byte swizzle layout: 8 K-rows x 128 bytes (64 MN elements) per atom,
// K-row groups 1024 B apart (SBO), MN atoms `lbo` bytes apart (LBO).
MESH_DEV uint64_t umma_desc_sw128_mn(uint32_t smem_addr, uint32_t lbo) {
    return uint64_t((smem_addr >> 4) & 0x3fffu) | (uint64_t((lbo >> 4) & 0x3fffu) << 16) |
           (uint64_t(1024 >> 4) << 32) | (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
MESH_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// 2-D tensor TMA load (tensor map in kernel-parameter space) completing on `bar`.
MESH_DEV void tma_load_2d(void* smem_dst, const void* tmap, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
            "r"(smem_u32(smem_dst)),
        "l"(tmap), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
// 4-D tensor TMA load.
MESH_DEV void tma_load_4d(void* smem_dst, const void* tmap, int x, int y, int z, int w, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::
            "r"(smem_u32(smem_dst)),
        "l"(tmap), "r"(x), "r"(y), "r"(z), "r"(w), "r"(smem_u32(bar))
        : "memory");
}
// Same, multicast: the box lands at the same smem offset of every CTA in
// `mask` and completes on the barrier at the same offset in each of them.
MESH_DEV void tma_load_2d_mc(void* smem_dst, const void* tmap, int x, int y, uint64_t* bar, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(smem_u32(smem_dst)),
        "l"(tmap), "r"(x), "r"(y), "r"(smem_u32(bar)), "h"(mask)
        : "memory");
}
// tcgen05.commit arriving on the barrier at this offset in every CTA of `mask`.
MESH_DEV void umma_commit_mc(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}
// ---- CTA pair (cta_group::2): one tcgen05.mma of M = 256 spans the TMEM and
// shared memory of both CTAs of a 2-CTA cluster; only rank 0 issues it.
MESH_DEV void tmem_alloc_2sm(uint32_t smem_dst, uint32_t ncols) {  // same warp id in both CTAs
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_dst), "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::: "memory");
}
MESH_DEV void tmem_dealloc_2sm(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(ncols) : "memory");
}
MESH_DEV void umma_bf16_2sm(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Arrive on the barrier at this offset in every CTA of `mask` once the pair's MMAs completed.
MESH_DEV void umma_commit_2sm_mc(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}
// Pair TMA loads: each CTA fills its own shared memory; the bytes complete on the
// barrier at the same offset in the rank-0 CTA (the peer bit of the address cleared).
constexpr uint32_t PAIR_PEER_MASK = 0xFEFFFFFFu;
MESH_DEV void tma_load_4d_2sm(void* smem_dst, const void* tmap, int x, int y, int z, int w, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(smem_u32(smem_dst)),
        "l"(tmap), "r"(x), "r"(y), "r"(z), "r"(w), "r"(smem_u32(bar) & PAIR_PEER_MASK)
        : "memory");
}
MESH_DEV void tma_load_2d_2sm(void* smem_dst, const void* tmap, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(smem_dst)),
        "l"(tmap), "r"(x), "r"(y), "r"(smem_u32(bar) & PAIR_PEER_MASK)
        : "memory");
}
// Arrive on the barrier at this offset in CTA `cta` of the cluster.
MESH_DEV void mbar_arrive_remote(uint64_t* bar, uint32_t cta) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(remote) : "r"(smem_u32(bar)), "r"(cta));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(remote) : "memory");
}
MESH_DEV uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
MESH_DEV void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// Bulk prefetch of global memory into L2 (no smem, no completion tracking).
MESH_DEV void bulk_prefetch_l2(const void* gsrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(gsrc), "r"(bytes) : "memory");
}
MESH_DEV void prefetch_tmap(const void* tmap) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(tmap) : "memory");
}

MESH_DEV void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

// ------------------------------------------------------------ grid barrier
// Sense-reversing barrier over all CTAs of a persistent launch. `count` returns
// to 0 after every barrier and `gen` only ever increments, so the pair needs no
// reset between launches. Called by ONE thread per CTA after a CTA-level
// bar.sync; the arrival is a gpu-scope release and the wait a gpu-scope acquire
// (the CTA's other threads are ordered by the surrounding bar.syncs), so no
// separate sequentially-consistent fences are needed.
MESH_DEV unsigned int ld_acquire_gpu(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
MESH_DEV int atom_add_acq_rel_gpu(int* p, int v) {
    int old;
    asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], %2;\n" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
// Monotonic grid barrier: barrier i of a launch completes when the counter
// reaches i * nblocks. Arrival is a fire-and-forget release reduction (no
// returned atomic, no last-arriver hop), so the chain is: last CTA's red lands
// in L2 -> every poller's next acquire load sees it. The counter is reset to 0
// by the launch's last CTA once every CTA is past its final barrier.
MESH_DEV void grid_barrier_mono(unsigned int* count, unsigned int target) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(count) : "memory");
    while (int(ld_acquire_gpu(count) - target) < 0) {
    }
}

MESH_DEV void grid_barrier(unsigned int* count, unsigned int* gen, unsigned int nblocks) {
    const unsigned int my_gen = ld_acquire_gpu(gen);
    unsigned int old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;\n" : "=r"(old) : "l"(count) : "memory");
    if (old == nblocks - 1) {
        asm volatile("st.relaxed.gpu.global.u32 [%0], 0;\n" ::"l"(count) : "memory");
        asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(gen), "r"(my_gen + 1) : "memory");
    } else {
        while (ld_acquire_gpu(gen) == my_gen) {
        }
    }
}

// ------------------------------------------------ weight tiling (T16 x SW128)
// Weight matrices [N][K] bf16 live in HBM as 16-row tiles; each tile is K/64
// blocks of 16 rows x 64 columns (2 KB) with the 128-byte swizzle, so a tile is
// contiguous and any run of blocks can be fetched with one bulk copy and read
// conflict-free by ldmatrix (and is the canonical SW128 K-major UMMA layout).
MESH_DEV uint32_t sw128_off(int r, int c) {  // byte offset of (r, c) inside a 16x64 block
    return uint32_t(r) * 128u + ((uint32_t((c >> 3) ^ (r & 7))) << 4) + uint32_t(c & 7) * 2u;
}
__host__ __device__ inline size_t tiled_index(int row, int col, int K) {
    // element index (not bytes) of logical (row, col) in the tiled layout
    size_t tile = size_t(row >> 4), kb = size_t(col >> 6);
    int r = row & 15, c = col & 63;
    size_t block = tile * size_t(K >> 6) + kb;
    size_t inblock = size_t(r) * 64 + size_t((((c >> 3) ^ (r & 7)) << 3) + (c & 7));
    return block * 1024 + inblock;
}

// Host: the current CUDA device, for per-device one-time launch configuration
// (function attributes and occupancy apply to the device current when they are
// set; one process may drive several devices through several mesh_gpu handles).
constexpr int MAX_DEVICES = 64;
inline int cur_device() {
    int d = 0;
    cudaGetDevice(&d);
    return (d >= 0 && d < MAX_DEVICES) ? d : 0;
}

}  // namespace meshgpu
