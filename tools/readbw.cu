// Read-bandwidth ceiling probe for the decode kernel's streaming design.
//   ldg   : grid-stride uint4 loads (8 in flight per thread), summed
//   ring  : persistent CTA per SM, one producer thread issuing cp.async.bulk
//           stages into an N-deep smem ring, 8 consumer warps wait + release
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/readbw tools/readbw.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(smem_u32(b)),
        "r"(par)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__global__ void ldg_kernel(const uint4* p, size_t n, unsigned long long* out) {
    size_t tid = blockIdx.x * size_t(blockDim.x) + threadIdx.x, nt = size_t(gridDim.x) * blockDim.x;
    uint32_t acc = 0;
    for (size_t i = tid; i < n; i += 8 * nt) {
        uint4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = (i + k * nt < n) ? __ldcs(p + i + k * nt) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int k = 0; k < 8; ++k) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
    }
    if (acc == 0x12345678) atomicAdd(out, 1ull);
}

// Each CTA streams a contiguous 1/G share of the buffer in `stage` byte stages
// made of `stage / piece` bulk copies.
__global__ void __launch_bounds__(288, 1) ring_kernel(const uint8_t* p, size_t bytes, int stage, int piece, int depth,
                                                      unsigned long long* out, int plan, size_t scatter = 0,
                                                      int gscatter = 0) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + size_t(depth) * stage);
    uint64_t* empty = full + depth;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < depth; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const size_t per = bytes / gridDim.x / stage * stage;
    const uint8_t* base = p + per * blockIdx.x;
    const int n = int(per / stage);
    if (warp == 8) {
        if (lane < plan) {  // lane L issues stages q = L (mod plan)
            for (int q = lane; q < n; q += plan) {
                const int slot = q % depth;
                const uint32_t par = (q / depth) & 1;
                mbar_wait(&empty[slot], par ^ 1u);
                mbar_expect_tx(&full[slot], stage);
                for (int o = 0; o < stage; o += piece) {
                    // scatter > 0: pieces `scatter` bytes apart (paged-KV-like), wrapping in the CTA's share
                    // scatter > 0: pieces `scatter` bytes apart (paged-KV-like), wrapping in the CTA's share;
                    // gscatter: the same stride wrapping over the whole buffer (a KV block stride of MBs:
                    // every piece on its own 2 MB page)
                    const size_t idx = size_t(q) * (stage / piece) + o / piece;
                    const uint8_t* src = scatter == 0 ? base + size_t(q) * stage + o
                                         : !gscatter ? base + idx * scatter % (per - piece)
                                                     : p + ((size_t(blockIdx.x) * 7919 + idx) * scatter) % (bytes - piece) / 4096 * 4096;
                    bulk_g2s(sm + size_t(slot) * stage + o, src, piece, &full[slot]);
                }
            }
        }
        return;
    }
    uint32_t acc = 0;
    for (int q = warp; q < n; q += 8) {
        const int slot = q % depth;
        mbar_wait(&full[slot], (q / depth) & 1);
        acc ^= reinterpret_cast<const uint32_t*>(sm + size_t(slot) * stage)[lane];
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
    }
    if (acc == 0x12345678) atomicAdd(out, 1ull);
}

int main(int argc, char** argv) {
    setvbuf(stdout, nullptr, _IONBF, 0);
    const size_t bytes = size_t(4) << 30;
    uint8_t* buf;
    unsigned long long* out;
    CK(cudaMalloc(&buf, bytes));
    CK(cudaMalloc(&out, 8));
    CK(cudaMemset(buf, 1, bytes));
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto timeit = [&](auto launch) {
        launch();
        CK(cudaDeviceSynchronize());
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            CK(cudaEventRecord(e0));
            launch();
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (ms < best) best = ms;
        }
        return best;
    };
    for (int bpsm : {8}) {
        float ms = timeit([&] { ldg_kernel<<<sms * bpsm, 256>>>((const uint4*)buf, bytes / 16, out); });
        printf("{\"kind\":\"ldg\",\"blocks_per_sm\":%d,\"GBps\":%.1f}\n", bpsm, bytes / ms / 1e6);
    }
    CK(cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    if (argc > 1 && std::string(argv[1]) == "grid") {
        // per-SM rate at lane quotas: 8 KB stages of 1..4 pieces, contiguous or scattered
        const bool tlb = argc > 2 && std::string(argv[2]) == "tlb";
        for (int g : {17, 56, 148})
            for (int piece : {2048, 4096, 8192})
                for (size_t sc : tlb ? std::vector<size_t>{0, 368640, 1835008} : std::vector<size_t>{0, 368640}) {
                    if (tlb && piece == 2048) continue;
                    const int gs = tlb && sc == 1835008;
                    const size_t smem = size_t(8192) * 16 + 16 * 16;
                    float ms = timeit([&] { ring_kernel<<<g, 288, smem>>>(buf, bytes / 148 * g, 8192, piece, 16, out, 8, sc, gs); });
                    const double gbs = double(bytes / 148 * g) / ms / 1e6;
                    printf("{\"kind\":\"ring-grid\",\"grid\":%d,\"piece\":%d,\"scatter\":%zu,\"global\":%d,\"GBps\":%.1f,\"GBps_per_sm\":%.1f}\n",
                           g, piece, sc, gs, gbs, gbs / g);
                }
        return 0;
    }
    int stages[] = {4096, 8192, 16384};
    int depths[] = {8, 16};  // multiples of 8: a warp always re-waits on its own slots
    for (int st : stages)
        for (int d : depths) {
            if (size_t(st) * d > 200 * 1024) continue;
            if (d < 8) continue;
            for (int piece : {4096, st}) {
                if (piece > st) continue;
                size_t smem = size_t(st) * d + 16 * d;
                for (int plan : {1, 2, 4, 8}) {
                    float ms = timeit([&] { ring_kernel<<<sms, 288, smem>>>(buf, bytes, st, piece, d, out, plan); });
                    printf("{\"kind\":\"ring\",\"stage\":%d,\"piece\":%d,\"depth\":%d,\"lanes\":%d,\"GBps\":%.1f}\n", st,
                           piece, d, plan, bytes / ms / 1e6);
                }
                if (piece == st) break;
            }
        }
    CK(cudaGetLastError());
    return 0;
}
