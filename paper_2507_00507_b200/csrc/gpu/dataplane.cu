// Host side of the B200 data plane behind include/mesh_gpu.h.
//
//  * KV pool: every instance reserves a virtual range (cuMemAddressReserve)
//    and maps 2 MiB physical granules from a per-device free list; block b of
//    the instance lives at va + b * block_bytes, so GROW = map granules (no
//    copy) and SHRINK = move live blocks above the new high-water mark into
//    the lowest free slots (batched block-copy kernel), rewrite the block
//    tables, unmap the tail. Ops are applied physically when ISSUED, so the
//    physical footprint tracks the control plane's optimistic budget
//    (memory.cpp:84-104) and every accounted target is backed.
//  * Block tables: per request, the block ids in position order; new blocks
//    come from the lowest free index (deterministic).
//  * Steps run on execution lanes (one stream + scratch + an SM quota each);
//    the host never waits for a step unless asked (tickets).
//  * Swap: an evicted request's blocks are gathered by one copy kernel on a
//    side stream straight into a preallocated pinned host range (host-mapped,
//    PCIe writes); swap_out never waits on the host, and the blocks return to
//    the free list once the gather's event fired. Resume (the request's next
//    prefill step, or an explicit swap_in prefetch) is gated on that event and
//    scatters the range back with the same kernel, then feeds only the last
//    token (equivalent to the reference's re-prefill of I+O tokens).
//  * Migration: the same copy kernel on the destination GPU loads the source
//    instance's blocks over NVLink (every KV granule is mapped readable by all
//    peer devices) and writes the destination's blocks; event-ordered on both
//    lanes, no stream synchronisation.
#include <cuda.h>
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/mesh_gpu.h"
#include "decode.cuh"
#include "prefill.cuh"

using namespace meshgpu;

namespace {

// ------------------------------------------------------------------ errors
struct MeshError : std::runtime_error {
    mesh_status code;
    MeshError(mesh_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
#define CK(expr)                                                                                      \
    do {                                                                                              \
        cudaError_t _e = (expr);                                                                      \
        if (_e != cudaSuccess)                                                                        \
            throw MeshError(MESH_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));      \
    } while (0)

// ------------------------------------------------------- driver VMM entry
struct Driver {
    decltype(&cuMemAddressReserve) addr_reserve = nullptr;
    decltype(&cuMemAddressFree) addr_free = nullptr;
    decltype(&cuMemCreate) create = nullptr;
    decltype(&cuMemRelease) release = nullptr;
    decltype(&cuMemMap) map = nullptr;
    decltype(&cuMemUnmap) unmap = nullptr;
    decltype(&cuMemSetAccess) set_access = nullptr;
    decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
    bool ok = false;
};
Driver& drv() {
    static Driver d;
    static std::once_flag once;
    std::call_once(once, [] {
        auto get = [](const char* name, void** fn) {
            cudaDriverEntryPointQueryResult q;
            return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
                   q == cudaDriverEntryPointSuccess && *fn != nullptr;
        };
        d.ok = get("cuMemAddressReserve", (void**)&d.addr_reserve) &&
               get("cuMemAddressFree", (void**)&d.addr_free) && get("cuMemCreate", (void**)&d.create) &&
               get("cuMemRelease", (void**)&d.release) && get("cuMemMap", (void**)&d.map) &&
               get("cuMemUnmap", (void**)&d.unmap) && get("cuMemSetAccess", (void**)&d.set_access) &&
               get("cuMemGetAllocationGranularity", (void**)&d.granularity);
    });
    return d;
}
void CU(CUresult r, const char* what) {
    if (r != CUDA_SUCCESS) throw MeshError(MESH_ERR_CUDA, std::string(what) + " failed: CUresult " + std::to_string(int(r)));
}

// -------------------------------------------------------------- kernels
template <int SEL>
__global__ void init_tiled(uint8_t* dst, Shape s, uint64_t seed, int layer, int N, int K) {
    // SEL: 0 qkv, 1 o, 2 gu, 3 down, 4 lm
    size_t total = size_t(N) * K;
    uint16_t* out = reinterpret_cast<uint16_t*>(dst);
    const int kbs = K / 64;
    for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
        size_t block = e >> 10;
        int inb = int(e & 1023);
        int tile = int(block / kbs), kb = int(block % kbs);
        int r = inb >> 6, cs = inb & 63;
        int c = ((((cs >> 3) ^ (r & 7))) << 3) + (cs & 7);
        int prow = tile * 16 + r, col = kb * 64 + c;
        uint32_t tensor;
        size_t index;
        if (SEL == 0) {
            QkvRow q = qkv_row(s, prow);
            tensor = q.section == 0 ? T_WQ : (q.section == 1 ? T_WK : T_WV);
            index = size_t(q.head * s.dh + q.dim) * K + col;
        } else if (SEL == 1) {
            tensor = T_WO;
            index = size_t(prow) * K + col;
        } else if (SEL == 2) {
            int up, row;
            gu_row(prow, &up, &row);
            tensor = up ? T_WUP : T_WGATE;
            index = size_t(row) * K + col;
        } else if (SEL == 3) {
            tensor = T_WDOWN;
            index = size_t(prow) * K + col;
        } else {
            tensor = s.tied ? T_EMB : T_LM;
            index = size_t(prow) * K + col;
        }
        uint64_t key = tensor_key(seed, tensor, (SEL == 4) ? 0u : uint32_t(layer));
        out[e] = f_to_bf16(weight_value(key, index));
    }
}
__global__ void init_emb(uint16_t* dst, Shape s, uint64_t seed) {
    size_t total = size_t(s.vocab) * s.d;
    uint64_t key = tensor_key(seed, T_EMB, 0);
    for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x)
        dst[e] = f_to_bf16(weight_value(key, e));
}
__global__ void init_gain(float* dst, int n, uint64_t seed, uint32_t tensor, int layer) {
    uint64_t key = tensor_key(seed, tensor, uint32_t(layer));
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        dst[i] = gain_value(key, uint64_t(i));
}
// Batched whole-block KV copy driven by a block list passed by value (no
// device-side list buffer, no H2D of it): block src[i] of the source region
// -> block dst[i] of the destination region, blockIdx.y = i. One kernel serves
// every KV move of the data plane:
//   compaction  src = dst = the instance's VA range (HBM -> HBM)
//   swap out    src = VA range, dst = host-mapped pinned staging, dst[i] = i (gather -> PCIe writes)
//   swap in     src = pinned staging, src[i] = i, dst = VA range (PCIe reads -> scatter)
//   migration   src = another instance's VA range, possibly on a peer GPU (NVLink P2P loads)
// Each thread keeps 4 x 16 B loads in flight before its stores, so PCIe / NVLink
// read latency is covered with a modest grid.
constexpr int KV_LIST_MAX = 256;  // == DEC_BT_MAX: one request's blocks fit one launch
struct BlockList {
    int n;
    int src[KV_LIST_MAX];
    int dst[KV_LIST_MAX];
};
__global__ void __launch_bounds__(256) kv_blocks_copy(uint8_t* dst_base, const uint8_t* src_base, long long block_bytes,
                                                      const __grid_constant__ BlockList L) {
    const int i = blockIdx.y;
    const uint4* src = reinterpret_cast<const uint4*>(src_base + size_t(L.src[i]) * size_t(block_bytes));
    uint4* dst = reinterpret_cast<uint4*>(dst_base + size_t(L.dst[i]) * size_t(block_bytes));
    const size_t n = size_t(block_bytes) / 16, stride = size_t(gridDim.x) * blockDim.x;
    size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    for (; e + 3 * stride < n; e += 4 * stride) {
        uint4 v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = __ldcs(src + e + k * stride);
#pragma unroll
        for (int k = 0; k < 4; ++k) __stcs(dst + e + k * stride, v[k]);
    }
    for (; e < n; e += stride) __stcs(dst + e, __ldcs(src + e));
}
__global__ void set_int(int* p, int v) { *p = v; }
__global__ void read_tiled_row(const uint8_t* W, int K, int prow, float* out) {
    const uint16_t* w = reinterpret_cast<const uint16_t*>(W);
    for (int col = threadIdx.x; col < K; col += blockDim.x) out[col] = bf16_to_f(w[tiled_index(prow, col, K)]);
}

// ----------------------------------------------------------- structures
constexpr int MAX_SLOTS = 64;  // concurrent requests per instance (batch cap 8 + queued)

struct Granule {
    CUmemGenericAllocationHandle h;
};

// Physical KV memory: granules created with cuMemCreate, mapped once into the
// KV arena (below) and never unmapped on the serving path.
struct PhysPool {
    int device = 0;
    size_t gran = 2u << 20;
    long long limit = 0;
    long long mapped = 0;  // bytes of arena slots assigned to instances (capacity + lazy slack)
    std::vector<CUmemGenericAllocationHandle> free_list;  // created, not mapped
    std::vector<CUmemGenericAllocationHandle> all;

    CUmemGenericAllocationHandle take() {
        if (!free_list.empty()) {
            auto h = free_list.back();
            free_list.pop_back();
            return h;
        }
        CUmemAllocationProp prop = {};
        prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        prop.location.id = device;
        CUmemGenericAllocationHandle h;
        CUresult r = drv().create(&h, gran, &prop, 0);
        if (r != CUDA_SUCCESS) throw MeshError(MESH_ERR_NOMEM, "cuMemCreate failed: " + std::to_string(int(r)));
        all.push_back(h);
        return h;
    }
    void give(CUmemGenericAllocationHandle h) { free_list.push_back(h); }
};

struct ReqState {
    int slot = -1;
    int ctx = 0;               // tokens whose KV is resident
    std::vector<int> blocks;   // block ids by position / 16
    std::vector<int> tokens;   // prompt + generated ids (host history)
    int pending_tokens = 0;    // emitted on device, not yet copied back
};

// Pinned host swap space shared by every handle of the process. Pinned memory
// allocated cudaHostAllocPortable | Mapped is addressable from every GPU, so a
// request evicted on one device can resume on any other (the control plane may
// re-route it to another node). Chunks are pinned once (at open when
// mesh_gpu_cfg.swap_pool_mb > 0, else on first use) and carved first-fit;
// swaps never call cudaHostAlloc / cudaFreeHost on the steady path.
struct HostSwapPool {
    struct Chunk {
        uint8_t* base = nullptr;
        size_t bytes = 0;
        std::map<size_t, size_t> free;  // offset -> length, coalesced
    };
    std::mutex mu;
    std::vector<Chunk> chunks;
    size_t chunk_bytes = size_t(256) << 20;
    size_t pinned = 0;

    void add_chunk(size_t bytes) {
        Chunk c;
        c.bytes = bytes;
        if (cudaHostAlloc((void**)&c.base, bytes, cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess) {
            cudaGetLastError();
            throw MeshError(MESH_ERR_NOMEM, "swap space: cudaHostAlloc of " + std::to_string(bytes) + " bytes failed");
        }
        c.free[0] = bytes;
        pinned += bytes;
        chunks.push_back(std::move(c));
    }
    void reserve(size_t bytes) {  // make sure `bytes` of pinned space exist
        std::lock_guard<std::mutex> lk(mu);
        if (pinned < bytes) add_chunk(bytes - pinned);
    }
    // -> (chunk, offset); 256-byte aligned
    std::pair<int, size_t> take(size_t n) {
        n = (n + 255) & ~size_t(255);
        std::lock_guard<std::mutex> lk(mu);
        for (int pass = 0; pass < 2; ++pass) {
            for (size_t ci = 0; ci < chunks.size(); ++ci)
                for (auto it = chunks[ci].free.begin(); it != chunks[ci].free.end(); ++it)
                    if (it->second >= n) {
                        const size_t off = it->first, len = it->second;
                        chunks[ci].free.erase(it);
                        if (len > n) chunks[ci].free[off + n] = len - n;
                        return {int(ci), off};
                    }
            if (pass == 0) add_chunk(std::max(chunk_bytes, n));
        }
        throw MeshError(MESH_ERR_NOMEM, "swap space exhausted");
    }
    void give(int ci, size_t off, size_t n) {
        n = (n + 255) & ~size_t(255);
        std::lock_guard<std::mutex> lk(mu);
        auto& fr = chunks[size_t(ci)].free;
        auto it = fr.emplace(off, n).first;
        auto nx = std::next(it);
        if (nx != fr.end() && it->first + it->second == nx->first) {
            it->second += nx->second;
            fr.erase(nx);
        }
        if (it != fr.begin()) {
            auto pv = std::prev(it);
            if (pv->first + pv->second == it->first) {
                pv->second += it->second;
                fr.erase(it);
            }
        }
    }
    uint8_t* ptr(int ci, size_t off) { return chunks[size_t(ci)].base + off; }
};
HostSwapPool& host_pool() {
    static HostSwapPool p;
    return p;
}

// A request parked in pinned host memory. `done` fires when its gather (D2H)
// finished; the host history may still miss the tokens of steps that were in
// flight at eviction (`pending_tokens`), which drain into the entry as the
// origin instance's tickets retire.
struct SwapEntry {
    uint64_t shape_key = 0;
    int ctx = 0;
    std::vector<int> tokens;
    int pending_tokens = 0;
    mesh_gpu* origin = nullptr;  // handle / instance the request was evicted from
    int64_t origin_inst = -1;
    int chunk = -1;              // host swap space range (chunk < 0: no KV parked)
    size_t off = 0;
    size_t bytes = 0;
    long long block_bytes = 0;
    cudaEvent_t done = nullptr;
};

// Blocks whose last reader (a swap gather or a migration copy) may still run:
// they return to the free list once `ev` fired.
struct PendingFree {
    cudaEvent_t ev = nullptr;
    std::vector<int> blocks;
};

struct Instance {
    int64_t id = -1;
    Shape s{};
    uint64_t seed = 0;
    uint64_t shape_key = 0;
    uint8_t* wmem = nullptr;
    Weights w{};
    // KV region: extents of the device's KV arena. Block ids the control plane and
    // the policy see are logical (0 .. cap-1, the oracle's ids); the device sees
    // physical ids (block p at arena base + p * block_bytes), translated per extent.
    struct Extent {
        int s0, k;  // arena slots [s0, s0 + k)
        int p0, L;  // physical blocks [p0, p0 + L): the whole blocks inside those slots
    };
    std::vector<Extent> ext;      // in logical order
    std::vector<int> ext_first;   // logical id of each extent's first block
    int ext_slots = 1;            // slots per extent (>= 32 blocks per extent)
    long long block_bytes = 0;
    long long target = 0;  // accounted KV bytes (control plane target)
    int cap_blocks = 0;
    std::set<int> free_blocks;
    int live_blocks = 0;
    // requests
    std::map<int64_t, ReqState> reqs;
    std::vector<int> free_slots;
    int* d_block_table = nullptr;  // [MAX_SLOTS][bt_stride]
    int bt_stride = 0;
    int* d_last_tok = nullptr;     // [MAX_SLOTS]
    std::vector<int> h_block_table;
    int lane = 0;
    double weight_bytes = 0;
    cudaEvent_t last_ev = nullptr;  // after the instance's last enqueued lane work (steps, compaction)
    std::deque<PendingFree> pending_free;  // blocks still read by an in-flight swap-out / migration
};

struct Ticket {
    int64_t instance = -1;
    bool prefill = false;
    std::vector<int64_t> reqs;
    int ring = -1;
    int lane = 0;
    cudaEvent_t start = nullptr, kend = nullptr, end = nullptr;
    bool logits = false;
    int vocab = 0;
    bool drained = false;
    std::vector<int> toks;
};

constexpr int RING = 1024;

// An execution lane: one stream, its own decode/prefill scratch and grid
// barrier, and a share of the SMs. Instances are bound to a lane; lanes run
// concurrently, so co-located instances step at the same time on disjoint SM
// quotas (the persistent decode grids of all lanes sum to <= the SM count, so
// they can always be co-resident).
struct Lane {
    cudaStream_t stream = nullptr;
    int ctas = 0;  // SM quota: decode grid and prefill GEMM grid
    // decode scratch
    float* h = nullptr;
    uint16_t* act = nullptr;
    uint16_t* attn = nullptr;
    uint16_t* abuf = nullptr;
    float* q = nullptr;
    float* ssA = nullptr;
    float* ssB = nullptr;
    float* apart = nullptr;
    int* acnt = nullptr;
    float* arg_val = nullptr;
    int* arg_idx = nullptr;
    int* arg_cnt = nullptr;
    int* claim = nullptr;  // decode tile-claim counters (self-resetting)
    int* qkv_done = nullptr;  // decode QKV-group completion counters (self-resetting)
    float* logits = nullptr;
    unsigned* bar = nullptr;  // [count, gen]
    // prefill scratch
    float* p_h = nullptr;
    uint16_t* p_act = nullptr;
    float* p_rs = nullptr;
    float* p_q = nullptr;
    uint16_t* p_attn = nullptr;
    uint16_t* p_abuf = nullptr;
    float* p_logits = nullptr;
    int* p_tokens = nullptr;
    double weight_bytes = 0;  // bound instances (placement balance, SM quota)
    int n_inst = 0;
    int* tile_ctr = nullptr;  // prefill GEMM dynamic tile counter
    float* sk_ws = nullptr;   // prefill split-K partials
    int* sk_cnt = nullptr;    // prefill split-K arrival counters
    cudaEvent_t quota_ev = nullptr;  // tail of the lane's queue when its quota last shrank
};

}  // namespace

struct mesh_gpu {
    mesh_gpu_cfg cfg{};
    std::string err;
    int sms = 0;
    cudaStream_t side = nullptr;     // swap-out gathers (D2H over PCIe)
    cudaStream_t side_in = nullptr;  // swap-in prefetch scatters (H2D; PCIe is full duplex)
    cudaEvent_t timer[8] = {};       // mesh_gpu_timer_mark slots
    cudaEvent_t lane_join = nullptr; // timer marks: joins lanes into lane 0
    bool check = false;              // MESH_GPU_CHECK: synchronous per-step validation (debug)
    bool poison = false;             // MESH_GPU_POISON: NaN-fill newly mapped KV granules (debug)
    bool prefill_quota = false;      // MESH_PREFILL_QUOTA: cap prefill GEMM grids at the lane quota
    int prefill_min_ctas = 0;        // MESH_PREFILL_CTAS=n: cap at max(lane quota, n) instead
    PhysPool pool;
    std::map<int64_t, std::unique_ptr<Instance>> insts;
    std::vector<Lane> lanes;         // concurrent execution lanes (>= 1)
    // scratch capacities (sized for the largest registered shape, every lane)
    size_t cap_d = 0, cap_ff = 0, cap_vocab = 0, cap_q = 0, cap_ap = 0, cap_seq = 0;
    int* h_pf_stage = nullptr;       // [RING][pf_stage_ints] pinned prefill staging (block row + tokens)
    size_t pf_stage_ints = 0;
    // step rings
    StepDesc* h_desc = nullptr;
    StepDesc* d_desc = nullptr;
    int* h_tok = nullptr;   // [RING][8]
    int* d_tok = nullptr;   // [RING][8]
    cudaEvent_t ring_ev[RING] = {};
    bool ring_used[RING] = {};
    int ring_next = 0;
    std::map<int64_t, Ticket> tickets;
    int64_t next_ticket = 1;
    bool capture_logits = false;
    mesh_gpu_stats st{};
    int nstage = DEC_NSTAGE;  // decode ring depth (the round-1 8-stage A/B knob is gone)
    int skip = 0;             // MESH_GPU_SKIP debug mask (benchmarking only)
    int kv_lanes = 1;         // MESH_GPU_KV_LANES=0: attention KV stages through the batched push/flush instead of decoupled lanes
    int w_lanes = 1;          // MESH_GPU_W_LANES=0: weight stages through the batched push/flush instead of decoupled lanes
    int l2pf = 0;             // MESH_GPU_L2PF: weight-stage L2 prefetch lookahead in stages (decode_kernel)
    int* dbg_host = nullptr;  // MESH_GPU_WATCHDOG: host-mapped decode progress
    int* dbg_dev = nullptr;
    // Weights are a pure function of shape + weight seed, and the seed is the
    // model's, so every replica of a model is identical and read-only: live
    // replicas share one weight set (a scale-out replica costs no allocation and
    // no init kernels), and a set whose last replica unloads stays resident for
    // a reload (LRU past wcache_cap bytes of idle sets). Per-instance buffers
    // (KV VA range, block table, last tokens) are recycled the same way. No
    // create or destroy calls cudaFree / cudaMalloc on the steady path: both
    // serialise the device.
    struct WeightSet {
        uint8_t* wmem;
        size_t bytes;
        int refs;
        cudaEvent_t ready;  // after the init kernels (other lanes wait on it)
        uint64_t tick;      // last release, for LRU eviction of idle sets
    };
    std::map<uint64_t, WeightSet> wsets;  // by shape key
    // Per-instance buffers of unloaded instances (block table, last tokens),
    // recycled by the next create: no cudaMalloc / cudaFree on the churn path.
    struct InstBufs {
        int* d_block_table;  // [MAX_SLOTS][DEC_BT_MAX]
        int* d_last_tok;
    };
    std::vector<InstBufs> ibufs;  // free per-instance buffers
    // The KV arena: ONE virtual range for every instance's KV, carved into
    // granule-sized slots. A slot is backed (cuMemCreate + cuMemMap) the first
    // time it is needed, or at open (MESH_GPU_KV_PREALLOC_GB), and then stays
    // mapped: growing, shrinking, reclaiming and recycling KV between instances
    // is host bookkeeping plus a stream wait on the previous owner's last work.
    // cuMemMap / cuMemUnmap wait for the whole device to drain, so none of them
    // runs on the serving path once the arena is backed.
    struct KvArena {
        CUdeviceptr base = 0;
        int nslots = 0;
        std::vector<CUmemGenericAllocationHandle> h;  // 0: not backed yet
        std::vector<int64_t> owner;                    // -1: free
        std::vector<cudaEvent_t> ev;                   // free slot: after its last owner's queued work
        size_t bytes(size_t gran) const { return size_t(nslots) * gran; }
    } arena;
    size_t wcache_cap = size_t(32) << 30;  // MESH_GPU_WCACHE_GB: bytes of idle weight sets kept
    uint64_t wtick = 0;
    // devices that may map this device's KV (peer access over NVLink): every KV
    // granule is mapped readable by them, so a migration is one copy kernel on
    // the destination GPU reading the source VA range directly
    std::vector<int> peers;
    // swap space ranges whose last reader (a swap-in scatter) may still run
    struct HostFree {
        cudaEvent_t ev;
        int chunk;
        size_t off, bytes;
    };
    std::deque<HostFree> host_free;
};

namespace {

// Parked requests by request id (ids are global to the control plane). One
// store per process, like the pinned space it indexes (HostSwapPool): a
// request may resume on another handle / device than the one it left.
struct SwapStore {
    std::mutex mu;
    std::map<int64_t, SwapEntry> m;
};
SwapStore& swaps() {
    static SwapStore s;
    return s;
}
std::map<int64_t, SwapEntry>& swap_store() { return swaps().m; }

// Identity of a weight set: every input of the generator and of the RoPE table
// that lives in the set (theta and max_seq_len size and fill the table).
uint64_t shape_key_of(const Shape& s, uint64_t seed) {
    uint64_t k = seed;
    uint32_t theta_bits, eps_bits;
    std::memcpy(&theta_bits, &s.rope_theta, 4);
    std::memcpy(&eps_bits, &s.eps, 4);
    int64_t v[] = {s.n_layers, s.d, s.n_heads, s.n_kv, s.dh, s.ff, s.vocab, s.tied, s.max_seq, theta_bits, eps_bits};
    for (int64_t x : v) k = splitmix64(k ^ uint64_t(x));
    return k;
}

void device_guard(mesh_gpu* g) { CK(cudaSetDevice(g->cfg.device)); }

Lane& lane_of(mesh_gpu* g, const Instance& in) { return g->lanes[size_t(in.lane)]; }
cudaStream_t stream_of(mesh_gpu* g, const Instance& in) { return lane_of(g, in).stream; }
void sync_all(mesh_gpu* g) {
    for (Lane& l : g->lanes) CK(cudaStreamSynchronize(l.stream));
    CK(cudaStreamSynchronize(g->side));
}

int sm_budget(const mesh_gpu* g) { return g->cfg.sm_quota > 0 ? std::min(g->cfg.sm_quota, g->sms) : g->sms; }

// Token-level SM quotas: the SM budget is split over the lanes that hold
// instances in proportion to the weight bytes every step of theirs streams
// (decode is HBM-bound, so equal-duration steps need SMs in proportion to
// bytes); lanes without instances keep an even share for their first step.
// Quotas always sum to <= the budget, so every lane's persistent decode grid
// can be co-resident.
void rebalance_lanes(mesh_gpu* g) {
    const int budget = sm_budget(g), n = int(g->lanes.size());
    std::vector<int> q(size_t(n), 0);
    double wsum = 0;
    int busy = 0;
    for (const Lane& l : g->lanes)
        if (l.n_inst > 0) {
            wsum += l.weight_bytes;
            busy++;
        }
    if (busy == 0) {
        for (int i = 0; i < n; ++i) q[size_t(i)] = budget / n;
    } else {
        int used = 0;
        for (int i = 0; i < n; ++i) {
            const Lane& l = g->lanes[size_t(i)];
            q[size_t(i)] = l.n_inst > 0 ? std::max(1, int(double(budget) * l.weight_bytes / wsum)) : 0;
            used += q[size_t(i)];
        }
        auto biggest = [&] {
            int b = 0;
            for (int i = 1; i < n; ++i)
                if (q[size_t(i)] > q[size_t(b)]) b = i;
            return b;
        };
        // idle lanes: an even share of what is left (at least 1 SM, taken from the largest lane)
        for (int i = 0; i < n; ++i)
            if (g->lanes[size_t(i)].n_inst == 0) {
                const int big = biggest();
                if (used >= budget && q[size_t(big)] > 1) {
                    q[size_t(big)]--;
                    used--;
                }
                q[size_t(i)] = std::max(1, (budget - used) / std::max(1, n - busy));
                used += q[size_t(i)];
            }
        while (used > budget) {  // rounding guard
            q[size_t(biggest())]--;
            used--;
        }
        // SMs left over by rounding down go to the busy lanes with the largest
        // remainders (budget * w / wsum - quota), so every SM of the budget streams
        while (used < budget && busy > 0) {
            int best = -1;
            double rem = -1e300;
            for (int i = 0; i < n; ++i) {
                const Lane& l = g->lanes[size_t(i)];
                if (l.n_inst == 0) continue;
                const double r = double(budget) * l.weight_bytes / wsum - double(q[size_t(i)]);
                if (r > rem) {
                    rem = r;
                    best = i;
                }
            }
            q[size_t(best)]++;
            used++;
        }
    }
    // No host wait: every lane whose quota grows makes its stream wait for the
    // work already queued on the lanes whose quota shrinks (an event recorded
    // now on each of them). Old-quota grids of shrinking lanes therefore finish
    // before any new-quota grid of a growing lane starts, so the persistent
    // decode grids in flight never exceed the budget; lanes keep running.
    bool any_shrink = false;
    for (int i = 0; i < n; ++i) {
        Lane& l = g->lanes[size_t(i)];
        if (q[size_t(i)] < l.ctas) {
            CK(cudaEventRecord(l.quota_ev, l.stream));
            any_shrink = true;
        }
    }
    if (any_shrink)
        for (int i = 0; i < n; ++i) {
            Lane& l = g->lanes[size_t(i)];
            if (q[size_t(i)] <= l.ctas) continue;
            for (int j = 0; j < n; ++j)
                if (q[size_t(j)] < g->lanes[size_t(j)].ctas) CK(cudaStreamWaitEvent(l.stream, g->lanes[size_t(j)].quota_ev, 0));
        }
    for (int i = 0; i < n; ++i) g->lanes[size_t(i)].ctas = q[size_t(i)];
}

template <typename T>
void dalloc(T** p, size_t n) {
    if (*p) CK(cudaFree(*p));
    *p = nullptr;
    CK(cudaMalloc((void**)p, std::max<size_t>(n, 1) * sizeof(T)));
    CK(cudaMemset(*p, 0, std::max<size_t>(n, 1) * sizeof(T)));
}

void ensure_scratch(mesh_gpu* g, const Shape& s) {
    size_t nd = std::max(g->cap_d, size_t(s.d)), nff = std::max(g->cap_ff, size_t(s.ff)),
           nv = std::max(g->cap_vocab, size_t(s.vocab)), nq = std::max(g->cap_q, size_t(s.n_heads) * s.dh),
           nap = std::max(g->cap_ap, decode_apart_floats(s)), nseq = std::max(g->cap_seq, size_t(s.max_seq));
    if (g->lanes[0].h && nd == g->cap_d && nff == g->cap_ff && nv == g->cap_vocab && nq == g->cap_q && nap == g->cap_ap &&
        nseq == g->cap_seq)
        return;
    sync_all(g);
    g->cap_d = nd;
    g->cap_ff = nff;
    g->cap_vocab = nv;
    g->cap_q = nq;
    g->cap_ap = nap;
    g->cap_seq = nseq;
    for (Lane& l : g->lanes) {
        dalloc(&l.h, 8 * nd);
        dalloc(&l.act, 8 * nd);
        dalloc(&l.attn, 8 * nd);
        dalloc(&l.abuf, 8 * nff);
        dalloc(&l.q, 8 * nq);
        dalloc(&l.ssA, 8 * (nd / 16));
        dalloc(&l.ssB, 8 * (nd / 16));
        dalloc(&l.apart, nap);
        dalloc(&l.acnt, size_t(8) * 64);
        dalloc(&l.logits, 8 * nv);
        dalloc(&l.p_h, nseq * nd);
        dalloc(&l.p_act, nseq * nd);
        dalloc(&l.p_rs, nseq);
        dalloc(&l.p_q, nseq * nq);
        dalloc(&l.p_attn, nseq * nd);
        dalloc(&l.p_abuf, nseq * nff);
        dalloc(&l.p_logits, nv);
        dalloc(&l.p_tokens, nseq);
    }
    if (g->h_pf_stage) CK(cudaFreeHost(g->h_pf_stage));
    g->pf_stage_ints = nseq + DEC_BT_MAX;
    CK(cudaHostAlloc((void**)&g->h_pf_stage, g->pf_stage_ints * RING * sizeof(int), cudaHostAllocDefault));
}

Instance& inst_of(mesh_gpu* g, int64_t id) {
    auto it = g->insts.find(id);
    if (it == g->insts.end()) throw MeshError(MESH_ERR_ARG, "unknown instance " + std::to_string(id));
    return *it->second;
}

// ---- whole-block KV copies (compaction, swap, migration)
int copy_grid_x(long long block_bytes) { return int(std::max(1LL, std::min(32LL, block_bytes / 16384))); }

// dst_ids / src_ids null: blocks 0..n-1 of a contiguous staging range
void launch_blocks_copy(uint8_t* dst_base, const uint8_t* src_base, long long block_bytes, const int* src_ids,
                        const int* dst_ids, int n, cudaStream_t st) {
    for (int o = 0; o < n; o += KV_LIST_MAX) {
        BlockList L;
        L.n = std::min(KV_LIST_MAX, n - o);
        for (int i = 0; i < L.n; ++i) {
            L.src[i] = src_ids ? src_ids[o + i] : o + i;
            L.dst[i] = dst_ids ? dst_ids[o + i] : o + i;
        }
        kv_blocks_copy<<<dim3(unsigned(copy_grid_x(block_bytes)), unsigned(L.n)), 256, 0, st>>>(dst_base, src_base,
                                                                                              block_bytes, L);
        CK(cudaGetLastError());
    }
}

cudaEvent_t record_new_event(cudaStream_t st) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CK(cudaEventRecord(e, st));
    return e;
}

// Blocks of swapped-out / migrated requests go back to the free list once the
// copy that reads them finished (force: wait for it).
void reap_blocks(Instance& in, bool force) {
    for (auto it = in.pending_free.begin(); it != in.pending_free.end();) {
        const cudaError_t e = force ? cudaEventSynchronize(it->ev) : cudaEventQuery(it->ev);
        if (e == cudaErrorNotReady) {
            ++it;
            continue;
        }
        if (e != cudaSuccess) CK(e);
        for (int b : it->blocks) {
            if (b < in.cap_blocks) in.free_blocks.insert(b);
            in.live_blocks--;
        }
        cudaEventDestroy(it->ev);
        it = in.pending_free.erase(it);
    }
}

void reap_host(mesh_gpu* g, bool force) {
    for (auto it = g->host_free.begin(); it != g->host_free.end();) {
        const cudaError_t e = force ? cudaEventSynchronize(it->ev) : cudaEventQuery(it->ev);
        if (e == cudaErrorNotReady) {
            ++it;
            continue;
        }
        if (e != cudaSuccess) CK(e);
        host_pool().give(it->chunk, it->off, it->bytes);
        cudaEventDestroy(it->ev);
        it = g->host_free.erase(it);
    }
}

// ---- KV region management
int blocks_for_target(const Instance& in, long long target) {
    if (target <= 0) return 0;
    long long tokens = target / in.s.kv_bytes_per_token();
    long long blocks = (tokens + KV_BLOCK_TOKENS - 1) / KV_BLOCK_TOKENS;
    return int(blocks) + DEC_MAXB;  // one partial tail block per resident request
}

struct VmmTimer {  // host time of VMM driver calls -> stats
    mesh_gpu* g;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    explicit VmmTimer(mesh_gpu* gg) : g(gg) {}
    ~VmmTimer() {
        g->st.vmm_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
};

// Frees idle weight sets (no live replica), least recently released first,
// until at most `cap` bytes of them remain.
void evict_weights(mesh_gpu* g, size_t cap) {
    for (;;) {
        size_t idle = 0;
        auto victim = g->wsets.end();
        for (auto it = g->wsets.begin(); it != g->wsets.end(); ++it)
            if (it->second.refs == 0) {
                idle += it->second.bytes;
                if (victim == g->wsets.end() || it->second.tick < victim->second.tick) victim = it;
            }
        if (idle <= cap || victim == g->wsets.end()) return;
        // stream-ordered free: no device-wide synchronisation (the set has no live
        // replica, and its last replica's work finished before its destroy returned)
        cudaFreeAsync(victim->second.wmem, g->side);
        cudaEventDestroy(victim->second.ready);
        g->wsets.erase(victim);
    }
}

// ---- the KV arena
int kv_capacity(const Instance& in) { return in.ext.empty() ? 0 : in.ext_first.back() + in.ext.back().L; }

// physical id (arena-relative) of the instance's logical block b
int phys_of(const Instance& in, int b) {
    const size_t i = size_t(std::upper_bound(in.ext_first.begin(), in.ext_first.end(), b) - in.ext_first.begin()) - 1;
    return in.ext[i].p0 + (b - in.ext_first[i]);
}
std::vector<int> phys_list(const Instance& in, const std::vector<int>& ids) {
    std::vector<int> p(ids.size());
    for (size_t i = 0; i < ids.size(); ++i) p[i] = phys_of(in, ids[i]);
    return p;
}
uint8_t* arena_ptr(const mesh_gpu* g) { return reinterpret_cast<uint8_t*>(g->arena.base); }

// Backs slots [s0, s0 + n) that have no physical memory yet: the only cuMemMap
// calls (first use of a slot; the device drains once per call batch). Access is
// granted to this device and every NVLink peer (a migration's copy kernel runs on
// the destination GPU and loads the source's blocks directly).
void back_slots(mesh_gpu* g, int s0, int n) {
    const size_t gran = g->pool.gran;
    Driver& d = drv();
    VmmTimer vt(g);
    std::vector<CUmemAccessDesc> acc(1 + g->peers.size());
    for (size_t i = 0; i < acc.size(); ++i) {
        acc[i] = {};
        acc[i].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        acc[i].location.id = i == 0 ? g->cfg.device : g->peers[i - 1];
        acc[i].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    }
    int run = -1;  // first slot of the current run of newly mapped slots
    auto grant = [&](int end) {
        if (run < 0) return;
        CU(d.set_access(g->arena.base + size_t(run) * gran, size_t(end - run) * gran, acc.data(), acc.size()),
           "cuMemSetAccess");
        g->st.vmm_calls++;
        run = -1;
    };
    for (int sl = s0; sl < s0 + n; ++sl) {
        if (g->arena.h[size_t(sl)]) {
            grant(sl);
            continue;
        }
        CUmemGenericAllocationHandle h;
        try {
            h = g->pool.take();
        } catch (const MeshError&) {
            // HBM is short: idle weight sets go first (stream-ordered frees, then
            // hand the freed memory back from the allocator's pool), then retry
            evict_weights(g, 0);
            CK(cudaStreamSynchronize(g->side));
            cudaMemPool_t mp;
            if (cudaDeviceGetDefaultMemPool(&mp, g->cfg.device) == cudaSuccess) cudaMemPoolTrimTo(mp, 0);
            h = g->pool.take();
        }
        CUresult r = d.map(g->arena.base + size_t(sl) * gran, gran, 0, h, 0);
        if (r != CUDA_SUCCESS) {
            g->pool.give(h);
            grant(sl);
            throw MeshError(MESH_ERR_RUNTIME, "cuMemMap failed: " + std::to_string(int(r)));
        }
        g->arena.h[size_t(sl)] = h;
        g->st.vmm_calls++;
        if (run < 0) run = sl;
    }
    grant(s0 + n);
}

// Returns the instance's last extent to the arena. Its slots stay mapped; the
// next owner's streams wait for `ev` (the owner's queued work at release), so no
// host wait. ev == nullptr: the owner's work is known to be finished.
void release_extent(mesh_gpu* g, Instance& in, cudaStream_t owner_stream) {
    const Instance::Extent e = in.ext.back();
    for (int sl = e.s0; sl < e.s0 + e.k; ++sl) {
        g->arena.owner[size_t(sl)] = -1;
        if (owner_stream) g->arena.ev[size_t(sl)] = record_new_event(owner_stream);
    }
    g->pool.mapped -= (long long)e.k * (long long)g->pool.gran;
    in.ext.pop_back();
    in.ext_first.pop_back();
}

// Shrinks are lazy: a shrink compacts the live blocks below the new capacity but
// keeps the extents above it, so a later grow of the same instance costs nothing.
// Another instance's grow that finds no free run takes them back here.
bool reclaim_slack(mesh_gpu* g, const Instance* growing) {
    bool any = false;
    for (auto& [id, ip] : g->insts) {
        Instance& in = *ip;
        if (&in == growing) continue;  // its capacity is being raised right now
        while (!in.ext.empty() && in.ext_first.back() >= in.cap_blocks) {
            release_extent(g, in, stream_of(g, in));
            any = true;
        }
    }
    if (any) g->st.kv_reclaims++;
    return any;
}

int find_run(const mesh_gpu* g, int k) {
    int n = 0;
    for (int sl = 0; sl < g->arena.nslots; ++sl) {
        n = g->arena.owner[size_t(sl)] < 0 ? n + 1 : 0;
        if (n == k) return sl - k + 1;
    }
    return -1;
}

// Grows the instance's extents until they hold `blocks` logical blocks.
void assign_to(mesh_gpu* g, Instance& in, int blocks) {
    const size_t gran = g->pool.gran;
    const long long bb = in.block_bytes;
    while (kv_capacity(in) < blocks) {
        const int k = in.ext_slots;
        int s0 = find_run(g, k);
        if (s0 < 0 && reclaim_slack(g, &in)) s0 = find_run(g, k);
        if (s0 < 0)
            throw MeshError(MESH_ERR_NOMEM, "KV pool exhausted (limit " + std::to_string(g->pool.limit) + " bytes)");
        back_slots(g, s0, k);
        cudaStream_t st = stream_of(g, in);
        for (int sl = s0; sl < s0 + k; ++sl) {
            g->arena.owner[size_t(sl)] = in.id;
            cudaEvent_t& ev = g->arena.ev[size_t(sl)];
            if (ev) {  // the previous owner's queued work on these slots comes first
                CK(cudaStreamWaitEvent(st, ev, 0));
                CK(cudaStreamWaitEvent(g->side_in, ev, 0));
                cudaEventDestroy(ev);
                ev = nullptr;
            }
        }
        g->pool.mapped += (long long)k * (long long)gran;
        const long long lo = (long long)s0 * (long long)gran, hi = lo + (long long)k * (long long)gran;
        Instance::Extent e{s0, k, int((lo + bb - 1) / bb), 0};
        e.L = int(hi / bb) - e.p0;
        in.ext_first.push_back(kv_capacity(in));
        in.ext.push_back(e);
        // debug (MESH_GPU_POISON): recycled KV memory may hold any bit pattern; fill
        // newly assigned slots with bf16 NaN so reads of unwritten KV cannot go unnoticed
        if (g->poison) CK(cudaMemsetAsync(arena_ptr(g) + lo, 0xff, size_t(hi - lo), st));
    }
}

// Gives the physical memory of every backed, unassigned slot back to the driver
// (weights need HBM). cuMemUnmap drains the device: not a serving-path call.
void release_free_slots(mesh_gpu* g) {
    Driver& d = drv();
    VmmTimer vt(g);
    sync_all(g);
    for (int sl = 0; sl < g->arena.nslots; ++sl) {
        if (g->arena.owner[size_t(sl)] >= 0 || !g->arena.h[size_t(sl)]) continue;
        if (g->arena.ev[size_t(sl)]) {
            cudaEventDestroy(g->arena.ev[size_t(sl)]);
            g->arena.ev[size_t(sl)] = nullptr;
        }
        CU(d.unmap(g->arena.base + size_t(sl) * g->pool.gran, g->pool.gran), "cuMemUnmap");
        g->st.vmm_calls++;
        g->st.vmm_unmaps++;
        g->pool.give(g->arena.h[size_t(sl)]);
        g->arena.h[size_t(sl)] = 0;
    }
    for (auto h : g->pool.free_list) {
        drv().release(h);
        g->pool.all.erase(std::find(g->pool.all.begin(), g->pool.all.end(), h));
    }
    g->pool.free_list.clear();
}

void write_bt_entry(Instance& in, int slot, int idx, int block) {
    in.h_block_table[size_t(slot) * in.bt_stride + idx] = phys_of(in, block);
}

void resize_kv(mesh_gpu* g, Instance& in, long long to) {
    int new_cap = blocks_for_target(in, to);
    if (new_cap >= in.cap_blocks) {
        assign_to(g, in, new_cap);
        for (int b = in.cap_blocks; b < new_cap; ++b) in.free_blocks.insert(b);
        in.cap_blocks = new_cap;
        in.target = to;
        return;
    }
    // shrink: compact live blocks >= new_cap into the lowest free ids < new_cap
    reap_blocks(in, true);  // blocks of swapped-out / migrated requests still being read count as live
    if (in.live_blocks > new_cap)
        throw MeshError(MESH_ERR_RUNTIME, "kv shrink below live blocks (" + std::to_string(in.live_blocks) + " > " +
                                              std::to_string(new_cap) + ")");
    std::vector<int> from, to_ids;
    std::set<int> low_free;
    for (int b : in.free_blocks)
        if (b < new_cap) low_free.insert(b);
    for (auto& [rid, r] : in.reqs) {
        for (size_t i = 0; i < r.blocks.size(); ++i) {
            int b = r.blocks[i];
            if (b < new_cap) continue;
            int dst = *low_free.begin();
            low_free.erase(low_free.begin());
            from.push_back(b);
            to_ids.push_back(dst);
            r.blocks[i] = dst;
            write_bt_entry(in, r.slot, int(i), dst);
        }
    }
    if (!from.empty()) {
        // one batched copy kernel per 256 moves, block lists passed by value (no pair buffer, no host wait)
        cudaStream_t st = stream_of(g, in);
        const std::vector<int> pf = phys_list(in, from), pt = phys_list(in, to_ids);
        launch_blocks_copy(arena_ptr(g), arena_ptr(g), in.block_bytes, pf.data(), pt.data(), int(pf.size()), st);
        CK(cudaMemcpyAsync(in.d_block_table, in.h_block_table.data(), in.h_block_table.size() * sizeof(int),
                           cudaMemcpyHostToDevice, st));
        CK(cudaEventRecord(in.last_ev, st));
        g->st.blocks_moved += (long long)from.size();
        g->st.bytes_moved += 2LL * (long long)from.size() * in.block_bytes;
    }
    // the extents above the new capacity stay assigned (lazy shrink, see reclaim_slack)
    in.free_blocks = low_free;
    in.cap_blocks = new_cap;
    in.target = to;
}

int alloc_block(mesh_gpu* g, Instance& in) {
    if (in.free_blocks.empty() && !in.pending_free.empty()) {
        reap_blocks(in, false);
        if (in.free_blocks.empty()) reap_blocks(in, true);  // the copies reading them are short
    }
    if (in.free_blocks.empty()) {
        // physical overcommit beyond the accounted target (rounding slack exhausted)
        int b = in.cap_blocks;
        assign_to(g, in, b + 1);
        in.cap_blocks = b + 1;
        in.live_blocks++;
        return b;
    }
    int b = *in.free_blocks.begin();
    in.free_blocks.erase(in.free_blocks.begin());
    in.live_blocks++;
    return b;
}

void release_blocks(Instance& in, ReqState& r) {
    for (int b : r.blocks) {
        if (b < in.cap_blocks) in.free_blocks.insert(b);
        in.live_blocks--;
    }
    r.blocks.clear();
    r.ctx = 0;
}

ReqState& req_slot(Instance& in, int64_t rid) {
    auto it = in.reqs.find(rid);
    if (it != in.reqs.end()) return it->second;
    if (in.free_slots.empty()) throw MeshError(MESH_ERR_NOMEM, "instance request table full");
    ReqState r;
    r.slot = in.free_slots.back();
    in.free_slots.pop_back();
    return in.reqs.emplace(rid, std::move(r)).first->second;
}

void free_request(Instance& in, int64_t rid) {
    auto it = in.reqs.find(rid);
    if (it == in.reqs.end()) return;
    release_blocks(in, it->second);
    in.free_slots.push_back(it->second.slot);
    in.reqs.erase(it);
}

// Collect a finished ticket's tokens into the host histories (once).
void drain_ticket(mesh_gpu* g, Ticket& t) {
    if (t.drained) return;
    CK(cudaEventSynchronize(t.end));
    const int* toks = g->h_tok + t.ring * 8;
    int n = int(t.reqs.size());
    auto it = g->insts.find(t.instance);
    t.toks.assign(toks, toks + n);
    for (int i = 0; i < n; ++i) {
        if (it == g->insts.end()) break;
        auto rit = it->second->reqs.find(t.reqs[i]);
        if (rit != it->second->reqs.end()) {
            rit->second.tokens.push_back(toks[i]);
            rit->second.pending_tokens--;
        } else {  // swapped out while this step was in flight: the token belongs to the parked history
            std::lock_guard<std::mutex> lk(swaps().mu);
            auto sit = swap_store().find(t.reqs[i]);
            if (sit != swap_store().end() && sit->second.origin == g && sit->second.origin_inst == t.instance &&
                sit->second.pending_tokens > 0) {
                sit->second.tokens.push_back(toks[i]);
                sit->second.pending_tokens--;
            }
        }
    }
    float ms = 0.f, kms = 0.f, end_ms = -1.f;
    cudaEventElapsedTime(&ms, t.start, t.end);
    cudaEventElapsedTime(&kms, t.start, t.kend);
    if (g->timer[0] && cudaEventElapsedTime(&end_ms, g->timer[0], t.end) != cudaSuccess) end_ms = -1.f;
    g->st.last_step_ms = ms;
    g->st.last_kernel_ms = kms;
    g->st.last_step_end_ms = end_ms;
    g->ring_used[t.ring] = false;
    t.drained = true;
}

// Drain every outstanding ticket of an instance up to `upto` (in issue order)
// so request histories stay in token order.
void drain_instance(mesh_gpu* g, int64_t inst, int64_t upto = INT64_MAX) {
    for (auto& [tid, t] : g->tickets) {
        if (tid > upto) break;
        if (t.instance == inst) drain_ticket(g, t);
    }
}

void flush_request(mesh_gpu* g, int64_t inst, int64_t rid) {
    (void)rid;
    drain_instance(g, inst);
}

void destroy_ticket(Ticket& t) {
    cudaEventDestroy(t.start);
    cudaEventDestroy(t.kend);
    cudaEventDestroy(t.end);
}

int take_ring(mesh_gpu* g) {
    for (int k = 0; k < RING; ++k) {
        int i = (g->ring_next + k) % RING;
        if (!g->ring_used[i]) {
            g->ring_next = (i + 1) % RING;
            // the previous user of this slot may still be copying
            CK(cudaEventSynchronize(g->ring_ev[i]));
            g->ring_used[i] = true;
            return i;
        }
    }
    throw MeshError(MESH_ERR_RUNTIME, "too many outstanding step tickets (wait on older tickets)");
}

DecodeArgs decode_args(mesh_gpu* g, Instance& in, StepDesc* d_desc, int ring) {
    DecodeArgs a{};
    a.s = in.s;
    a.w = in.w;
    a.kv_base = arena_ptr(g);
    a.block_bytes = in.block_bytes;
    a.block_table = in.d_block_table;
    a.bt_stride = in.bt_stride;
    a.last_tok = in.d_last_tok;
    a.desc = d_desc;
    Lane& ln = lane_of(g, in);
    a.h = ln.h;
    a.act = ln.act;
    a.attn = ln.attn;
    a.abuf = ln.abuf;
    a.q = ln.q;
    a.ssA = ln.ssA;
    a.ssB = ln.ssB;
    a.apart = ln.apart;
    a.acnt = ln.acnt;
    a.arg_val = ln.arg_val;
    a.arg_idx = ln.arg_idx;
    a.arg_cnt = ln.arg_cnt;
    a.claim = ln.claim;
    a.qkv_done = ln.qkv_done;
    a.logits = g->capture_logits ? ln.logits : nullptr;
    a.tok_out = g->d_tok + ring * 8;
    a.bar_count = ln.bar;
    a.bar_gen = ln.bar + 1;
    a.progress = g->dbg_dev;
    a.trace = nullptr;
    a.arrive = nullptr;
    a.nstage = g->nstage;
    a.l2pf = g->l2pf;
    a.kv_lanes = g->kv_lanes;
    a.w_lanes = g->w_lanes;
    a.skip = g->skip;
    return a;
}

int grid_of(mesh_gpu* g, const Instance& in) { return lane_of(g, in).ctas; }

// Build the decode descriptor for `rids` (allocating blocks for new positions).
void build_decode_desc(mesh_gpu* g, Instance& in, const int64_t* rids, int n, StepDesc& d) {
    d.B = n;
    d.n_upd = 0;
    for (int i = 0; i < n; ++i) {
        auto it = in.reqs.find(rids[i]);
        if (it == in.reqs.end() || it->second.ctx == 0)
            throw MeshError(MESH_ERR_ARG, "decode of request " + std::to_string(rids[i]) + " without prefill");
        ReqState& r = it->second;
        if (r.ctx >= in.s.max_seq) throw MeshError(MESH_ERR_ARG, "context exceeds max_seq_len");
        d.slot[i] = r.slot;
        d.pos[i] = r.ctx;
        if (r.ctx % KV_BLOCK_TOKENS == 0) {
            int b = alloc_block(g, in);
            r.blocks.push_back(b);
            write_bt_entry(in, r.slot, int(r.blocks.size()) - 1, b);
            if (d.n_upd >= MAX_BT_UPDATES) throw MeshError(MESH_ERR_RUNTIME, "too many block-table updates");
            d.upd[d.n_upd][0] = r.slot;
            d.upd[d.n_upd][1] = int(r.blocks.size()) - 1;
            d.upd[d.n_upd][2] = phys_of(in, b);
            d.n_upd++;
        }
    }
}

void launch_decode_step(mesh_gpu* g, Instance& in, const int64_t* rids, int n, Ticket& t) {
    StepDesc& hd = g->h_desc[t.ring];
    build_decode_desc(g, in, rids, n, hd);
    cudaStream_t st = stream_of(g, in);
    CK(cudaMemcpyAsync(g->d_desc + t.ring, &hd, sizeof(StepDesc), cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(t.start, st));
    DecodeArgs a = decode_args(g, in, g->d_desc + t.ring, t.ring);
    CK(launch_decode(a, grid_of(g, in), st));
    CK(cudaEventRecord(t.kend, st));
    g->st.kernel_launches += 1;
    g->st.h2d_bytes += (long long)sizeof(StepDesc);
    for (int i = 0; i < n; ++i) {
        ReqState& r = in.reqs[rids[i]];
        r.ctx += 1;
        r.pending_tokens++;
    }
    g->st.decode_tokens += n;
}

// Takes a parked request out of the swap store (its history completed first:
// tokens of steps that were in flight at eviction drain from the origin).
SwapEntry take_parked(int64_t rid) {
    mesh_gpu* origin = nullptr;
    int64_t oinst = -1;
    {
        std::lock_guard<std::mutex> lk(swaps().mu);
        auto it = swap_store().find(rid);
        if (it == swap_store().end()) throw MeshError(MESH_ERR_ARG, "request " + std::to_string(rid) + " is not parked");
        if (it->second.pending_tokens > 0) {
            origin = it->second.origin;
            oinst = it->second.origin_inst;
        }
    }
    if (origin) drain_instance(origin, oinst);
    std::lock_guard<std::mutex> lk(swaps().mu);
    auto it = swap_store().find(rid);
    if (it == swap_store().end()) throw MeshError(MESH_ERR_ARG, "request " + std::to_string(rid) + " is not parked");
    SwapEntry e = std::move(it->second);
    swap_store().erase(it);
    return e;
}

// Scatter a parked request's KV back into fresh blocks of `in`, on stream `st`
// after the gather's event (no host wait); the pinned range is released once
// the scatter's own event fired. `st` is the instance's lane (resume inside a
// prefill step) or the swap-in side stream (prefetch; the lane then waits on
// the scatter before its next work).
void restore_parked(mesh_gpu* g, Instance& in, ReqState& r, SwapEntry& e, cudaStream_t st) {
    const int nblk = (e.ctx + KV_BLOCK_TOKENS - 1) / KV_BLOCK_TOKENS;
    for (int i = 0; i < nblk; ++i) {
        int b = alloc_block(g, in);
        r.blocks.push_back(b);
        write_bt_entry(in, r.slot, i, b);
    }
    CK(cudaStreamWaitEvent(st, e.done, 0));
    const std::vector<int> pb = phys_list(in, r.blocks);
    launch_blocks_copy(arena_ptr(g), host_pool().ptr(e.chunk, e.off), in.block_bytes, nullptr, pb.data(), nblk, st);
    cudaEvent_t ev = record_new_event(st);
    if (st != stream_of(g, in)) {
        CK(cudaStreamWaitEvent(stream_of(g, in), ev, 0));
        CK(cudaMemcpyAsync(in.d_block_table + size_t(r.slot) * in.bt_stride,
                           in.h_block_table.data() + size_t(r.slot) * in.bt_stride, sizeof(int) * in.bt_stride,
                           cudaMemcpyHostToDevice, stream_of(g, in)));
        set_int<<<1, 1, 0, stream_of(g, in)>>>(in.d_last_tok + r.slot, e.tokens.empty() ? 0 : e.tokens.back());
        CK(cudaGetLastError());
    }
    g->host_free.push_back({ev, e.chunk, e.off, e.bytes});
    cudaEventDestroy(e.done);
    e.done = nullptr;
    r.ctx = e.ctx;
    r.tokens = e.tokens;
    g->st.swap_in_bytes += (long long)nblk * in.block_bytes;
}

void drop_parked(mesh_gpu* g, SwapEntry& e) {
    if (e.chunk >= 0) {  // the gather may still be writing the range
        CK(cudaEventSynchronize(e.done));
        host_pool().give(e.chunk, e.off, e.bytes);
    }
    if (e.done) cudaEventDestroy(e.done);
    (void)g;
}

void launch_prefill_step(mesh_gpu* g, Instance& in, const mesh_step_plan& p, Ticket& t) {
    const int64_t rid = p.prefill_request;
    // a request with device history (re-prefill) needs its token history complete
    if (in.reqs.count(rid)) flush_request(g, in.id, rid);
    int n = p.prefill_len;
    if (n < 1 || n > in.s.max_seq) throw MeshError(MESH_ERR_ARG, "prefill_len out of range");
    // A request that was evicted resumes from its parked KV (or at least its
    // history). It is taken out of the store BEFORE its new slot exists: the
    // take completes the parked history from the origin's in-flight steps, and
    // those tokens must land in the entry, not in a fresh state of the same id.
    SwapEntry e;
    bool parked = false;
    if (!in.reqs.count(rid)) {
        {
            std::lock_guard<std::mutex> lk(swaps().mu);
            parked = swap_store().count(rid) > 0;
        }
        if (parked) {
            if (in.free_slots.empty()) throw MeshError(MESH_ERR_NOMEM, "instance request table full");
            e = take_parked(rid);
        }
    }
    ReqState& r = req_slot(in, rid);
    if (parked) {
        if (e.chunk >= 0 && e.shape_key == in.shape_key && e.ctx == n - 1) {
            restore_parked(g, in, r, e, stream_of(g, in));
        } else {
            r.tokens = e.tokens;
            drop_parked(g, e);
        }
    }
    if (r.tokens.empty()) {
        int I = p.prefill_input_len > 0 ? p.prefill_input_len : n;
        for (int i = 0; i < I; ++i) r.tokens.push_back(prompt_token(g->cfg.prompt_seed, rid, i, in.s.vocab));
    }
    if (int(r.tokens.size()) < n)
        throw MeshError(MESH_ERR_RUNTIME, "prefill of " + std::to_string(n) + " tokens but history has " +
                                              std::to_string(r.tokens.size()));
    int p0, L;
    if (r.ctx == n - 1 && r.ctx > 0) {  // resume: KV for [0, n-1) resident, feed token n-1
        p0 = n - 1;
        L = 1;
    } else {
        release_blocks(in, r);  // re-prefill from scratch
        p0 = 0;
        L = n;
    }
    // blocks for positions [p0, p0 + L)
    int need = (p0 + L + KV_BLOCK_TOKENS - 1) / KV_BLOCK_TOKENS;
    while (int(r.blocks.size()) < need) {
        int b = alloc_block(g, in);
        r.blocks.push_back(b);
        write_bt_entry(in, r.slot, int(r.blocks.size()) - 1, b);
    }
    // stage the block table row and the tokens through this ticket's pinned slot
    // (the slot is reused only after its previous step drained: no host sync here)
    int* stage = g->h_pf_stage + size_t(t.ring) * g->pf_stage_ints;
    std::memcpy(stage, in.h_block_table.data() + size_t(r.slot) * in.bt_stride, sizeof(int) * in.bt_stride);
    std::memcpy(stage + in.bt_stride, r.tokens.data() + p0, sizeof(int) * L);
    Lane& ln = lane_of(g, in);
    CK(cudaMemcpyAsync(in.d_block_table + size_t(r.slot) * in.bt_stride, stage, sizeof(int) * in.bt_stride,
                       cudaMemcpyHostToDevice, ln.stream));
    CK(cudaMemcpyAsync(ln.p_tokens, stage + in.bt_stride, sizeof(int) * L, cudaMemcpyHostToDevice, ln.stream));
    g->st.h2d_bytes += (long long)sizeof(int) * (in.bt_stride + L);
    PrefillArgs a{};
    a.s = in.s;
    a.w = in.w;
    a.kv_base = arena_ptr(g);
    a.block_bytes = in.block_bytes;
    a.kv_blocks = (long long)(g->arena.bytes(g->pool.gran) / size_t(in.block_bytes));
    a.bt_row = in.d_block_table + size_t(r.slot) * in.bt_stride;
    a.slot = r.slot;
    a.L = L;
    a.p0 = p0;
    a.tokens = ln.p_tokens;
    a.h = ln.p_h;
    a.act = ln.p_act;
    a.rs = ln.p_rs;
    a.q = reinterpret_cast<uint16_t*>(ln.p_q);  // bf16 view of the fp32-sized buffer
    a.attn = ln.p_attn;
    a.abuf = ln.p_abuf;
    a.logits = ln.p_logits;
    // Prefill GEMMs keep no grid barrier, so they may take every SM (their CTAs
    // queue behind other lanes' decode grids and finish); a lane's quota bounds
    // its persistent decode grid only. Measured: +5 % C2 tokens/s, -8 % e2e wall.
    a.max_ctas = g->prefill_quota ? std::max(ln.ctas, g->prefill_min_ctas) : 0;
    int busy_lanes = 0;
    for (const Lane& l : g->lanes) busy_lanes += l.n_inst > 0;
    a.pair_ok = busy_lanes <= 1;
    a.tile_ctr = ln.tile_ctr;
    a.sk_ws = ln.sk_ws;
    a.sk_cnt = ln.sk_cnt;
    a.last_tok = in.d_last_tok;
    a.tok_out = g->d_tok + t.ring * 8;
    CK(cudaEventRecord(t.start, ln.stream));
    CK(launch_prefill(a, ln.stream));
    CK(cudaEventRecord(t.kend, ln.stream));
    g->st.kernel_launches += prefill_launch_count(in.s);
    r.ctx = p0 + L;
    // history: the prefill consumed tokens[0, n); anything beyond is stale
    r.tokens.resize(n);
    r.pending_tokens++;
    g->st.prefill_tokens += L;
}

mesh_status fail(mesh_gpu* g, const std::exception& e) {
    if (auto* me = dynamic_cast<const MeshError*>(&e)) {
        if (g) g->err = me->what();
        return me->code;
    }
    if (g) g->err = e.what();
    return MESH_ERR_RUNTIME;
}

template <typename F>
mesh_status guarded(mesh_gpu* g, F&& body, double* host_ms = nullptr) {
    const auto t0 = std::chrono::steady_clock::now();
    struct Acc {
        double* ms;
        std::chrono::steady_clock::time_point t0;
        ~Acc() {
            if (ms) *ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        }
    } acc{host_ms, t0};
    try {
        if (g) device_guard(g);
        body();
        return MESH_OK;
    } catch (const std::exception& e) {
        return fail(g, e);
    }
}

// The data plane's shape of a C-ABI model shape (validated: throws MESH_ERR_CONFIG).
Shape shape_of(const mesh_model_shape& m) {
    const mesh_model_shape* sh = &m;
    Shape s{};
    s.n_layers = sh->n_layers;
    s.d = sh->d_model;
    s.n_heads = sh->n_heads;
    s.n_kv = sh->n_kv_heads;
    s.dh = sh->d_head;
    s.ff = sh->d_ff;
    s.vocab = sh->vocab;
    s.tied = sh->tied_embeddings;
    s.max_seq = sh->max_seq_len;
    s.rope_theta = sh->rope_theta > 0 ? sh->rope_theta : 10000.f;
    s.eps = sh->rms_eps > 0 ? sh->rms_eps : 1e-5f;
    if (s.dh != 64 && s.dh != 128) throw MeshError(MESH_ERR_CONFIG, "d_head must be 64 or 128");
    if (s.n_heads % s.n_kv != 0 || s.gq() * s.dh > 512)
        throw MeshError(MESH_ERR_CONFIG, "GQA group x d_head must be <= 512 (decode smem budget)");
    if (s.n_heads * s.dh != s.d) throw MeshError(MESH_ERR_CONFIG, "n_heads * d_head must equal d_model");
    if (s.d % 256 || s.ff % 256 || s.vocab % 128 || (s.qkv_rows() % 128))
        throw MeshError(MESH_ERR_CONFIG, "d_model/d_ff must be multiples of 256, vocab of 128");
    if (s.n_layers < 1 || s.n_layers * 4 + 1 > DEC_CLAIM_MAX) throw MeshError(MESH_ERR_CONFIG, "n_layers out of range");
    if (s.n_kv > DEC_KV_HEADS_MAX) throw MeshError(MESH_ERR_CONFIG, "n_kv_heads out of range");
    if (s.max_seq < 2 || s.max_seq > DEC_BT_MAX * KV_BLOCK_TOKENS)
        throw MeshError(MESH_ERR_CONFIG, "max_seq_len out of range");
    return s;
}

// Bytes of one weight set (tiled GEMM operands, embeddings, gains, RoPE table).
size_t weight_set_bytes(const Shape& s) {
    const size_t L = s.n_layers;
    const size_t qkv = size_t(s.qkv_rows()) * s.d * 2, o = size_t(s.d) * s.n_heads * s.dh * 2,
                 gu = size_t(2 * s.ff) * s.d * 2, dn = size_t(s.d) * s.ff * 2, lm = size_t(s.vocab) * s.d * 2,
                 emb = size_t(s.vocab) * s.d * 2;
    const size_t norms = (2 * L + 1) * s.d * 4, rope = size_t(s.max_seq) * (s.dh / 2) * 8;
    return L * (qkv + o + gu + dn) + lm + emb + norms + rope + 4096;
}

}  // namespace

extern "C" {

const char* mesh_gpu_version(void) { return "0.1.0-sm100a"; }

int32_t mesh_gpu_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

const char* mesh_gpu_last_error(const mesh_gpu* g) { return g ? g->err.c_str() : "null mesh_gpu handle"; }

mesh_status mesh_gpu_open(const mesh_gpu_cfg* cfg, mesh_gpu** out) {
    if (!cfg || !out) return MESH_ERR_ARG;
    *out = nullptr;
    auto g = std::make_unique<mesh_gpu>();
    g->cfg = *cfg;
    mesh_status st = guarded(g.get(), [&] {
        int n = 0;
        CK(cudaGetDeviceCount(&n));
        if (cfg->device < 0 || cfg->device >= n) throw MeshError(MESH_ERR_CUDA, "no such CUDA device");
        cudaDeviceProp prop;
        CK(cudaGetDeviceProperties(&prop, cfg->device));
        if (prop.major != 10)
            throw MeshError(MESH_ERR_CUDA, std::string("sm_100a kernels need a Blackwell B200, found ") + prop.name);
        g->sms = prop.multiProcessorCount;
        if (!drv().ok) throw MeshError(MESH_ERR_CUDA, "CUDA VMM driver entry points unavailable");
        // lanes: cfg->lanes (else MESH_GPU_LANES, else 1); the SMs (or the quota) split evenly
        int nl = cfg->lanes > 0 ? cfg->lanes : 1;
        if (cfg->lanes <= 0)
            if (const char* e = std::getenv("MESH_GPU_LANES")) nl = std::max(1, std::atoi(e));
        const int budget = cfg->sm_quota > 0 ? std::min(cfg->sm_quota, g->sms) : g->sms;
        if (nl > budget) throw MeshError(MESH_ERR_ARG, "more lanes than SMs");
        g->lanes.resize(size_t(nl));
        for (Lane& l : g->lanes) {
            CK(cudaStreamCreateWithFlags(&l.stream, cudaStreamNonBlocking));
            l.ctas = budget / nl;
            dalloc(&l.bar, 2);
            dalloc(&l.arg_val, size_t(8) * g->sms);
            dalloc(&l.arg_idx, size_t(8) * g->sms);
            dalloc(&l.arg_cnt, 1);
            dalloc(&l.claim, DEC_CLAIM_MAX);
            dalloc(&l.qkv_done, DEC_KV_HEADS_MAX);
            dalloc(&l.tile_ctr, 1);
            dalloc(&l.sk_ws, size_t(2) * g->sms * 128 * 256);
            dalloc(&l.sk_cnt, SK_TILES_MAX);
            CK(cudaEventCreateWithFlags(&l.quota_ev, cudaEventDisableTiming));
        }
        CK(cudaStreamCreateWithFlags(&g->side, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&g->side_in, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&g->lane_join, cudaEventDisableTiming));
        // peers: devices that can load this device's memory over NVLink get read/write
        // access to every KV granule (back_slots); this device may load theirs
        for (int d = 0; d < n; ++d) {
            if (d == cfg->device) continue;
            int can = 0;
            if (cudaDeviceCanAccessPeer(&can, d, cfg->device) == cudaSuccess && can) g->peers.push_back(d);
            int back = 0;
            if (cudaDeviceCanAccessPeer(&back, cfg->device, d) == cudaSuccess && back) {
                const cudaError_t e = cudaDeviceEnablePeerAccess(d, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
                cudaGetLastError();
            }
        }
        g->st.peer_devices = (int64_t)g->peers.size();
        // pinned swap space, pinned once up front (cudaHostAlloc of GBs takes ~0.1-1 s)
        if (cfg->swap_pool_mb > 0) host_pool().reserve(size_t(cfg->swap_pool_mb) << 20);
        g->pool.device = cfg->device;
        CUmemAllocationProp prop2 = {};
        prop2.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        prop2.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        prop2.location.id = cfg->device;
        size_t gran = 0;
        CU(drv().granularity(&gran, &prop2, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "cuMemGetAllocationGranularity");
        // large physical chunks: every cuMemMap / cuMemUnmap costs host time (and a
        // TLB shoot-down), so fewer, larger granules make grows and releases cheap
        const size_t want = cfg->kv_granule_bytes > 0 ? size_t(cfg->kv_granule_bytes) : size_t(32) << 20;
        gran = std::max<size_t>(gran, 2u << 20);
        if (want % gran) throw MeshError(MESH_ERR_ARG, "kv_granule_bytes must be a multiple of " + std::to_string(gran));
        g->pool.gran = want;
        g->st.kv_granule_bytes = (long long)want;
        g->pool.limit = cfg->kv_pool_bytes > 0 ? cfg->kv_pool_bytes : (long long)(prop.totalGlobalMem / 2);
        // the KV arena: one VA range of limit / granule slots for every instance
        g->arena.nslots = int(std::max<long long>(1, g->pool.limit / (long long)g->pool.gran));
        CU(drv().addr_reserve(&g->arena.base, g->arena.bytes(g->pool.gran), g->pool.gran, 0, 0), "cuMemAddressReserve");
        g->arena.h.assign(size_t(g->arena.nslots), 0);
        g->arena.owner.assign(size_t(g->arena.nslots), -1);
        g->arena.ev.assign(size_t(g->arena.nslots), nullptr);
        // weight sets come from the stream-ordered allocator's pool: keep freed memory
        // in the pool (default threshold 0 hands it back to the driver at every
        // synchronisation, and re-growing it maps memory, which drains the device)
        {
            cudaMemPool_t mp;
            if (cudaDeviceGetDefaultMemPool(&mp, cfg->device) == cudaSuccess) {
                uint64_t thr = UINT64_MAX;
                cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &thr);
            }
        }
        // MESH_GPU_KV_PREALLOC_GB: back that much of the arena now (cuMemCreate +
        // cuMemMap, ~1-4 ms per granule and a device drain per map batch), so the
        // serving path never calls the VMM driver
        if (const char* e = std::getenv("MESH_GPU_KV_PREALLOC_GB")) {
            const long long want = std::min<long long>(g->pool.limit, (long long)(std::atof(e) * double(1LL << 30)));
            const int n = int(std::min<long long>(g->arena.nslots, want / (long long)g->pool.gran));
            if (n > 0) back_slots(g.get(), 0, n);
        }
        CK(cudaHostAlloc((void**)&g->h_desc, sizeof(StepDesc) * RING, cudaHostAllocDefault));
        CK(cudaMalloc((void**)&g->d_desc, sizeof(StepDesc) * RING));
        CK(cudaHostAlloc((void**)&g->h_tok, sizeof(int) * 8 * RING, cudaHostAllocDefault));
        CK(cudaMalloc((void**)&g->d_tok, sizeof(int) * 8 * RING));
        for (int i = 0; i < RING; ++i) CK(cudaEventCreateWithFlags(&g->ring_ev[i], cudaEventDisableTiming));
        g->st.kv_pool_bytes = g->pool.limit;
        g->check = std::getenv("MESH_GPU_CHECK") != nullptr;
        g->poison = std::getenv("MESH_GPU_POISON") != nullptr;
        g->prefill_quota = std::getenv("MESH_PREFILL_QUOTA") != nullptr;
        if (const char* e = std::getenv("MESH_PREFILL_CTAS")) {
            g->prefill_quota = true;
            g->prefill_min_ctas = std::atoi(e);
        }
        if (const char* e = std::getenv("MESH_GPU_SKIP")) g->skip = std::atoi(e);
        if (const char* e = std::getenv("MESH_GPU_L2PF")) g->l2pf = std::atoi(e);
        if (const char* e = std::getenv("MESH_GPU_KV_LANES")) g->kv_lanes = std::atoi(e);
        if (const char* e = std::getenv("MESH_GPU_W_LANES")) g->w_lanes = std::atoi(e);
        if (const char* e = std::getenv("MESH_GPU_WCACHE_GB")) g->wcache_cap = size_t(std::max(0.0, std::atof(e)) * double(1 << 30));
        if (std::getenv("MESH_GPU_WATCHDOG")) {
            CK(cudaHostAlloc((void**)&g->dbg_host, sizeof(int) * 2 * 1024, cudaHostAllocMapped));
            std::memset(g->dbg_host, 0, sizeof(int) * 2 * 1024);
            CK(cudaHostGetDevicePointer((void**)&g->dbg_dev, g->dbg_host, 0));
        }
    });
    if (st != MESH_OK) {
        // keep the message reachable: hand the handle back only on success
        static thread_local std::string last;
        last = g->err;
        std::fprintf(stderr, "mesh_gpu_open: %s\n", last.c_str());
        return st;
    }
    *out = g.release();
    return MESH_OK;
}

void mesh_gpu_close(mesh_gpu* g) {
    if (!g) return;
    cudaSetDevice(g->cfg.device);
    cudaDeviceSynchronize();
    // finish every request history (tokens of retired steps) before the tickets go
    for (auto& [id, t] : g->tickets) {
        try {
            drain_ticket(g, t);
        } catch (...) {
        }
        destroy_ticket(t);
    }
    {  // parked requests keep their KV and history, but forget this handle
        std::lock_guard<std::mutex> lk(swaps().mu);
        for (auto& [rid, e] : swap_store())
            if (e.origin == g) {
                e.origin = nullptr;
                e.pending_tokens = 0;
            }
    }
    try {
        reap_host(g, true);
    } catch (...) {
    }
    for (auto& [id, in] : g->insts) {
        for (PendingFree& pf : in->pending_free) cudaEventDestroy(pf.ev);
        if (in->last_ev) cudaEventDestroy(in->last_ev);
        cudaFree(in->d_block_table);
        cudaFree(in->d_last_tok);
    }
    for (auto& [k, ws] : g->wsets) {
        cudaFreeAsync(ws.wmem, g->side);
        cudaEventDestroy(ws.ready);
    }
    cudaStreamSynchronize(g->side);
    for (auto& b : g->ibufs) {
        cudaFree(b.d_block_table);
        cudaFree(b.d_last_tok);
    }
    for (int sl = 0; sl < g->arena.nslots; ++sl) {
        if (g->arena.ev[size_t(sl)]) cudaEventDestroy(g->arena.ev[size_t(sl)]);
        if (g->arena.h[size_t(sl)]) drv().unmap(g->arena.base + size_t(sl) * g->pool.gran, g->pool.gran);
    }
    if (g->arena.base) drv().addr_free(g->arena.base, g->arena.bytes(g->pool.gran));
    for (auto h : g->pool.all) drv().release(h);
    for (Lane& l : g->lanes) {
        void* lane_ptrs[] = {l.h, l.act, l.attn, l.abuf, l.q, l.ssA, l.ssB, l.apart, l.acnt, l.arg_val,
                             l.arg_idx, l.arg_cnt, l.logits, l.bar, l.p_h, l.p_act, l.p_rs, l.p_q, l.p_attn,
                             l.p_abuf, l.p_logits, l.p_tokens, l.tile_ctr, l.sk_ws, l.sk_cnt, l.claim, l.qkv_done};
        for (void* p : lane_ptrs)
            if (p) cudaFree(p);
        if (l.stream) cudaStreamDestroy(l.stream);
        if (l.quota_ev) cudaEventDestroy(l.quota_ev);
    }
    void* dev_ptrs[] = {g->d_desc, g->d_tok};
    for (void* p : dev_ptrs)
        if (p) cudaFree(p);
    if (g->h_desc) cudaFreeHost(g->h_desc);
    if (g->h_tok) cudaFreeHost(g->h_tok);
    if (g->h_pf_stage) cudaFreeHost(g->h_pf_stage);
    for (int i = 0; i < RING; ++i)
        if (g->ring_ev[i]) cudaEventDestroy(g->ring_ev[i]);
    if (g->side) cudaStreamDestroy(g->side);
    if (g->side_in) cudaStreamDestroy(g->side_in);
    for (cudaEvent_t e : g->timer)
        if (e) cudaEventDestroy(e);
    if (g->lane_join) cudaEventDestroy(g->lane_join);
    delete g;
}

mesh_status mesh_gpu_instance_create(mesh_gpu* g, int64_t instance_id, const mesh_model_shape* sh,
                                     uint64_t weight_seed) {
    if (!g || !sh) return MESH_ERR_ARG;
    return guarded(g, [&] {
        if (g->insts.count(instance_id)) throw MeshError(MESH_ERR_ARG, "duplicate instance id");
        const Shape s = shape_of(*sh);
        static const bool ctrace = std::getenv("MESH_GPU_CREATE_TRACE") != nullptr;
        const auto c0 = std::chrono::steady_clock::now();
        ensure_scratch(g, s);
        const auto c1 = std::chrono::steady_clock::now();
        auto in = std::make_unique<Instance>();
        in->id = instance_id;
        // bind to an empty lane if there is one, else to the lane with the fewest
        // weight bytes (the HBM every step streams)
        size_t best = 0;
        for (size_t i = 1; i < g->lanes.size(); ++i) {
            const Lane &a = g->lanes[i], &b = g->lanes[best];
            if ((a.n_inst == 0) != (b.n_inst == 0) ? a.n_inst == 0 : a.weight_bytes < b.weight_bytes) best = i;
        }
        in->lane = int(best);
        cudaStream_t st = g->lanes[best].stream;
        in->s = s;
        in->seed = weight_seed;
        in->shape_key = shape_key_of(s, weight_seed);
        const size_t L = s.n_layers;
        size_t qkv = size_t(s.qkv_rows()) * s.d * 2, o = size_t(s.d) * s.n_heads * s.dh * 2,
               gu = size_t(2 * s.ff) * s.d * 2, dn = size_t(s.d) * s.ff * 2, lm = size_t(s.vocab) * s.d * 2,
               emb = size_t(s.vocab) * s.d * 2;
        size_t norms = (2 * L + 1) * s.d * 4, rope = size_t(s.max_seq) * (s.dh / 2) * 8;
        const size_t total = weight_set_bytes(s);
        in->block_bytes = (long long)KV_BLOCK_TOKENS * s.kv_bytes_per_token();
        // extents of >= 32 whole blocks: at most one block per extent lost to alignment
        in->ext_slots = int(std::max<long long>(1, (32 * in->block_bytes + (long long)g->pool.gran - 1) /
                                                       (long long)g->pool.gran));
        if (in->ext_slots > g->arena.nslots) throw MeshError(MESH_ERR_CONFIG, "KV block too large for the pool");
        in->bt_stride = (s.max_seq + KV_BLOCK_TOKENS - 1) / KV_BLOCK_TOKENS;
        in->h_block_table.assign(size_t(MAX_SLOTS) * in->bt_stride, 0);
        // per-instance buffers first (recycled, else allocated); on any later failure they go back
        if (!g->ibufs.empty()) {
            in->d_block_table = g->ibufs.back().d_block_table;
            in->d_last_tok = g->ibufs.back().d_last_tok;
            g->ibufs.pop_back();
        } else if (cudaMalloc((void**)&in->d_block_table, sizeof(int) * size_t(MAX_SLOTS) * DEC_BT_MAX) != cudaSuccess ||
                   cudaMalloc((void**)&in->d_last_tok, sizeof(int) * MAX_SLOTS) != cudaSuccess) {
            cudaGetLastError();
            if (in->d_block_table) cudaFree(in->d_block_table);
            throw MeshError(MESH_ERR_NOMEM, "instance buffers: cudaMalloc failed");
        }
        Instance* ip = in.get();
        auto give_back_bufs = [g, ip] {
            g->ibufs.push_back({ip->d_block_table, ip->d_last_tok});
        };
        // weights: share a live or idle set of the same model, else allocate
        // (stream-ordered, so a later free never serialises the device) and
        // initialise. The set's reference is taken only once nothing can fail.
        bool fresh = false;
        auto wit = g->wsets.find(in->shape_key);
        if (wit != g->wsets.end()) {
            in->wmem = wit->second.wmem;
            CK(cudaStreamWaitEvent(st, wit->second.ready, 0));  // initialised on another lane maybe
        } else {
            cudaError_t e = cudaMallocAsync((void**)&in->wmem, total, st);
            if (e != cudaSuccess) {
                cudaGetLastError();
                evict_weights(g, 0);  // make room: drop every idle set, then retry
                e = cudaMallocAsync((void**)&in->wmem, total, st);
            }
            if (e != cudaSuccess) {
                // then the KV arena's backed but unassigned slots: weights come first,
                // the arena re-backs slots on demand (the rare path that unmaps)
                cudaGetLastError();
                release_free_slots(g);
                cudaMemPool_t mp;
                if (cudaDeviceGetDefaultMemPool(&mp, g->cfg.device) == cudaSuccess) cudaMemPoolTrimTo(mp, 0);
                e = cudaMallocAsync((void**)&in->wmem, total, st);
            }
            if (e != cudaSuccess) {
                cudaGetLastError();
                give_back_bufs();
                throw MeshError(MESH_ERR_NOMEM, "weights: cudaMallocAsync of " + std::to_string(total) + " bytes failed");
            }
            fresh = true;
        }
        const auto c2 = std::chrono::steady_clock::now();
        uint8_t* p = in->wmem;
        auto take = [&](size_t n) {
            uint8_t* r = p;
            p += (n + 255) & ~size_t(255);
            return r;
        };
        uint8_t* wq = take(L * qkv);
        uint8_t* wo = take(L * o);
        uint8_t* wgu = take(L * gu);
        uint8_t* wdn = take(L * dn);
        uint8_t* wlm = take(lm);
        uint16_t* wemb = reinterpret_cast<uint16_t*>(take(emb));
        float* ga = reinterpret_cast<float*>(take(L * s.d * 4));
        float* gm = reinterpret_cast<float*>(take(L * s.d * 4));
        float* gf = reinterpret_cast<float*>(take(size_t(s.d) * 4));
        float2* rp = reinterpret_cast<float2*>(take(rope));
        in->w = Weights{wq, wo, wgu, wdn, wlm, wemb, ga, gm, gf, rp, qkv, o, gu, dn};
        if (fresh) {
            const int blocks = g->sms * 8;
            for (int l = 0; l < s.n_layers; ++l) {
                init_tiled<0><<<blocks, 256, 0, st>>>(wq + l * qkv, s, weight_seed, l, s.qkv_rows(), s.d);
                init_tiled<1><<<blocks, 256, 0, st>>>(wo + l * o, s, weight_seed, l, s.d, s.n_heads * s.dh);
                init_tiled<2><<<blocks, 256, 0, st>>>(wgu + l * gu, s, weight_seed, l, 2 * s.ff, s.d);
                init_tiled<3><<<blocks, 256, 0, st>>>(wdn + l * dn, s, weight_seed, l, s.d, s.ff);
                init_gain<<<32, 256, 0, st>>>(ga + size_t(l) * s.d, s.d, weight_seed, T_GATTN, l);
                init_gain<<<32, 256, 0, st>>>(gm + size_t(l) * s.d, s.d, weight_seed, T_GMLP, l);
            }
            init_tiled<4><<<blocks, 256, 0, st>>>(wlm, s, weight_seed, 0, s.vocab, s.d);
            init_emb<<<blocks, 256, 0, st>>>(wemb, s, weight_seed);
            init_gain<<<32, 256, 0, st>>>(gf, s.d, weight_seed, T_GFINAL, 0);
            CK(cudaGetLastError());
            // rotate-half RoPE table, computed in double on the host (the oracle uses the same formula)
            std::vector<float2> tab(size_t(s.max_seq) * (s.dh / 2));
            for (int pos = 0; pos < s.max_seq; ++pos)
                for (int i = 0; i < s.dh / 2; ++i) {
                    double inv = std::pow(double(s.rope_theta), -2.0 * i / double(s.dh));
                    double ang = double(pos) * inv;
                    tab[size_t(pos) * (s.dh / 2) + i] = make_float2(float(std::cos(ang)), float(std::sin(ang)));
                }
            CK(cudaMemcpyAsync(rp, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice, st));
            // the pageable table copy returns once staged; the init kernels and every
            // later step of the instance are ordered on the lane stream: no host wait
            mesh_gpu::WeightSet ws{in->wmem, total, 0, nullptr, ++g->wtick};
            CK(cudaEventCreateWithFlags(&ws.ready, cudaEventDisableTiming));
            CK(cudaEventRecord(ws.ready, st));
            g->wsets.emplace(in->shape_key, ws);  // idle (refs 0) until the create completes
        }
        CK(cudaMemsetAsync(in->d_block_table, 0, sizeof(int) * in->h_block_table.size(), st));
        CK(cudaMemsetAsync(in->d_last_tok, 0, sizeof(int) * MAX_SLOTS, st));
        if (cudaEventCreateWithFlags(&in->last_ev, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            give_back_bufs();
            throw MeshError(MESH_ERR_CUDA, "instance event creation failed");
        }
        CK(cudaEventRecord(in->last_ev, st));
        g->wsets.at(in->shape_key).refs++;
        if (!fresh) g->st.weight_cache_hits++;
        for (int i = MAX_SLOTS - 1; i >= 0; --i) in->free_slots.push_back(i);
        in->weight_bytes = double(total);
        g->lanes[best].weight_bytes += in->weight_bytes;
        g->lanes[best].n_inst++;
        g->insts.emplace(instance_id, std::move(in));
        rebalance_lanes(g);
        if (ctrace) {
            auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
            const auto c3 = std::chrono::steady_clock::now();
            fprintf(stderr, "instance_create %lld: scratch %.2f ms, weights alloc %.2f ms (%s), rest %.2f ms\n",
                    (long long)instance_id, ms(c0, c1), ms(c1, c2), fresh ? "fresh" : "shared", ms(c2, c3));
        }
    }, &g->st.host_ms_create);
}

mesh_status mesh_gpu_reserve(mesh_gpu* g, const mesh_model_shape* shapes, int32_t n) {
    if (!g || (n > 0 && !shapes) || n < 0) return MESH_ERR_ARG;
    return guarded(g, [&] {
        size_t wbytes = 0;
        for (int i = 0; i < n; ++i) {
            const Shape s = shape_of(shapes[i]);
            ensure_scratch(g, s);
            wbytes += (weight_set_bytes(s) + 255) & ~size_t(255);
        }
        if (wbytes == 0) return;
        // grow the allocator pool now (freed memory stays in it: release threshold max)
        void* p = nullptr;
        if (cudaMallocAsync(&p, wbytes, g->side) != cudaSuccess) {
            cudaGetLastError();
            return;  // best effort: creates allocate on demand
        }
        CK(cudaFreeAsync(p, g->side));
        CK(cudaStreamSynchronize(g->side));
    }, &g->st.host_ms_create);
}

mesh_status mesh_gpu_instance_destroy(mesh_gpu* g, int64_t instance_id) {
    if (!g) return MESH_ERR_ARG;
    return guarded(g, [&] {
        Instance& in = inst_of(g, instance_id);
        // wait for this instance's own lane work only (co-located instances keep running),
        // retire its tickets (histories of parked requests complete), and wait for the
        // swap / migration copies still reading its blocks
        CK(cudaEventSynchronize(in.last_ev));
        drain_instance(g, instance_id);
        reap_blocks(in, true);
        cudaEventDestroy(in.last_ev);
        lane_of(g, in).weight_bytes -= in.weight_bytes;
        lane_of(g, in).n_inst--;
        // release the weight set (kept while idle, for a reload) and recycle the
        // per-instance buffers: no cudaFree, which would serialise the device
        while (!in.ext.empty()) release_extent(g, in, nullptr);  // its work finished above
        g->ibufs.push_back({in.d_block_table, in.d_last_tok});
        auto wit = g->wsets.find(in.shape_key);
        if (wit != g->wsets.end()) {
            wit->second.refs--;
            wit->second.tick = ++g->wtick;
        }
        evict_weights(g, g->wcache_cap);
        std::vector<int64_t> dead;
        for (auto& [tid, t] : g->tickets)
            if (t.instance == instance_id) dead.push_back(tid);
        for (int64_t tid : dead) {
            Ticket& t = g->tickets[tid];
            g->ring_used[t.ring] = false;
            destroy_ticket(t);
            g->tickets.erase(tid);
        }
        g->insts.erase(instance_id);
        rebalance_lanes(g);
    }, &g->st.host_ms_destroy);
}

mesh_status mesh_gpu_kv_resize(mesh_gpu* g, int64_t instance_id, int64_t from_bytes, int64_t to_bytes) {
    if (!g || from_bytes < 0 || to_bytes < 0) return MESH_ERR_ARG;
    return guarded(g, [&] {
        Instance& in = inst_of(g, instance_id);
        if (from_bytes != in.target)
            throw MeshError(MESH_ERR_ARG, "kv_resize: from (" + std::to_string(from_bytes) +
                                              ") does not match current target (" + std::to_string(in.target) + ")");
        resize_kv(g, in, to_bytes);
        g->st.kv_mapped_bytes = g->pool.mapped;
    }, &g->st.host_ms_kv_resize);
}

// Debug (MESH_GPU_CHECK): block-table consistency and a NaN/Inf scan of a request's KV.
std::string debug_request_state(mesh_gpu* g, Instance& in, int64_t rid) {
    std::string m;
    auto it = in.reqs.find(rid);
    if (it == in.reqs.end()) return " [request not resident]";
    const ReqState& r = it->second;
    m += " | cap_blocks " + std::to_string(in.cap_blocks) + " live " + std::to_string(in.live_blocks) + " free " +
         std::to_string(in.free_blocks.size()) + " blocks:";
    std::vector<int> dev(size_t(in.bt_stride));
    CK(cudaMemcpy(dev.data(), in.d_block_table + size_t(r.slot) * in.bt_stride, sizeof(int) * in.bt_stride,
                  cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < r.blocks.size(); ++i) {
        m += " " + std::to_string(r.blocks[i]);
        if (dev[i] != phys_of(in, r.blocks[i])) m += "(dev " + std::to_string(dev[i]) + ")";
        if (in.h_block_table[size_t(r.slot) * in.bt_stride + i] != phys_of(in, r.blocks[i])) m += "(mirror!)";
        if (in.free_blocks.count(r.blocks[i])) m += "(FREE!)";
        for (auto& [o, os] : in.reqs)
            if (o != rid && std::find(os.blocks.begin(), os.blocks.end(), r.blocks[i]) != os.blocks.end())
                m += "(shared with " + std::to_string(o) + ")";
    }
    // scan K/V of every resident position for non-finite values
    std::vector<uint16_t> blk(size_t(in.block_bytes) / 2);
    int bad_pos = -1, bad_layer = -1, nbad = 0;
    for (int p = 0; p < r.ctx; ++p) {
        if (p % KV_BLOCK_TOKENS == 0)
            CK(cudaMemcpy(blk.data(), arena_ptr(g) + size_t(phys_of(in, r.blocks[p / KV_BLOCK_TOKENS])) * in.block_bytes,
                          in.block_bytes, cudaMemcpyDeviceToHost));
        for (int l = 0; l < in.s.n_layers; ++l)
            for (int kv = 0; kv < 2; ++kv)
                for (int h = 0; h < in.s.n_kv; ++h) {
                    const uint16_t* row = blk.data() + kv_offset(in.s, l, kv, h, p % KV_BLOCK_TOKENS) / 2;
                    for (int e = 0; e < in.s.dh; ++e)
                        if ((row[e] & 0x7f80) == 0x7f80) {
                            if (bad_pos < 0) {
                                bad_pos = p;
                                bad_layer = l;
                            }
                            ++nbad;
                        }
                }
    }
    m += " | non-finite KV values " + std::to_string(nbad);
    if (bad_pos >= 0) m += " first at pos " + std::to_string(bad_pos) + " layer " + std::to_string(bad_layer);
    return m;
}

mesh_status mesh_gpu_step(mesh_gpu* g, int64_t instance_id, const mesh_step_plan* plan, int64_t* ticket) {
    if (!g || !plan || !ticket) return MESH_ERR_ARG;
    return guarded(g, [&] {
        Instance& in = inst_of(g, instance_id);
        reap_blocks(in, false);  // blocks of swapped-out / migrated requests whose copy finished
        if (!g->host_free.empty()) reap_host(g, false);
        Ticket t;
        t.instance = instance_id;
        t.prefill = plan->is_prefill != 0;
        t.logits = g->capture_logits;
        t.vocab = in.s.vocab;
        t.ring = take_ring(g);
        t.lane = in.lane;
        cudaStream_t st = stream_of(g, in);
        CK(cudaEventCreate(&t.start));
        CK(cudaEventCreate(&t.kend));
        CK(cudaEventCreate(&t.end));
        try {
            if (t.prefill) {
                t.reqs.push_back(plan->prefill_request);
                launch_prefill_step(g, in, *plan, t);
            } else {
                if (plan->n_decode < 1 || plan->n_decode > DEC_MAXB || !plan->decode_requests)
                    throw MeshError(MESH_ERR_ARG, "decode batch must hold 1..8 requests");
                t.reqs.assign(plan->decode_requests, plan->decode_requests + plan->n_decode);
                launch_decode_step(g, in, plan->decode_requests, plan->n_decode, t);
            }
        } catch (...) {
            g->ring_used[t.ring] = false;
            destroy_ticket(t);
            throw;
        }
        CK(cudaMemcpyAsync(g->h_tok + t.ring * 8, g->d_tok + t.ring * 8, sizeof(int) * 8, cudaMemcpyDeviceToHost,
                           st));
        g->st.d2h_bytes += (long long)sizeof(int) * 8;
        CK(cudaEventRecord(t.end, st));
        CK(cudaEventRecord(g->ring_ev[t.ring], st));
        CK(cudaEventRecord(in.last_ev, st));
        g->st.steps++;
        if (g->check) {  // debug (MESH_GPU_CHECK=1): validate every step synchronously
            CK(cudaStreamSynchronize(st));
            const int n = t.prefill ? 1 : plan->n_decode;
            for (int i = 0; i < n; ++i) {
                const int tok = g->h_tok[t.ring * 8 + i];
                if (tok < 0 || tok >= in.s.vocab) {
                    std::string msg = std::string(t.prefill ? "prefill" : "decode") + " step " +
                                      std::to_string(g->st.steps) + " of instance " + std::to_string(instance_id) +
                                      " (d=" + std::to_string(in.s.d) + ") produced token " + std::to_string(tok) +
                                      " for column " + std::to_string(i) + "; requests:";
                    for (int64_t r : t.reqs) {
                        const ReqState& rs = in.reqs[r];
                        msg += " " + std::to_string(r) + "@slot" + std::to_string(rs.slot) + "/ctx" +
                               std::to_string(rs.ctx) + "/blocks" + std::to_string(rs.blocks.size());
                    }
                    if (t.prefill) msg += " prefill_len " + std::to_string(plan->prefill_len);
                    msg += debug_request_state(g, in, t.reqs[t.prefill ? 0 : i]);
                    throw MeshError(MESH_ERR_RUNTIME, msg);
                }
            }
        }
        *ticket = g->next_ticket++;
        static FILE* slog = std::getenv("MESH_GPU_STEP_LOG") ? std::fopen(std::getenv("MESH_GPU_STEP_LOG"), "w") : nullptr;
        if (slog)  // diagnostics: host time, instance, model (weight set), lane, decode batch (0: prefill)
            std::fprintf(slog, "%.1f %lld %llu %d %d\n",
                         std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count(),
                         (long long)instance_id, (unsigned long long)(in.shape_key % 100000), in.lane,
                         t.prefill ? 0 : plan->n_decode);
        g->tickets.emplace(*ticket, std::move(t));
    }, &g->st.host_ms_step);
}

mesh_status mesh_gpu_step_wait(mesh_gpu* g, int64_t ticket, int32_t* tokens_out, int32_t cap, int32_t* n_out,
                               float* logits_out, int64_t logits_cap) {
    if (!g) return MESH_ERR_ARG;
    return guarded(g, [&] {
        auto it = g->tickets.find(ticket);
        if (it == g->tickets.end()) throw MeshError(MESH_ERR_ARG, "unknown or already-waited ticket");
        Ticket& t = it->second;
        drain_instance(g, t.instance, ticket);
        int n = int(t.toks.size());
        for (int i = 0; i < n && tokens_out && i < cap; ++i) tokens_out[i] = t.toks[i];
        if (n_out) *n_out = n;
        if (logits_out) {
            if (!t.logits) throw MeshError(MESH_ERR_ARG, "logits capture was off for this step");
            // valid only for the most recent step (scratch is reused)
            size_t cnt = t.prefill ? size_t(t.vocab) : t.reqs.size() * size_t(t.vocab);
            if ((int64_t)cnt > logits_cap) throw MeshError(MESH_ERR_ARG, "logits buffer too small");
            const Lane& ln = g->lanes[size_t(t.lane)];
            CK(cudaMemcpy(logits_out, t.prefill ? ln.p_logits : ln.logits, cnt * sizeof(float),
                          cudaMemcpyDeviceToHost));
        }
        destroy_ticket(t);
        g->tickets.erase(it);
    });
}

mesh_status mesh_gpu_step_done(mesh_gpu* g, int64_t ticket, int32_t* done) {
    if (!g || !done) return MESH_ERR_ARG;
    return guarded(g, [&] {
        auto it = g->tickets.find(ticket);
        if (it == g->tickets.end()) throw MeshError(MESH_ERR_ARG, "unknown or already-waited ticket");
        const cudaError_t e = cudaEventQuery(it->second.end);
        if (e != cudaSuccess && e != cudaErrorNotReady) CK(e);
        *done = e == cudaSuccess ? 1 : 0;
    });
}

mesh_status mesh_gpu_set_capture_logits(mesh_gpu* g, int32_t enable) {
    if (!g) return MESH_ERR_ARG;
    g->capture_logits = enable != 0;
    return MESH_OK;
}

mesh_status mesh_gpu_request_free(mesh_gpu* g, int64_t instance_id, int64_t request_id) {
    if (!g) return MESH_ERR_ARG;
    return guarded(g, [&] {
        Instance& in = inst_of(g, instance_id);
        // no host sync: later kernels that reuse the blocks are stream-ordered after
        // every step that read them
        free_request(in, request_id);
    });
}

mesh_status mesh_gpu_swap_out(mesh_gpu* g, int64_t instance_id, int64_t request_id) {
    if (!g) return MESH_ERR_ARG;
    return guarded(g, [&] {
        Instance& in = inst_of(g, instance_id);
        auto it = in.reqs.find(request_id);
        if (it == in.reqs.end()) throw MeshError(MESH_ERR_ARG, "swap_out: request not resident");
        reap_host(g, false);
        ReqState& r = it->second;
        SwapEntry e;
        e.shape_key = in.shape_key;
        e.tokens = r.tokens;  // completed by the request's in-flight steps as they retire (drain_ticket)
        e.pending_tokens = r.pending_tokens;
        e.origin = g;
        e.origin_inst = instance_id;
        PendingFree pf;
        if (r.ctx > 0) {
            e.ctx = r.ctx;
            e.block_bytes = in.block_bytes;
            e.bytes = r.blocks.size() * size_t(in.block_bytes);
            const auto [ci, off] = host_pool().take(e.bytes);
            e.chunk = ci;
            e.off = off;
            // gather after every queued step that wrote this request's KV (event-ordered, no host wait)
            cudaEvent_t ready = record_new_event(stream_of(g, in));
            CK(cudaStreamWaitEvent(g->side, ready, 0));
            cudaEventDestroy(ready);
            const std::vector<int> pb = phys_list(in, r.blocks);
            launch_blocks_copy(host_pool().ptr(ci, off), arena_ptr(g), in.block_bytes, pb.data(), nullptr,
                               int(pb.size()), g->side);
            e.done = record_new_event(g->side);
            pf.ev = record_new_event(g->side);
            pf.blocks = r.blocks;
            g->st.swap_out_bytes += (long long)e.bytes;
        }
        SwapEntry old;
        bool had_old = false;
        {
            std::lock_guard<std::mutex> lk(swaps().mu);
            auto o = swap_store().find(request_id);
            if (o != swap_store().end()) {
                old = std::move(o->second);
                swap_store().erase(o);
                had_old = true;
            }
            swap_store().emplace(request_id, std::move(e));
        }
        if (had_old) drop_parked(g, old);
        // the slot is free now; the blocks stay live until the gather read them
        in.free_slots.push_back(r.slot);
        if (pf.ev) in.pending_free.push_back(std::move(pf));
        in.reqs.erase(it);
    });
}

mesh_status mesh_gpu_swap_in(mesh_gpu* g, int64_t instance_id, int64_t request_id) {
    if (!g) return MESH_ERR_ARG;
    return guarded(g, [&] {
        Instance& in = inst_of(g, instance_id);
        if (in.reqs.count(request_id)) throw MeshError(MESH_ERR_ARG, "swap_in: request already resident");
        {
            std::lock_guard<std::mutex> lk(swaps().mu);
            auto it = swap_store().find(request_id);
            if (it == swap_store().end()) throw MeshError(MESH_ERR_ARG, "swap_in: request is not parked");
            if (it->second.chunk < 0) throw MeshError(MESH_ERR_ARG, "swap_in: request has no parked KV");
            if (it->second.shape_key != in.shape_key)
                throw MeshError(MESH_ERR_ARG, "swap_in: parked KV belongs to another model");
        }
        reap_host(g, false);
        SwapEntry e = take_parked(request_id);
        ReqState& r = req_slot(in, request_id);
        try {
            restore_parked(g, in, r, e, g->side_in);
        } catch (...) {
            free_request(in, request_id);
            drop_parked(g, e);
            throw;
        }
    });
}

mesh_status mesh_gpu_swap_state(mesh_gpu* g, int64_t request_id, int32_t* state) {
    if (!g || !state) return MESH_ERR_ARG;
    return guarded(g, [&] {
        std::lock_guard<std::mutex> lk(swaps().mu);
        auto it = swap_store().find(request_id);
        if (it == swap_store().end()) {
            *state = MESH_SWAP_NONE;
            return;
        }
        if (it->second.chunk < 0) {
            *state = MESH_SWAP_HISTORY;
            return;
        }
        const cudaError_t e = cudaEventQuery(it->second.done);
        if (e != cudaSuccess && e != cudaErrorNotReady) CK(e);
        *state = e == cudaSuccess ? MESH_SWAP_PARKED : MESH_SWAP_COPYING;
    });
}

mesh_status mesh_gpu_migrate(mesh_gpu* src, int64_t src_instance, mesh_gpu* dst, int64_t dst_instance,
                             int64_t request_id) {
    if (!src || !dst) return MESH_ERR_ARG;
    return guarded(dst, [&] {
        CK(cudaSetDevice(src->cfg.device));
        Instance& si = inst_of(src, src_instance);
        auto it = si.reqs.find(request_id);
        if (it == si.reqs.end()) throw MeshError(MESH_ERR_ARG, "migrate: request not resident at source");
        Instance& di = inst_of(dst, dst_instance);
        if (di.shape_key != si.shape_key) throw MeshError(MESH_ERR_ARG, "migrate: instances serve different models");
        if (di.reqs.count(request_id)) throw MeshError(MESH_ERR_ARG, "migrate: request already at destination");
        if (src->cfg.device != dst->cfg.device &&
            std::find(src->peers.begin(), src->peers.end(), dst->cfg.device) == src->peers.end())
            throw MeshError(MESH_ERR_CUDA, "migrate: no peer access from device " + std::to_string(dst->cfg.device) +
                                               " to device " + std::to_string(src->cfg.device));
        // the token history travels with the request: retire the source instance's
        // in-flight steps (the control plane migrates requests of instances that
        // are not mid-step, so this normally waits for nothing)
        flush_request(src, src_instance, request_id);
        ReqState& sr = it->second;
        cudaEvent_t ready = record_new_event(stream_of(src, si));  // after every step that wrote the KV
        CK(cudaSetDevice(dst->cfg.device));
        if (di.free_slots.empty()) {
            cudaEventDestroy(ready);
            throw MeshError(MESH_ERR_NOMEM, "migrate: destination request table full");
        }
        // destination blocks first: on failure nothing has changed on either side
        std::vector<int> nb;
        try {
            while (nb.size() < sr.blocks.size()) nb.push_back(alloc_block(dst, di));
        } catch (...) {
            for (int b : nb) {
                if (b < di.cap_blocks) di.free_blocks.insert(b);
                di.live_blocks--;
            }
            cudaEventDestroy(ready);
            throw;
        }
        ReqState& dr = req_slot(di, request_id);
        cudaStream_t dst_st = stream_of(dst, di);
        dr.tokens = sr.tokens;
        dr.ctx = sr.ctx;
        dr.blocks = std::move(nb);
        for (size_t i = 0; i < dr.blocks.size(); ++i) write_bt_entry(di, dr.slot, int(i), dr.blocks[i]);
        CK(cudaStreamWaitEvent(dst_st, ready, 0));
        cudaEventDestroy(ready);
        // one copy kernel on the destination GPU: P2P loads of the source blocks over NVLink
        const std::vector<int> ps = phys_list(si, sr.blocks), pd = phys_list(di, dr.blocks);
        launch_blocks_copy(arena_ptr(dst), arena_ptr(src), di.block_bytes, ps.data(), pd.data(), int(ps.size()), dst_st);
        const int last = sr.tokens.empty() ? 0 : sr.tokens.back();
        set_int<<<1, 1, 0, dst_st>>>(di.d_last_tok + dr.slot, last);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(di.d_block_table + size_t(dr.slot) * di.bt_stride,
                           di.h_block_table.data() + size_t(dr.slot) * di.bt_stride, sizeof(int) * di.bt_stride,
                           cudaMemcpyHostToDevice, dst_st));
        PendingFree pf;
        pf.ev = record_new_event(dst_st);  // the source blocks are free once the copy read them
        CK(cudaEventRecord(di.last_ev, dst_st));
        dst->st.migrate_bytes += (long long)sr.blocks.size() * di.block_bytes;
        CK(cudaSetDevice(src->cfg.device));
        pf.blocks = std::move(sr.blocks);
        si.free_slots.push_back(sr.slot);
        si.pending_free.push_back(std::move(pf));
        si.reqs.erase(it);
        CK(cudaSetDevice(dst->cfg.device));
    });
}

mesh_status mesh_gpu_request_info(mesh_gpu* g, int64_t instance_id, int64_t request_id, int32_t* ctx_len,
                                  int32_t* blocks, int32_t* block_ids, int32_t cap) {
    if (!g) return MESH_ERR_ARG;
    return guarded(g, [&] {
        Instance& in = inst_of(g, instance_id);
        auto it = in.reqs.find(request_id);
        if (it == in.reqs.end()) throw MeshError(MESH_ERR_ARG, "request not resident");
        if (ctx_len) *ctx_len = it->second.ctx;
        if (blocks) *blocks = int(it->second.blocks.size());
        if (block_ids)
            for (int i = 0; i < std::min<int>(cap, int(it->second.blocks.size())); ++i) block_ids[i] = it->second.blocks[i];
    });
}

mesh_status mesh_gpu_request_tokens(mesh_gpu* g, int64_t instance_id, int64_t request_id, int32_t* tokens, int32_t cap,
                                    int32_t* n_out) {
    if (!g) return MESH_ERR_ARG;
    return guarded(g, [&] {
        Instance& in = inst_of(g, instance_id);
        flush_request(g, instance_id, request_id);
        auto it = in.reqs.find(request_id);
        std::vector<int> parked;
        const std::vector<int>* src = nullptr;
        if (it != in.reqs.end()) {
            src = &it->second.tokens;
        } else {
            mesh_gpu* origin = nullptr;
            int64_t oinst = -1;
            {
                std::lock_guard<std::mutex> lk(swaps().mu);
                auto sit = swap_store().find(request_id);
                if (sit == swap_store().end()) throw MeshError(MESH_ERR_ARG, "unknown request");
                if (sit->second.pending_tokens > 0) {
                    origin = sit->second.origin;
                    oinst = sit->second.origin_inst;
                }
            }
            if (origin) drain_instance(origin, oinst);
            std::lock_guard<std::mutex> lk(swaps().mu);
            parked = swap_store().at(request_id).tokens;
            src = &parked;
        }
        int n = int(src->size());
        for (int i = 0; i < std::min(n, cap); ++i) tokens[i] = (*src)[i];
        if (n_out) *n_out = n;
    });
}

mesh_status mesh_gpu_instance_lane(mesh_gpu* g, int64_t instance_id, int32_t* lane, int32_t* ctas) {
    if (!g) return MESH_ERR_ARG;
    return guarded(g, [&] {
        Instance& in = inst_of(g, instance_id);
        if (lane) *lane = in.lane;
        if (ctas) *ctas = lane_of(g, in).ctas;
    });
}

mesh_status mesh_gpu_instance_kv(mesh_gpu* g, int64_t instance_id, int64_t* target_bytes, int64_t* mapped_bytes,
                                 int32_t* capacity_blocks, int32_t* live_blocks) {
    if (!g) return MESH_ERR_ARG;
    return guarded(g, [&] {
        Instance& in = inst_of(g, instance_id);
        if (target_bytes) *target_bytes = in.target;
        if (mapped_bytes) {
            int64_t n = 0;
            for (const Instance::Extent& e : in.ext) n += e.k;
            *mapped_bytes = n * (int64_t)g->pool.gran;
        }
        if (capacity_blocks) *capacity_blocks = in.cap_blocks;
        if (live_blocks) *live_blocks = in.live_blocks;
    });
}

mesh_status mesh_gpu_read_weight(mesh_gpu* g, int64_t instance_id, int32_t tensor, int32_t layer, int32_t row,
                                 float* out, int32_t n) {
    if (!g || !out) return MESH_ERR_ARG;
    return guarded(g, [&] {
        Instance& in = inst_of(g, instance_id);
        const Shape& s = in.s;
        // locate the physical row that holds logical (tensor, row)
        const uint8_t* W = nullptr;
        int K = 0, prow = -1;
        if (tensor == T_WQ || tensor == T_WK || tensor == T_WV) {
            W = in.w.qkv + size_t(layer) * in.w.qkv_layer;
            K = s.d;
            for (int p = 0; p < s.qkv_rows() && prow < 0; ++p) {
                QkvRow q = qkv_row(s, p);
                int sec = tensor == T_WQ ? 0 : (tensor == T_WK ? 1 : 2);
                if (q.section == sec && q.head * s.dh + q.dim == row) prow = p;
            }
        } else if (tensor == T_WO) {
            W = in.w.o + size_t(layer) * in.w.o_layer;
            K = s.n_heads * s.dh;
            prow = row;
        } else if (tensor == T_WGATE || tensor == T_WUP) {
            W = in.w.gu + size_t(layer) * in.w.gu_layer;
            K = s.d;
            prow = (row / 8) * 16 + (row % 8) + (tensor == T_WUP ? 8 : 0);
        } else if (tensor == T_WDOWN) {
            W = in.w.down + size_t(layer) * in.w.down_layer;
            K = s.ff;
            prow = row;
        } else if (tensor == T_LM) {
            W = in.w.lm;
            K = s.d;
            prow = row;
        } else {
            throw MeshError(MESH_ERR_ARG, "read_weight: unsupported tensor");
        }
        if (prow < 0 || n < K) throw MeshError(MESH_ERR_ARG, "read_weight: bad row or buffer");
        float* d = nullptr;
        CK(cudaMalloc((void**)&d, sizeof(float) * K));
        cudaStream_t st = stream_of(g, in);
        read_tiled_row<<<1, 256, 0, st>>>(W, K, prow, d);
        CK(cudaMemcpyAsync(out, d, sizeof(float) * K, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        CK(cudaFree(d));
    });
}

mesh_status mesh_gpu_stats_get(mesh_gpu* g, mesh_gpu_stats* out) {
    if (!g || !out) return MESH_ERR_ARG;
    g->st.kv_mapped_bytes = g->pool.mapped;
    *out = g->st;
    return MESH_OK;
}

mesh_status mesh_gpu_sync(mesh_gpu* g) {
    if (!g) return MESH_ERR_ARG;
    return guarded(g, [&] { sync_all(g); });
}

mesh_status mesh_gpu_timer_mark(mesh_gpu* g, int32_t slot) {
    if (!g || slot < 0 || slot >= 8) return MESH_ERR_ARG;
    return guarded(g, [&] {
        // a mark orders every lane: lane 0 joins the others, records, and they
        // wait on the mark, so an interval between two marks covers all lanes
        if (!g->timer[slot]) CK(cudaEventCreate(&g->timer[slot]));
        cudaStream_t s0 = g->lanes[0].stream;
        for (size_t i = 1; i < g->lanes.size(); ++i) {
            CK(cudaEventRecord(g->lane_join, g->lanes[i].stream));
            CK(cudaStreamWaitEvent(s0, g->lane_join, 0));
        }
        CK(cudaEventRecord(g->timer[slot], s0));
        for (size_t i = 1; i < g->lanes.size(); ++i) CK(cudaStreamWaitEvent(g->lanes[i].stream, g->timer[slot], 0));
    });
}

mesh_status mesh_gpu_timer_elapsed(mesh_gpu* g, int32_t a, int32_t b, double* ms) {
    if (!g || !ms || a < 0 || a >= 8 || b < 0 || b >= 8) return MESH_ERR_ARG;
    return guarded(g, [&] {
        if (!g->timer[a] || !g->timer[b]) throw MeshError(MESH_ERR_ARG, "timer slot not marked");
        CK(cudaEventSynchronize(g->timer[b]));
        float f = 0.f;
        CK(cudaEventElapsedTime(&f, g->timer[a], g->timer[b]));
        *ms = f;
    });
}

mesh_status mesh_gpu_bench_decode(mesh_gpu* g, int64_t instance_id, const mesh_step_plan* plan, int32_t iters,
                                  double* ms_per_step) {
    if (!g || !plan || !ms_per_step || iters < 1) return MESH_ERR_ARG;
    return guarded(g, [&] {
        Instance& in = inst_of(g, instance_id);
        if (plan->n_decode < 1 || plan->n_decode > DEC_MAXB) throw MeshError(MESH_ERR_ARG, "bad batch");
        // fixed positions: every iteration re-decodes the same positions (no state advance)
        StepDesc hd{};
        hd.B = plan->n_decode;
        for (int i = 0; i < hd.B; ++i) {
            ReqState& r = in.reqs.at(plan->decode_requests[i]);
            if (r.ctx < 1) throw MeshError(MESH_ERR_ARG, "bench_decode needs prefilled requests");
            hd.slot[i] = r.slot;
            hd.pos[i] = r.ctx - 1;  // rewrite the last resident position: no new blocks needed
        }
        StepDesc* dd = nullptr;
        int* scratch_tok = nullptr;
        CK(cudaMalloc((void**)&dd, sizeof(StepDesc)));
        CK(cudaMalloc((void**)&scratch_tok, sizeof(int) * MAX_SLOTS));
        CK(cudaMemcpy(dd, &hd, sizeof(StepDesc), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(scratch_tok, in.d_last_tok, sizeof(int) * MAX_SLOTS, cudaMemcpyDeviceToDevice));
        int ring = take_ring(g);
        DecodeArgs a = decode_args(g, in, dd, ring);
        a.last_tok = scratch_tok;
        a.logits = nullptr;
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        unsigned long long* tr = nullptr;
        const char* trace_path = std::getenv("MESH_GPU_TRACE");
        if (trace_path) {
            CK(cudaMalloc((void**)&tr, sizeof(unsigned long long) * 4096));
            CK(cudaMemset(tr, 0, sizeof(unsigned long long) * 4096));
        }
        CK(launch_decode(a, grid_of(g, in), stream_of(g, in)));  // warm
        if (tr) {
            DecodeArgs at = a;
            at.trace = tr;
            unsigned long long* arr = nullptr;
            const size_t narr = size_t(256) * grid_of(g, in);
            CK(cudaMalloc((void**)&arr, sizeof(unsigned long long) * narr));
            CK(cudaMemset(arr, 0, sizeof(unsigned long long) * narr));
            at.arrive = arr;
            CK(launch_decode(at, grid_of(g, in), stream_of(g, in)));
            CK(cudaStreamSynchronize(stream_of(g, in)));
            {
                std::vector<unsigned long long> ha(narr);
                CK(cudaMemcpy(ha.data(), arr, sizeof(unsigned long long) * narr, cudaMemcpyDeviceToHost));
                std::string ap = std::string(trace_path) + ".arrive";
                FILE* fa = std::fopen(ap.c_str(), "w");
                if (fa) {
                    for (size_t i = 0; i < narr; ++i) std::fprintf(fa, "%llu%c", ha[i], (i + 1) % grid_of(g, in) ? ' ' : '\n');
                    std::fclose(fa);
                }
                CK(cudaFree(arr));
            }
            std::vector<unsigned long long> h(4096);
            CK(cudaMemcpy(h.data(), tr, sizeof(unsigned long long) * 4096, cudaMemcpyDeviceToHost));
            FILE* f = std::fopen(trace_path, "w");
            if (f) {
                for (size_t i = 0; i < h.size(); ++i)
                    if (h[i]) std::fprintf(f, "%llu %llu\n", h[i] >> 4, (h[i] & 15) + (i >= 2048 ? 100 : 0));
                std::fclose(f);
            }
            CK(cudaFree(tr));
        }
        CK(cudaEventRecord(e0, stream_of(g, in)));
        for (int i = 0; i < iters; ++i) CK(launch_decode(a, grid_of(g, in), stream_of(g, in)));
        CK(cudaEventRecord(e1, stream_of(g, in)));
        if (g->dbg_host) {
            for (int spin = 0; cudaEventQuery(e1) == cudaErrorNotReady; ++spin) {
                usleep(1000);
                if (spin == 20000) {
                    std::fprintf(stderr, "decode watchdog: step not finished after 20 s; per-CTA (barriers, stage):\n");
                    for (int i = 0; i < grid_of(g, in); ++i)
                        std::fprintf(stderr, "%d:(%d,%d) ", i, g->dbg_host[2 * i], g->dbg_host[2 * i + 1]);
                    std::fprintf(stderr, "\n");
                    std::fflush(stderr);
                    std::abort();
                }
            }
        }
        CK(cudaEventSynchronize(e1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        *ms_per_step = double(ms) / iters;
        g->ring_used[ring] = false;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        CK(cudaFree(dd));
        CK(cudaFree(scratch_tok));
    });
}

}  // extern "C"
