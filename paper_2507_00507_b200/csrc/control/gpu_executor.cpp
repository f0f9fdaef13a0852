#include <cstdlib>
#include "gpu_executor.hpp"

#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cstring>

#include "../../../include/mesh_gpu.h"

namespace mesh {

const LlamaShape& llama_shape_for(const std::string& sc) {
    static const std::map<std::string, LlamaShape> shapes = {
        {"1b", {22, 2048, 32, 4, 64, 5632, 32000, 0, 2048, 10000.f, 1e-5f}},     // TinyLlama-1.1B
        {"3b", {28, 3072, 24, 8, 128, 8192, 128256, 1, 4096, 500000.f, 1e-5f}},  // Llama-3.2-3B
        {"7b", {32, 4096, 32, 32, 128, 11008, 32000, 0, 4096, 10000.f, 1e-5f}},  // Llama-2-7B
        {"13b", {40, 5120, 40, 40, 128, 13824, 32000, 0, 4096, 10000.f, 1e-5f}}, // Llama-2-13B
        {"tiny", {2, 256, 4, 2, 64, 512, 512, 0, 512, 10000.f, 1e-5f}},          // tests
    };
    auto it = shapes.find(sc);
    if (it == shapes.end()) throw ConfigError("no Llama shape for size class `" + sc + "` on the GPU data plane");
    return it->second;
}

struct GpuExecutor::Api {
    decltype(&mesh_gpu_open) open;
    decltype(&mesh_gpu_close) close;
    decltype(&mesh_gpu_last_error) last_error;
    decltype(&mesh_gpu_instance_create) instance_create;
    decltype(&mesh_gpu_instance_destroy) instance_destroy;
    decltype(&mesh_gpu_kv_resize) kv_resize;
    decltype(&mesh_gpu_step) step;
    decltype(&mesh_gpu_step_wait) step_wait;
    decltype(&mesh_gpu_request_free) request_free;
    decltype(&mesh_gpu_swap_out) swap_out;
    decltype(&mesh_gpu_stats_get) stats_get;
    decltype(&mesh_gpu_step_done) step_done;
    decltype(&mesh_gpu_timer_mark) timer_mark;
    decltype(&mesh_gpu_migrate) migrate;
    decltype(&mesh_gpu_reserve) reserve;
};

namespace {
// Steps the host may have in flight before it retires the oldest: deep enough
// that every execution lane stays fed while one lane runs a long step (the
// data plane's ticket ring holds 1024). MESH_HOST_WINDOW overrides it: 240,
// 600 and 1000 gave the same e2e wall within run-to-run noise (24.7-26.5 s),
// because a deeper window only fills the launch queue further.
std::size_t max_pending() {
    static const std::size_t n = [] {
        const char* e = std::getenv("MESH_HOST_WINDOW");
        const long v = e ? std::atol(e) : 0;
        return v > 0 ? std::min<std::size_t>(std::size_t(v), 1000) : std::size_t(240);
    }();
    return n;
}
struct HostTimer {  // adds the scope's wall time (ms) to `acc`
    double& acc;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    explicit HostTimer(double& a) : acc(a) {}
    ~HostTimer() { acc += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(); }
};
uint64_t weight_seed(const std::string& model_id) {  // every instance of a model is the same replica
    uint64_t h = 1469598103934665603ULL;
    for (unsigned char ch : model_id) {
        h ^= ch;
        h *= 1099511628211ULL;
    }
    return h;
}
}  // namespace

GpuExecutor::GpuExecutor(const std::string& lib_path, std::vector<int> devices, long long kv_pool_bytes)
    : devices_(std::move(devices)), pool_bytes_(kv_pool_bytes) {
    if (devices_.empty()) throw ConfigError("attach_gpu: no devices given");
    dl_ = dlopen(lib_path.c_str(), RTLD_NOW | RTLD_LOCAL);
    if (!dl_) throw SimError(std::string("attach_gpu: cannot load ") + lib_path + ": " + dlerror());
    api_ = new Api();
    auto sym = [&](const char* n) {
        void* p = dlsym(dl_, n);
        if (!p) throw SimError(std::string("attach_gpu: missing symbol ") + n);
        return p;
    };
#define BIND(field, name) api_->field = reinterpret_cast<decltype(api_->field)>(sym(name))
    BIND(open, "mesh_gpu_open");
    BIND(close, "mesh_gpu_close");
    BIND(last_error, "mesh_gpu_last_error");
    BIND(instance_create, "mesh_gpu_instance_create");
    BIND(instance_destroy, "mesh_gpu_instance_destroy");
    BIND(kv_resize, "mesh_gpu_kv_resize");
    BIND(step, "mesh_gpu_step");
    BIND(step_wait, "mesh_gpu_step_wait");
    BIND(request_free, "mesh_gpu_request_free");
    BIND(swap_out, "mesh_gpu_swap_out");
    BIND(stats_get, "mesh_gpu_stats_get");
    BIND(step_done, "mesh_gpu_step_done");
    BIND(timer_mark, "mesh_gpu_timer_mark");
    BIND(migrate, "mesh_gpu_migrate");
    BIND(reserve, "mesh_gpu_reserve");
#undef BIND
    if (const char* e = std::getenv("MESH_MIGRATE")) migrate_ = std::atoi(e) != 0;
    for (int dev : devices_) {
        mesh_gpu_cfg cfg{};
        cfg.device = dev;
        cfg.sm_quota = 0;
        cfg.kv_pool_bytes = pool_bytes_;
        cfg.prompt_seed = 1234;
        if (const char* e = std::getenv("MESH_GPU_KV_GRANULE_MB")) cfg.kv_granule_bytes = std::atoll(e) << 20;
        // pinned swap space pinned at open (evictions then never pin on the serving path)
        if (const char* e = std::getenv("MESH_GPU_SWAP_POOL_MB")) cfg.swap_pool_mb = std::max(0, std::atoi(e));
        mesh_gpu* h = nullptr;
        if (api_->open(&cfg, &h) != MESH_OK) throw SimError("attach_gpu: mesh_gpu_open failed on device " + std::to_string(dev));
        handles_.push_back(h);
    }
}

GpuExecutor::~GpuExecutor() {
    if (api_)
        for (mesh_gpu* h : handles_) api_->close(h);
    delete api_;
    if (dl_) dlclose(dl_);
}

void GpuExecutor::check(mesh_gpu* h, int status, const char* what) {
    if (status != MESH_OK) throw SimError(std::string("gpu data plane: ") + what + ": " + api_->last_error(h));
}

mesh_gpu* GpuExecutor::handle_for_node(NodeId node) {
    return handles_[static_cast<std::size_t>(node) % handles_.size()];
}

namespace {
mesh_model_shape c_shape(const LlamaShape& L, int max_seq) {
    return mesh_model_shape{L.n_layers, L.d_model, L.n_heads, L.n_kv_heads, L.d_head, L.d_ff, L.vocab, L.tied,
                            std::min(L.max_seq_len, max_seq), L.rope_theta, L.rms_eps};
}
}  // namespace

// Every model's weight set and scratch reserved on every device before the clock
// starts: instance starts on the serving path then neither resize scratch (a
// device-wide sync) nor grow the weight allocator's pool (a device drain).
void GpuExecutor::prepare(const Cluster& c) {
    HostTimer ht(host_ms_create_);
    std::vector<mesh_model_shape> shapes;
    for (const auto& [id, m] : c.models()) shapes.push_back(c_shape(llama_shape_for(m.spec.size_class), m.spec.max_seq_len));
    if (shapes.empty()) return;
    for (mesh_gpu* h : handles_) check(h, api_->reserve(h, shapes.data(), int32_t(shapes.size())), "reserve");
}

void GpuExecutor::instance_start(const Cluster&, const Instance& inst) {
    HostTimer ht(host_ms_create_);
    ++instance_starts_;
    const mesh_model_shape s = c_shape(llama_shape_for(inst.model->size_class), inst.model->max_seq_len);
    mesh_gpu* h = handle_for_node(inst.node_id);
    inst_dev_[inst.id] = static_cast<int>(static_cast<std::size_t>(inst.node_id) % handles_.size());
    check(h, api_->instance_create(h, inst.id, &s, weight_seed(inst.model->model_id)), "instance_create");
}

void GpuExecutor::kv_issue(const Cluster&, const Instance& inst, const ScaleOp& op) {
    HostTimer ht(host_ms_kv_);
    mesh_gpu* h = handle_for_node(inst.node_id);
    check(h, api_->kv_resize(h, inst.id, op.from_bytes, op.to_bytes), "kv_resize");
}

void GpuExecutor::iteration_start(const Cluster& c, const Node& nd, const Instance& inst, const IterationPlan& p) {
    HostTimer ht(host_ms_step_);
    mesh_gpu* h = handle_for_node(nd.id);
    std::vector<Pending>& tk = tickets_[nd.id];
    if (p.is_prefill) {
        const Request& r = c.requests().get(p.prefill_request);
        mesh_step_plan sp{1, p.prefill_request, p.kind.input_len, r.input_len, 0, nullptr};
        int64_t t = 0;
        check(h, api_->step(h, inst.id, &sp, &t), "prefill step");
        (wall_ ? live_[inst.id] : tk).push_back({h, t, inst.id});
        prefill_tokens_ += p.kind.input_len;
        return;
    }
    std::vector<int64_t> rids;
    for (RequestId rid : inst.batch)
        if (c.requests().get(rid).prefill_done) rids.push_back(rid);
    for (std::size_t o = 0; o < rids.size(); o += 8) {  // the decode kernel takes <= 8 columns
        const int n = static_cast<int>(std::min<std::size_t>(8, rids.size() - o));
        mesh_step_plan sp{0, -1, 0, 0, n, rids.data() + o};
        int64_t t = 0;
        check(h, api_->step(h, inst.id, &sp, &t), "decode step");
        (wall_ ? live_[inst.id] : tk).push_back({h, t, inst.id});
    }
    decode_tokens_ += static_cast<long long>(rids.size());
}

void GpuExecutor::clock_start() {
    wall_ = true;
    for (mesh_gpu* h : handles_) check(h, api_->timer_mark(h, 0), "timer_mark");
}

// Wall-clock mode: an instance's step is done when all of its tickets are
// (a batch wider than the kernel's 8 columns is several launches). Tokens are
// then collected without blocking; the end time is the CUDA event of the
// step's last launch on the device timeline of clock_start's mark.
void GpuExecutor::poll_finished(std::vector<std::pair<InstanceId, double>>& done) {
    for (auto it = live_.begin(); it != live_.end();) {
        bool all = true;
        for (const Pending& p : it->second) {
            int32_t d = 0;
            check(p.h, api_->step_done(p.h, p.ticket, &d), "step_done");
            if (!d) {
                all = false;
                break;
            }
        }
        if (!all) {
            ++it;
            continue;
        }
        HostTimer ht(host_ms_wait_);
        double end_s = 0.0;
        for (const Pending& p : it->second) {
            int32_t toks[8];
            int32_t n = 0;
            check(p.h, api_->step_wait(p.h, p.ticket, toks, 8, &n, nullptr, 0), "step_wait");
            mesh_gpu_stats st{};
            api_->stats_get(p.h, &st);
            device_ms_ += st.last_step_ms;
            lane_busy_s_ += st.last_step_ms / 1e3;
            end_s = std::max(end_s, st.last_step_end_ms / 1e3);
            ++steps_;
        }
        done.emplace_back(it->first, end_s);
        it = live_.erase(it);
    }
}

void GpuExecutor::iteration_done(const Cluster&, const Node& nd, const IterationPlan&, const IterationOutcome&) {
    if (wall_) return;  // retired by poll_finished
    // Steps stay asynchronous: their tickets are retired lazily (bounded by the
    // data plane's ticket ring), so the host keeps scheduling while the GPU runs.
    auto it = tickets_.find(nd.id);
    if (it == tickets_.end()) return;
    for (const Pending& p : it->second) pending_.push_back(p);
    it->second.clear();
    while (pending_.size() > max_pending()) retire_one();
}

void GpuExecutor::retire_one() { retire_at(0); }

void GpuExecutor::retire_at(std::size_t i) {
    HostTimer ht(host_ms_wait_);
    const Pending p = pending_[i];
    pending_.erase(pending_.begin() + static_cast<long>(i));
    mesh_gpu* h = p.h;
    const long long t = p.ticket;
    int32_t toks[8];
    int32_t n = 0;
    check(h, api_->step_wait(h, t, toks, 8, &n, nullptr, 0), "step_wait");
    mesh_gpu_stats st{};
    api_->stats_get(h, &st);
    device_ms_ += st.last_step_ms;
    ++steps_;
}

void GpuExecutor::drain() {
    while (!pending_.empty()) retire_one();
}

void GpuExecutor::request_evicted(const Cluster&, InstanceId inst, const Request& r) {
    auto d = inst_dev_.find(inst);
    if (d == inst_dev_.end()) return;
    mesh_gpu* h = handles_[static_cast<std::size_t>(d->second)];
    // a request that never ran a prefill has no device state: nothing to park
    (void)api_->swap_out(h, inst, r.id);
}

mesh_gpu* GpuExecutor::handle_of_instance(InstanceId inst) {
    auto d = inst_dev_.find(inst);
    return d == inst_dev_.end() ? nullptr : handles_[static_cast<std::size_t>(d->second)];
}

// Displacement (commit_preemption, cluster.cpp:413-465): the reference drops the
// request's KV and re-prefills it at the plan's target. Here the KV moves to the
// target instance right away (one copy kernel on the target's GPU, NVLink P2P
// when the nodes differ); the target's re-prefill step then finds ctx = I+O-1
// resident and feeds one token. Decisions are untouched (the control plane
// still prices the re-prefill); only the executed work differs.
void GpuExecutor::request_displaced(const Cluster& c, InstanceId from, InstanceId planned_to, const Request& r) {
    mesh_gpu* src = handle_of_instance(from);
    mesh_gpu* dst = planned_to >= 0 ? handle_of_instance(planned_to) : nullptr;
    if (!src) return;
    if (migrate_ && dst) {
        HostTimer ht(host_ms_migrate_);
        if (api_->migrate(src, from, dst, planned_to, r.id) == MESH_OK) {
            moved_[r.id] = planned_to;
            ++migrations_;
            return;
        }
        ++migrate_fallbacks_;  // not resident (never prefilled), or no room / peer path: park it instead
    }
    request_evicted(c, from, r);
}

void GpuExecutor::request_placed(const Cluster& c, InstanceId to, const Request& r) {
    auto it = moved_.find(r.id);
    if (it == moved_.end()) return;
    const InstanceId at = it->second;
    moved_.erase(it);
    if (to != at) request_evicted(c, at, r);  // landed elsewhere: park the migrated KV for its re-prefill
}

void GpuExecutor::request_finished(const Cluster&, InstanceId inst, const Request& r) {
    auto d = inst_dev_.find(inst);
    if (d == inst_dev_.end()) return;
    (void)api_->request_free(handles_[static_cast<std::size_t>(d->second)], inst, r.id);
}

void GpuExecutor::instance_unloaded(const Cluster&, InstanceId inst) {
    auto d = inst_dev_.find(inst);
    if (d == inst_dev_.end()) return;
    if (auto lv = live_.find(inst); lv != live_.end()) {  // not expected: unloads happen between steps
        for (const Pending& p : lv->second) check(p.h, api_->step_wait(p.h, p.ticket, nullptr, 0, nullptr, nullptr, 0), "step_wait");
        live_.erase(lv);
    }
    // retire the instance's own outstanding tickets before it (and they) go away;
    // other instances' steps keep running
    for (std::size_t i = 0; i < pending_.size();)
        if (pending_[i].inst == inst)
            retire_at(i);
        else
            ++i;
    HostTimer ht(host_ms_destroy_);
    mesh_gpu* h = handles_[static_cast<std::size_t>(d->second)];
    check(h, api_->instance_destroy(h, inst), "instance_destroy");
    inst_dev_.erase(d);
}

std::map<std::string, double> GpuExecutor::metrics() const {
    std::map<std::string, double> m;
    m["gpu.steps"] = static_cast<double>(steps_);
    m["gpu.decode_tokens"] = static_cast<double>(decode_tokens_);
    m["gpu.prefill_tokens"] = static_cast<double>(prefill_tokens_);
    m["gpu.device_ms"] = device_ms_;
    m["gpu.instance_starts"] = static_cast<double>(instance_starts_);
    m["gpu.host_ms.instance_create"] = host_ms_create_;
    m["gpu.host_ms.instance_destroy"] = host_ms_destroy_;
    m["gpu.host_ms.kv_resize"] = host_ms_kv_;
    m["gpu.host_ms.step_issue"] = host_ms_step_;
    m["gpu.host_ms.step_wait"] = host_ms_wait_;
    double swap = 0, swap_in = 0, mig = 0, moved = 0, launches = 0, h2d = 0, d2h = 0, vmm_calls = 0, vmm_ms = 0, reclaims = 0,
           wcache = 0, unmaps = 0, dp_create = 0, dp_destroy = 0, dp_kv = 0, dp_step = 0;
    for (mesh_gpu* h : handles_) {
        mesh_gpu_stats st{};
        api_->stats_get(h, &st);
        swap += static_cast<double>(st.swap_out_bytes);
        swap_in += static_cast<double>(st.swap_in_bytes);
        mig += static_cast<double>(st.migrate_bytes);
        moved += static_cast<double>(st.blocks_moved);
        launches += static_cast<double>(st.kernel_launches);
        h2d += static_cast<double>(st.h2d_bytes);
        d2h += static_cast<double>(st.d2h_bytes);
        vmm_calls += static_cast<double>(st.vmm_calls);
        vmm_ms += st.vmm_ms;
        reclaims += static_cast<double>(st.kv_reclaims);
        wcache += static_cast<double>(st.weight_cache_hits);
        unmaps += static_cast<double>(st.vmm_unmaps);
        dp_create += st.host_ms_create;
        dp_destroy += st.host_ms_destroy;
        dp_kv += st.host_ms_kv_resize;
        dp_step += st.host_ms_step;
    }
    m["gpu.weight_cache_hits"] = wcache;
    m["gpu.lane_busy_s"] = lane_busy_s_;
    m["gpu.vmm_calls"] = vmm_calls;
    m["gpu.vmm_unmaps"] = unmaps;
    m["gpu.dp_ms.instance_create"] = dp_create;
    m["gpu.dp_ms.instance_destroy"] = dp_destroy;
    m["gpu.dp_ms.kv_resize"] = dp_kv;
    m["gpu.dp_ms.step"] = dp_step;
    m["gpu.host_ms.vmm"] = vmm_ms;
    m["gpu.kv_reclaims"] = reclaims;
    m["gpu.swap_out_bytes"] = swap;
    m["gpu.swap_in_bytes"] = swap_in;
    m["gpu.migrate_bytes"] = mig;
    m["gpu.migrations"] = static_cast<double>(migrations_);
    m["gpu.migrate_fallbacks"] = static_cast<double>(migrate_fallbacks_);
    m["gpu.host_ms.migrate"] = host_ms_migrate_;
    m["gpu.blocks_moved"] = moved;
    m["gpu.kernel_launches"] = launches;
    m["gpu.h2d_bytes"] = h2d;
    m["gpu.d2h_bytes"] = d2h;
    return m;
}

}  // namespace mesh
