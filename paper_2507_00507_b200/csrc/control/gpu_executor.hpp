// DataPlane that executes the control plane's actions on B200s through the
// mesh_gpu C ABI (libmesh_gpu.so, loaded with dlopen so the control plane
// builds and runs without CUDA). Node i -> device devices[i % n].
#pragma once

#include <deque>
#include <map>
#include <string>
#include <vector>

#include "mesh_cluster.hpp"

struct mesh_gpu;

namespace mesh {

struct LlamaShape {
    int n_layers, d_model, n_heads, n_kv_heads, d_head, d_ff, vocab, tied, max_seq_len;
    float rope_theta, rms_eps;
};
// Llama-family shapes per size class; unknown classes throw.
const LlamaShape& llama_shape_for(const std::string& size_class);

class GpuExecutor : public DataPlane {
public:
    GpuExecutor(const std::string& lib_path, std::vector<int> devices, long long kv_pool_bytes);
    ~GpuExecutor() override;

    void prepare(const Cluster&) override;
    void instance_start(const Cluster&, const Instance&) override;
    void kv_issue(const Cluster&, const Instance&, const ScaleOp&) override;
    void iteration_start(const Cluster&, const Node&, const Instance&, const IterationPlan&) override;
    void iteration_done(const Cluster&, const Node&, const IterationPlan&, const IterationOutcome&) override;
    void request_evicted(const Cluster&, InstanceId, const Request&) override;
    void request_displaced(const Cluster&, InstanceId from, InstanceId planned_to, const Request&) override;
    void request_placed(const Cluster&, InstanceId to, const Request&) override;
    void request_finished(const Cluster&, InstanceId, const Request&) override;
    void instance_unloaded(const Cluster&, InstanceId) override;

    // wall-clock mode (Cluster::set_wall_clock): steps complete on device events
    bool supports_wall_clock() const override { return true; }
    void clock_start() override;
    void poll_finished(std::vector<std::pair<InstanceId, double>>& done) override;
    std::size_t steps_in_flight() const override { return live_.size(); }

    std::map<std::string, double> metrics() const;
    void drain();  // wait for every launched step

private:
    struct Api;
    Api* api_ = nullptr;
    void* dl_ = nullptr;
    std::vector<int> devices_;
    long long pool_bytes_;
    std::vector<mesh_gpu*> handles_;                 // per device index
    std::map<InstanceId, int> inst_dev_;             // instance -> device index
    struct Pending {
        mesh_gpu* h;
        long long ticket;
        InstanceId inst;
    };
    std::map<NodeId, std::vector<Pending>> tickets_;  // in-flight step of each node
    double device_ms_ = 0.0;
    long long steps_ = 0, decode_tokens_ = 0, prefill_tokens_ = 0, instance_starts_ = 0;
    // host wall time spent inside each data-plane hook (e2e breakdown)
    double host_ms_create_ = 0, host_ms_destroy_ = 0, host_ms_kv_ = 0, host_ms_step_ = 0, host_ms_wait_ = 0;
    std::deque<Pending> pending_;  // launched, not yet retired (oldest first)
    bool wall_ = false;
    std::map<InstanceId, std::vector<Pending>> live_;  // wall-clock mode: the step in flight per instance
    double lane_busy_s_ = 0.0;                          // wall-clock mode: sum of step device times
    // live KV migration of displaced requests (MESH_MIGRATE=0 turns it off: they
    // are swapped out and resume from pinned host memory, like evictions)
    bool migrate_ = true;
    std::map<RequestId, InstanceId> moved_;  // displaced request -> instance its KV was migrated to
    long long migrations_ = 0, migrate_fallbacks_ = 0;
    double host_ms_migrate_ = 0;
    mesh_gpu* handle_of_instance(InstanceId inst);
    void retire_one();
    void retire_at(std::size_t i);
    mesh_gpu* handle_for_node(NodeId node);
    void check(mesh_gpu* h, int status, const char* what);
};

}  // namespace mesh
