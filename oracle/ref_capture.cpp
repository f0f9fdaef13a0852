// TEST INFRASTRUCTURE ONLY — links the UNMODIFIED reference simulator sources
// (/root/reference/proj/src, compiled by oracle/Makefile into oracle/_ref/) and
// dumps its decisions so tests/ can byte-compare our control plane against it.
// Nothing in the product path links this file.
//
//   ref_capture run  <config.json> <out_dir> [key=value ...]
//        writes summary.json, requests.csv, ttft_cdf.csv, events.jsonl (always on),
//        plus ops.csv (ScaleOp transcript, memory.hpp:69-81), steps.csv (one row per
//        launched iteration, cluster.cpp:556-572) and hash.txt (state_hash,
//        cluster.cpp:908-931).
//   ref_capture time <config.json> <reps> [key=value ...]
//        times the reference's simulate() (simulation.cpp:116-124) with the event
//        log off, best of <reps>, and prints one JSON line.
//
// The driver below restates simulation.cpp:32-114 (execute) through the
// reference's public headers only so that the Cluster object stays reachable.

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <limits>
#include <map>
#include <memory>
#include <random>
#include <set>
#include <string>
#include <vector>

#include "cluster.hpp"
#include "config.hpp"
#include "metrics.hpp"
#include "simcore.hpp"
#include "simulation.hpp"
#include "workload.hpp"

using namespace mesh;
namespace fs = std::filesystem;

namespace {

struct Harness {
    Engine engine;
    RequestStore store;
    MetricsCollector metrics;
    std::mt19937_64 rng;
    std::unique_ptr<Cluster> cluster;
    std::vector<std::string> step_rows;
    std::vector<SimTime> last_busy_until;
};

void build(const ExperimentConfig& cfg, Harness& h, bool record_steps) {
    int max_total = 2;
    for (const auto& t : cfg.templates) max_total = std::max(max_total, t.max_seq_len);
    LengthDataset ds = load_length_dataset(cfg.lengths_path, max_total);
    TraceSpec trace = load_trace(cfg.trace_path, cfg.window_s, cfg.sample_functions, cfg.seed);
    std::map<std::string, const ModelTemplateCfg*> tpl_by_name;
    for (const auto& t : cfg.templates) tpl_by_name[t.name] = &t;
    std::vector<std::pair<std::string, const ModelTemplateCfg*>> bound;
    std::map<std::string, int> caps;
    std::size_t k = 0;
    for (auto& [fn, mid] : trace.model_map) {
        const ModelTemplateCfg* tpl = tpl_by_name.at(cfg.assignment[k++ % cfg.assignment.size()]);
        mid = tpl->name + ":" + fn;
        caps[mid] = tpl->max_seq_len;
        bound.emplace_back(mid, tpl);
    }
    h.store.all = build_request_stream(trace, ds, caps, cfg.seed ^ 0x517cc1b727220a95ULL);
    h.engine.set_log_enabled(cfg.event_log);
    h.rng.seed(cfg.seed);
    Policy pol = cfg.policy;
    h.cluster = std::make_unique<Cluster>(h.engine, h.store, h.metrics, cfg.slo, pol,
                                          cfg.cost_params(HwClass::Cpu),
                                          cfg.cost_params(HwClass::Gpu), h.rng);
    std::set<HwClass> classes;
    for (const auto& g : cfg.node_groups) {
        for (int i = 0; i < g.count; ++i)
            h.cluster->add_node(g.cls, static_cast<Bytes>(std::llround(g.mem_gb * double(GB))));
        classes.insert(g.cls);
    }
    std::set<std::string> scs;
    for (const auto& [mid, tpl] : bound) scs.insert(tpl->size_class);
    for (const auto& sc : scs) {
        for (HwClass hw : classes) {
            auto it = cfg.table_paths.find(sc + ":" + hw_name(hw));
            if (it != cfg.table_paths.end())
                h.cluster->register_table(sc, hw, load_perf_table(it->second, sc, hw));
            else
                h.cluster->register_table(sc, hw,
                                          make_synthetic_table(sc, hw, default_synthetic_perf(sc, hw),
                                                               cfg.grid_max_len, cfg.grid_max_batch));
        }
    }
    double mean_out = ds.mean_output();
    for (const auto& [mid, tpl] : bound) {
        ModelSpec s;
        s.model_id = mid;
        s.size_class = tpl->size_class;
        s.param_bytes = static_cast<Bytes>(std::llround(tpl->param_gb * double(GB)));
        s.kv_bytes_per_token = tpl->kv_kib_per_token * KiB;
        s.max_seq_len = tpl->max_seq_len;
        s.max_batch = tpl->max_batch;
        s.min_total_len = tpl->min_total_len > 0 ? tpl->min_total_len : tpl->max_seq_len;
        s.avg_output = std::max(1.0, tpl->avg_output_seed > 0 ? tpl->avg_output_seed : mean_out);
        s.avg_output_fixed = tpl->avg_output_fixed;
        h.cluster->add_model(std::move(s));
    }
    Cluster* c = h.cluster.get();
    h.last_busy_until.assign(c->nodes().size(), -1.0);
    Harness* hp = &h;
    h.engine.set_handler([c, hp, record_steps](const Event& ev) {
        c->on_event(ev);
        if (!record_steps) return;
        // A node whose busy_until moved has launched a new iteration in this handler.
        for (const Node& nd : c->nodes()) {
            auto idx = static_cast<std::size_t>(nd.id);
            if (!nd.busy || nd.busy_until == hp->last_busy_until[idx]) continue;
            hp->last_busy_until[idx] = nd.busy_until;
            const IterationPlan& p = nd.current_plan;
            char buf[256];
            std::snprintf(buf, sizeof(buf), "%.9f,%lld,%lld,%d,%lld,%d,%d,%d,%.12g", ev.time,
                          (long long)nd.id, (long long)p.instance_id, p.is_prefill ? 1 : 0,
                          (long long)p.prefill_request, p.kind.input_len, p.kind.batch,
                          p.kind.avg_len, p.predicted_duration);
            std::string row = buf;
            row += ",";
            const Instance* inst = c->find_instance(p.instance_id);
            bool first = true;
            if (inst) {
                for (RequestId rid : inst->batch) {
                    const Request& r = c->requests().get(rid);
                    if (p.is_prefill ? rid != p.prefill_request : !r.prefill_done) continue;
                    if (!first) row += ";";
                    row += std::to_string(rid) + ":" + std::to_string(r.input_len + r.tokens_generated);
                    first = false;
                }
            }
            hp->step_rows.push_back(row);
        }
    });
    for (const Request& r : h.store.all) h.engine.schedule(r.arrival_time, EventKind::RequestArrival, r.id);
}

int cmd_run(const std::string& cfg_path, const std::string& out, std::vector<std::string> ov) {
    ov.push_back("output.event_log=true");
    ExperimentConfig cfg = load_config(cfg_path, ov, std::nullopt, out);
    Harness h;
    build(cfg, h, true);
    h.engine.run_until(std::numeric_limits<double>::infinity());
    h.cluster->finalize(h.engine.now());
    SummaryReport rep = h.metrics.finalize(h.store, cfg.slo, h.engine.now());
    fs::create_directories(out);
    write_summary(rep, out + "/summary.json");
    write_requests_csv(h.metrics.request_records(h.store, cfg.slo), out + "/requests.csv");
    write_cdf_csv(rep, out + "/ttft_cdf.csv");
    {
        std::ofstream ev(out + "/events.jsonl");
        ev << format_event_log(h.engine.log());
    }
    {
        std::ofstream os(out + "/ops.csv");
        os << "op_id,instance,kind,from,to,state,latency,exec_started,exec_ends,setup,teardown\n";
        for (const auto& [id, op] : h.cluster->ops()) {
            char buf[320];
            std::snprintf(buf, sizeof(buf), "%lld,%lld,%s,%lld,%lld,%d,%.12g,%.9f,%.9f,%d,%d\n",
                          (long long)id, (long long)op.instance_id, scale_kind_name(op.kind),
                          (long long)op.from_bytes, (long long)op.to_bytes, (int)op.state,
                          op.latency, op.exec_started, op.exec_ends, op.setup ? 1 : 0,
                          op.teardown ? 1 : 0);
            os << buf;
        }
    }
    {
        std::ofstream ss(out + "/steps.csv");
        ss << "time,node,instance,is_prefill,prefill_request,input_len,batch,avg_len,predicted,members\n";
        for (const auto& r : h.step_rows) ss << r << "\n";
    }
    {
        std::ofstream hs(out + "/hash.txt");
        hs << h.cluster->state_hash() << "\n";
    }
    return 0;
}

int cmd_time(const std::string& cfg_path, int reps, std::vector<std::string> ov) {
    ov.push_back("output.event_log=false");
    ExperimentConfig cfg = load_config(cfg_path, ov, std::nullopt, std::nullopt);
    double best = 1e30;
    long long events = 0, decode_tokens = 0, steps = 0, total_tokens = 0;
    for (int i = 0; i < reps; ++i) {
        Harness h;
        auto t0 = std::chrono::steady_clock::now();
        build(cfg, h, false);
        SimulationReport r = h.engine.run_until(std::numeric_limits<double>::infinity());
        h.cluster->finalize(h.engine.now());
        double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        best = std::min(best, dt);
        events = r.events_processed;
        SummaryReport rep = h.metrics.finalize(h.store, cfg.slo, h.engine.now());
        decode_tokens = (long long)std::llround(rep.gpu_throughput * rep.gpu_nodes_avg * rep.run_length +
                                                rep.cpu_throughput * rep.cpu_nodes_avg * rep.run_length);
        total_tokens = 0;
        steps = 0;
        for (const Request& q : h.store.all) total_tokens += (long long)q.emission_times.size();
        (void)steps;
    }
    std::printf("{\"best_s\": %.6f, \"events\": %lld, \"tokens\": %lld, \"decode_tokens\": %lld}\n",
                best, events, total_tokens, decode_tokens);
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 4) {
        std::fprintf(stderr, "usage: ref_capture run <cfg> <out> [k=v..] | time <cfg> <reps> [k=v..]\n");
        return 2;
    }
    std::string cmd = argv[1];
    std::vector<std::string> ov(argv + 4, argv + argc);
    try {
        if (cmd == "run") return cmd_run(argv[2], argv[3], ov);
        if (cmd == "time") return cmd_time(argv[2], std::atoi(argv[3]), ov);
    } catch (const ConfigError& e) {
        std::fprintf(stderr, "config error: %s\n", e.what());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "runtime error: %s\n", e.what());
        return 3;
    }
    return 2;
}
