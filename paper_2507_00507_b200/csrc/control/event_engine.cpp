#include "event_engine.hpp"

#include <algorithm>
#include <cstdio>

namespace mesh {

const char* event_kind_name(EventKind k) {
    static const char* const names[] = {"request_arrival", "iteration_complete", "scale_op_complete",
                                        "keep_alive_check", "cold_start_complete"};
    const int i = static_cast<int>(k);
    return (i >= 0 && i < 5) ? names[i] : "unknown";
}

void Engine::push(const Event& e) {
    heap_.push_back(e);
    std::push_heap(heap_.begin(), heap_.end(), after);
}

Event Engine::pop() {
    std::pop_heap(heap_.begin(), heap_.end(), after);
    Event e = heap_.back();
    heap_.pop_back();
    return e;
}

void Engine::schedule(SimTime when, EventKind kind, std::int64_t subject) {
    if (when < now_) {
        throw SimError("schedule: event time " + std::to_string(when) + " precedes clock " + std::to_string(now_));
    }
    push(Event{when, seq_++, kind, subject});
}

SimulationReport Engine::run_until(SimTime horizon) {
    SimulationReport rep;
    while (!heap_.empty() && heap_.front().time <= horizon) {
        const Event e = pop();
        now_ = e.time;
        if (logging_) log_.push_back(e);
        ++rep.events_processed;
        if (handler_) handler_(e);
    }
    // an exhausted queue lets the clock reach a finite horizon
    if (heap_.empty() && now_ < horizon && horizon < std::numeric_limits<double>::infinity()) now_ = horizon;
    rep.end_time = now_;
    return rep;
}

std::string format_event_log(const std::vector<EventLogRecord>& log) {
    std::string out;
    out.reserve(log.size() * 72);
    char line[192];
    for (const Event& e : log) {
        int n = std::snprintf(line, sizeof(line), "{\"time\":%.9f,\"seq\":%lld,\"kind\":\"%s\",\"subject\":%lld}\n",
                              e.time, static_cast<long long>(e.seq), event_kind_name(e.kind),
                              static_cast<long long>(e.subject));
        out.append(line, static_cast<std::size_t>(n));
    }
    return out;
}

}  // namespace mesh
