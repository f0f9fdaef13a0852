// Discrete-event engine: a virtual clock over a (time, seq) min-heap.
// Same ordering contract as proj/src/simcore.hpp:55-101 — equal-time events
// run in insertion order, scheduling into the past is an error — so event
// logs replay byte-identically.
#pragma once

#include <cstdint>
#include <functional>
#include <limits>
#include <string>
#include <vector>

#include "core_types.hpp"

namespace mesh {

enum class EventKind { RequestArrival, IterationComplete, ScaleOpComplete, KeepAliveCheck, ColdStartComplete };
const char* event_kind_name(EventKind k);

struct Event {
    SimTime time = 0.0;
    std::int64_t seq = 0;
    EventKind kind = EventKind::RequestArrival;
    std::int64_t subject = -1;  // request / node / op / instance id by kind
};
using EventLogRecord = Event;

struct SimulationReport {
    std::int64_t events_processed = 0;
    SimTime end_time = 0.0;
};

class Engine {
public:
    using Handler = std::function<void(const Event&)>;

    void set_handler(Handler h) { handler_ = std::move(h); }
    void set_log_enabled(bool on) { logging_ = on; }
    SimTime now() const { return now_; }
    bool empty() const { return heap_.empty(); }
    std::size_t pending() const { return heap_.size(); }
    SimTime next_time() const { return heap_.empty() ? std::numeric_limits<double>::infinity() : heap_.front().time; }

    void schedule(SimTime when, EventKind kind, std::int64_t subject);
    SimulationReport run_until(SimTime horizon);
    const std::vector<EventLogRecord>& log() const { return log_; }

private:
    static bool after(const Event& x, const Event& y) {
        return x.time != y.time ? x.time > y.time : x.seq > y.seq;
    }
    void push(const Event& e);
    Event pop();

    std::vector<Event> heap_;  // binary heap ordered by `after`
    SimTime now_ = 0.0;
    std::int64_t seq_ = 0;
    Handler handler_;
    bool logging_ = false;
    std::vector<EventLogRecord> log_;
};

// {"time":%.9f,"seq":..,"kind":"..","subject":..} per line (simcore.cpp:8-20 format).
std::string format_event_log(const std::vector<EventLogRecord>& log);

}  // namespace mesh
