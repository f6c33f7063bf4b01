// Executor — the multi-lane resource pool (Alg. 4) in front of
// GpuIndex, mirroring the reference's Executor contract
// (include/blockivf/executor.hpp:21-196, src/executor.cpp):
//   * search lanes: one worker thread + one GPU lease each (stream, device
//     workspace, pinned staging); fail-fast reject when every lane is busy,
//     never queue (executor.cpp:165-170); the whole request batch (<= 10
//     queries) is ONE device search, not a per-query loop
//   * two-tier scratch accounting: lane cache + central grants (executor.cpp:267-284)
//   * one data lane with the insertion batcher: flush at >= batch_multiple
//     pending vectors, manual flush, the flush interval, or shutdown; chunks of
//     <= batch_cap with one id-mode per batch; post_insert_maintenance after
//     every batch (executor.cpp:331-445)
//   * serialized FIFO mode on one lane (executor.cpp:447-472)
//   * tickets with submit/start/end stamps (executor.hpp:39-72)
#pragma once

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "index.h"

namespace bivf {

using Clock = std::chrono::steady_clock;

enum class TicketStatus { Pending = 0, Done = 1, Rejected = 2, Error = 3 };
enum class RequestType { Search = 0, Insert = 1 };

struct ExecConfig {
    uint32_t num_lanes = 32;
    uint64_t lane_cache_bytes = 512 * 1024;
    uint64_t central_grant_bytes = 2 * 1024 * 1024;
    uint32_t central_grants = 4;
    uint32_t flush_interval_ms = 1000;
    uint32_t batch_multiple = 128;
    uint32_t batch_cap = 1024;
    uint32_t max_search_batch = 10;
    bool serialized = false;
};

struct TicketState {
    std::mutex mu;
    std::condition_variable cv;
    bool ready = false;
    TicketStatus status = TicketStatus::Pending;
    RequestType type = RequestType::Search;
    std::string error;
    int lane = -1;
    uint32_t nq = 0, k = 0;
    std::vector<int64_t> ids;  // search: nq*k; insert: one per vector
    std::vector<float> dists;
    std::vector<uint32_t> counts;
    Clock::time_point submit, start, end;
    double latency_us() const { return std::chrono::duration<double, std::micro>(end - submit).count(); }
    double queue_us() const { return std::chrono::duration<double, std::micro>(start - submit).count(); }
    double exec_us() const { return std::chrono::duration<double, std::micro>(end - start).count(); }
    void wait() {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return ready; });
    }
};
using Ticket = std::shared_ptr<TicketState>;

class Executor {
public:
    Executor(GpuIndex& index, const ExecConfig& cfg);
    ~Executor();

    Ticket submit_search(const float* q, uint32_t nq, uint32_t k, uint32_t nprobe);
    Ticket submit_insert(const float* x, uint64_t n, const int64_t* ids);
    void flush_insertions();
    void set_mode(bool serialized);
    void shutdown();

    // rejected, completed, in_flight, grants_outstanding, grants_total,
    // lane_cache_allocations, lane_double_hold_violations, largest_flush
    void stats(uint64_t out[8]) const;
    const ExecConfig& config() const { return cfg_; }
    GpuIndex& index() { return index_; }

private:
    struct SearchTask {
        Ticket t;
        std::vector<float> q;
        uint32_t nq, k, nprobe;
    };
    struct PendingInsert {
        Ticket t;
        std::vector<float> x;
        std::vector<int64_t> ids;
        uint64_t count = 0, flushed = 0, completed = 0;
        bool failed = false;
        std::string error;
    };
    struct Lane {
        std::thread worker;
        std::mutex mu;
        std::condition_variable cv;
        std::unique_ptr<SearchTask> task;
        std::atomic<bool> busy{false};
        bool stop = false;
    };
    struct SerialTask {
        RequestType type;
        std::unique_ptr<SearchTask> search;
        std::shared_ptr<PendingInsert> insert;
    };

    Ticket make_ticket(RequestType t);
    void resolve(const Ticket& t, TicketStatus s, const std::string& err = {});
    void reject(const Ticket& t, const std::string& why);
    void lane_main(uint32_t id);
    void run_search(SearchTask& task, int lane);
    void insertion_main();
    void flush_locked(std::unique_lock<std::mutex>& lk);
    void serial_main();
    bool pop_free_lane(uint32_t& id);
    void push_free_lane(uint32_t id);

    GpuIndex& index_;
    ExecConfig cfg_;
    std::vector<std::unique_ptr<Lane>> lanes_;
    std::mutex free_mu_;
    std::deque<uint32_t> free_lanes_;

    std::thread insertion_thread_, serial_thread_;
    std::mutex batch_mu_;
    std::condition_variable batch_cv_;
    std::deque<std::shared_ptr<PendingInsert>> pending_;
    uint64_t pending_vectors_ = 0;
    bool manual_flush_ = false;
    Clock::time_point last_flush_;

    std::mutex serial_mu_;
    std::condition_variable serial_cv_;
    std::deque<SerialTask> serial_queue_;

    std::atomic<bool> accepting_{true}, stopping_{false};
    std::atomic<uint64_t> in_flight_{0}, rejected_{0}, completed_{0};
    std::atomic<uint64_t> grants_outstanding_{0}, grants_total_{0}, grants_available_{0};
    std::atomic<uint64_t> double_hold_{0}, largest_flush_{0};
    uint64_t lane_cache_allocations_ = 0;
};

// Open-loop replay (workload.cpp:114-269 subset): deterministic schedule
// (fixed or Poisson arrivals from mt19937_64(seed)), search requests of
// search_batch queries and insert requests of insert_batch vectors, every
// ticket awaited.  Outputs per-request latencies (us; -1 rejected, -2 error).
struct ReplaySpec {
    double qps_search = 0, qps_insert = 0, duration_s = 1;
    uint32_t search_batch = 1, insert_batch = 1, k = 10, nprobe = 8;
    uint64_t seed = 1;
    bool poisson = false;
};
struct ReplayOut {
    std::vector<double> search_us, insert_us;
    uint64_t rejected = 0, errors = 0;
};
ReplayOut replay(Executor& ex, const ReplaySpec& spec, const float* queries, uint64_t nqueries,
                 const float* inserts, uint64_t ninserts);

}  // namespace bivf
