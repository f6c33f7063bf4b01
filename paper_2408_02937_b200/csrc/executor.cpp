// Executor + replay implementation (see executor.h for the contract).
#include "executor.h"

#include <algorithm>
#include <cstring>
#include <random>

namespace bivf {

namespace {
constexpr uint64_t kCandidateRecordBytes = sizeof(float) + sizeof(int64_t);  // executor.cpp:18
}

Executor::Executor(GpuIndex& index, const ExecConfig& cfg) : index_(index), cfg_(cfg) {
    // ExecutorConfig::validate (executor.cpp:22-30)
    if (cfg_.num_lanes < 1) throw Error(BIVF_EINVAL, "ExecutorConfig: num_lanes must be >= 1");
    if (cfg_.batch_multiple < 1) throw Error(BIVF_EINVAL, "ExecutorConfig: batch_multiple must be >= 1");
    if (cfg_.batch_cap < cfg_.batch_multiple)
        throw Error(BIVF_EINVAL, "ExecutorConfig: batch_cap must be >= batch_multiple");
    if (cfg_.max_search_batch < 1)
        throw Error(BIVF_EINVAL, "ExecutorConfig: max_search_batch must be >= 1");
    grants_available_ = cfg_.central_grants;
    for (uint32_t i = 0; i < cfg_.num_lanes; ++i) {
        lanes_.push_back(std::make_unique<Lane>());
        ++lane_cache_allocations_;
        free_lanes_.push_back(i);
    }
    for (uint32_t i = 0; i < cfg_.num_lanes; ++i)
        lanes_[i]->worker = std::thread(&Executor::lane_main, this, i);
    last_flush_ = Clock::now();
    insertion_thread_ = std::thread(&Executor::insertion_main, this);
    serial_thread_ = std::thread(&Executor::serial_main, this);
}

Executor::~Executor() { shutdown(); }

Ticket Executor::make_ticket(RequestType t) {
    auto s = std::make_shared<TicketState>();
    s->type = t;
    s->submit = Clock::now();
    return s;
}

void Executor::resolve(const Ticket& t, TicketStatus s, const std::string& err) {
    {
        std::lock_guard<std::mutex> lk(t->mu);
        t->status = s;
        t->error = err;
        t->ready = true;
    }
    t->cv.notify_all();
    completed_.fetch_add(1);
}

void Executor::reject(const Ticket& t, const std::string& why) {
    t->start = t->end = Clock::now();
    rejected_.fetch_add(1);
    {
        std::lock_guard<std::mutex> lk(t->mu);
        t->status = TicketStatus::Rejected;
        t->error = why;
        t->ready = true;
    }
    t->cv.notify_all();
}

bool Executor::pop_free_lane(uint32_t& id) {
    std::lock_guard<std::mutex> lk(free_mu_);
    if (free_lanes_.empty()) return false;
    id = free_lanes_.front();
    free_lanes_.pop_front();
    return true;
}

void Executor::push_free_lane(uint32_t id) {
    std::lock_guard<std::mutex> lk(free_mu_);
    free_lanes_.push_back(id);
}

Ticket Executor::submit_search(const float* q, uint32_t nq, uint32_t k, uint32_t nprobe) {
    // executor.cpp:128-179
    if (nq < 1 || nq > cfg_.max_search_batch)
        throw Error(BIVF_EINVAL, "submit_search: batch size out of [1, max_search_batch]");
    if (k < 1) throw Error(BIVF_EINVAL, "submit_search: k must be >= 1");
    if (nprobe < 1 || nprobe > index_.C())
        throw Error(BIVF_EINVAL, "submit_search: nprobe out of [1, num_clusters]");
    // the device path's limits (INTEGRATION.md "Limits"), rejected at submission
    // rather than in the lane: the reference accepts any k and nprobe <= C
    if (k > 256) throw Error(BIVF_EINVAL, "submit_search: k above the device top-k capacity (256)");
    if (nprobe > 256 && nprobe != index_.C())
        throw Error(BIVF_EINVAL, "submit_search: nprobe must be <= 256 or == num_clusters");
    Ticket t = make_ticket(RequestType::Search);
    if (!accepting_.load()) {
        t->start = t->end = Clock::now();
        resolve(t, TicketStatus::Error, "executor is shut down");
        return t;
    }
    auto task = std::make_unique<SearchTask>();
    task->t = t;
    task->q.assign(q, q + (size_t)nq * index_.D());
    task->nq = nq;
    task->k = k;
    task->nprobe = nprobe;
    if (cfg_.serialized) {
        in_flight_.fetch_add(1);
        {
            std::lock_guard<std::mutex> lk(serial_mu_);
            serial_queue_.push_back({RequestType::Search, std::move(task), nullptr});
        }
        serial_cv_.notify_one();
        return t;
    }
    uint32_t lane;
    if (!pop_free_lane(lane)) {
        reject(t, "all search lanes busy");  // fail fast, never queue
        return t;
    }
    in_flight_.fetch_add(1);
    Lane& L = *lanes_[lane];
    {
        std::lock_guard<std::mutex> lk(L.mu);
        L.task = std::move(task);
    }
    L.cv.notify_one();
    return t;
}

Ticket Executor::submit_insert(const float* x, uint64_t n, const int64_t* ids) {
    // executor.cpp:181-222
    if (n < 1) throw Error(BIVF_EINVAL, "submit_insert: empty batch");
    Ticket t = make_ticket(RequestType::Insert);
    if (!accepting_.load()) {
        t->start = t->end = Clock::now();
        resolve(t, TicketStatus::Error, "executor is shut down");
        return t;
    }
    auto item = std::make_shared<PendingInsert>();
    item->t = t;
    item->x.assign(x, x + n * index_.D());
    if (ids) item->ids.assign(ids, ids + n);
    item->count = n;
    t->ids.assign(n, -1);
    in_flight_.fetch_add(1);
    if (cfg_.serialized) {
        {
            std::lock_guard<std::mutex> lk(serial_mu_);
            serial_queue_.push_back({RequestType::Insert, nullptr, std::move(item)});
        }
        serial_cv_.notify_one();
        return t;
    }
    {
        std::lock_guard<std::mutex> lk(batch_mu_);
        pending_.push_back(std::move(item));
        pending_vectors_ += n;
    }
    batch_cv_.notify_one();
    return t;
}

void Executor::flush_insertions() {
    {
        std::lock_guard<std::mutex> lk(batch_mu_);
        if (pending_.empty()) return;
        manual_flush_ = true;
    }
    batch_cv_.notify_one();
}

void Executor::set_mode(bool serialized) {
    if (in_flight_.load() != 0) throw Error(BIVF_ELOGIC, "set_mode: executor is busy");
    cfg_.serialized = serialized;
}

void Executor::lane_main(uint32_t id) {
    Lane& L = *lanes_[id];
    for (;;) {
        std::unique_ptr<SearchTask> task;
        {
            std::unique_lock<std::mutex> lk(L.mu);
            L.cv.wait(lk, [&] { return L.stop || L.task; });
            if (L.stop && !L.task) return;
            task = std::move(L.task);
        }
        if (L.busy.exchange(true)) double_hold_.fetch_add(1);
        run_search(*task, (int)id);
        // hand the lane back before resolving (executor.cpp:253-256)
        L.busy.store(false);
        push_free_lane(id);
        in_flight_.fetch_sub(1);
        resolve(task->t, task->t->error.empty() ? TicketStatus::Done : TicketStatus::Error,
                task->t->error);
    }
}

void Executor::run_search(SearchTask& task, int lane) {
    Ticket& t = task.t;
    t->lane = lane;
    t->start = Clock::now();
    // two-tier scratch: a central grant backs requests whose candidate volume
    // exceeds the lane cache (executor.cpp:267-284)
    const uint64_t clusters = std::max<uint64_t>(index_.C(), 1);
    const uint64_t avg_list = index_.size() / clusters + 1;
    const uint64_t demand = (uint64_t)task.nq * task.nprobe * avg_list * kCandidateRecordBytes;
    bool grant = false;
    if (demand > cfg_.lane_cache_bytes) {
        uint64_t avail = grants_available_.load();
        while (avail > 0 && !grants_available_.compare_exchange_weak(avail, avail - 1)) {
        }
        if (avail > 0) {
            grant = true;
            grants_outstanding_.fetch_add(1);
            grants_total_.fetch_add(1);
        }
    }
    try {
        t->nq = task.nq;
        t->k = task.k;
        t->ids.resize((size_t)task.nq * task.k);
        t->dists.resize((size_t)task.nq * task.k);
        t->counts.resize(task.nq);
        index_.search(task.q.data(), task.nq, task.k, task.nprobe, t->ids.data(), t->dists.data(),
                      t->counts.data());
    } catch (const std::exception& e) {
        t->error = e.what();
    }
    if (grant) {
        grants_available_.fetch_add(1);
        grants_outstanding_.fetch_sub(1);
    }
    t->end = Clock::now();
}

void Executor::flush_locked(std::unique_lock<std::mutex>& lk) {
    // executor.cpp:331-413
    if (pending_.empty()) return;
    struct Part {
        std::shared_ptr<PendingInsert> item;
        uint64_t from, count, batch_from;
    };
    const uint32_t D = index_.D();
    std::vector<Part> parts;
    std::vector<float> batch;
    std::vector<int64_t> batch_ids;
    const bool with_ids = !pending_.front()->ids.empty();
    uint64_t taken = 0;
    while (!pending_.empty() && taken < cfg_.batch_cap) {
        auto item = pending_.front();
        if ((!item->ids.empty()) != with_ids) break;  // one id-mode per batch
        const uint64_t avail = item->count - item->flushed;
        const uint64_t take = std::min<uint64_t>(avail, cfg_.batch_cap - taken);
        batch.insert(batch.end(), item->x.begin() + item->flushed * D,
                     item->x.begin() + (item->flushed + take) * D);
        if (with_ids)
            batch_ids.insert(batch_ids.end(), item->ids.begin() + item->flushed,
                             item->ids.begin() + item->flushed + take);
        parts.push_back({item, item->flushed, take, taken});
        item->flushed += take;
        taken += take;
        if (item->flushed == item->count) pending_.pop_front();
        else break;  // cap hit mid-request
    }
    pending_vectors_ -= taken;
    uint64_t prev = largest_flush_.load();
    while (taken > prev && !largest_flush_.compare_exchange_weak(prev, taken)) {
    }
    lk.unlock();
    const auto start = Clock::now();
    std::vector<int64_t> out(taken, -1);
    bool failed = false;
    std::string error;
    try {
        index_.insert(batch.data(), taken, with_ids ? batch_ids.data() : nullptr, out.data());
        index_.rearrange_sweep();  // post_insert_maintenance (ivf_index.hpp:82)
    } catch (const std::exception& e) {
        failed = true;
        error = e.what();
    }
    const auto end = Clock::now();
    for (auto& p : parts) {
        auto& it = *p.item;
        if (failed) {
            it.failed = true;
            it.error = error;
        } else {
            for (uint64_t i = 0; i < p.count; ++i) it.t->ids[p.from + i] = out[p.batch_from + i];
        }
        it.completed += p.count;
        if (it.completed == it.count) {
            it.t->lane = (int)cfg_.num_lanes;  // the dedicated data lane
            it.t->start = start;
            it.t->end = end;
            in_flight_.fetch_sub(1);
            resolve(it.t, it.failed ? TicketStatus::Error : TicketStatus::Done, it.error);
        }
    }
    lk.lock();
}

void Executor::insertion_main() {
    // executor.cpp:415-445
    std::unique_lock<std::mutex> lk(batch_mu_);
    last_flush_ = Clock::now();
    for (;;) {
        if (stopping_.load() && pending_.empty()) return;
        if (pending_vectors_ == 0 && !manual_flush_) {
            batch_cv_.wait(lk, [&] { return stopping_.load() || pending_vectors_ > 0 || manual_flush_; });
            last_flush_ = Clock::now();
            continue;
        }
        const auto deadline = last_flush_ + std::chrono::milliseconds(cfg_.flush_interval_ms);
        if (pending_vectors_ < cfg_.batch_multiple && !manual_flush_ && !stopping_.load()) {
            batch_cv_.wait_until(lk, deadline, [&] {
                return stopping_.load() || manual_flush_ || pending_vectors_ >= cfg_.batch_multiple;
            });
        }
        const bool timer_due = Clock::now() >= deadline;
        if (pending_vectors_ >= cfg_.batch_multiple || manual_flush_ || timer_due ||
            stopping_.load()) {
            manual_flush_ = false;
            while (!pending_.empty()) flush_locked(lk);
            last_flush_ = Clock::now();
        }
    }
}

void Executor::serial_main() {
    // executor.cpp:447-472: FIFO on one lane
    for (;;) {
        SerialTask task;
        {
            std::unique_lock<std::mutex> lk(serial_mu_);
            serial_cv_.wait(lk, [&] { return stopping_.load() || !serial_queue_.empty(); });
            if (serial_queue_.empty()) {
                if (stopping_.load()) return;
                continue;
            }
            task = std::move(serial_queue_.front());
            serial_queue_.pop_front();
        }
        if (task.type == RequestType::Search) {
            run_search(*task.search, 0);
            in_flight_.fetch_sub(1);
            resolve(task.search->t,
                    task.search->t->error.empty() ? TicketStatus::Done : TicketStatus::Error,
                    task.search->t->error);
        } else {
            auto& it = *task.insert;
            it.t->lane = 0;
            it.t->start = Clock::now();
            std::string err;
            try {
                index_.insert(it.x.data(), it.count, it.ids.empty() ? nullptr : it.ids.data(),
                              it.t->ids.data());
                index_.rearrange_sweep();
            } catch (const std::exception& e) {
                err = e.what();
            }
            it.t->end = Clock::now();
            in_flight_.fetch_sub(1);
            resolve(it.t, err.empty() ? TicketStatus::Done : TicketStatus::Error, err);
        }
    }
}

void Executor::shutdown() {
    bool expected = true;
    if (!accepting_.compare_exchange_strong(expected, false)) return;
    stopping_.store(true);
    batch_cv_.notify_all();
    serial_cv_.notify_all();
    if (insertion_thread_.joinable()) insertion_thread_.join();
    if (serial_thread_.joinable()) serial_thread_.join();
    for (auto& l : lanes_) {
        {
            std::lock_guard<std::mutex> lk(l->mu);
            l->stop = true;
        }
        l->cv.notify_one();
    }
    for (auto& l : lanes_)
        if (l->worker.joinable()) l->worker.join();
}

void Executor::stats(uint64_t out[8]) const {
    out[0] = rejected_.load();
    out[1] = completed_.load();
    out[2] = in_flight_.load();
    out[3] = grants_outstanding_.load();
    out[4] = grants_total_.load();
    out[5] = lane_cache_allocations_;
    out[6] = double_hold_.load();
    out[7] = largest_flush_.load();
}

ReplayOut replay(Executor& ex, const ReplaySpec& spec, const float* queries, uint64_t nqueries,
                 const float* inserts, uint64_t ninserts) {
    // WorkloadSpec::validate (workload.cpp:17-25)
    if (spec.qps_search < 0 || spec.qps_insert < 0) throw Error(BIVF_EINVAL, "replay: rates must be >= 0");
    if (spec.duration_s <= 0) throw Error(BIVF_EINVAL, "replay: duration must be > 0");
    if (spec.search_batch < 1 || spec.search_batch > 10)
        throw Error(BIVF_EINVAL, "replay: search_batch out of [1, 10]");
    if (spec.insert_batch < 1) throw Error(BIVF_EINVAL, "replay: insert_batch must be >= 1");
    if (spec.qps_search > 0 && nqueries == 0) throw Error(BIVF_EINVAL, "replay: no queries");
    if (spec.qps_insert > 0 && ninserts == 0) throw Error(BIVF_EINVAL, "replay: no insertion vectors");
    struct Ev {
        double at;
        bool search;
    };
    std::vector<Ev> evs;
    std::mt19937_64 rng(spec.seed);
    auto schedule = [&](double qps, bool s) {  // workload.cpp:136-146
        if (qps <= 0) return;
        std::exponential_distribution<double> gap(qps);
        double t = 0;
        for (;;) {
            t += spec.poisson ? gap(rng) : 1.0 / qps;
            if (t >= spec.duration_s) break;
            evs.push_back({t, s});
        }
    };
    schedule(spec.qps_search, true);
    schedule(spec.qps_insert, false);
    std::stable_sort(evs.begin(), evs.end(), [](const Ev& a, const Ev& b) { return a.at < b.at; });
    const uint32_t D = ex.index().D();
    std::vector<float> qb((size_t)spec.search_batch * D), ib((size_t)spec.insert_batch * D);
    std::vector<std::pair<Ticket, bool>> issued;
    issued.reserve(evs.size());
    uint64_t qc = 0, ic = 0;
    const auto t0 = Clock::now();
    for (const Ev& e : evs) {
        std::this_thread::sleep_until(t0 + std::chrono::duration_cast<Clock::duration>(
                                               std::chrono::duration<double>(e.at)));
        if (e.search) {
            for (uint32_t i = 0; i < spec.search_batch; ++i, ++qc)
                std::memcpy(qb.data() + (size_t)i * D, queries + (qc % nqueries) * D, D * 4);
            issued.push_back({ex.submit_search(qb.data(), spec.search_batch, spec.k, spec.nprobe), true});
        } else {
            for (uint32_t i = 0; i < spec.insert_batch; ++i, ++ic)
                std::memcpy(ib.data() + (size_t)i * D, inserts + (ic % ninserts) * D, D * 4);
            issued.push_back({ex.submit_insert(ib.data(), spec.insert_batch, nullptr), false});
        }
    }
    ex.flush_insertions();
    ReplayOut out;
    for (auto& it : issued) {
        it.first->wait();
        const auto st = it.first->status;
        double v = it.first->latency_us();
        if (st == TicketStatus::Rejected) {
            ++out.rejected;
            v = -1;
        } else if (st == TicketStatus::Error) {
            ++out.errors;
            v = -2;
        }
        (it.second ? out.search_us : out.insert_us).push_back(v);
    }
    return out;
}

}  // namespace bivf
