// group.cpp -- single-process multi-GPU driver (prx_group_*, include/prx.h).
//
// The reference's one Engine object over a machine's GPUs: the paths are split into
// contiguous shards (one engine each, on the given devices), the engines are attached to the
// in-process local collectives (comm.cpp) and every frame is each engine's own prx_run_frame,
// run concurrently by one persistent host thread per shard -- the exchanges happen inside the
// engines, so the frame is bit-identical to one engine and has one read-back per shard.
#include "group.h"

namespace prx {

EngineGroup::EngineGroup(std::vector<Engine*> engines, std::vector<std::unique_ptr<Comm>> comms)
    : engines_(std::move(engines)), comms_(std::move(comms)) {
    for (size_t r = 0; r < engines_.size(); ++r) {
        prx_collectives t{};
        comms_[r]->table(&t);
        engines_[r]->set_collectives(&t);
    }
    errors_.resize(engines_.size());
    for (size_t r = 0; r < engines_.size(); ++r) threads_.emplace_back(&EngineGroup::worker, this, static_cast<int>(r));
}

EngineGroup::~EngineGroup() {
    {
        std::lock_guard<std::mutex> lk(m_);
        stop_ = true;
    }
    cv_task_.notify_all();
    for (std::thread& t : threads_) t.join();
}

void EngineGroup::worker(int rank) {
    uint64_t seen = 0;
    for (;;) {
        std::function<void(int, Engine&)> task;
        {
            std::unique_lock<std::mutex> lk(m_);
            cv_task_.wait(lk, [&] { return stop_ || generation_ != seen; });
            if (stop_) return;
            seen = generation_;
            task = task_;
        }
        std::exception_ptr err;
        try {
            task(rank, *engines_[rank]);
        } catch (...) {
            err = std::current_exception();
        }
        std::lock_guard<std::mutex> lk(m_);
        errors_[rank] = err;
        if (--pending_ == 0) cv_done_.notify_all();
    }
}

void EngineGroup::run_all(const std::function<void(int, Engine&)>& fn) {
    std::unique_lock<std::mutex> lk(m_);
    task_ = fn;
    pending_ = static_cast<int>(engines_.size());
    ++generation_;
    cv_task_.notify_all();
    cv_done_.wait(lk, [&] { return pending_ == 0; });
    for (const std::exception_ptr& e : errors_)
        if (e) std::rethrow_exception(e);
}

}  // namespace prx
