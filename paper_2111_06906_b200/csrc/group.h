// group.h -- one process driving several path-sharded engines (group.cpp).
#pragma once

#include <condition_variable>
#include <exception>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "comm.h"
#include "engine.h"

namespace prx {

// `world` engines over contiguous path shards (devices may repeat), attached to in-process
// local collectives, each driven by its own persistent host thread: run_all() runs one
// collective call (run_frame, splat, ...) on every engine concurrently and rethrows the first
// error in the caller.
class EngineGroup {
public:
    EngineGroup(std::vector<Engine*> engines, std::vector<std::unique_ptr<Comm>> comms);
    ~EngineGroup();
    EngineGroup(const EngineGroup&) = delete;
    EngineGroup& operator=(const EngineGroup&) = delete;

    int size() const { return static_cast<int>(engines_.size()); }
    void run_all(const std::function<void(int rank, Engine& e)>& fn);

private:
    void worker(int rank);

    std::vector<Engine*> engines_;
    std::vector<std::unique_ptr<Comm>> comms_;
    std::vector<std::thread> threads_;
    std::mutex m_;
    std::condition_variable cv_task_, cv_done_;
    std::function<void(int, Engine&)> task_;
    std::vector<std::exception_ptr> errors_;
    uint64_t generation_ = 0;
    int pending_ = 0;
    bool stop_ = false;
};

}  // namespace prx
