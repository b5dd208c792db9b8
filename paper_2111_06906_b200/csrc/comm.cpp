// comm.cpp -- collective backends for path-sharded engines (include/prx.h).
//
// An engine with a prx_collectives table enqueues its frame's exchanges (DM_C all-reduce,
// prune-count and dead-slot all-gathers, counter and image all-reduces) on its own stream
// between its kernels, so a sharded frame has the single-engine frame's one host read-back.
// Two backends implement the table:
//   * NCCL (one rank per process or per device): libnccl is loaded at run time (dlopen), so
//     _prx.so has no link dependency on it; every call is an ncclAllReduce / ncclAllGather
//     on the caller's stream.
//   * local: `world` engines driven by `world` host threads of one process (any mix of
//     devices, including several shards on one device -- the GPU tests' configuration).
//     Each collective is two host barriers and stream-ordered device work: the ranks publish
//     their buffers and an event, wait on every peer's event, reduce (kernel over peer
//     pointers) or copy (peer memcpy) into their own destination, and publish a second event
//     so no buffer is overwritten before every peer has read it.  No kernel ever waits on
//     another rank's kernel; ordering is by events only.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "comm.h"
#include "engine.h"

namespace prx {

// ------------------------------------------------------------------------------ NCCL
namespace {

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static std::once_flag once;
    static NcclApi api;
    static std::string err;
    std::call_once(once, [] {
        const char* env = std::getenv("PRX_NCCL_LIB");
        void* h = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = std::string("cannot load NCCL (") + (env ? env : "libnccl.so.2") + "): " + dlerror();
            return;
        }
        auto sym = [&](const char* name) {
            void* p = dlsym(h, name);
            if (!p) err = std::string("NCCL symbol missing: ") + name;
            return p;
        };
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
        api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
        api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
        api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(sym("ncclAllReduce"));
        api.all_gather = reinterpret_cast<decltype(api.all_gather)>(sym("ncclAllGather"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
    });
    if (!err.empty()) throw std::runtime_error(err);
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw std::runtime_error(std::string(what) + ": " + nccl().error_string(r));
}

}  // namespace

struct NcclComm final : Comm {
    ncclComm_t comm = nullptr;
    int device = 0;

    ~NcclComm() override {
        if (comm) nccl().comm_destroy(comm);
    }
    static int reduce(void* ctx, void* buf, size_t n, ncclDataType_t t, void* stream) {
        auto* c = static_cast<NcclComm*>(ctx);
        return nccl().all_reduce(buf, buf, n, t, ncclSum, c->comm, static_cast<cudaStream_t>(stream)) == ncclSuccess
                   ? 0
                   : 1;
    }
    void table(prx_collectives* out) override {
        out->ctx = this;
        out->rank = rank;
        out->world = world;
        out->all_reduce_sum_u32 = [](void* ctx, uint32_t* b, size_t n, void* s) { return reduce(ctx, b, n, ncclUint32, s); };
        out->all_reduce_sum_u64 = [](void* ctx, uint64_t* b, size_t n, void* s) { return reduce(ctx, b, n, ncclUint64, s); };
        out->all_reduce_sum_f32 = [](void* ctx, float* b, size_t n, void* s) { return reduce(ctx, b, n, ncclFloat32, s); };
        out->all_gather_u32 = [](void* ctx, const uint32_t* send, uint32_t* recv, size_t n, void* s) {
            auto* c = static_cast<NcclComm*>(ctx);
            return nccl().all_gather(send, recv, n, ncclUint32, c->comm, static_cast<cudaStream_t>(s)) == ncclSuccess
                       ? 0
                       : 1;
        };
    }
};

void nccl_unique_id(uint8_t out[128]) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof(id));
}

std::unique_ptr<Comm> nccl_comm(const uint8_t id[128], int rank, int world, int device) {
    if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("nccl comm: bad rank / world");
    auto c = std::make_unique<NcclComm>();
    c->rank = rank;
    c->world = world;
    c->device = device;
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    PRX_CUDA(cudaSetDevice(device));
    nccl_check(nccl().comm_init_rank(&c->comm, world, uid, rank), "ncclCommInitRank");
    return c;
}

// ------------------------------------------------------------------------------ local
struct LocalShared {
    int world = 0;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t generation = 0;
    struct Slot {
        const void* buf = nullptr;
        cudaEvent_t ev_a = nullptr, ev_b = nullptr;
    };
    std::vector<Slot> slots;

    void barrier() {
        std::unique_lock<std::mutex> lk(m);
        const uint64_t gen = generation;
        if (++arrived == world) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != gen; });
        }
    }
};

struct LocalComm final : Comm {
    std::shared_ptr<LocalShared> sh;
    cudaEvent_t ev_a = nullptr, ev_b = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    int tmp_device = -1;
    bool peers_checked = false;

    ~LocalComm() override {
        if (ev_a) cudaEventDestroy(ev_a);
        if (ev_b) cudaEventDestroy(ev_b);
        if (tmp) cudaFree(tmp);
    }

    void ensure(size_t bytes) {
        int dev = 0;
        PRX_CUDA(cudaGetDevice(&dev));
        if (!ev_a) {
            PRX_CUDA(cudaEventCreateWithFlags(&ev_a, cudaEventDisableTiming));
            PRX_CUDA(cudaEventCreateWithFlags(&ev_b, cudaEventDisableTiming));
        }
        if (bytes > tmp_bytes || dev != tmp_device) {
            if (tmp) PRX_CUDA(cudaFree(tmp));
            PRX_CUDA(cudaMalloc(&tmp, bytes));
            tmp_bytes = bytes;
            tmp_device = dev;
        }
    }

    // phase A: publish `buf` + an event after this rank's producers; wait on every peer's
    void publish_and_wait(const void* buf, cudaStream_t s) {
        PRX_CUDA(cudaEventRecord(ev_a, s));
        sh->slots[rank].buf = buf;
        sh->slots[rank].ev_a = ev_a;
        sh->barrier();
        if (!peers_checked) enable_peers();
        for (int h = 0; h < world; ++h)
            if (h != rank) PRX_CUDA(cudaStreamWaitEvent(s, sh->slots[h].ev_a, 0));
    }
    // phase B: every peer has finished reading every published buffer
    void finish(cudaStream_t s) {
        PRX_CUDA(cudaEventRecord(ev_b, s));
        sh->slots[rank].ev_b = ev_b;
        sh->barrier();
        for (int h = 0; h < world; ++h)
            if (h != rank) PRX_CUDA(cudaStreamWaitEvent(s, sh->slots[h].ev_b, 0));
    }
    void enable_peers() {  // direct loads of peer buffers across devices
        peers_checked = true;
        int dev = 0, n = 0;
        PRX_CUDA(cudaGetDevice(&dev));
        PRX_CUDA(cudaGetDeviceCount(&n));
        for (int d = 0; d < n; ++d) {
            if (d == dev) continue;
            int ok = 0;
            cudaDeviceCanAccessPeer(&ok, dev, d);
            if (ok) {
                const cudaError_t e = cudaDeviceEnablePeerAccess(d, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) PRX_CUDA(e);
                cudaGetLastError();
            }
        }
    }

    template <typename T>
    int reduce(T* buf, size_t n, void* stream) {
        try {
            const cudaStream_t s = static_cast<cudaStream_t>(stream);
            ensure(sizeof(T) * std::max<size_t>(n, 1));
            publish_and_wait(buf, s);
            const void* peers[kMaxLocalRanks];
            for (int h = 0; h < world; ++h) peers[h] = sh->slots[h].buf;
            launch_local_reduce(peers, world, tmp, n, sizeof(T) == 8 ? 2 : (std::is_same<T, float>::value ? 1 : 0), s);
            finish(s);
            PRX_CUDA(cudaMemcpyAsync(buf, tmp, sizeof(T) * n, cudaMemcpyDeviceToDevice, s));
            return 0;
        } catch (const std::exception&) {
            return 1;
        }
    }
    int gather(const uint32_t* send, uint32_t* recv, size_t n, void* stream) {
        try {
            const cudaStream_t s = static_cast<cudaStream_t>(stream);
            ensure(4);
            publish_and_wait(send, s);
            for (int h = 0; h < world; ++h)
                PRX_CUDA(cudaMemcpyAsync(recv + static_cast<size_t>(h) * n, sh->slots[h].buf, 4 * n,
                                         cudaMemcpyDeviceToDevice, s));
            finish(s);
            return 0;
        } catch (const std::exception&) {
            return 1;
        }
    }

    void table(prx_collectives* out) override {
        out->ctx = this;
        out->rank = rank;
        out->world = world;
        out->all_reduce_sum_u32 = [](void* c, uint32_t* b, size_t n, void* s) { return static_cast<LocalComm*>(c)->reduce(b, n, s); };
        out->all_reduce_sum_u64 = [](void* c, uint64_t* b, size_t n, void* s) { return static_cast<LocalComm*>(c)->reduce(b, n, s); };
        out->all_reduce_sum_f32 = [](void* c, float* b, size_t n, void* s) { return static_cast<LocalComm*>(c)->reduce(b, n, s); };
        out->all_gather_u32 = [](void* c, const uint32_t* send, uint32_t* recv, size_t n, void* s) {
            return static_cast<LocalComm*>(c)->gather(send, recv, n, s);
        };
    }
};

std::vector<std::unique_ptr<Comm>> local_comms(int world) {
    if (world < 1 || world > kMaxLocalRanks) throw std::invalid_argument("local comm: world must be 1..16");
    auto sh = std::make_shared<LocalShared>();
    sh->world = world;
    sh->slots.resize(world);
    std::vector<std::unique_ptr<Comm>> out;
    for (int r = 0; r < world; ++r) {
        auto c = std::make_unique<LocalComm>();
        c->rank = r;
        c->world = world;
        c->sh = sh;
        out.push_back(std::move(c));
    }
    return out;
}

}  // namespace prx
