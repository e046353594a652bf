// Transports of the mesh-partitioned multi-GPU schedule (see dist.h).
#include "dist.h"

#include <dlfcn.h>

#include <condition_variable>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <tuple>

namespace mrab {

// ------------------------------------------------------------------------------------
// NCCL through dlopen (ABI of nccl.h 2.x: opaque comm, 128-byte unique id, int results)
// ------------------------------------------------------------------------------------
namespace {
struct NcclApi {
    typedef struct { char internal[128]; } UniqueId;
    void* lib = nullptr;
    int (*GetUniqueId)(UniqueId*) = nullptr;
    int (*CommInitRank)(void**, int, UniqueId, int) = nullptr;
    int (*CommDestroy)(void*) = nullptr;
    int (*Send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*Recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*GroupStart)() = nullptr;
    int (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(int) = nullptr;
    bool load(std::string* err) {
        if (lib) return true;
        lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) {
            if (err) *err = std::string("libnccl not found: ") + dlerror();
            return false;
        }
        auto sym = [&](const char* n) { return dlsym(lib, n); };
        GetUniqueId = (decltype(GetUniqueId))sym("ncclGetUniqueId");
        CommInitRank = (decltype(CommInitRank))sym("ncclCommInitRank");
        CommDestroy = (decltype(CommDestroy))sym("ncclCommDestroy");
        Send = (decltype(Send))sym("ncclSend");
        Recv = (decltype(Recv))sym("ncclRecv");
        GroupStart = (decltype(GroupStart))sym("ncclGroupStart");
        GroupEnd = (decltype(GroupEnd))sym("ncclGroupEnd");
        GetErrorString = (decltype(GetErrorString))sym("ncclGetErrorString");
        if (!GetUniqueId || !CommInitRank || !Send || !Recv || !GroupStart || !GroupEnd) {
            if (err) *err = "libnccl lacks a required symbol";
            return false;
        }
        return true;
    }
};
NcclApi& nccl() {
    static NcclApi a;
    return a;
}

struct NcclTransport : Transport {
    void* comm = nullptr;
    bool ck(int r, const char* what) {
        if (r == 0) return true;
        err = std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error");
        return false;
    }
    ~NcclTransport() override {
        if (comm && nccl().CommDestroy) nccl().CommDestroy(comm);
    }
    bool begin() override { return ck(nccl().GroupStart(), "ncclGroupStart"); }
    // bytes as ncclInt8 (= 0)
    bool send(const void* dev, size_t bytes, int peer, int, cudaStream_t st) override {
        return ck(nccl().Send(dev, bytes, 0, peer, comm, st), "ncclSend");
    }
    bool recv(void* dev, size_t bytes, int peer, int, cudaStream_t st) override {
        return ck(nccl().Recv(dev, bytes, 0, peer, comm, st), "ncclRecv");
    }
    bool end(cudaStream_t) override { return ck(nccl().GroupEnd(), "ncclGroupEnd"); }
};
}  // namespace

bool nccl_unique_id(void* out128, std::string* err) {
    if (!nccl().load(err)) return false;
    NcclApi::UniqueId id;
    const int r = nccl().GetUniqueId(&id);
    if (r != 0) {
        if (err) *err = "ncclGetUniqueId failed";
        return false;
    }
    std::memcpy(out128, &id, 128);
    return true;
}

std::unique_ptr<Transport> make_nccl_transport(const void* unique_id, int rank, int nranks, std::string* err) {
    if (!nccl().load(err)) return nullptr;
    std::unique_ptr<NcclTransport> t(new NcclTransport());
    NcclApi::UniqueId id;
    std::memcpy(&id, unique_id, 128);
    const int r = nccl().CommInitRank(&t->comm, nranks, id, rank);
    if (r != 0) {
        if (err) *err = std::string("ncclCommInitRank: ") + (nccl().GetErrorString ? nccl().GetErrorString(r) : "error");
        return nullptr;
    }
    return t;
}

// ------------------------------------------------------------------------------------
// loopback: sends are buffered (device copy into a hub-owned buffer, event recorded), receives
// block the calling host thread until the matching send has been posted, then wait on its event
// in stream order.  Messages of one (source, destination, tag) are matched in FIFO order.
// ------------------------------------------------------------------------------------
namespace {
struct Hub {
    struct Msg {
        void* buf;
        size_t bytes;
        cudaEvent_t ev;
    };
    std::mutex mu;
    std::condition_variable cv;
    std::map<std::tuple<int, int, int>, std::deque<Msg>> box;
};
std::mutex g_hub_mu;
std::map<int, std::shared_ptr<Hub>> g_hubs;

struct LoopbackTransport : Transport {
    std::shared_ptr<Hub> hub;
    int rank = 0;
    bool begin() override { return true; }
    bool send(const void* dev, size_t bytes, int peer, int tag, cudaStream_t st) override {
        Hub::Msg m{nullptr, bytes, nullptr};
        if (cudaMalloc(&m.buf, bytes) != cudaSuccess || cudaEventCreateWithFlags(&m.ev, cudaEventDisableTiming) != cudaSuccess ||
            cudaMemcpyAsync(m.buf, dev, bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess ||
            cudaEventRecord(m.ev, st) != cudaSuccess) {
            err = "loopback send failed";
            return false;
        }
        {
            std::lock_guard<std::mutex> l(hub->mu);
            hub->box[std::make_tuple(rank, peer, tag)].push_back(m);
        }
        hub->cv.notify_all();
        return true;
    }
    bool recv(void* dev, size_t bytes, int peer, int tag, cudaStream_t st) override {
        Hub::Msg m;
        {
            std::unique_lock<std::mutex> l(hub->mu);
            auto key = std::make_tuple(peer, rank, tag);
            hub->cv.wait(l, [&] { return !hub->box[key].empty(); });
            m = hub->box[key].front();
            hub->box[key].pop_front();
        }
        if (m.bytes != bytes) {
            err = "loopback recv: size mismatch";
            return false;
        }
        if (cudaStreamWaitEvent(st, m.ev, 0) != cudaSuccess ||
            cudaMemcpyAsync(dev, m.buf, bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess) {
            err = "loopback recv failed";
            return false;
        }
        // the buffer is released once the copy has run
        cudaStreamSynchronize(st);
        cudaFree(m.buf);
        cudaEventDestroy(m.ev);
        return true;
    }
    bool end(cudaStream_t) override { return true; }
};
}  // namespace

std::unique_ptr<Transport> make_loopback_transport(int world_id, int rank, int) {
    std::unique_ptr<LoopbackTransport> t(new LoopbackTransport());
    {
        std::lock_guard<std::mutex> l(g_hub_mu);
        auto& h = g_hubs[world_id];
        if (!h) h = std::make_shared<Hub>();
        t->hub = h;
    }
    t->rank = rank;
    return t;
}

}  // namespace mrab
