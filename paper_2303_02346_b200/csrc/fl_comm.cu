// fl_comm.cu -- ThreadTransport and NcclTransport (see fl_comm.h).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstring>
#include <string>

#include "fl_comm.h"
#include "fl_host.h"

namespace fl {

// ---------------------------------------------------------------------------
// in-process group
// ---------------------------------------------------------------------------
ThreadGroup::ThreadGroup(int n_) : n(n_), slots(n_) {}

ThreadGroup::~ThreadGroup() {
    for (auto& s : slots) {
        if (s.ready) cudaEventDestroy(s.ready);
        if (s.done) cudaEventDestroy(s.done);
    }
}

void ThreadGroup::barrier() {
    std::unique_lock<std::mutex> lk(m);
    if (aborted) throw FlumeError(FLUME_E_ENGINE, "slab group aborted by a failing rank");
    const long gen = generation;
    if (++arrived == n) {
        arrived = 0;
        generation++;
        cv.notify_all();
        return;
    }
    cv.wait(lk, [&] { return generation != gen || aborted; });
    if (generation == gen) throw FlumeError(FLUME_E_ENGINE, "slab group aborted by a failing rank");
}

void ThreadGroup::abort() {
    std::lock_guard<std::mutex> lk(m);
    aborted = true;
    cv.notify_all();
}

template <class T, int OP>
__global__ void k_stack_reduce(const T* __restrict__ stack, size_t count, int nr, T* __restrict__ out) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < count; i += size_t(gridDim.x) * blockDim.x) {
        T a = stack[i];
        for (int r = 1; r < nr; r++) {  // rank order: identical bits on every rank
            const T b = stack[size_t(r) * count + i];
            if (OP == 0) a = a + b;
            if (OP == 1) a = b < a ? b : a;
            if (OP == 2) a = b > a ? b : a;
        }
        out[i] = a;
    }
}

template <class T>
static void stack_reduce_t(const void* stack, size_t count, int nr, ROp op, void* out, cudaStream_t s) {
    const int grid = int(std::min<size_t>((count + 255) / 256, 1184));
    const T* in = static_cast<const T*>(stack);
    T* o = static_cast<T*>(out);
    if (op == ROp::Sum) k_stack_reduce<T, 0><<<grid, 256, 0, s>>>(in, count, nr, o);
    if (op == ROp::Min) k_stack_reduce<T, 1><<<grid, 256, 0, s>>>(in, count, nr, o);
    if (op == ROp::Max) k_stack_reduce<T, 2><<<grid, 256, 0, s>>>(in, count, nr, o);
}

void launch_stack_reduce(const void* stack, size_t count, int nr, DType t, ROp op, void* out, cudaStream_t s) {
    if (count == 0) return;
    if (t == DType::F64) stack_reduce_t<double>(stack, count, nr, op, out, s);
    if (t == DType::U64) stack_reduce_t<unsigned long long>(stack, count, nr, op, out, s);
    if (t == DType::I32) stack_reduce_t<int>(stack, count, nr, op, out, s);
}

static size_t dtype_size(DType t) { return t == DType::I32 ? 4 : 8; }

namespace {

struct ThreadTransport final : Transport {
    std::shared_ptr<ThreadGroup> g;
    int r, dev;
    DevArr<unsigned char> stack;
    ThreadTransport(std::shared_ptr<ThreadGroup> grp, int rank_, int device) : g(std::move(grp)), r(rank_), dev(device) {
        auto& s = g->slots[r];
        s.device = dev;
        CK(cudaEventCreateWithFlags(&s.ready, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
    }
    int rank() const override { return r; }
    int size() const override { return g->n; }
    void barrier() override { g->barrier(); }
    void abort() override { g->abort(); }

    void exchange_counts(const long send[2], long recv[2], cudaStream_t) override {
        auto& me = g->slots[r];
        me.counts[0] = send[0];
        me.counts[1] = send[1];
        g->barrier();
        recv[0] = r > 0 ? g->slots[r - 1].counts[1] : 0;
        recv[1] = r + 1 < g->n ? g->slots[r + 1].counts[0] : 0;
        g->barrier();
    }

    void neighbor_exchange(const void* const sbuf[2], const size_t sbytes[2], void* const rbuf[2],
                           const size_t rbytes[2], cudaStream_t s) override {
        auto& me = g->slots[r];
        for (int d = 0; d < 2; d++) {
            me.sbuf[d] = sbuf[d];
            me.sbytes[d] = sbytes[d];
        }
        CK(cudaEventRecord(me.ready, s));
        g->barrier();
        for (int d = 0; d < 2; d++) {
            const int peer = d == 0 ? r - 1 : r + 1;
            if (peer < 0 || peer >= g->n || rbytes[d] == 0) continue;
            const auto& p = g->slots[peer];
            if (p.sbytes[1 - d] != rbytes[d])
                throw FlumeError(FLUME_E_ENGINE, "slab exchange: message size mismatch between ranks");
            CK(cudaStreamWaitEvent(s, p.ready, 0));
            CK(cudaMemcpyPeerAsync(rbuf[d], dev, p.sbuf[1 - d], p.device, rbytes[d], s));
        }
        CK(cudaEventRecord(me.done, s));
        g->barrier();
        // do not let this rank overwrite its send buffers before the peers copied them
        for (int d = 0; d < 2; d++) {
            const int peer = d == 0 ? r - 1 : r + 1;
            if (peer < 0 || peer >= g->n || sbytes[d] == 0) continue;
            CK(cudaStreamWaitEvent(s, g->slots[peer].done, 0));
        }
    }

    void allreduce(void* buf, size_t count, DType t, ROp op, cudaStream_t s) override {
        const size_t bytes = count * dtype_size(t);
        auto& me = g->slots[r];
        me.red = buf;
        me.red_bytes = bytes;
        stack.alloc(bytes * size_t(g->n));
        CK(cudaEventRecord(me.ready, s));
        g->barrier();
        for (int q = 0; q < g->n; q++) {
            const auto& p = g->slots[q];
            if (p.red_bytes != bytes) throw FlumeError(FLUME_E_ENGINE, "slab all-reduce: size mismatch");
            if (q != r) CK(cudaStreamWaitEvent(s, p.ready, 0));
            if (bytes) CK(cudaMemcpyPeerAsync(stack.p + size_t(q) * bytes, dev, p.red, p.device, bytes, s));
        }
        CK(cudaEventRecord(me.done, s));
        g->barrier();
        for (int q = 0; q < g->n; q++)
            if (q != r) CK(cudaStreamWaitEvent(s, g->slots[q].done, 0));
        launch_stack_reduce(stack.p, count, g->n, t, op, buf, s);
        CK(cudaGetLastError());
    }
};

// ---------------------------------------------------------------------------
// NCCL (dlopen'ed; only the handful of entry points the slabs use)
// ---------------------------------------------------------------------------
typedef struct ncclComm* ncclComm_t;
struct ncclUniqueId {
    char internal[128];
};
enum { nccl_Int32 = 2, nccl_Uint8 = 1, nccl_Uint64 = 5, nccl_Float64 = 8 };
enum { nccl_Sum = 0, nccl_Max = 2, nccl_Min = 3 };

struct NcclApi {
    void* h = nullptr;
    int (*GetUniqueId)(ncclUniqueId*) = nullptr;
    int (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    int (*CommDestroy)(ncclComm_t) = nullptr;
    int (*GroupStart)() = nullptr;
    int (*GroupEnd)() = nullptr;
    int (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    int (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    int (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(int) = nullptr;
    static NcclApi& get() {
        static NcclApi api;
        static std::once_flag once;
        std::call_once(once, [] { api.load(); });
        if (!api.h) throw FlumeError(FLUME_E_CUDA, "libnccl.so.2 not found (multi-process slabs need NCCL)");
        return api;
    }
    void load() {
        h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        auto sym = [&](const char* n) { return dlsym(h, n); };
        GetUniqueId = reinterpret_cast<decltype(GetUniqueId)>(sym("ncclGetUniqueId"));
        CommInitRank = reinterpret_cast<decltype(CommInitRank)>(sym("ncclCommInitRank"));
        CommDestroy = reinterpret_cast<decltype(CommDestroy)>(sym("ncclCommDestroy"));
        GroupStart = reinterpret_cast<decltype(GroupStart)>(sym("ncclGroupStart"));
        GroupEnd = reinterpret_cast<decltype(GroupEnd)>(sym("ncclGroupEnd"));
        Send = reinterpret_cast<decltype(Send)>(sym("ncclSend"));
        Recv = reinterpret_cast<decltype(Recv)>(sym("ncclRecv"));
        AllReduce = reinterpret_cast<decltype(AllReduce)>(sym("ncclAllReduce"));
        GetErrorString = reinterpret_cast<decltype(GetErrorString)>(sym("ncclGetErrorString"));
        if (!GetUniqueId || !CommInitRank || !CommDestroy || !GroupStart || !GroupEnd || !Send || !Recv ||
            !AllReduce)
            h = nullptr;
    }
};

#define NK(expr)                                                                                   \
    do {                                                                                           \
        int r_ = (expr);                                                                           \
        if (r_ != 0)                                                                               \
            throw FlumeError(FLUME_E_CUDA, std::string("nccl: ") +                                 \
                                               (api.GetErrorString ? api.GetErrorString(r_) : "?") + \
                                               " at " + __FILE__ + ":" + std::to_string(__LINE__)); \
    } while (0)

struct NcclTransport final : Transport {
    ncclComm_t comm = nullptr;
    int r, n;
    DevArr<long> cnt;
    NcclTransport(const unsigned char uid[128], int rank_, int nranks, int device) : r(rank_), n(nranks) {
        NcclApi& api = NcclApi::get();
        CK(cudaSetDevice(device));
        ncclUniqueId id;
        std::memcpy(id.internal, uid, 128);
        NK(api.CommInitRank(&comm, n, id, r));
        cnt.alloc(4);
    }
    ~NcclTransport() override {
        if (comm) NcclApi::get().CommDestroy(comm);
    }
    int rank() const override { return r; }
    int size() const override { return n; }
    void barrier() override {
        // an all-reduce of one int on a private stream is the barrier
        NcclApi& api = NcclApi::get();
        cudaStream_t s;
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        NK(api.AllReduce(cnt.p, cnt.p, 1, nccl_Int32, nccl_Sum, comm, s));
        CK(cudaStreamSynchronize(s));
        CK(cudaStreamDestroy(s));
    }
    void exchange_counts(const long send[2], long recv[2], cudaStream_t s) override {
        NcclApi& api = NcclApi::get();
        long h[4] = {send[0], send[1], 0, 0};
        CK(cudaMemcpyAsync(cnt.p, h, 2 * sizeof(long), cudaMemcpyHostToDevice, s));
        NK(api.GroupStart());
        if (r > 0) {
            NK(api.Send(cnt.p, sizeof(long), nccl_Uint8, r - 1, comm, s));
            NK(api.Recv(cnt.p + 2, sizeof(long), nccl_Uint8, r - 1, comm, s));
        }
        if (r + 1 < n) {
            NK(api.Send(cnt.p + 1, sizeof(long), nccl_Uint8, r + 1, comm, s));
            NK(api.Recv(cnt.p + 3, sizeof(long), nccl_Uint8, r + 1, comm, s));
        }
        NK(api.GroupEnd());
        CK(cudaMemcpyAsync(h, cnt.p, 4 * sizeof(long), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        recv[0] = r > 0 ? h[2] : 0;
        recv[1] = r + 1 < n ? h[3] : 0;
    }
    void neighbor_exchange(const void* const sbuf[2], const size_t sbytes[2], void* const rbuf[2],
                           const size_t rbytes[2], cudaStream_t s) override {
        NcclApi& api = NcclApi::get();
        NK(api.GroupStart());
        for (int d = 0; d < 2; d++) {
            const int peer = d == 0 ? r - 1 : r + 1;
            if (peer < 0 || peer >= n) continue;
            if (sbytes[d]) NK(api.Send(sbuf[d], sbytes[d], nccl_Uint8, peer, comm, s));
            if (rbytes[d]) NK(api.Recv(rbuf[d], rbytes[d], nccl_Uint8, peer, comm, s));
        }
        NK(api.GroupEnd());
    }
    void allreduce(void* buf, size_t count, DType t, ROp op, cudaStream_t s) override {
        NcclApi& api = NcclApi::get();
        if (count == 0) return;
        const int dt = t == DType::F64 ? nccl_Float64 : (t == DType::U64 ? nccl_Uint64 : nccl_Int32);
        const int o = op == ROp::Sum ? nccl_Sum : (op == ROp::Min ? nccl_Min : nccl_Max);
        NK(api.AllReduce(buf, buf, count, dt, o, comm, s));
    }
};

}  // namespace

std::unique_ptr<Transport> make_thread_transport(std::shared_ptr<ThreadGroup> g, int rank, int device) {
    return std::unique_ptr<Transport>(new ThreadTransport(std::move(g), rank, device));
}

std::unique_ptr<Transport> make_nccl_transport(const unsigned char uid[128], int rank, int nranks, int device) {
    return std::unique_ptr<Transport>(new NcclTransport(uid, rank, nranks, device));
}

void nccl_unique_id(unsigned char out[128]) {
    NcclApi& api = NcclApi::get();
    ncclUniqueId id;
    NK(api.GetUniqueId(&id));
    std::memcpy(out, id.internal, 128);
}

}  // namespace fl
