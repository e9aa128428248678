// fl_comm.cu -- ThreadTransport and NcclTransport (see fl_comm.h).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <sys/stat.h>

#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <thread>

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

// ---------------------------------------------------------------------------
// CUDA IPC between the processes of one node (one or more ranks per GPU)
// ---------------------------------------------------------------------------
// Every rank owns two device inboxes (from below / from above) and an all-reduce slot,
// exported with cudaIpcGetMemHandle; peers copy straight into them (NVLink peer copies
// between GPUs, a device copy when two ranks share one) and order everything on the
// device with interprocess events.  The host side is a POSIX shared-memory segment with
// the handles and a sense-reversing barrier -- two host barriers per exchange, no stream
// synchronisation.  Inboxes grow on demand (a new handle and a generation number).

constexpr int kIpcMaxRanks = 64;
constexpr uint32_t kIpcMagic = 0x464c4950u;  // "FLIP"

struct IpcRankShm {
    cudaIpcMemHandle_t inbox[2];
    cudaIpcMemHandle_t red;
    cudaIpcEventHandle_t sent[2], freed[2], red_ready, red_done;
    size_t inbox_cap[2];
    size_t red_cap;
    uint32_t inbox_gen[2], red_gen;
    int device;
    long counts[2];
};

struct IpcShm {
    std::atomic<uint32_t> magic;
    std::atomic<int> arrived;
    std::atomic<long> generation;
    std::atomic<int> aborted;
    std::atomic<int> attached;
    int n;
    IpcRankShm rank[kIpcMaxRanks];
};

struct IpcTransport final : Transport {
    int r, n, dev;
    std::string name;
    IpcShm* shm = nullptr;
    DevArr<unsigned char> inbox[2], red, stack;
    cudaEvent_t ev_sent[2] = {}, ev_freed[2] = {}, ev_red_ready = nullptr, ev_red_done = nullptr;
    // peers' exported objects, opened lazily (by generation)
    struct Peer {
        void* inbox[2] = {nullptr, nullptr};
        uint32_t inbox_gen[2] = {0, 0};
        void* red = nullptr;
        uint32_t red_gen = 0;
        cudaEvent_t sent[2] = {}, freed[2] = {}, red_ready = nullptr, red_done = nullptr;
    };
    std::vector<Peer> peers;

    IpcTransport(const std::string& nm, int rank_, int nranks, int device) : r(rank_), n(nranks), dev(device), name(nm) {
        if (n > kIpcMaxRanks) throw FlumeError(FLUME_E_ARG, "IPC slabs: at most 64 ranks");
        CK(cudaSetDevice(dev));
        const bool creator = r == 0;
        int fd = -1;
        for (int tries = 0; fd < 0; tries++) {
            fd = shm_open(name.c_str(), creator ? (O_CREAT | O_RDWR) : O_RDWR, 0600);
            if (fd < 0) {
                if (creator || tries > 30000) throw FlumeError(FLUME_E_ENGINE, "IPC slabs: shm_open failed: " + name);
                std::this_thread::sleep_for(std::chrono::milliseconds(1));
            }
        }
        if (creator && ftruncate(fd, sizeof(IpcShm)) != 0) {
            close(fd);
            throw FlumeError(FLUME_E_ENGINE, "IPC slabs: ftruncate failed");
        }
        // (the others wait for the creator's size and magic before touching it)
        for (int tries = 0;; tries++) {
            struct stat st {};
            if (fstat(fd, &st) == 0 && size_t(st.st_size) >= sizeof(IpcShm)) break;
            if (tries > 30000) throw FlumeError(FLUME_E_ENGINE, "IPC slabs: shared segment never sized");
            std::this_thread::sleep_for(std::chrono::milliseconds(1));
        }
        void* m = mmap(nullptr, sizeof(IpcShm), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
        close(fd);
        if (m == MAP_FAILED) throw FlumeError(FLUME_E_ENGINE, "IPC slabs: mmap failed");
        shm = static_cast<IpcShm*>(m);
        if (creator) {
            shm->arrived.store(0);
            shm->generation.store(0);
            shm->aborted.store(0);
            shm->attached.store(0);
            shm->n = n;
            shm->magic.store(kIpcMagic, std::memory_order_release);
        } else {
            for (int tries = 0; shm->magic.load(std::memory_order_acquire) != kIpcMagic; tries++) {
                if (tries > 30000) throw FlumeError(FLUME_E_ENGINE, "IPC slabs: group never initialised");
                std::this_thread::sleep_for(std::chrono::milliseconds(1));
            }
        }
        IpcRankShm& me = shm->rank[r];
        std::memset(static_cast<void*>(&me), 0, sizeof(me));
        me.device = dev;
        auto mk = [&](cudaEvent_t& e, cudaIpcEventHandle_t& h) {
            CK(cudaEventCreateWithFlags(&e, cudaEventInterprocess | cudaEventDisableTiming));
            CK(cudaIpcGetEventHandle(&h, e));
        };
        for (int d = 0; d < 2; d++) {
            mk(ev_sent[d], me.sent[d]);
            mk(ev_freed[d], me.freed[d]);
        }
        mk(ev_red_ready, me.red_ready);
        mk(ev_red_done, me.red_done);
        peers.resize(n);
        shm->attached.fetch_add(1);
        barrier();
        if (r == 0) shm_unlink(name.c_str());  // every rank has it mapped: the name can go
        for (int q = 0; q < n; q++) {
            if (q == r) continue;
            const IpcRankShm& o = shm->rank[q];
            Peer& p = peers[q];
            for (int d = 0; d < 2; d++) {
                CK(cudaIpcOpenEventHandle(&p.sent[d], o.sent[d]));
                CK(cudaIpcOpenEventHandle(&p.freed[d], o.freed[d]));
            }
            CK(cudaIpcOpenEventHandle(&p.red_ready, o.red_ready));
            CK(cudaIpcOpenEventHandle(&p.red_done, o.red_done));
        }
    }
    ~IpcTransport() override {
        for (auto& p : peers) {
            for (int d = 0; d < 2; d++)
                if (p.inbox[d]) cudaIpcCloseMemHandle(p.inbox[d]);
            if (p.red) cudaIpcCloseMemHandle(p.red);
        }
        if (shm) munmap(shm, sizeof(IpcShm));
    }
    int rank() const override { return r; }
    int size() const override { return n; }
    void abort() override {
        if (shm) shm->aborted.store(1);
    }
    void barrier() override {
        const long gen = shm->generation.load(std::memory_order_acquire);
        if (shm->arrived.fetch_add(1, std::memory_order_acq_rel) == n - 1) {
            shm->arrived.store(0, std::memory_order_relaxed);
            shm->generation.fetch_add(1, std::memory_order_acq_rel);
            return;
        }
        for (long spins = 0; shm->generation.load(std::memory_order_acquire) == gen; spins++) {
            if (shm->aborted.load()) throw FlumeError(FLUME_E_ENGINE, "slab group aborted by a failing rank");
            if (spins > 64) std::this_thread::sleep_for(std::chrono::microseconds(spins > 10000 ? 200 : 5));
        }
    }
    // grow an exported buffer; peers reopen it when they see the new generation
    static void grow(DevArr<unsigned char>& a, size_t need, cudaIpcMemHandle_t& h, size_t& cap, uint32_t& gen) {
        if (need <= cap && a.p) return;
        size_t c = std::max<size_t>(need, 1 << 16);
        c = std::max(c, cap * 2);
        a.alloc(c);
        CK(cudaIpcGetMemHandle(&h, a.p));
        cap = c;
        gen++;
    }
    void* open_peer(void*& ptr, uint32_t& have, uint32_t gen, const cudaIpcMemHandle_t& h) {
        if (have != gen) {
            if (ptr) CK(cudaIpcCloseMemHandle(ptr));
            CK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
            have = gen;
        }
        return ptr;
    }

    void exchange_counts(const long send[2], long recv[2], cudaStream_t) override {
        IpcRankShm& me = shm->rank[r];
        me.counts[0] = send[0];
        me.counts[1] = send[1];
        barrier();
        recv[0] = r > 0 ? shm->rank[r - 1].counts[1] : 0;
        recv[1] = r + 1 < n ? shm->rank[r + 1].counts[0] : 0;
        barrier();
    }

    void neighbor_exchange(const void* const sbuf[2], const size_t sbytes[2], void* const rbuf[2],
                           const size_t rbytes[2], cudaStream_t s) override {
        IpcRankShm& me = shm->rank[r];
        for (int d = 0; d < 2; d++)
            if (rbytes[d]) grow(inbox[d], rbytes[d], me.inbox[d], me.inbox_cap[d], me.inbox_gen[d]);
        barrier();  // inboxes published; the peers' "freed" events of the last exchange recorded
        for (int d = 0; d < 2; d++) {
            const int q = d == 0 ? r - 1 : r + 1;
            if (q < 0 || q >= n || sbytes[d] == 0) continue;
            const IpcRankShm& o = shm->rank[q];
            Peer& p = peers[q];
            // my message toward d lands in the peer's inbox from the other side
            const int pd = 1 - d;
            if (o.inbox_cap[pd] < sbytes[d])
                throw FlumeError(FLUME_E_ENGINE, "slab exchange: message size mismatch between ranks");
            void* dst = open_peer(p.inbox[pd], p.inbox_gen[pd], o.inbox_gen[pd], o.inbox[pd]);
            CK(cudaStreamWaitEvent(s, p.freed[pd], 0));  // the peer has copied its last message out
            CK(cudaMemcpyAsync(dst, sbuf[d], sbytes[d], cudaMemcpyDeviceToDevice, s));
            CK(cudaEventRecord(ev_sent[d], s));
        }
        barrier();  // every "sent" event recorded
        for (int d = 0; d < 2; d++) {
            const int q = d == 0 ? r - 1 : r + 1;
            if (q < 0 || q >= n || rbytes[d] == 0) continue;
            CK(cudaStreamWaitEvent(s, peers[q].sent[1 - d], 0));
            CK(cudaMemcpyAsync(rbuf[d], inbox[d].p, rbytes[d], cudaMemcpyDeviceToDevice, s));
            CK(cudaEventRecord(ev_freed[d], s));
        }
    }

    void allreduce(void* buf, size_t count, DType t, ROp op, cudaStream_t s) override {
        const size_t bytes = count * dtype_size(t);
        IpcRankShm& me = shm->rank[r];
        if (bytes) grow(red, bytes, me.red, me.red_cap, me.red_gen);
        barrier();  // slots published; the last round's "done" events recorded
        for (int q = 0; q < n; q++)
            if (q != r) CK(cudaStreamWaitEvent(s, peers[q].red_done, 0));  // nobody still reads my slot
        if (bytes) CK(cudaMemcpyAsync(red.p, buf, bytes, cudaMemcpyDeviceToDevice, s));
        CK(cudaEventRecord(ev_red_ready, s));
        barrier();
        stack.alloc(std::max<size_t>(bytes * size_t(n), 1));
        for (int q = 0; q < n && bytes; q++) {
            const void* src = red.p;
            if (q != r) {
                Peer& p = peers[q];
                const IpcRankShm& o = shm->rank[q];
                src = open_peer(p.red, p.red_gen, o.red_gen, o.red);
                CK(cudaStreamWaitEvent(s, p.red_ready, 0));
            }
            CK(cudaMemcpyAsync(stack.p + size_t(q) * bytes, src, bytes, cudaMemcpyDeviceToDevice, s));
        }
        CK(cudaEventRecord(ev_red_done, s));
        launch_stack_reduce(stack.p, count, n, t, op, buf, s);  // rank order: identical bits everywhere
        CK(cudaGetLastError());
    }
};

}  // namespace

std::unique_ptr<Transport> make_thread_transport(std::shared_ptr<ThreadGroup> g, int rank, int device) {
    return std::unique_ptr<Transport>(new ThreadTransport(std::move(g), rank, device));
}

std::unique_ptr<Transport> make_nccl_transport(const unsigned char uid[128], int rank, int nranks, int device) {
    return std::unique_ptr<Transport>(new NcclTransport(uid, rank, nranks, device));
}

bool is_ipc_unique_id(const unsigned char uid[128]) { return std::memcmp(uid, "IPC:", 4) == 0; }

std::unique_ptr<Transport> make_ipc_transport(const unsigned char uid[128], int rank, int nranks, int device) {
    char name[128];
    std::memcpy(name, uid + 4, 120);
    name[119] = 0;
    return std::unique_ptr<Transport>(new IpcTransport(std::string("/") + name, rank, nranks, device));
}

void ipc_unique_id(unsigned char out[128]) {
    std::memset(out, 0, 128);
    std::random_device rd;
    char name[64];
    std::snprintf(name, sizeof(name), "flume_b200_%d_%08x%08x", int(getpid()), unsigned(rd()), unsigned(rd()));
    std::memcpy(out, "IPC:", 4);
    std::memcpy(out + 4, name, std::strlen(name));
}

void nccl_unique_id(unsigned char out[128]) {
    NcclApi& api = NcclApi::get();
    ncclUniqueId id;
    NK(api.GetUniqueId(&id));
    std::memcpy(out, id.internal, 128);
}

}  // namespace fl
