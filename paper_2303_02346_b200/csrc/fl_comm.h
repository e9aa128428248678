// fl_comm.h -- rank-to-rank transport for the x-slab decomposition.
//
// A multi-rank context owns one slab of particle-block columns.  Per substep it
// needs exactly three kinds of communication:
//   * neighbour exchange   halo planes of the scatter tiles (P2G, G2P adjoint)
//                          and migrating particles / their cotangents,
//   * count exchange       sizes of the migration messages (host values),
//   * all-reduce           rigid-member positions and bars (disjoint support,
//                          so the sum is exact), loss partials, effector bars,
//                          error flags.
// Three implementations:
//   ThreadTransport  one process, one host thread per rank (ranks may share a
//                    device); copies are stream-ordered cudaMemcpyPeerAsync
//                    behind cross-stream events, reductions are summed in rank
//                    order, so every rank gets identical bits.
//   NcclTransport    one process per GPU (torchrun); NCCL send/recv and
//                    all-reduce on the context stream.  libnccl is dlopen'ed
//                    (the copy torch already loaded when present).
//   IpcTransport     processes of one node (one or several per GPU): peer copies
//                    into CUDA-IPC-exported inboxes (NVLink between GPUs), ordered
//                    by interprocess events, host barrier in POSIX shared memory.
// All calls are collective over the group and must be issued in the same order
// on every rank.
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <mutex>
#include <vector>

namespace fl {

enum class DType { F64 = 0, U64 = 1, I32 = 2 };
enum class ROp { Sum = 0, Min = 1, Max = 2 };

struct Transport {
    virtual ~Transport() = default;
    virtual int rank() const = 0;
    virtual int size() const = 0;
    // host values: send[d] to the neighbour below (d = 0, rank-1) / above (d = 1, rank+1),
    // recv[d] from the same neighbours (0 where a neighbour is missing)
    virtual void exchange_counts(const long send[2], long recv[2], cudaStream_t s) = 0;
    // device buffers, stream-ordered; byte counts must match the peer's
    virtual void neighbor_exchange(const void* const sbuf[2], const size_t sbytes[2], void* const rbuf[2],
                                   const size_t rbytes[2], cudaStream_t s) = 0;
    // in-place all-reduce of a device buffer, stream-ordered, identical result on every rank
    virtual void allreduce(void* buf, size_t count, DType t, ROp op, cudaStream_t s) = 0;
    // host barrier (setup / teardown only)
    virtual void barrier() = 0;
    // a failing rank releases its peers (ThreadTransport: their barriers throw)
    virtual void abort() {}
};

// shared state of an in-process group
struct ThreadGroup {
    explicit ThreadGroup(int n);
    ~ThreadGroup();
    int n;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    long generation = 0;
    bool aborted = false;
    struct Slot {
        int device = 0;
        const void* sbuf[2] = {nullptr, nullptr};
        size_t sbytes[2] = {0, 0};
        long counts[2] = {0, 0};
        void* red = nullptr;
        size_t red_bytes = 0;
        cudaEvent_t ready = nullptr, done = nullptr;
    };
    std::vector<Slot> slots;
    void barrier();  // throws FlumeError when the group was aborted
    void abort();
};

std::unique_ptr<Transport> make_thread_transport(std::shared_ptr<ThreadGroup> g, int rank, int device);
std::unique_ptr<Transport> make_nccl_transport(const unsigned char uid[128], int rank, int nranks, int device);
void nccl_unique_id(unsigned char out[128]);
// CUDA-IPC transport between the processes of one node ("IPC:" group ids)
bool is_ipc_unique_id(const unsigned char uid[128]);
std::unique_ptr<Transport> make_ipc_transport(const unsigned char uid[128], int rank, int nranks, int device);
void ipc_unique_id(unsigned char out[128]);

// dtype/op reduction of `nr` stacked copies (rank order) into out (ThreadTransport)
void launch_stack_reduce(const void* stack, size_t count, int nr, DType t, ROp op, void* out, cudaStream_t s);

}  // namespace fl
