// fl_spill.h -- the file tier of the checkpoint store (checkpoint.hpp:11-50,
// PAPER.md's NVMe offload): grad_trajectory snapshots that fit neither HBM nor pinned host
// memory go to a file on local storage.
//
// A snapshot leaves the device by a D2H copy into one of a few pinned staging buffers on
// the caller's stream; a worker thread waits for that copy and pwrite()s the buffer at the
// snapshot's offset, then frees the buffer -- the forward only waits when every staging
// buffer is still in flight.  The backward reads a snapshot back with pread() into a
// staging buffer and an H2D copy on its stream, and prefetches the next older snapshot on
// the worker while the current segment replays.  The file is unlinked as soon as it is
// created, so it disappears with the context.  Bytes round-trip exactly: gradients are
// identical to the HBM and pinned-host stores.
#pragma once

#include <cuda_runtime.h>
#include <fcntl.h>
#include <unistd.h>

#include <condition_variable>
#include <deque>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "fl_host.h"

namespace fl {

class FileSpill {
   public:
    FileSpill(const std::string& dir, size_t slot_bytes, int nstage = 3) : slot(slot_bytes) {
        std::string tmpl = dir + "/flume_spill_XXXXXX";
        std::vector<char> path(tmpl.begin(), tmpl.end());
        path.push_back('\0');
        fd = mkstemp(path.data());
        if (fd < 0) throw FlumeError(FLUME_E_ARG, "checkpoint spill: cannot create a file in " + dir);
        unlink(path.data());  // anonymous: gone with the descriptor
        stage.resize(nstage);
        for (auto& s : stage) {
            CK(cudaMallocHost(&s.buf, slot));
            CK(cudaEventCreateWithFlags(&s.ev, cudaEventDisableTiming));
        }
        worker = std::thread([this] { run(); });
    }
    ~FileSpill() {
        {
            std::lock_guard<std::mutex> lk(m);
            stop = true;
        }
        cv.notify_all();
        if (worker.joinable()) worker.join();
        for (auto& s : stage) {
            if (s.buf) cudaFreeHost(s.buf);
            if (s.ev) cudaEventDestroy(s.ev);
        }
        if (fd >= 0) close(fd);
    }
    FileSpill(const FileSpill&) = delete;
    FileSpill& operator=(const FileSpill&) = delete;

    size_t slot_bytes() const { return slot; }
    void reset() {  // a new trajectory: offsets from the start of the file
        drain();
        std::unique_lock<std::mutex> lk(m);
        for (auto& kv : prefetched) {  // unclaimed prefetches: let their reads land, free the buffers
            cv.wait(lk, [&] { return stage[kv.second].ready || failed; });
            stage[kv.second].busy = false;
            stage[kv.second].ready = false;
        }
        prefetched.clear();
        next_off = 0;
    }

    // snapshot of `bytes` device bytes (D2H ordered after the work already on s); returns its offset
    off_t put(const void* dev, size_t bytes, cudaStream_t s) {
        if (bytes > slot) throw FlumeError(FLUME_E_ENGINE, "checkpoint spill: snapshot larger than its slot");
        const int i = acquire();
        CK(cudaMemcpyAsync(stage[i].buf, dev, bytes, cudaMemcpyDeviceToHost, s));
        CK(cudaEventRecord(stage[i].ev, s));
        off_t off;
        {
            std::lock_guard<std::mutex> lk(m);
            off = next_off;
            next_off += off_t(bytes);
            jobs.push_back(Job{true, i, off, bytes});
            pending_writes++;
        }
        cv.notify_all();
        return off;
    }

    // read a snapshot back into device memory (H2D on s)
    void get(off_t off, void* dev, size_t bytes, cudaStream_t s) {
        wait_writes();
        int i = -1;
        {
            std::unique_lock<std::mutex> lk(m);
            auto it = prefetched.find(off);
            if (it != prefetched.end()) {
                cv.wait(lk, [&] { return stage[it->second].ready || failed; });
                i = it->second;
                prefetched.erase(it);
            }
        }
        check_failed();
        if (i < 0) {
            i = acquire();
            read_into(stage[i].buf, off, bytes);
        }
        CK(cudaMemcpyAsync(dev, stage[i].buf, bytes, cudaMemcpyHostToDevice, s));
        CK(cudaEventRecord(stage[i].ev, s));  // the buffer is free again once this copy ran
        std::lock_guard<std::mutex> lk(m);
        stage[i].busy = false;
        stage[i].ready = false;
        stage[i].h2d = true;
    }

    // start reading a snapshot into a staging buffer (the worker); get() picks it up
    void prefetch(off_t off, size_t bytes) {
        {
            std::lock_guard<std::mutex> lk(m);
            if (prefetched.count(off)) return;
        }
        const int i = acquire();
        std::lock_guard<std::mutex> lk(m);
        prefetched[off] = i;
        stage[i].ready = false;
        jobs.push_back(Job{false, i, off, bytes});
        cv.notify_all();
    }

   private:
    struct Stage {
        void* buf = nullptr;
        cudaEvent_t ev = nullptr;
        bool busy = false;   // owned by a put/get/prefetch in flight
        bool ready = false;  // a prefetched read landed
        bool h2d = false;    // last use was an H2D copy: free once ev completed
    };
    struct Job {
        bool write;
        int stage;
        off_t off;
        size_t bytes;
    };
    size_t slot;
    int fd = -1;
    std::vector<Stage> stage;
    std::deque<Job> jobs;
    std::map<off_t, int> prefetched;
    off_t next_off = 0;
    int pending_writes = 0;
    bool stop = false, failed = false;
    std::string fail_msg;
    std::mutex m;
    std::condition_variable cv;
    std::thread worker;

    int acquire() {
        std::unique_lock<std::mutex> lk(m);
        for (;;) {
            for (size_t i = 0; i < stage.size(); i++) {
                Stage& s = stage[i];
                if (s.busy) continue;
                if (s.h2d) {  // the H2D reading it must have run
                    lk.unlock();
                    CK(cudaEventSynchronize(s.ev));
                    lk.lock();
                    s.h2d = false;
                }
                s.busy = true;
                return int(i);
            }
            cv.wait(lk);
            if (failed) break;
        }
        lk.unlock();
        check_failed();
        return -1;
    }
    void read_into(void* dst, off_t off, size_t bytes) {
        size_t done = 0;
        while (done < bytes) {
            const ssize_t r = pread(fd, static_cast<char*>(dst) + done, bytes - done, off + off_t(done));
            if (r <= 0) throw FlumeError(FLUME_E_ENGINE, "checkpoint spill: read failed");
            done += size_t(r);
        }
    }
    void wait_writes() {
        std::unique_lock<std::mutex> lk(m);
        cv.wait(lk, [&] { return pending_writes == 0 || failed; });
        lk.unlock();
        check_failed();
    }
    void drain() {
        std::unique_lock<std::mutex> lk(m);
        cv.wait(lk, [&] { return (jobs.empty() && pending_writes == 0) || failed; });
    }
    void check_failed() {
        std::lock_guard<std::mutex> lk(m);
        if (failed) throw FlumeError(FLUME_E_ENGINE, "checkpoint spill: " + fail_msg);
    }
    void run() {
        for (;;) {
            Job j;
            {
                std::unique_lock<std::mutex> lk(m);
                cv.wait(lk, [&] { return stop || !jobs.empty(); });
                if (stop && jobs.empty()) return;
                j = jobs.front();
                jobs.pop_front();
            }
            bool ok = true;
            std::string why;
            if (j.write) {
                if (cudaEventSynchronize(stage[j.stage].ev) != cudaSuccess) {
                    ok = false;
                    why = "device copy failed";
                }
                size_t done = 0;
                while (ok && done < j.bytes) {
                    const ssize_t w = pwrite(fd, static_cast<const char*>(stage[j.stage].buf) + done, j.bytes - done,
                                             j.off + off_t(done));
                    if (w <= 0) {
                        ok = false;
                        why = "write failed (disk full?)";
                    } else {
                        done += size_t(w);
                    }
                }
            } else {
                size_t done = 0;
                while (ok && done < j.bytes) {
                    const ssize_t r = pread(fd, static_cast<char*>(stage[j.stage].buf) + done, j.bytes - done,
                                            j.off + off_t(done));
                    if (r <= 0) {
                        ok = false;
                        why = "read failed";
                    } else {
                        done += size_t(r);
                    }
                }
            }
            {
                std::lock_guard<std::mutex> lk(m);
                if (!ok) {
                    failed = true;
                    fail_msg = why;
                }
                if (j.write) {
                    stage[j.stage].busy = false;
                    pending_writes--;
                } else {
                    stage[j.stage].ready = true;
                }
            }
            cv.notify_all();
        }
    }
};

}  // namespace fl
