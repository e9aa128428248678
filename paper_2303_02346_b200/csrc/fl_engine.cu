// fl_engine.cu -- host runtime behind the C ABI (include/flume_b200.h).
//
// Owns the device-resident trajectory store and drives the kernels:
//   substep()          = mpm_substep          (mpm.hpp:455-473)
//   rollout_loss()     = rollout_loss         (grad.hpp:15-41)
//   grad_trajectory()  = grad_trajectory      (grad.hpp:61-134) with the
//                        CheckpointStore policy (checkpoint.hpp:11-50): snapshots
//                        at stride multiples, each segment replayed once into an
//                        HBM cache.  Unlike the reference there is no
//                        capture_forward re-run: the cache already holds every
//                        pre-state of the segment.
//   adjoint_substep()  = adjoint_substep      (adjoint.hpp:476-548)
// Effector kinematics (advance_effectors, mpm.hpp:418-433) and the effector
// pose adjoint (adjoint.hpp:522-545) are tiny and open-loop, so they run on the
// host in fp64; everything per-particle / per-node runs on the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/flume_b200.h"
#include "fl_comm.h"
#include "fl_host.h"
#include "fl_kernels.h"
#include "fl_scatter.cuh"
#include "fl_spill.h"

namespace fl {

// ---------------------------------------------------------------------------
// trajectory storage
// ---------------------------------------------------------------------------
struct StateBuf {
    void* mem = nullptr;
    PBuf p{};
    size_t bytes = 0;
    int n = 0;  // occupied slots (active + parked + arrivals + departed holes; N on one rank;
                // an upper bound on slabs, whose exact counts are `cnt` on the device)
    int* cnt = nullptr;  // device [StateCnt]: n_active, n_stored, park_base (slab contexts)
    StateBuf(int cap, int nmem) {
        size_t pbytes = (size_t(cap) * (24 * sizeof(float) + 3 * sizeof(uint32_t)) + 255) & ~size_t(255);
        const size_t mbytes = (size_t(std::max(nmem, 1)) * 3 * sizeof(double) + 255) & ~size_t(255);
        bytes = pbytes + mbytes + SC_N * sizeof(int);  // the counts travel with every copy / spill
        CK(cudaMalloc(&mem, bytes));
        p.cap = cap;
        p.f = static_cast<float*>(mem);
        p.meta = reinterpret_cast<uint32_t*>(p.f + size_t(24) * cap);
        p.id = p.meta + cap;
        p.key = p.id + cap;
        p.mx = reinterpret_cast<double*>(static_cast<char*>(mem) + pbytes);
        cnt = reinterpret_cast<int*>(static_cast<char*>(mem) + pbytes + mbytes);
    }
    ~StateBuf() { cudaFree(mem); }
};
using StatePtr = std::shared_ptr<StateBuf>;

// a trajectory snapshot spilled to pinned host memory (CheckpointStore, checkpoint.hpp:11-50,
// for horizons beyond HBM)
struct HostState {
    void* mem = nullptr;
    size_t bytes = 0;
    int n = 0;
    cudaEvent_t done = nullptr;  // D2H completion on the copy stream
    explicit HostState(size_t b) : bytes(b) {
        CK(cudaMallocHost(&mem, b));
        CK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    }
    ~HostState() {
        if (mem) cudaFreeHost(mem);
        if (done) cudaEventDestroy(done);
    }
};
using HostPtr = std::shared_ptr<HostState>;

struct EffState {
    V3<double> t;
    M3<double> R;
    V3<double> vlin;
    V3<double> w;
};

// everything the backward of one substep needs besides its pre-state buffer
struct Record {
    void* mem = nullptr;
    uint32_t* perm = nullptr;
    BlockRec* recs = nullptr;
    int* n_blocks = nullptr;
    int* nb_list = nullptr;
    int* n_nb = nullptr;
    int* mslot = nullptr;
    double* mstart = nullptr;
    double* mid = nullptr;
    double* mact = nullptr;
    double* fit = nullptr;
    uint16_t* celltab = nullptr;
    float4* gridv = nullptr;   // grid velocity after contact (G2P input), dense block-major
    float4* gridv0 = nullptr;  // (p/m, m) before gravity/walls/contact (grid-update adjoint input)
    uint8_t* cmask = nullptr;  // per node: effectors within contact range (bit e)
    int* blockmap = nullptr;   // particle block -> list slot + 1 (0 = none), incl. slab ghost blocks
    EffK<float>* effx = nullptr;  // replica contexts: this substep's effector set (EffSet::ext)
    // host counts: exact on one rank; upper bounds on slabs, where `dcnt` (device,
    // [RecCnt]) holds the exact ones, the migration's message counts among them
    int n_active = 0;
    int n_keep = 0;    // active + parked slots of the pre-state (= N on one rank)
    int n_stored = 0;  // all slots of the pre-state, departed holes included
    int* dcnt = nullptr;
    // slabs: dcnt read back into pinned memory as the forward runs (no wait); the
    // backward sizes the cotangent return messages from it
    int* hcnt = nullptr;
    cudaEvent_t hcnt_ev = nullptr;
    // slab migration after this substep's G2P: slots of the departed particles
    // (by direction, in message order)
    uint32_t* mig_src = nullptr;
    int mig_cap = 0;
    long substep = 0;
    bool scratch = false;  // a scratch record (forward only): no adjoint inputs kept
    std::vector<ActEntry> act;
    std::vector<EmitAdjEntry> emit;
    EffSet effk{};
    Record(int N, int maxb, int nbtot, int nmem, int nbody, int migcap, int neffx = 0) {
        size_t off = 0;
        auto carve = [&](size_t bytes) {
            size_t o = off;
            off += (bytes + 255) & ~size_t(255);
            return o;
        };
        size_t o_perm = carve(size_t(N) * 4), o_recs = carve(size_t(maxb) * sizeof(BlockRec)), o_nb = carve(size_t(work_order_ints(maxb)) * 4),
               o_nbl = carve(size_t(nbtot) * 4), o_nnb = carve(16), o_ms = carve(size_t(nmem) * 4),
               o_mst = carve(size_t(nmem) * 24), o_mid = carve(size_t(nmem) * 32),
               o_fit = carve(size_t(nbody) * 24 * 8), o_ct = carve(size_t(maxb) * kCellTab * 2),
               o_gv = carve(size_t(nbtot) * 64 * sizeof(float4)), o_gv0 = carve(size_t(nbtot) * 64 * sizeof(float4)),
               o_mig = carve(size_t(2) * migcap * 4), o_cm = carve(size_t(nbtot) * 64), o_bm = carve(size_t(nbtot) * 4),
               o_dc = carve(RC_N * sizeof(int)), o_ex = carve(size_t(neffx) * sizeof(EffK<float>));
        CK(cudaMalloc(&mem, off));
        char* b = static_cast<char*>(mem);
        perm = reinterpret_cast<uint32_t*>(b + o_perm);
        recs = reinterpret_cast<BlockRec*>(b + o_recs);
        n_blocks = reinterpret_cast<int*>(b + o_nb);
        nb_list = reinterpret_cast<int*>(b + o_nbl);
        n_nb = reinterpret_cast<int*>(b + o_nnb);
        mslot = reinterpret_cast<int*>(b + o_ms);
        mstart = reinterpret_cast<double*>(b + o_mst);
        mid = reinterpret_cast<double*>(b + o_mid);
        mact = mid + 3 * size_t(nmem);
        fit = reinterpret_cast<double*>(b + o_fit);
        celltab = reinterpret_cast<uint16_t*>(b + o_ct);
        gridv = reinterpret_cast<float4*>(b + o_gv);
        gridv0 = reinterpret_cast<float4*>(b + o_gv0);
        mig_src = migcap > 0 ? reinterpret_cast<uint32_t*>(b + o_mig) : nullptr;
        cmask = reinterpret_cast<uint8_t*>(b + o_cm);
        blockmap = reinterpret_cast<int*>(b + o_bm);
        dcnt = reinterpret_cast<int*>(b + o_dc);
        effx = neffx > 0 ? reinterpret_cast<EffK<float>*>(b + o_ex) : nullptr;
        mig_cap = migcap;
        CK(cudaMemset(gridv, 0, size_t(nbtot) * 64 * sizeof(float4)));
        CK(cudaMemset(gridv0, 0, size_t(nbtot) * 64 * sizeof(float4)));
    }
    ~Record() {
        cudaFree(mem);
        if (hcnt) cudaFreeHost(hcnt);
        if (hcnt_ev) cudaEventDestroy(hcnt_ev);
    }
    void readback_counts(cudaStream_t s) {
        if (!hcnt) {
            CK(cudaMallocHost(&hcnt, RC_N * sizeof(int)));
            CK(cudaEventCreateWithFlags(&hcnt_ev, cudaEventDisableTiming));
        }
        CK(cudaMemcpyAsync(hcnt, dcnt, RC_N * sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaEventRecord(hcnt_ev, s));
    }
    const int* host_counts() const {  // (long complete when the backward asks)
        CK(cudaEventSynchronize(hcnt_ev));
        return hcnt;
    }
};
using RecordPtr = std::shared_ptr<Record>;

static int bits_for(uint64_t v) {
    int b = 0;
    while ((uint64_t(1) << b) <= v) b++;
    return b < 1 ? 1 : b;
}

// per-kernel CUDA-event timing (enabled by flume_profile): events are recorded on
// the context stream around each launch and summed after the next sync
enum KId { K_P2G = 0, K_GRID = 1, K_G2P = 2, K_SORT = 3, K_ADJ_G2P = 4, K_ADJ_GRID = 5, K_ADJ_P2G = 6,
           K_RIGID = 7, K_OTHER = 8, K_COMM = 9, K_COUNT = 10 };

struct Prof {
    bool on = false;
    std::vector<cudaEvent_t> pool;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
    double ms[K_COUNT] = {};
    long count[K_COUNT] = {};
    cudaEvent_t ev() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        return e;
    }
    cudaEvent_t begin(cudaStream_t s) {
        if (!on) return nullptr;
        cudaEvent_t e = ev();
        CK(cudaEventRecord(e, s));
        return e;
    }
    void end(int id, cudaEvent_t b, cudaStream_t s) {
        if (!on || !b) return;
        cudaEvent_t e = ev();
        CK(cudaEventRecord(e, s));
        pending.push_back({id, {b, e}});
        if (pending.size() > 4096) collect(s);
    }
    void collect(cudaStream_t s) {
        if (pending.empty()) return;
        CK(cudaStreamSynchronize(s));
        for (auto& p : pending) {
            float t = 0;
            CK(cudaEventElapsedTime(&t, p.second.first, p.second.second));
            ms[p.first] += t;
            count[p.first]++;
            pool.push_back(p.second.first);
            pool.push_back(p.second.second);
        }
        pending.clear();
    }
    void reset() {
        for (int k = 0; k < K_COUNT; k++) {
            ms[k] = 0;
            count[k] = 0;
        }
    }
    ~Prof() {
        for (auto& p : pending) {
            cudaEventDestroy(p.second.first);
            cudaEventDestroy(p.second.second);
        }
        for (auto e : pool) cudaEventDestroy(e);
    }
};

#define PROF(id, call)                          \
    do {                                        \
        cudaEvent_t pb_ = prof.begin(stream);   \
        call;                                   \
        prof.end(id, pb_, stream);              \
    } while (0)

// ---------------------------------------------------------------------------
// context
// ---------------------------------------------------------------------------
struct Ctx {
    Prof prof;
    cudaEvent_t marks[8] = {};
    // light (plain-liquid) and heavy (SVD / rigid) block variants run concurrently
    cudaStream_t s2 = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    DevArr<int> wq;  // rolling work counters for dynamically scheduled kernels
    int wq_next = 0;
    static constexpr int kWq = 256;
    // n zeroed counters.  All n come from the same pool epoch: a counter handed out
    // before a wrap's memset but used after it would start the next epoch dirty.
    int* take_wq(int n = 1) {
        if (wq_next + n > kWq) {
            CK(cudaMemsetAsync(wq.p, 0, kWq * sizeof(int), stream));
            wq_next = 0;
        }
        int* p = wq.p + wq_next;
        wq_next += n;
        return p;
    }
    // The SVD/rigid ("heavy") and plain-liquid ("light") variants of a scatter/gather kernel.
    // dual_mode 1 (default): one stream, the heavy grid first, releasing the light grid as
    // soon as its CTAs are resident (DualScope, fl_layout.cuh), so the few long heavy blocks
    // run beside the light ones.  dual_mode 0 (rounds 1-2): the heavy grid on a second stream
    // -- but the light grid, launched early by programmatic serialization, filled every SM
    // first and the heavy grid mostly ran after it (c4 grad_trajectory 175.9 -> 162.4 ms).
    template <class Fn>
    void dual(Fn&& fn) {
        if (!classes_heavy && !upload_full) {  // no SVD/rigid particle can exist: light kernel only
            fn(false, take_wq(1), stream);
            launches += 1;
            return;
        }
        launches += 2;
        int* wh = take_wq(2);
        int* wl = wh + 1;
        if (dual_mode == 1) {
            dual_role() = 1;
            fn(true, wh, stream);
            dual_role() = 2;
            fn(false, wl, stream);
            dual_role() = 0;
            return;
        }
        CK(cudaEventRecord(ev_fork, stream));
        CK(cudaStreamWaitEvent(s2, ev_fork, 0));
        fn(true, wh, s2);
        fn(false, wl, stream);
        CK(cudaEventRecord(ev_join, s2));
        CK(cudaStreamWaitEvent(stream, ev_join, 0));
    }
    int dual_mode = 1;
    int device = 0;
    cudaStream_t stream = nullptr;
    flume_error_info last_err{};
    flume_timing timing{};
    long launches = 0;

    // scene
    flume_config cfg{};
    Geom geom{};
    int N = 0;
    int maxb = 0;
    std::vector<flume_material> mats;
    std::vector<flume_effector_shape> eff_shapes;
    std::vector<int> p_mat, p_body;
    std::vector<double> p_mass, p_vol0;
    std::vector<long> p_act;
    std::vector<uint32_t> p_class;
    std::vector<ClassInfo> classes;
    // rigid
    int nbody = 0, nmem = 0;
    std::vector<int> rb_off, rb_id, member_body, mrank_by_id;
    std::vector<long> rb_members;
    std::vector<double> rb_rest, rb_mass, rb_smrest, rb_total;
    std::vector<int> chunk_body, chunk_m0, chunk_m1;
    // emitters by particle id
    std::vector<int> emitter_of;
    std::vector<flume_emitter> emitters;
    std::map<long, std::vector<int>> pending;  // activation substep -> ids (sorted)

    // device constants
    DevArr<ClassInfo> d_cls;
    DevArr<int> d_member_id;
    DevArr<int> d_rb_off, d_rb_id, d_member_body, d_mrank, d_chunk_body, d_chunk_m0, d_chunk_m1, d_act;
    DevArr<double> d_rb_rest, d_rb_mass, d_rb_smrest, d_rb_total;

    // scratch
    DevArr<int> bzero, bstart;  // bzero = [bcount | bheavy | bfill], zeroed per sort
    int *bcount = nullptr, *bheavy = nullptr, *bfill = nullptr, *nbflag = nullptr;
    DevArr<int> nbflag_arr;
    bool counters_clean = false;  // what the grid update clears is zero (all of bzero, or bfill when counts are kept)
    // incremental sort (fl_sort.cu): the block counts persist from sort to sort, okey[okey_cur]
    // holds the last sort's keys by sorted position, and chain_rec is the record whose sort
    // order chain_out (the G2P output of that substep) is stored in
    bool inc_sort = true;  // flume_set_incremental_sort
    DevArr<uint32_t> okey[2];
    int okey_cur = 0;
    DevArr<int> isort_blk;  // [dirty | acnt | overflow count | its copy], zero between sorts
    DevArr<int4> rold;
    DevArr<uint32_t> mov, inbox;
    const Record* chain_rec = nullptr;
    const StateBuf* chain_out = nullptr;
    long n_inc_sorts = 0, n_full_sorts = 0;
    bool keep_counts() const { return inc_sort && !comm && uint64_t(geom.key_departed) < 0x80000000ull; }
    void chain_break() {
        chain_rec = nullptr;
        chain_out = nullptr;
    }
    // what the grid update clears for the next sort
    int* clear_ptr() { return keep_counts() ? bfill : bzero.p; }
    int clear_n() const { return keep_counts() ? geom.nbtot + 2 : int(bzero.n); }
    // checkpoint spill: snapshots of grad_trajectory in pinned host memory (D2H on a
    // copy stream overlapping the forward; H2D when the backward replays a segment)
    int spill = 0;  // 0 HBM, 1 pinned host memory, 2 a file in spill_dir (FileSpill)
    std::string spill_dir;
    std::unique_ptr<FileSpill> fspill;
    int chamfer_mode = 0;  // flume_set_chamfer_mode
    cudaStream_t cstream = nullptr;
    cudaEvent_t ev_snap = nullptr;
    std::vector<HostPtr> host_pool;
    HostPtr get_host(size_t bytes) {
        for (size_t i = 0; i < host_pool.size(); i++)
            if (host_pool[i]->bytes == bytes) {
                HostPtr h = host_pool[i];
                host_pool.erase(host_pool.begin() + long(i));
                return h;
            }
        return std::make_shared<HostState>(bytes);
    }
    HostPtr spill_state(const StateBuf& st) {
        if (!cstream) {
            CK(cudaStreamCreateWithFlags(&cstream, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&ev_snap, cudaEventDisableTiming));
        }
        HostPtr h = get_host(st.bytes);
        CK(cudaEventRecord(ev_snap, stream));
        CK(cudaStreamWaitEvent(cstream, ev_snap, 0));
        CK(cudaMemcpyAsync(h->mem, st.mem, st.bytes, cudaMemcpyDeviceToHost, cstream));
        CK(cudaEventRecord(h->done, cstream));
        h->n = st.n;
        return h;
    }
    void unspill(const HostState& h, StateBuf& dst) {
        CK(cudaStreamWaitEvent(stream, h.done, 0));
        CK(cudaMemcpyAsync(dst.mem, h.mem, h.bytes, cudaMemcpyHostToDevice, stream));
        dst.n = h.n;
    }
    DevArr<int> nbpos;
    DevArr<int4> tile_sum;
    DevArr<uint32_t> skey, sslot, gk, gv;
    DevArr<float4> staging, staging_bar, gridbar;
    DevArr<unsigned long long> d_err;
    DevArr<int> d_nonfinite;
    DevArr<double> rig_partial, abar, eff_partial, eff_out, em_out, loss_partial, loss_out;
    DevArr<float> start_bar, xbar_tmp, Fbar_tmp, barsA, barsB;
    cudaEvent_t tev[3] = {nullptr, nullptr, nullptr};
    DevArr<ActEntry> d_act_list;
    DevArr<EmitAdjEntry> d_emit_list;
    DevArr<double> d_up[4];
    DevArr<uint32_t> d_upmeta;
    DevArr<uint8_t> d_upactive;
    DevArr<int> d_anyfull;
    // the upload's active / parked split, kept for the substep index it was made at
    long up_substep = -1;
    bool up_active_dev = false;
    std::vector<uint8_t> up_active;
    std::vector<uint32_t> up_inactive;
    std::map<long, std::vector<int>> up_pending;
    int up_n_active = 0;
    DevArr<float> d_x0;  // [3][N] positions by particle id at upload (LossSet.x0)
    int hvar = 1;  // heavy kernel variant (occupancy_grid): 1 beside liquid, 2 dominant, 3 few beside liquid
    int grid_p2g = 0, grid_g2p = 0, grid_upd = 0, grid_sort = 0, grid_adj = 0;
    int eff_blocks = kEffBlocks;
    // effector-bar partial rows per substep: one per grid-adjoint CTA, twice on slabs
    // (interior and edge launches)
    int eff_rows() const { return slab() ? 2 * eff_blocks : eff_blocks; }
    int grid_p2g_h = 0, grid_g2p_h = 0, grid_adj_h = 0, grid_ap = 0, grid_ap_h = 0;

    // live state
    StatePtr cur;
    std::vector<uint32_t> inactive_ids;  // tail of cur's storage, sorted by id
    int n_active = 0;
    long substep_index = 0;
    double time = 0;
    std::vector<EffState> eff;
    std::vector<StatePtr> pool;
    std::vector<RecordPtr> rec_pool;
    RecordPtr scratch_rec, scratch_alt;  // alternating, so a chained sort reads the previous tables
    Record& next_scratch() {
        std::swap(scratch_rec, scratch_alt);
        return *scratch_rec;
    }
    void new_scratch() {
        scratch_rec = get_record();
        scratch_alt = get_record();
        scratch_rec->scratch = scratch_alt->scratch = true;
        chain_break();
    }

    // x-slab decomposition; comm == nullptr on one rank
    std::unique_ptr<Transport> comm;
    int rank = 0, nranks = 1;
    int n_stored = 0;  // slots of cur: active + parked + arrivals + departed holes (= N on one rank)
    int park_base = 0;  // first parked slot of cur (= n_active on one rank)
    int mig_cap = 0;
    DevArr<unsigned char> halo_send[2], halo_recv[2], mig_send[2], mig_recv[2];
    DevArr<int> d_ovf;  // migration / store overflow flag (checked once per call)
    DevArr<int> mig_bcnt;
    void set_mig_cap(int cap);
    DevArr<double> mbar;
    std::vector<float> parked_x;  // positions of parked particles by id (ownership of their activation)
    bool slab() const { return comm != nullptr; }
    int n_parked() const { return int(inactive_ids.size()); }
    void set_transport(std::unique_ptr<Transport> t);
    void partition(const std::vector<uint32_t>& keys, const std::vector<uint8_t>& active);
    void halo_exchange(int* blockmap, float4* stg, int* flags, cudaStream_t st = nullptr);
    cudaStream_t s_comm = nullptr;  // slabs: halo exchange overlapping the interior grid update
    cudaEvent_t ev_halo_fork = nullptr, ev_halo_join = nullptr;
    void migrate(StateBuf& out, Record& r);
    void return_bars(Record& r, BarBuf post);
    // slab contexts keep the exact particle counts on the device (StateBuf::cnt,
    // Record::dcnt); the host holds upper bounds between calls and the exact values
    // after sync_counts() (one stream sync, at call boundaries)
    void state_counts_from_host(StateBuf& st) {
        const int h[SC_N] = {n_active, n_stored, park_base, 0};
        CK(cudaMemcpyAsync(st.cnt, h, sizeof(h), cudaMemcpyHostToDevice, stream));
        CK(cudaStreamSynchronize(stream));
    }
    void rec_counts_from_host(Record& r, int pb) {
        int h[RC_N] = {};
        h[RC_ACTIVE] = r.n_active;
        h[RC_KEEP] = r.n_keep;
        h[RC_STORED] = r.n_stored;
        h[RC_PARK] = pb;
        CK(cudaMemcpyAsync(r.dcnt, h, sizeof(h), cudaMemcpyHostToDevice, stream));
        CK(cudaStreamSynchronize(stream));
    }
    void sync_counts() {
        if (!slab() || !cur) return;
        int h[SC_N] = {};
        CK(cudaMemcpyAsync(h, cur->cnt, sizeof(h), cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        n_active = h[SC_ACTIVE];
        n_stored = h[SC_STORED];
        park_base = h[SC_PARK];
        cur->n = n_stored;
    }
    // A slab call whose migration overflowed its fixed-size messages is re-run from the
    // same starting point with 4x the capacity (mutates = the call advances the context:
    // its starting state and host bookkeeping are kept for the re-run).  The canonical
    // order makes the result independent of the capacity.
    template <class Fn>
    void slab_retry(bool mutates, Fn&& fn) {
        if (!slab()) {
            fn();
            return;
        }
        for (;;) {
            StatePtr backup;
            const long s0 = substep_index;
            const double t0 = time;
            const int na0 = n_active, ns0 = n_stored, pb0 = park_base;
            const std::vector<EffState> eff0 = eff;
            const std::vector<uint32_t> inact0 = inactive_ids;
            const auto pend0 = pending;
            if (mutates) {
                backup = get_state();
                copy_state(*backup, *cur);
            }
            // an overflowed attempt lost migrants, so it may also have raised a (collective,
            // all-reduced) engine error: the overflow decides
            bool failed = false;
            FlumeError err(FLUME_E_ENGINE, "");
            try {
                fn();
            } catch (const FlumeError& e) {
                if (e.code == FLUME_E_CUDA || e.code == FLUME_E_ARG) throw;
                failed = true;
                err = e;
            }
            const bool ovf = migration_overflowed();
            if (!ovf) {
                put_state(backup);
                if (failed) throw err;
                sync_counts();
                return;
            }
            if (mig_cap >= N) throw FlumeError(FLUME_E_ENGINE, "slab store overflow");
            if (mutates) {
                put_state(cur);
                cur = backup;
            }
            // (a pure call that raised midway skipped its own host restore)
            substep_index = s0;
            time = t0;
            n_active = na0;
            n_stored = ns0;
            park_base = pb0;
            eff = eff0;
            inactive_ids = inact0;
            pending = pend0;
            set_mig_cap(4 * mig_cap);
            mig_retries++;
        }
    }
    long mig_retries = 0;
    // after a slab call: did any rank's migration exceed the message capacity (or the
    // store)?  Collective; resets the flag.
    bool migration_overflowed() {
        if (!slab()) return false;
        allreduce(d_ovf.p, 1, DType::I32, ROp::Max);
        int h = 0;
        CK(cudaMemcpyAsync(&h, d_ovf.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        if (h) CK(cudaMemsetAsync(d_ovf.p, 0, sizeof(int), stream));
        return h != 0;
    }
    // effector-bar final sums are deferred and batched (kEffRing substeps per launch);
    // the backward runs t downwards, so the pending substeps are [eff_lo, eff_hi]
    long eff_lo = -1, eff_hi = -1;
    void eff_flush() {
        if (eff_lo < 0) return;
        launch_eff_final(eff_partial.p, eff_rows(), int(eff.size()), eff_lo, int(eff_hi - eff_lo + 1), eff_out.p,
                         eslots() * 18, stream);
        launches++;
        eff_lo = eff_hi = -1;
    }
    void eff_pending(long t) {
        if (eff_lo >= 0 && (t != eff_lo - 1 || eff_hi - t + 1 > kEffRing)) eff_flush();
        if (eff_lo < 0) eff_hi = t;
        eff_lo = t;
        if (eff_hi - eff_lo + 1 == kEffRing) eff_flush();
    }
    void allreduce(void* p, size_t n, DType t, ROp op) {
        if (comm) comm->allreduce(p, n, t, op, stream);
    }

    // -------------------------------------------------------------------
    StatePtr get_state() {
        if (!pool.empty()) {
            StatePtr s = pool.back();
            pool.pop_back();
            return s;
        }
        return std::make_shared<StateBuf>(N, nmem);
    }
    void put_state(StatePtr s) {
        if (s.get() == chain_out) chain_break();  // about to be reused for something else
        if (s) pool.push_back(std::move(s));
    }
    RecordPtr get_record() {
        if (!rec_pool.empty()) {
            RecordPtr r = rec_pool.back();
            rec_pool.pop_back();
            return r;
        }
        return std::make_shared<Record>(N, maxb, geom.nbtot, std::max(nmem, 1), std::max(nbody, 1), mig_cap,
                                        nrep > 1 ? int(eff_shapes.size()) : 0);  // ~2 KB/node block
    }
    void put_record(RecordPtr r) {
        if (r) rec_pool.push_back(std::move(r));
    }

    RigidDev rigid_dev(Record& r) {
        RigidDev d{};
        d.nbody = nbody;
        d.nmem = nmem;
        d.off = d_rb_off.p;
        d.mrank = d_mrank.p;
        d.rest = d_rb_rest.p;
        d.mass = d_rb_mass.p;
        d.smrest = d_rb_smrest.p;
        d.total = d_rb_total.p;
        d.body_id = d_rb_id.p;
        d.member_body = d_member_body.p;
        d.member_id = d_member_id.p;
        d.mslot = r.mslot;
        d.mstart = r.mstart;
        d.mid = r.mid;
        d.mact = r.mact;
        d.fit = r.fit;
        return d;
    }

    void init(const flume_scene_desc* desc, int dev, int n_replicas = 1);
    // replica contexts (the CMA-ES population of optimize.hpp:383-418): n_rep
    // copies of one scene in one grid (Geom::rstride), every kernel launch covering all of them.
    // Particle i of replica r is id r * n1 + i, effector e is r * e1 + e, body b is
    // r * body_stride + b; actions are n_rep x 6 per substep.
    int nrep = 1, n1 = 0, e1 = 0, body_stride = 0;
    int act_stride() const { return 6 * nrep; }
    void require_single(const char* what) const {
        if (nrep > 1) throw FlumeError(FLUME_E_ARG, std::string(what) + ": not available on a replica context");
    }
    // replica contexts: the effector set travels in device memory, in the substep's record
    // (the grid update and, later, its adjoint read it), copied from a ring of pinned
    // staging slots (a slot is reused once its copy has run)
    static constexpr int kEffRingRep = 64;
    EffK<float>* h_effring = nullptr;
    std::vector<cudaEvent_t> effring_ev;
    int effring_i = 0;
    void fill_effk(size_t i, const EffState& e, EffK<float>& k) const;
    EffSet replica_effset(Record& r);
    EffSet effset_now(Record& r) { return nrep > 1 ? replica_effset(r) : make_effset(eff); }
    void check_error(long substep_base = 0);
    EffSet make_effset(const std::vector<EffState>& es) const;
    void advance_effectors(const double* action);
    bool empty = false;  // no particles at all (N == 0)
#ifndef FL_CAP_GRID
#define FL_CAP_GRID 1
#endif
#ifndef FL_CAP_HEAVY
#define FL_CAP_HEAVY 0  // (1: the cap below; it paid while the pair ran on two streams)
#endif
    // persistent block-list kernels: no more CTAs than ~one per 256 active particles (a
    // block holds ~8 particles per cell x 64 cells), so small scenes do not launch hundreds
    // of CTAs that only find the work counter exhausted
    int sm_count = 148;
    int light_grid(int grid, int active) const {
        if (!FL_CAP_GRID) return grid;
        return std::min(grid, std::max(sm_count, (active + 255) / 256));
    }
    int light_grid(int grid) const { return light_grid(grid, n_active); }
    // heavy (SVD / rigid) kernels: persistent CTAs beyond the heavy blocks only hold SM
    // resources the concurrent light kernel needs (a CTA of the 256-thread variant takes
    // half an SM's registers), so the grid follows the heavy particle count (~2 blocks
    // per 512 particles, partial blocks at the bodies' faces); the work counter keeps any
    // underestimate correct.  Not after an upload that handed in full liquid F (those
    // particles take the heavy path for a substep).
    long n_heavy = 0;
    int heavy_grid(int grid) const {
        if (upload_full || !FL_CAP_HEAVY) return grid;
        return std::min(grid, int(std::max<long>(sm_count / 4, 2 * ((n_heavy + 511) / 512) + 16)));
    }
    // heavy (SVD / rigid) blocks are possible: a heavy class is present, or the last upload
    // (or an adjoint_substep call) handed in a liquid with a full F (kMetaFull)
    bool classes_heavy = true, upload_full = true;
    void upload(const flume_state_view* view);
    void download(flume_state_view* view);
    void set_effectors(const flume_state_view* view);
    void download_meta(flume_state_view* view);
    void require_particles() const {
        if (empty) throw FlumeError(FLUME_E_SCENE, "scene has no particles");
    }
    void sort_and_lists(StateBuf& st, Record& r, const Record* prev = nullptr);
    void forward_substep(const double* action, StatePtr in, StatePtr out, Record& r);
    void substep(const double* action, int count);
    void stage_grid(double* mass, double* vel);
    LossSet make_lossset(const flume_loss_desc* loss, std::vector<std::shared_ptr<void>>& keep);
    // one loss set per replica: the scene's terms on that replica's bodies
    std::vector<LossSet> replica_lossets(const flume_loss_desc* loss, std::vector<std::shared_ptr<void>>& keep) {
        std::vector<LossSet> lss;
        lss.push_back(make_lossset(loss, keep));
        for (int r = 1; r < nrep; r++) {
            if (loss->attraction_weight > 0 && loss->n_prev > 0)
                throw FlumeError(FLUME_E_ARG, "the attraction term is not available on a replica context");
            flume_loss_desc dr = *loss;
            std::vector<flume_loss_term> terms(loss->terms, loss->terms + loss->n_terms);
            for (auto& t : terms) t.body += r * body_stride;
            dr.terms = terms.data();
            lss.push_back(make_lossset(&dr, keep));
        }
        return lss;
    }
    // effector-bar slots per substep (partials, final sums, spawn bars): at least kMaxEff
    int eslots() const { return std::max<int>(kMaxEff, int(eff_shapes.size())); }
    PointLossScratch pls;  // trajectory_chamfer / mixing_spread scratch (fl_loss.cu)
    void point_losses(StateBuf& st, const LossSet& ls, uint32_t mask, int seg, double* out_dev, BarBuf* bars);
    void make_attraction(const flume_loss_desc* loss, LossSet& ls, std::vector<std::shared_ptr<void>>& keep);
    void per_particle(const flume_loss_desc* loss, double* out);
    // ls evaluated on a state at `substep` (activation semantics of parked particles)
    static LossSet at_substep(const LossSet& ls, long substep) {
        LossSet l = ls;
        l.substep = substep;
        return l;
    }
    uint32_t loss_mask(const flume_loss_desc* loss, int seg, int nseg) const;
    void eval_loss(StateBuf& st, const LossSet& ls, uint32_t mask, double* out_dev, int seg, long substep);
    // rep_total (replica contexts): the n_rep losses; per_seg then holds n_rep x n_segments
    double rollout_loss(const flume_actions* a, const flume_loss_desc* loss, long window, double* per_seg,
                        bool keep_final = false, double* rep_total = nullptr);
    void adjoint_step(StateBuf& pre, StateBuf& post_st, Record& r, DevArr<float>& bars_post, DevArr<float>& bars_pre,
                      int t_slot);
    void grad_trajectory(const flume_actions* a, const flume_loss_desc* loss, long stride, long window,
                         double* grad, double* loss_out, double* full_loss, double* per_seg, long* snapshots);
    void adjoint_substep_api(const double* action, double* xb, double* vb, double* Fb, double* Cb, double* eb,
                             double* abar_out);
    void copy_state(StateBuf& dst, const StateBuf& src) {
        dst.n = src.n;
        CK(cudaMemcpyAsync(dst.mem, src.mem, src.bytes, cudaMemcpyDeviceToDevice, stream));
    }
};

// ---------------------------------------------------------------------------
void Ctx::init(const flume_scene_desc* desc, int dev, int n_replicas) {
    device = dev;
    CK(cudaSetDevice(dev));
    CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    if (const char* dm = getenv("FL_DUAL_MODE")) dual_mode = atoi(dm);  // A/B experiments (tools/dual_probe.py)
    CK(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    wq.alloc(kWq);
    CK(cudaMemsetAsync(wq.p, 0, kWq * sizeof(int), stream));
    cfg = desc->config;
    N = int(desc->n_particles);
    if (N < 0) throw FlumeError(FLUME_E_ARG, "negative particle count");
    nrep = n_replicas;
    n1 = N / nrep;
    e1 = desc->n_effectors / nrep;
    mats.assign(desc->materials, desc->materials + desc->n_materials);
    eff_shapes.assign(desc->effectors, desc->effectors + desc->n_effectors);
    if (e1 > kMaxEff) throw FlumeError(FLUME_E_ARG, "at most 8 effectors are supported");

    // geometry (types.hpp:67-95)
    const double dx = cfg.domain[0] / cfg.grid_resolution;
    Geom& g = geom;
    for (int a = 0; a < 3; a++) {
        g.nd[a] = int(std::lround(cfg.domain[a] / dx)) + 1;
        g.NB[a] = (g.nd[a] + 3) / 4;
        g.lo[a] = float(dx);
        g.hi[a] = float(cfg.domain[a] - dx);
        g.gdt[a] = float(cfg.gravity[a] * cfg.dt_substep);
    }
    g.rstride = 0;
    if (nrep > 1) {  // replicas side by side along x, one empty block column between them
        g.rstride = g.NB[0] + 1;
        g.NB[0] = nrep * g.rstride - 1;
    }
    g.nbtot = g.NB[0] * g.NB[1] * g.NB[2];
    g.key_inactive = uint32_t(g.nbtot) << 6;
    g.key_departed = uint32_t(g.nbtot + 1) << 6;
    g.keybits = bits_for(g.key_departed);
    g.colblocks = g.NB[1] * g.NB[2];
    g.sx0 = 0;
    g.sx1 = g.NB[0];
    if (N == 0) {
        // an empty scene (no bodies): substeps only move the effectors and the clock,
        // like the reference's particle loops over nothing (test_cli.cpp:75-84)
        empty = true;
        eff.resize(eff_shapes.size());
        return;
    }
    g.idbits = bits_for(uint64_t(N - 1));
    if (g.keybits + g.idbits > 64) throw FlumeError(FLUME_E_ARG, "grid too large for 64-bit sort keys");
    g.dx = float(dx);
    g.inv_dx = float(1.0 / dx);
    g.dt = float(cfg.dt_substep);
    g.bw = cfg.boundary_width;
    g.vmax = float(cfg.cfl_fraction * dx / cfg.dt_substep);
    g.mass_eps = float(cfg.mass_epsilon);
    g.eps_cells = float(cfg.contact_eps_cells);
    g.hard = cfg.hard_contact;
    g.k4 = float(4.0 / (dx * dx));
    g.stress_coeff = float(cfg.dt_substep * 4.0 / (dx * dx));
    maxb = std::min(g.nbtot, N);
    g.maxb = maxb;

    // per-particle immutable fields and the class table
    p_mat.assign(desc->material_id, desc->material_id + N);
    p_body.assign(desc->body_id, desc->body_id + N);
    p_mass.assign(desc->mass, desc->mass + N);
    p_vol0.assign(desc->volume0, desc->volume0 + N);
    p_act.assign(N, 0);
    if (desc->activation_substep) p_act.assign(desc->activation_substep, desc->activation_substep + N);

    // rigid bodies
    nbody = desc->n_rigid;
    rb_off.assign(1, 0);
    mrank_by_id.assign(N, -1);
    std::vector<int> rigid_of_id(N, -1);
    for (int b = 0; b < nbody; b++) {
        const flume_rigid_body& rb = desc->rigid[b];
        if (rb.n_members < 3) throw FlumeError(FLUME_E_RIGIDITY, "rigid_shape_match: bad point lists");
        rb_id.push_back(rb.body_id);
        rb_total.push_back(rb.total_mass);
        double sm[3] = {0, 0, 0};
        for (long j = 0; j < rb.n_members; j++) {
            long pid = rb.members[j];
            if (pid < 0 || pid >= N) throw FlumeError(FLUME_E_ARG, "rigid member out of range");
            mrank_by_id[pid] = int(rb_members.size());
            rigid_of_id[pid] = b;
            rb_members.push_back(pid);
            member_body.push_back(b);
            for (int a = 0; a < 3; a++) rb_rest.push_back(rb.rest_offsets[3 * j + a]);
            rb_mass.push_back(p_mass[pid]);
            for (int a = 0; a < 3; a++) sm[a] += p_mass[pid] * rb.rest_offsets[3 * j + a];
        }
        for (int a = 0; a < 3; a++) rb_smrest.push_back(sm[a]);
        rb_off.push_back(int(rb_members.size()));
        for (long m0 = 0; m0 < rb.n_members; m0 += kRigidChunk) {
            chunk_body.push_back(b);
            chunk_m0.push_back(rb_off[b] + int(m0));
            chunk_m1.push_back(rb_off[b] + int(std::min<long>(rb.n_members, m0 + kRigidChunk)));
        }
    }
    nmem = int(rb_members.size());

    std::map<std::tuple<int, int, double, double, int, int>, uint32_t> cmap;
    p_class.resize(N);
    for (int i = 0; i < N; i++) {
        if (p_mat[i] < 0 || p_mat[i] >= int(mats.size())) throw FlumeError(FLUME_E_SCENE, "bad material id");
        const int rep = i / std::max(n1, 1);
        auto key = std::make_tuple(p_mat[i], p_body[i], p_mass[i], p_vol0[i], rigid_of_id[i], rep);
        auto it = cmap.find(key);
        if (it == cmap.end()) {
            const flume_material& m = mats[p_mat[i]];
            ClassInfo ci{};
            ci.kind = m.kind;
            ci.body = p_body[i];
            ci.rigid = rigid_of_id[i];
            ci.heavy = (m.kind != MK_LIQUID || m.mu != 0.0 || rigid_of_id[i] >= 0) ? 1 : 0;
            ci.iso = ((m.kind == MK_LIQUID || m.kind == MK_VISCOUS) && rigid_of_id[i] < 0) ? 1 : 0;
            ci.mass = float(p_mass[i]);
            ci.vol0 = float(p_vol0[i]);
            ci.mu = float(m.mu);
            ci.lambda = float(m.lambda);
            ci.theta_c = float(m.theta_c);
            ci.theta_s = float(m.theta_s);
            ci.sigma_y = float(m.sigma_y);
            ci.rep = rep;
            it = cmap.emplace(key, uint32_t(classes.size())).first;
            classes.push_back(ci);
        }
        p_class[i] = it->second;
    }

    // emitters
    emitter_of.assign(N, -1);
    emitters.assign(desc->emitters, desc->emitters + desc->n_emitters);
    for (size_t k = 0; k < emitters.size(); k++) emitter_of[emitters[k].particle] = int(k);

    // device constants
    d_cls.upload(classes, stream);
    d_rb_off.upload(rb_off, stream);
    d_rb_id.upload(rb_id, stream);
    d_member_body.upload(member_body, stream);
    {
        std::vector<int> mid32(rb_members.begin(), rb_members.end());
        d_member_id.upload(mid32, stream);
    }
    d_mrank.upload(mrank_by_id, stream);
    d_chunk_body.upload(chunk_body, stream);
    d_chunk_m0.upload(chunk_m0, stream);
    d_chunk_m1.upload(chunk_m1, stream);
    d_rb_rest.upload(rb_rest, stream);
    d_rb_mass.upload(rb_mass, stream);
    d_rb_smrest.upload(rb_smrest, stream);
    d_rb_total.upload(rb_total, stream);
    std::vector<int> act32(N);
    for (int i = 0; i < N; i++) act32[i] = int(std::min<long>(p_act[i], 0x7fffffff));
    d_act.upload(act32, stream);

    // scratch
    if (N >= (1 << 26)) throw FlumeError(FLUME_E_ARG, "at most 2^26-1 particles per context");
    // one zero-memset per sort covers counts, heavy flags and fill cursors (with two
    // virtual blocks: parked, departed); node-block flags and the block map are
    // written in full by the list scan
    const size_t bz = size_t(g.nbtot) + 2;
    bzero.alloc(3 * bz);
    bcount = bzero.p;
    bheavy = bzero.p + bz;
    bfill = bzero.p + 2 * bz;
    isort_blk.alloc(2 * bz + 2);
    CK(cudaMemsetAsync(isort_blk.p, 0, isort_blk.n * sizeof(int), stream));
    inbox.alloc(bz * kInbox);
    mov.alloc(N);
    rold.alloc(maxb);
    for (int k = 0; k < 2; k++) okey[k].alloc(N);
    nbflag_arr.alloc(g.nbtot);
    nbflag = nbflag_arr.p;
    nbpos.alloc(g.nbtot);
    tile_sum.alloc(sort_list_tiles(g));
    bstart.alloc(g.nbtot + 2);
    skey.alloc(N);
    sslot.alloc(N);
    gk.alloc(2 * size_t(N) + 2);
    gv.alloc(2 * size_t(N) + 2);
    staging.alloc(size_t(maxb) * kTile);
    staging_bar.alloc(size_t(maxb) * kTile);
    gridbar.alloc(size_t(g.nbtot) * 64);
    d_err.alloc(1);
    CK(cudaMemsetAsync(d_err.p, 0xff, sizeof(unsigned long long), stream));
    d_nonfinite.alloc(1);
    rig_partial.alloc(std::max<size_t>(chunk_body.size(), 1) * 17);
    abar.alloc(std::max(nbody, 1) * 13);
    start_bar.alloc(std::max(nmem, 1) * 3);
    mbar.alloc(std::max(nmem, 1) * 6);
    loss_partial.alloc(size_t(kLossBlocks) * kMaxLossTerms);
    d_act_list.alloc(64);
    d_emit_list.alloc(64);
    CK(cudaMemsetAsync(gridbar.p, 0, gridbar.n * sizeof(float4), stream));



    // heavy kernels: a scene dominated by SVD/rigid particles (c3) wants them at high
    // occupancy; a mostly-liquid one (c4) at low occupancy beside the light kernel
    {
        long nh = 0;
        for (int i = 0; i < N; i++) nh += classes[p_class[i]].heavy;
        classes_heavy = nh > 0;
        n_heavy = nh;
        hvar = 2 * nh >= N ? 2 : 1;
        // fewer SVD/rigid blocks than SMs beside a liquid scene (c4's floater): they are the
        // dual launches' tail -> variant 3, 256-thread CTAs (a full block in fewer rounds)
        int nsm = 148;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        if (hvar == 1 && nh < long(nsm) * 512) hvar = 3;
        if (const char* hv = getenv("FL_HVAR")) hvar = atoi(hv);  // A/B experiments
    }
    grid_p2g = occupancy_grid(KG_P2G, 0);
    grid_p2g_h = occupancy_grid(KG_P2G, hvar);
    grid_g2p = occupancy_grid(KG_G2P, 0);
    grid_g2p_h = occupancy_grid(KG_G2P, hvar);
    grid_adj = occupancy_grid(KG_ADJ_G2P, 0);
    grid_adj_h = occupancy_grid(KG_ADJ_G2P, hvar);
    grid_ap = occupancy_grid(KG_ADJ_P2G, 0);
    grid_ap_h = occupancy_grid(KG_ADJ_P2G, hvar);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    sm_count = sms;
    grid_upd = sms * 8;
    // grid adjoint: one 64-thread CTA per node block up to kEffBlocks; small scenes get fewer
    // (every CTA writes its effector-bar partials, which the final sums then read).  Sized by
    // the scene (grid-stride loop over the touched node blocks: never more CTAs than node
    // blocks or ~1 per 64 particles), at least one CTA per SM.
    eff_blocks = std::max(sm_count, std::min({kEffBlocks, g.nbtot, (N + 63) / 64}));
    if (nrep > 1) eff_blocks = std::min(eff_blocks, 4 * sm_count);  // rows of every replica's effectors
    eff_partial.alloc(size_t(kEffRing) * 2 * eff_blocks * eslots() * 18);  // (slabs: interior + edge rows)
#ifndef FL_SORT_CTAS
#define FL_SORT_CTAS 16  // per-block sort CTAs per SM (round-2 end: 8 -> 16, c4 sort 29.2 -> 27.5 us)
#endif
    grid_sort = sms * FL_SORT_CTAS;


    // initial effector state from the shapes' defaults is set by upload()
    eff.resize(eff_shapes.size());
    new_scratch();
    cur = get_state();
    CK(cudaStreamSynchronize(stream));
}

EffSet Ctx::make_effset(const std::vector<EffState>& es) const {
    EffSet s{};
    s.n = int(es.size());
    for (size_t i = 0; i < es.size(); i++) fill_effk(i, es[i], s.e[i]);
    return s;
}

EffSet Ctx::replica_effset(Record& r) {
    const size_t ne = eff.size();
    if (!h_effring) {
        CK(cudaMallocHost(&h_effring, size_t(kEffRingRep) * ne * sizeof(EffK<float>)));
        effring_ev.assign(kEffRingRep, nullptr);
    }
    const int slot = effring_i;
    effring_i = (effring_i + 1) % kEffRingRep;
    if (effring_ev[slot]) CK(cudaEventSynchronize(effring_ev[slot]));  // its last copy has run
    else CK(cudaEventCreateWithFlags(&effring_ev[slot], cudaEventDisableTiming));
    EffK<float>* h = h_effring + size_t(slot) * ne;
    for (size_t i = 0; i < ne; i++) fill_effk(i, eff[i], h[i]);
    EffK<float>* d = r.effx;
    CK(cudaMemcpyAsync(d, h, ne * sizeof(EffK<float>), cudaMemcpyHostToDevice, stream));
    CK(cudaEventRecord(effring_ev[slot], stream));
    EffSet s{};
    s.n = int(ne);
    s.per_rep = e1;
    s.ext = d;
    return s;
}

void Ctx::fill_effk(size_t i, const EffState& e, EffK<float>& k) const {
    const flume_effector_shape& sh = eff_shapes[i];
    k.shape.kind = sh.shape_kind;
    k.shape.radius = float(sh.radius);
    k.shape.half = V3<float>{float(sh.half_extents[0]), float(sh.half_extents[1]), float(sh.half_extents[2])};
    k.shape.seg_a = V3<float>{float(sh.seg_a[0]), float(sh.seg_a[1]), float(sh.seg_a[2])};
    k.shape.seg_b = V3<float>{float(sh.seg_b[0]), float(sh.seg_b[1]), float(sh.seg_b[2])};
    k.shape.normal = V3<float>{float(sh.plane_normal[0]), float(sh.plane_normal[1]), float(sh.plane_normal[2])};
    k.shape.offset = float(sh.plane_offset);
    k.shape.half_height = float(sh.half_height);
    // world shape pose = compose(pose, sdf.pose) in fp64 (sdf.hpp:17-22)
    M3<double> sR;
    for (int q = 0; q < 9; q++) sR.m[q] = sh.shape_R[q];
    V3<double> st = {sh.shape_t[0], sh.shape_t[1], sh.shape_t[2]};
    V3<double> wt = e.t + e.R * st;
    M3<double> wR = e.R * sR;
    k.wt = V3<float>{float(wt.x), float(wt.y), float(wt.z)};
    for (int q = 0; q < 9; q++) {
        k.wR.m[q] = float(wR.m[q]);
        k.shapeR.m[q] = float(sR.m[q]);
    }
    k.shapet = V3<float>{float(st.x), float(st.y), float(st.z)};
    k.pt = V3<float>{float(e.t.x), float(e.t.y), float(e.t.z)};
    k.vlin = V3<float>{float(e.vlin.x), float(e.vlin.y), float(e.vlin.z)};
    k.wang = V3<float>{float(e.w.x), float(e.w.y), float(e.w.z)};
    k.sticky = std::isinf(sh.friction_mu) ? 1 : 0;
    k.mu = k.sticky ? 0.f : float(sh.friction_mu);
}

// mpm.hpp:418-433, fp64 on the host
void Ctx::advance_effectors(const double* action) {
    const double dt = cfg.dt_substep;
    for (size_t i = 0; i < eff.size(); i++) {
        const flume_effector_shape& sh = eff_shapes[i];
        EffState& e = eff[i];
        const double* act = action + 6 * (nrep > 1 ? int(i) / e1 : 0);  // replicas: their own actions
        for (int a = 0; a < 3; a++)
            if (sh.action_mask[a]) e.vlin[a] = act[a];
        for (int a = 0; a < 3; a++)
            if (sh.action_mask[3 + a]) e.w[a] = act[3 + a];
        e.t = e.t + e.vlin * dt;
        e.R = advance_rotation(e.R, e.w, dt);
    }
}

void Ctx::check_error(long /*substep_base*/) {
    check_launch();  // a rejected <<<>>> launch (invalid config, resources) must not pass silently
    unsigned long long h = 0;
    allreduce(d_err.p, 1, DType::U64, ROp::Min);  // slabs: every rank raises the same error
    CK(cudaMemcpyAsync(&h, d_err.p, sizeof(h), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    if (h == ~0ull) return;
    uint32_t who = uint32_t(h & 0xffffffffull);
    uint32_t stage = uint32_t((h >> 32) & 0xf);
    long sub = long(h >> 36);
    unsigned long long reset = ~0ull;
    CK(cudaMemcpy(d_err.p, &reset, sizeof(reset), cudaMemcpyHostToDevice));
    switch (stage) {
        case ES_P2G_ESCAPE: {
            FlumeError e(FLUME_E_ENGINE, "p2g: particle " + std::to_string(who) + " escaped the clamped region");
            e.pid = who;
            e.substep = sub;
            throw e;
        }
        case ES_P2G_STRESS: {
            FlumeError e(FLUME_E_DEGENERATE, "corotated_stress: det(F) <= 0");
            e.pid = who;
            e.substep = sub;
            throw e;
        }
        case ES_G2P_PROJECT: {
            FlumeError e(FLUME_E_DEGENERATE, "g2p return map: det(F) <= 0 or singular value <= 0");
            e.pid = who;
            e.substep = sub;
            throw e;
        }
        case ES_RIGID: {
            FlumeError e(FLUME_E_RIGIDITY, "rigid_shape_match: degenerate covariance");
            e.body = int(who);
            e.substep = sub;
            throw e;
        }
        case ES_LOSS_EMPTY:
            throw FlumeError(FLUME_E_ENGINE, who == 0 ? "chamfer_distance: empty point set"
                                                      : "mixing_spread_loss: need at least 2 particles");
        default: throw FlumeError(FLUME_E_ENGINE, "device error");
    }
}

// upload a SimState<3> view; canonical store order is established here
void Ctx::upload(const flume_state_view* view) {
    // upload_full (a liquid handed in with a full F, kMetaFull) is k_upload's device flag,
    // read back with the upload's final synchronisation
    upload_full = false;
    if (empty) {
        substep_index = view->substep_index;
        time = view->time;
        set_effectors(view);
        return;
    }
    for (int k = 0; k < 4; k++) d_up[k].alloc(size_t(N) * (k < 2 ? 3 : 9));
    CK(cudaMemcpyAsync(d_up[0].p, view->x, size_t(N) * 3 * 8, cudaMemcpyHostToDevice, stream));
    CK(cudaMemcpyAsync(d_up[1].p, view->v, size_t(N) * 3 * 8, cudaMemcpyHostToDevice, stream));
    CK(cudaMemcpyAsync(d_up[2].p, view->F, size_t(N) * 9 * 8, cudaMemcpyHostToDevice, stream));
    CK(cudaMemcpyAsync(d_up[3].p, view->C, size_t(N) * 9 * 8, cudaMemcpyHostToDevice, stream));
    substep_index = view->substep_index;
    time = view->time;
    // particles activating at or after this substep are parked in the tail; the
    // substep that reaches their activation index brings them in (mpm.hpp:435-449).
    // The split depends on the substep index alone: kept from the last upload at the same one.
    std::vector<uint8_t>& active = up_active;
    if (up_substep != substep_index || slab()) {
        active.assign(N, 0);
        up_pending.clear();
        up_inactive.clear();
        up_n_active = 0;
        for (int i = 0; i < N; i++) {
            bool act = p_act[i] < substep_index || (p_act[i] <= substep_index && emitter_of[i] < 0);
            active[i] = act ? 1 : 0;
            if (act)
                up_n_active++;
            else {
                up_inactive.push_back(uint32_t(i));
                up_pending[p_act[i]].push_back(i);
            }
        }
        up_substep = slab() ? -1 : substep_index;
        up_active_dev = false;
    }
    pending = up_pending;
    inactive_ids = up_inactive;
    n_active = up_n_active;
    if (slab()) {
        // split the columns by the uploaded positions (the same on every rank), keep
        // this slab's active particles; parked ones stay replicated on all slabs
        std::vector<uint32_t> keys(N, 0);
        parked_x.assign(size_t(N) * 3, 0.f);
        for (int i = 0; i < N; i++) {
            const float p[3] = {float(view->x[3 * size_t(i)]), float(view->x[3 * size_t(i) + 1]),
                                float(view->x[3 * size_t(i) + 2])};
            for (int a = 0; a < 3; a++) parked_x[3 * size_t(i) + a] = p[a];
            if (active[i]) cell_key(geom, p[0], p[1], p[2], keys[i]);
        }
        partition(keys, active);
        n_active = 0;
        for (int i = 0; i < N; i++) {
            if (!active[i]) continue;
            const int col = key_col(geom, keys[i]);
            if (col < geom.sx0 || col >= geom.sx1)
                active[i] = 2;
            else
                n_active++;
        }
    }
    if (!d_upmeta.p) d_upmeta.upload(p_class, stream);  // (fixed per context)
    if (!up_active_dev || slab()) {
        d_upactive.upload(active, stream);
        up_active_dev = true;
    }
    d_anyfull.alloc(1);
    CK(cudaMemsetAsync(d_anyfull.p, 0, sizeof(int), stream));
    StatePtr raw = get_state();
    launch_upload(geom, raw->p, N, d_up[0].p, d_up[1].p, d_up[2].p, d_up[3].p, d_upmeta.p, d_upactive.p, d_cls.p,
                  d_anyfull.p, stream);
    launches++;
    // positions by id at upload: a parked particle keeps them until its activation substep,
    // which is where a loss evaluated at that substep sees it (emission happens in place)
    d_x0.alloc(size_t(N) * 3);
    CK(cudaMemcpyAsync(d_x0.p, raw->p.f, size_t(N) * 3 * sizeof(float), cudaMemcpyDeviceToDevice, stream));
    scratch_rec->n_active = n_active;
    scratch_rec->n_keep = n_active + n_parked();
    scratch_rec->n_stored = N;
    if (slab()) rec_counts_from_host(*scratch_rec, 0);
    sort_and_lists(*raw, *scratch_rec);
    launch_gather(raw->p, cur->p, scratch_rec->perm, scratch_rec->n_keep, stream);
    n_stored = scratch_rec->n_keep;
    // cur is stored in this sort's order: the first substep can sort incrementally
    chain_rec = keep_counts() ? scratch_rec.get() : nullptr;
    chain_out = chain_rec ? cur.get() : nullptr;
    cur->n = n_stored;
    park_base = n_active;
    if (slab()) state_counts_from_host(*cur);
    launch_upload_rigid(cur->p, nmem, d_member_id.p, d_up[0].p, stream);
    launches += 3;
    put_state(raw);
    set_effectors(view);
    unsigned long long reset = ~0ull;
    CK(cudaMemcpyAsync(d_err.p, &reset, sizeof(reset), cudaMemcpyHostToDevice, stream));
    int anyfull = 0;
    CK(cudaMemcpyAsync(&anyfull, d_anyfull.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
    // escape check of the uploaded positions happens in the first P2G
    CK(cudaStreamSynchronize(stream));
    upload_full = anyfull != 0;
}

void Ctx::set_effectors(const flume_state_view* view) {
    for (size_t i = 0; i < eff.size(); i++) {
        const flume_effector_state& es = view->effectors[i];
        eff[i].t = V3<double>{es.pose_t[0], es.pose_t[1], es.pose_t[2]};
        for (int q = 0; q < 9; q++) eff[i].R.m[q] = es.pose_R[q];
        eff[i].vlin = V3<double>{es.linear_velocity[0], es.linear_velocity[1], es.linear_velocity[2]};
        eff[i].w = V3<double>{es.angular_velocity[0], es.angular_velocity[1], es.angular_velocity[2]};
    }
}

void Ctx::download(flume_state_view* view) {
    if (empty) {
        download_meta(view);
        return;
    }
    for (int k = 0; k < 4; k++) d_up[k].alloc(size_t(N) * (k < 2 ? 3 : 9));
    if (slab()) {
        sync_counts();
        // every rank fills its own particles (rank 0 also the parked ones) into
        // zeroed arrays; the all-reduce assembles the whole state on every rank
        for (int k = 0; k < 4; k++) CK(cudaMemsetAsync(d_up[k].p, 0, d_up[k].n * 8, stream));
        launch_download(cur->p, n_stored, d_up[0].p, d_up[1].p, d_up[2].p, d_up[3].p, rank == 0,
                        geom.key_inactive, d_cls.p, stream);
        for (int k = 0; k < 4; k++) allreduce(d_up[k].p, size_t(N) * (k < 2 ? 3 : 9), DType::F64, ROp::Sum);
    } else {
        launch_download(cur->p, N, d_up[0].p, d_up[1].p, d_up[2].p, d_up[3].p, 1, geom.key_inactive, d_cls.p,
                        stream);
    }
    launch_download_rigid(cur->p, nmem, d_member_id.p, d_up[0].p, stream);
    launches += 2;
    if (view->x) CK(cudaMemcpyAsync(view->x, d_up[0].p, size_t(N) * 3 * 8, cudaMemcpyDeviceToHost, stream));
    if (view->v) CK(cudaMemcpyAsync(view->v, d_up[1].p, size_t(N) * 3 * 8, cudaMemcpyDeviceToHost, stream));
    if (view->F) CK(cudaMemcpyAsync(view->F, d_up[2].p, size_t(N) * 9 * 8, cudaMemcpyDeviceToHost, stream));
    if (view->C) CK(cudaMemcpyAsync(view->C, d_up[3].p, size_t(N) * 9 * 8, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    download_meta(view);
}

void Ctx::download_meta(flume_state_view* view) {
    view->time = time;
    view->substep_index = substep_index;
    if (view->effectors)
        for (size_t i = 0; i < eff.size(); i++) {
            flume_effector_state& es = view->effectors[i];
            for (int a = 0; a < 3; a++) {
                es.pose_t[a] = eff[i].t[a];
                es.linear_velocity[a] = eff[i].vlin[a];
                es.angular_velocity[a] = eff[i].w[a];
            }
            for (int q = 0; q < 9; q++) es.pose_R[q] = eff[i].R.m[q];
        }
}

// keys -> canonical order + particle-block list (fl_sort.cu)
// prev: the record of the substep that produced st (st is stored in its sort order) --
// the incremental sort; nullptr: the full sort
void Ctx::sort_and_lists(StateBuf& st, Record& r, const Record* prev) {
    Geom& g = geom;
    const DN n = dn(r.n_stored, slab() ? r.dcnt + RC_STORED : nullptr);
    const bool keep = keep_counts();
    const size_t bz = size_t(g.nbtot) + 2;
    if (prev) {
        const IncSort is{prev->recs, prev->blockmap, prev->celltab, okey[okey_cur].p, okey[okey_cur ^ 1].p,
                         isort_blk.p, isort_blk.p + bz, inbox.p, isort_blk.p + 2 * bz, isort_blk.p + 2 * bz + 1,
                         mov.p, rold.p};
        launch_isort_diff(g, st.p, r.n_stored, d_cls.p, bcount, bheavy, is, upload_full, stream);
        launch_sort_lists(g, maxb, bcount, bheavy, bstart.p, nbflag, r.nb_list, r.n_nb, r.recs, r.blockmap,
                          r.n_blocks, tile_sum.p, &is, stream);
        launch_isort_place(g, st.p, d_cls.p, bcount, bstart.p, r.recs, r.n_blocks, maxb, is, sslot.p, r.perm,
                           r.celltab, gk.p, gv.p, grid_sort, 2 * sm_count, stream);
        okey_cur ^= 1;
        counters_clean = false;
        n_inc_sorts++;
        launches += 4;  // diff, list sums, list write, per-block sort
        return;
    }
    // the grid update clears bfill (counts kept) or all three arrays
    if (!counters_clean)
        CK(cudaMemsetAsync(bzero.p, 0, bzero.n * sizeof(int), stream));
    else if (keep)
        CK(cudaMemsetAsync(bzero.p, 0, 2 * bz * sizeof(int), stream));
    counters_clean = false;
    launch_sort_count(g, st.p, n, d_cls.p, bcount, bheavy, stream);
    launch_sort_lists(g, maxb, bcount, bheavy, bstart.p, nbflag, r.nb_list, r.n_nb, r.recs, r.blockmap, r.n_blocks,
                      tile_sum.p, nullptr, stream);
    launch_sort_scatter(g, st.p, n, bstart.p, bfill, skey.p, sslot.p, keep ? d_cls.p : nullptr, stream);
    launch_sort_blocks(g, bcount, bstart.p, r.recs, r.n_blocks, maxb, skey.p, sslot.p, r.perm, r.celltab, gk.p, gv.p,
                       keep ? okey[okey_cur ^ 1].p : nullptr, grid_sort, stream);
    if (keep) okey_cur ^= 1;
    n_full_sorts++;
    launches += 5;  // count, list sums, list write, scatter, per-block sort
}

// ---------------------------------------------------------------------------
// x-slabs: halo exchange of scatter tiles, particle migration, cotangent return
// ---------------------------------------------------------------------------
void Ctx::set_transport(std::unique_ptr<Transport> t) {
    comm = std::move(t);
    counters_clean = false;  // the sort counts were kept on one rank: clear them all
    chain_break();
    rank = comm->rank();
    nranks = comm->size();
    if (nranks > geom.NB[0]) throw FlumeError(FLUME_E_ARG, "more slab ranks than 4-cell columns along x");
    // ghost particle blocks of the two neighbour columns live past the block list
    staging.alloc((size_t(maxb) + 2 * size_t(geom.colblocks)) * kTile);
    staging_bar.alloc((size_t(maxb) + 2 * size_t(geom.colblocks)) * kTile);
    for (int d = 0; d < 2; d++) {
        halo_send[d].alloc(halo_bytes(geom));
        halo_recv[d].alloc(halo_bytes(geom));
    }
    // fixed-size migration messages: the CFL bound (< 1 cell per substep) lets only the
    // particles near a slab face leave, a small fraction of a slab; a substep that sends
    // more sets the overflow flag and the call is re-run with 4x the capacity
    set_mig_cap(4096);
    d_ovf.alloc(1);
    mig_bcnt.alloc(kMigCountInts);
    if (!s_comm) {
        CK(cudaStreamCreateWithFlags(&s_comm, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&ev_halo_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ev_halo_join, cudaEventDisableTiming));
    }
    CK(cudaMemsetAsync(d_ovf.p, 0, sizeof(int), stream));
    CK(cudaStreamSynchronize(stream));
}

void Ctx::set_mig_cap(int cap) {
    mig_cap = std::min(cap, N);
    for (int d = 0; d < 2; d++) {
        mig_send[d].alloc(mig_msg_bytes(mig_cap));
        mig_recv[d].alloc(mig_msg_bytes(mig_cap));
    }
    rec_pool.clear();  // records carry per-capacity migration slot lists
    new_scratch();
}

// Columns [cut[r], cut[r+1]) per rank, cut nearest to equal weight, at least
// one column each (flume_slab_split exposes it to the host tests).
static void slab_split(const double* w, int nc, int nranks, int* cut) {
    double tot = 0;
    for (int c = 0; c < nc; c++) tot += w[c];
    cut[0] = 0;
    cut[nranks] = nc;
    double acc = 0;
    int c = 0;
    for (int r = 1; r < nranks; r++) {
        const double want = tot * r / nranks;
        while (c < nc && acc + 0.5 * w[c] <= want) acc += w[c++];
        cut[r] = std::max(cut[r - 1] + 1, std::min(c, nc - (nranks - r)));
        while (c < cut[r]) acc += w[c++];
    }
}

// every rank computes the same split from the same uploaded state
void Ctx::partition(const std::vector<uint32_t>& keys, const std::vector<uint8_t>& active) {
    const int nc = geom.NB[0];
    std::vector<double> w(nc, 0.0);
    for (size_t i = 0; i < keys.size(); i++)
        if (active[i]) w[key_col(geom, keys[i])] += 1.0;
    std::vector<int> cut(nranks + 1, 0);
    slab_split(w.data(), nc, nranks, cut.data());
    geom.sx0 = cut[rank];
    geom.sx1 = cut[rank + 1];
}

// After a scatter into `stg` (P2G tiles or the G2P-adjoint grid cotangent):
// send tile planes 0,1 of the bottom column down and 4,5 of the top column up,
// install the received planes as ghost blocks.  flags != nullptr (forward):
// also flag the owned node blocks reached only by the lower neighbour's tiles.
void Ctx::halo_exchange(int* blockmap, float4* stg, int* flags, cudaStream_t st) {
    Geom& g = geom;
    if (!st) st = stream;
    const bool lo = rank > 0, hi = rank + 1 < nranks;
    if (lo) launch_halo_pack(g, blockmap, stg, g.sx0, 0, halo_send[0].p, st);
    if (hi) launch_halo_pack(g, blockmap, stg, g.sx1 - 1, 4, halo_send[1].p, st);
    const size_t hb = halo_bytes(g);
    const void* sb[2] = {halo_send[0].p, halo_send[1].p};
    void* rb[2] = {halo_recv[0].p, halo_recv[1].p};
    const size_t sz[2] = {lo ? hb : 0, hi ? hb : 0};
    comm->neighbor_exchange(sb, sz, rb, sz, st);
    if (lo)
        launch_halo_unpack(g, halo_recv[0].p, g.sx0 - 1, 4, maxb, blockmap, stg, flags, flags ? g.sx0 : -1, st);
    if (hi) launch_halo_unpack(g, halo_recv[1].p, g.sx1, 0, maxb + g.colblocks, blockmap, stg, nullptr, -1, st);
    launches += 2 * (int(lo) + int(hi));
}

// Particles whose post-G2P base cell left the slab go to the neighbour (CFL:
// < 1 cell per substep, so never further); arrivals are appended after the
// parked tail.  Fixed-size messages carry their counts in a header, and one thread
// turns the headers into the record's and the post-state's device counts: no host
// round trip.  The host keeps upper bounds for launch sizes (tightened from the
// device counts read back asynchronously, host_bounds()).
void Ctx::migrate(StateBuf& out, Record& r) {
    const bool lo = rank > 0, hi = rank + 1 < nranks;
    launch_mig_pack(geom, out.p, dn(r.n_active, r.dcnt + RC_ACTIVE), lo ? mig_send[0].p : nullptr,
                    hi ? mig_send[1].p : nullptr, r.mig_src, mig_cap, mig_bcnt.p, d_ovf.p, stream);
    const size_t mb = mig_msg_bytes(mig_cap);
    const void* sb[2] = {mig_send[0].p, mig_send[1].p};
    void* rb[2] = {mig_recv[0].p, mig_recv[1].p};
    const size_t sz[2] = {lo ? mb : 0, hi ? mb : 0};
    comm->neighbor_exchange(sb, sz, rb, sz, stream);
    launch_mig_counts(lo ? mig_send[0].p : nullptr, hi ? mig_send[1].p : nullptr, lo ? mig_recv[0].p : nullptr,
                      hi ? mig_recv[1].p : nullptr, r.dcnt, out.cnt, mig_cap, N, d_ovf.p, stream);
    if (lo) launch_mig_unpack(out.p, mig_recv[0].p, r.dcnt, 0, mig_cap, stream);
    if (hi) launch_mig_unpack(out.p, mig_recv[1].p, r.dcnt, 1, mig_cap, stream);
    r.readback_counts(stream);
    launches += 3 + int(lo) + int(hi);
    // host upper bounds: every neighbour sends at most mig_cap
    const int in_max = (int(lo) + int(hi)) * mig_cap;
    n_active = std::min(N, n_active + in_max);
    n_stored = std::min(N, r.n_keep + in_max);
}

// Backward of migrate(): before the adjoint of substep r, the cotangents of the
// particles that arrived here travel back into the departed slots of their
// previous slab (message order = the forward's; counts from the record).
void Ctx::return_bars(Record& r, BarBuf post) {
    const bool lo = rank > 0, hi = rank + 1 < nranks;
    if (lo) launch_bars_pack(post, r.dcnt, 0, mig_cap, mig_send[0].p, stream);
    if (hi) launch_bars_pack(post, r.dcnt, 1, mig_cap, mig_send[1].p, stream);
    // exact sizes: the forward's counts came back to the host while it ran
    const int* hc = r.host_counts();
    auto bytes = [](int n) { return size_t(16 + 24 * size_t(n)) * sizeof(float); };
    const void* sb[2] = {mig_send[0].p, mig_send[1].p};
    void* rb[2] = {mig_recv[0].p, mig_recv[1].p};
    const size_t ss[2] = {lo ? bytes(hc[RC_RECV]) : 0, hi ? bytes(hc[RC_RECV + 1]) : 0};
    const size_t rs[2] = {lo ? bytes(hc[RC_SENT]) : 0, hi ? bytes(hc[RC_SENT + 1]) : 0};
    comm->neighbor_exchange(sb, ss, rb, rs, stream);
    if (lo) launch_bars_scatter(post, mig_recv[0].p, r.mig_src, r.dcnt, 0, mig_cap, stream);
    if (hi) launch_bars_scatter(post, mig_recv[1].p, r.mig_src + r.mig_cap, r.dcnt, 1, mig_cap, stream);
    launches += 2 * (int(lo) + int(hi));
}

void Ctx::forward_substep(const double* action, StatePtr in, StatePtr out, Record& r) {
    advance_effectors(action);
    r.substep = substep_index;
    r.effk = effset_now(r);
    // activation (mpm.hpp:435-449): ids reaching their activation substep
    r.act.clear();
    r.emit.clear();
    auto it = pending.find(substep_index);
    // slabs: activation slots are relative to the parked tail, whose first slot only the
    // device counts know (the record's RC_PARK)
    const int slot0 = slab() ? 0 : park_base;
    const int* slot_base = slab() ? r.dcnt + RC_PARK : nullptr;
    int gained = 0;
    if (it != pending.end()) {
        for (int id : it->second) {
            auto pos_it = std::lower_bound(inactive_ids.begin(), inactive_ids.end(), uint32_t(id));
            int slot = slot0 + int(pos_it - inactive_ids.begin());
            ActEntry a{};
            a.slot = slot;
            a.rep = nrep > 1 ? id / n1 : 0;
            int em = emitter_of[id];
            float px[3] = {parked_x.empty() ? 0.f : parked_x[3 * size_t(id)],
                           parked_x.empty() ? 0.f : parked_x[3 * size_t(id) + 1],
                           parked_x.empty() ? 0.f : parked_x[3 * size_t(id) + 2]};
            EmitAdjEntry ea{};
            bool has_emit = false;
            if (em >= 0) {
                const flume_emitter& e = emitters[em];
                V3<double> lp = {e.local_pos[0], e.local_pos[1], e.local_pos[2]};
                V3<double> lv = {e.local_vel[0], e.local_vel[1], e.local_vel[2]};
                V3<double> raw = lp, vel = lv;
                if (e.effector >= 0) {
                    const EffState& es = eff[e.effector];
                    raw = es.R * lp + es.t;
                    vel = es.R * lv;
                }
                ea.slot = slot;
                ea.eff = e.effector;
                a.has_xv = 1;
                for (int d = 0; d < 3; d++) {
                    double cl = clamp_ref(raw[d], double(geom.lo[d]), double(geom.hi[d]));
                    a.x[d] = float(cl);
                    a.v[d] = float(vel[d]);
                    px[d] = a.x[d];
                    ea.mask[d] = (cl != raw[d]) ? 1 : 0;
                    ea.local_pos[d] = lp[d];
                    ea.local_vel[d] = lv[d];
                }
                has_emit = true;
            }
            if (slab()) {  // the slab owning the activation cell takes the particle
                uint32_t key;
                cell_key(geom, px[0], px[1], px[2], key);
                const int col = key_col(geom, key);
                a.departed = (col < geom.sx0 || col >= geom.sx1) ? 1 : 0;
            }
            if (has_emit && !a.departed) r.emit.push_back(ea);
            if (!a.departed) gained++;
            r.act.push_back(a);
        }
        for (int id : it->second) {
            auto pos_it = std::lower_bound(inactive_ids.begin(), inactive_ids.end(), uint32_t(id));
            inactive_ids.erase(pos_it);
        }
        // parked slots are [n_active, n_active + parked): the activated ones are
        // re-keyed in place and sorted in; departed ones drop out at the next sort
        n_active += gained;
    }
    r.n_active = n_active;
    r.n_keep = n_active + n_parked();
    r.n_stored = n_stored;
    if (slab()) {  // the record's exact counts, from the pre-state's device counts
        launch_slab_counts_pre(in->cnt, r.dcnt, gained, n_parked(), mig_send[0].p, mig_send[1].p, stream);
        launches++;
    }
    if (!r.act.empty()) {
        if (r.act.size() <= size_t(kActInline)) {
            launch_activate_inline(geom, in->p, r.act.data(), int(r.act.size()), slot_base, stream);
        } else {
            d_act_list.alloc(r.act.size());
            CK(cudaMemcpyAsync(d_act_list.p, r.act.data(), r.act.size() * sizeof(ActEntry),
                               cudaMemcpyHostToDevice, stream));
            launch_activate(geom, in->p, d_act_list.p, int(r.act.size()), slot_base, stream);
            // the activation list buffer is reused next substep: order the copy
            CK(cudaStreamSynchronize(stream));
        }
        launches++;
    }
    const Record* prev = (keep_counts() && r.act.empty() && chain_rec && chain_rec != &r && chain_out == in.get())
                             ? chain_rec
                             : nullptr;
    PROF(K_SORT, sort_and_lists(*in, r, prev));
    PROF(K_P2G, dual([&](bool hv, int* w, cudaStream_t s) {
             launch_p2g(geom, in->p, r.perm, r.recs, r.n_blocks, r.celltab, hv ? heavy_grid(grid_p2g_h) : light_grid(grid_p2g), d_cls.p,
                        staging.p, d_err.p, uint32_t(substep_index), hv ? hvar : 0, w, s);
         }));
    // the adjoint's inputs (v0 = p/m, contact mask) only for substeps that keep a record
    const bool keep = !r.scratch;
    if (slab()) {
        // the halo planes travel on the comm stream while the interior node columns update
        // (they read no ghost tile); then the node-block list gains the blocks reached only
        // by ghost tiles and the two edge columns update
        const int c0 = rank > 0 ? geom.sx0 : -1, c1 = rank + 1 < nranks ? geom.sx1 : -1;
        CK(cudaEventRecord(ev_halo_fork, stream));
        CK(cudaStreamWaitEvent(s_comm, ev_halo_fork, 0));
        halo_exchange(r.blockmap, staging.p, nbflag, s_comm);
        CK(cudaEventRecord(ev_halo_join, s_comm));
        PROF(K_GRID, launch_grid_update(geom, r.nb_list, r.n_nb, grid_upd, r.blockmap, staging.p, r.gridv,
                                        keep ? r.gridv0 : nullptr, r.effk, keep ? r.cmask : nullptr, bzero.p,
                                        int(bzero.n), stream, 1, c0, c1));
        PROF(K_COMM, CK(cudaStreamWaitEvent(stream, ev_halo_join, 0)));
        launch_flag_list(nbflag, geom.nbtot, r.nb_list, r.n_nb, nbpos.p, stream);
        PROF(K_GRID, launch_grid_update(geom, r.nb_list, r.n_nb, grid_upd, r.blockmap, staging.p, r.gridv,
                                        keep ? r.gridv0 : nullptr, r.effk, keep ? r.cmask : nullptr, nullptr, 0,
                                        stream, 2, c0, c1));
        launches += 3;
    } else {
        PROF(K_GRID, launch_grid_update(geom, r.nb_list, r.n_nb, grid_upd, r.blockmap, staging.p, r.gridv,
                                        keep ? r.gridv0 : nullptr, r.effk, keep ? r.cmask : nullptr, clear_ptr(),
                                        clear_n(), stream));
    }
    counters_clean = true;
    RigidDev rd = rigid_dev(r);
    if (nbody > 0) {
        CK(cudaMemsetAsync(r.mslot, 0xff, size_t(nmem) * sizeof(int), stream));
        CK(cudaMemsetAsync(r.mid, 0, size_t(nmem) * 4 * sizeof(double), stream));
        CK(cudaMemcpyAsync(out->p.mx, in->p.mx, size_t(nmem) * 3 * sizeof(double), cudaMemcpyDeviceToDevice,
                           stream));
    }
    PROF(K_G2P, dual([&](bool hv, int* w, cudaStream_t s) {
             launch_g2p(geom, in->p, out->p, r.perm, r.recs, r.n_blocks, hv ? heavy_grid(grid_g2p_h) : light_grid(grid_g2p), d_cls.p, r.gridv,
                        rd, d_err.p, uint32_t(substep_index), hv ? hvar : 0, w, s);
         }));
    PROF(K_OTHER, launch_tail_copy(geom, in->p, out->p, r.perm, dn(r.n_active, slab() ? r.dcnt + RC_ACTIVE : nullptr),
                                   dn(r.n_keep, slab() ? r.dcnt + RC_KEEP : nullptr), n_parked(), stream));
    launches += 1 + (n_parked() > 0 ? 1 : 0);  // grid update, tail copy if any (dual() counts p2g, g2p)
    if (nbody > 0) {
        // slabs: every rank contributes its members' positions (disjoint support,
        // exact sum) so all ranks fit identical rigid transforms
        if (slab()) allreduce(r.mid, size_t(nmem) * 4, DType::F64, ROp::Sum);
        PROF(K_RIGID, launch_rigid(geom, out->p, rd, int(chunk_body.size()), d_chunk_body.p, d_chunk_m0.p,
                                   d_chunk_m1.p, rig_partial.p, d_err.p, uint32_t(substep_index), stream));
        launches += 3;
    }
    park_base = r.n_active;
    if (keep_counts()) {  // out is stored in r's sort order
        chain_rec = &r;
        chain_out = out.get();
    } else {
        chain_break();
    }
    if (slab()) {
        PROF(K_COMM, migrate(*out, r));
    } else {
        n_stored = r.n_keep;
    }
    out->n = n_stored;
    time += cfg.dt_substep;
    substep_index++;
    check_launch();
}

void Ctx::substep(const double* action, int count) {
    if (empty) {  // mpm_substep over no particles: effectors and clock only (mpm.hpp:455-473)
        for (int i = 0; i < count; i++) {
            advance_effectors(action);
            time += cfg.dt_substep;
            substep_index++;
        }
        return;
    }
    for (int i = 0; i < count; i++) {
        StatePtr nxt = get_state();
        forward_substep(action, cur, nxt, next_scratch());
        put_state(cur);
        cur = nxt;
    }
    check_error();
}

// p2g + grid_update on the live state without advancing (KAT harness)
void Ctx::stage_grid(double* mass, double* vel) {
    require_single("stage_grid");
    if (empty) {
        const size_t nn = size_t(geom.nd[0]) * geom.nd[1] * geom.nd[2];
        if (mass) std::fill(mass, mass + nn, 0.0);
        if (vel) std::fill(vel, vel + 3 * nn, 0.0);
        return;
    }
    Record& r = *scratch_rec;
    chain_break();  // this sort replaces the chained tables
    sync_counts();
    r.n_active = n_active;
    r.n_keep = n_active + n_parked();
    r.n_stored = n_stored;
    if (slab()) rec_counts_from_host(r, park_base);
    sort_and_lists(*cur, r);
    EffSet es = make_effset(eff);
    dual([&](bool hv, int* w, cudaStream_t s) {
        launch_p2g(geom, cur->p, r.perm, r.recs, r.n_blocks, r.celltab, hv ? heavy_grid(grid_p2g_h) : light_grid(grid_p2g), d_cls.p,
                   staging.p, d_err.p, uint32_t(substep_index), hv ? hvar : 0, w, s);
    });
    if (slab()) {
        halo_exchange(r.blockmap, staging.p, nbflag);
        launch_flag_list(nbflag, geom.nbtot, r.nb_list, r.n_nb, nbpos.p, stream);
    }
    launch_grid_update(geom, r.nb_list, r.n_nb, grid_upd, r.blockmap, staging.p, r.gridv, r.gridv0, es, r.cmask,
                       clear_ptr(), clear_n(), stream);
    counters_clean = true;
    std::vector<float4> h(size_t(geom.nbtot) * 64);
    std::vector<int> bm(geom.nbtot);
    CK(cudaMemcpyAsync(h.data(), r.gridv, h.size() * sizeof(float4), cudaMemcpyDeviceToHost, stream));
    CK(cudaMemcpyAsync(bm.data(), r.blockmap, bm.size() * sizeof(int), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    check_error();
    // node blocks the grid update wrote (the rest of the dense array is stale)
    std::vector<char> touched(geom.nbtot, 0);
    for (int b = 0; b < geom.nbtot; b++) {
        if (bm[b] <= 0) continue;
        int bx, by, bz;
        block_unlin(geom, b, bx, by, bz);
        for (int d = 0; d < 8; d++) {
            int x = bx + (d >> 2), y = by + ((d >> 1) & 1), z = bz + (d & 1);
            if (x < geom.NB[0] && y < geom.NB[1] && z < geom.NB[2]) touched[block_lin(geom, x, y, z)] = 1;
        }
    }
    const int* nd = geom.nd;
    // slabs: each rank writes the node planes it owns
    const int i0 = slab() ? 4 * geom.sx0 : 0, i1 = slab() ? std::min(nd[0], 4 * geom.sx1) : nd[0];
    for (int i = i0; i < i1; i++)
        for (int j = 0; j < nd[1]; j++)
            for (int k = 0; k < nd[2]; k++) {
                size_t flat = (size_t(i) * nd[1] + j) * nd[2] + k;
                int blk = block_lin(geom, i >> 2, j >> 2, k >> 2);
                float4 v = touched[blk] ? h[node_index(geom, i, j, k)] : make_float4(0, 0, 0, 0);
                if (mass) mass[flat] = v.w;
                if (vel) {
                    vel[3 * flat] = v.x;
                    vel[3 * flat + 1] = v.y;
                    vel[3 * flat + 2] = v.z;
                }
            }
}

LossSet Ctx::make_lossset(const flume_loss_desc* loss, std::vector<std::shared_ptr<void>>& keep) {
    LossSet ls{};
    if (!loss || loss->n_terms <= 0) throw FlumeError(FLUME_E_SCENE, "scene has no loss specification");
    if (loss->n_terms > kMaxLossTerms) throw FlumeError(FLUME_E_ARG, "too many loss terms");
    ls.n = loss->n_terms;
    ls.act = d_act.p;
    ls.x0 = d_x0.p;
    ls.n_all = N;
    ls.count_parked = rank == 0 ? 1 : 0;
    ls.substep = substep_index;
    for (int k = 0; k < ls.n; k++) {
        const flume_loss_term& t = loss->terms[k];
        LossTermDev& d = ls.t[k];
        d.kind = t.kind;
        d.body = t.body;
        d.squared = t.squared;
        d.weight = t.weight;
        for (int a = 0; a < 3; a++) d.goal[a] = t.goal[a];
        d.init = nullptr;
        if (t.kind == FLUME_LOSS_HOLD_INITIAL) {
            // initial positions by particle id from the current (state0) store
            auto arr = std::make_shared<DevArr<float>>();
            arr->alloc(size_t(N) * 3);
            d_up[0].alloc(size_t(N) * 3);
            if (slab()) {
                sync_counts();
                CK(cudaMemsetAsync(d_up[0].p, 0, size_t(N) * 3 * 8, stream));
            }
            launch_download(cur->p, n_stored, d_up[0].p, nullptr, nullptr, nullptr, rank == 0, geom.key_inactive,
                            d_cls.p, stream);
            if (slab()) allreduce(d_up[0].p, size_t(N) * 3, DType::F64, ROp::Sum);
            std::vector<double> hx(size_t(N) * 3);
            CK(cudaMemcpyAsync(hx.data(), d_up[0].p, hx.size() * 8, cudaMemcpyDeviceToHost, stream));
            CK(cudaStreamSynchronize(stream));
            std::vector<float> fx(hx.begin(), hx.end());
            arr->upload(fx, stream);
            d.init = arr->p;
            keep.push_back(arr);
        } else if (t.kind == FLUME_LOSS_MIXING_SPREAD || t.kind == FLUME_LOSS_TRAJECTORY_CHAMFER) {
            if (slab()) throw FlumeError(FLUME_E_ARG, "point-set losses run on single-rank contexts only");
            int max_goals = 1;
            if (t.kind == FLUME_LOSS_TRAJECTORY_CHAMFER) {
                if (t.n_goal_steps < 1 || !t.goal_step_offsets || !t.goal_points)
                    throw FlumeError(FLUME_E_SCENE, "trajectory_chamfer: empty goal_trajectory");
                const long np = t.goal_step_offsets[t.n_goal_steps];
                for (int q = 0; q < t.n_goal_steps; q++) {
                    const long m = t.goal_step_offsets[q + 1] - t.goal_step_offsets[q];
                    if (m <= 0) throw FlumeError(FLUME_E_ENGINE, "chamfer_distance: empty point set");
                    max_goals = std::max<long>(max_goals, m);
                }
                auto arr = std::make_shared<DevArr<double>>();
                arr->alloc(size_t(np) * 3);
                CK(cudaMemcpyAsync(arr->p, t.goal_points, size_t(np) * 3 * 8, cudaMemcpyHostToDevice, stream));
                d.gpts = arr->p;
                d.goff_h = t.goal_step_offsets;
                d.nsteps = t.n_goal_steps;
                d.last_g0 = int(t.goal_step_offsets[t.n_goal_steps - 1]);
                d.last_ng = int(np - t.goal_step_offsets[t.n_goal_steps - 1]);
                keep.push_back(arr);
            }
            d.kind = t.kind == FLUME_LOSS_MIXING_SPREAD ? LK_SPREAD : LK_CHAMFER;
            pls.reserve(N, max_goals);
        } else if (t.kind != FLUME_LOSS_TARGET_POINT) {
            throw FlumeError(FLUME_E_SCENE, "loss kind not supported on device");
        }
    }
    if (loss->attraction_weight > 0 && loss->n_prev > 0) make_attraction(loss, ls, keep);
    return ls;
}

// LossEvaluator::enable_attraction + the prev_losses_ refresh_attraction stored
// (losses.hpp:350-363); tau as attraction_tau (losses.hpp:159-166)
void Ctx::make_attraction(const flume_loss_desc* loss, LossSet& ls, std::vector<std::shared_ptr<void>>& keep) {
    if (slab()) throw FlumeError(FLUME_E_ARG, "the attraction term runs on single-rank contexts only");
    if (!loss->prev_losses) throw FlumeError(FLUME_E_ARG, "attraction: prev_losses is null");
    if (!(loss->attraction_radius > 0)) throw FlumeError(FLUME_E_ARG, "attraction: radius must be positive");
    AttractionDev& A = ls.attr;
    const int body = loss->attraction_body < 0 ? loss->terms[0].body : loss->attraction_body;
    auto mrank = std::make_shared<DevArr<int>>();
    std::vector<int> hr(size_t(N), -1);
    int nm = 0;
    for (int i = 0; i < N; i++)
        if (p_body[size_t(i)] == body) hr[size_t(i)] = nm++;
    if (long(nm) != loss->n_prev) throw FlumeError(FLUME_E_ENGINE, "attraction_loss: loss list size mismatch");
    if (nm >= (1 << 24)) throw FlumeError(FLUME_E_ARG, "attraction: more than 2^24 members");
    std::vector<double> tmp(loss->prev_losses, loss->prev_losses + nm);
    double tau = loss->attraction_tau;
    if (!(tau > 0)) {
        std::nth_element(tmp.begin(), tmp.begin() + tmp.size() / 2, tmp.end());
        tau = std::max(0.1 * tmp[tmp.size() / 2], 1e-9);
    }
    unsigned long long ncell = 1;
    for (int a = 0; a < 3; a++) {
        // cells floor(x / radius) over the domain plus one pad cell on each side
        const double span = std::floor(cfg.domain[a] / loss->attraction_radius) + 3.0;
        if (span > double(1 << 20)) throw FlumeError(FLUME_E_ARG, "attraction: radius too small for the hash");
        A.nc[a] = int(span);
        ncell *= (unsigned long long)A.nc[a];
    }
    int bits = 1;
    while ((1ull << bits) < ncell) bits++;
    if (bits > 40) throw FlumeError(FLUME_E_ARG, "attraction: radius too small for the hash");
    mrank->upload(hr, stream);
    auto prev = std::make_shared<DevArr<double>>();
    prev->alloc(size_t(nm));
    CK(cudaMemcpyAsync(prev->p, loss->prev_losses, size_t(nm) * 8, cudaMemcpyHostToDevice, stream));
    CK(cudaStreamSynchronize(stream));  // the host copies above are temporaries
    keep.push_back(mrank);
    keep.push_back(prev);
    A.on = 1;
    A.n_members = nm;
    A.weight = loss->attraction_weight;
    A.radius = loss->attraction_radius;
    A.tau = tau;
    A.prev = prev->p;
    A.mrank = mrank->p;
    A.key_bits = bits;
    pls.reserve_attraction(std::max(nm, 1));
}

// LossEvaluator::per_particle (losses.hpp:367-390) of the current state, by particle id
void Ctx::per_particle(const flume_loss_desc* loss, double* out) {
    require_single("loss_per_particle");
    if (slab()) throw FlumeError(FLUME_E_ARG, "per_particle runs on single-rank contexts only");
    std::vector<std::shared_ptr<void>> keep;
    flume_loss_desc plain = *loss;
    plain.attraction_weight = 0;  // the surrogate is not part of per_particle
    const LossSet ls = at_substep(make_lossset(&plain, keep), substep_index);
    d_up[0].alloc(size_t(N));
    CK(cudaMemsetAsync(d_up[0].p, 0, size_t(N) * 8, stream));
    launch_per_particle(cur->p, cur->n, d_cls.p, ls, geom.key_departed, d_up[0].p, stream);
    launches += 1;
    CK(cudaMemcpyAsync(out, d_up[0].p, size_t(N) * 8, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    check_error();
}

// trajectory_chamfer / mixing_spread terms of `mask` (losses.hpp:474-551): eval adds
// weight * value into *out_dev (after the per-particle terms), grad adds into bars
void Ctx::point_losses(StateBuf& st, const LossSet& ls, uint32_t mask, int seg, double* out_dev, BarBuf* bars) {
    for (int k = 0; k < ls.n; k++) {
        if (!((mask >> k) & 1u) || ls.t[k].kind < LK_SPREAD) continue;
        launch_point_loss(pls, st.p, st.n, d_cls.p, ls, ls.t[k], seg, geom.key_inactive, out_dev, bars, d_err.p,
                          chamfer_mode, stream);
        launches += 5;
    }
    // attraction: every segment boundary, independent of the terms' eval mode (losses.hpp:332-345)
    if (ls.attr.on) {
        launch_attraction(pls, st.p, st.n, ls, geom.key_departed, out_dev, bars, stream);
        launches += 4;
    }
}

uint32_t Ctx::loss_mask(const flume_loss_desc* loss, int seg, int nseg) const {
    uint32_t m = 0;
    for (int k = 0; k < loss->n_terms; k++)
        if (!loss->terms[k].final_only || seg == nseg - 1) m |= 1u << k;
    return m;
}

void Ctx::eval_loss(StateBuf& st, const LossSet& ls0, uint32_t mask, double* out_dev, int seg, long substep) {
    const LossSet ls = at_substep(ls0, substep);
    // per-slab partial; the segment losses are all-reduced once after the rollout
    launch_loss(st.p, dn(st.n, slab() ? st.cnt + SC_STORED : nullptr), d_cls.p, ls, mask, loss_partial.p, out_dev,
                geom.key_inactive, stream);
    launches += 2;
    point_losses(st, ls, mask, seg, out_dev, nullptr);
}

double Ctx::rollout_loss(const flume_actions* a, const flume_loss_desc* loss, long window, double* per_seg,
                         bool keep_final, double* rep_total) {
    const long T = long(a->n_segments) * a->segment_length;
    if (window <= 0) window = T;
    std::vector<std::shared_ptr<void>> keep;
    std::vector<LossSet> lss = replica_lossets(loss, keep);
    const int nseg = a->n_segments;
    loss_out.alloc(size_t(nrep) * nseg);
    // state0 is const: work on a copy
    const long s0 = substep_index;
    const double time0 = time;
    const int na0 = n_active, ns0 = n_stored, pb0 = park_base;
    const std::vector<EffState> eff0 = eff;
    const std::vector<uint32_t> inact0 = inactive_ids;
    const auto pend0 = pending;
    StatePtr st = get_state();
    copy_state(*st, *cur);
    for (long t = 0; t < T; t++) {
        StatePtr nxt = get_state();
        forward_substep(a->values + act_stride() * (t / a->segment_length), st, nxt, next_scratch());
        put_state(st);
        st = nxt;
        if ((t + 1) % a->segment_length == 0) {
            int seg = int((t + 1) / a->segment_length) - 1;
            for (int r = 0; r < nrep; r++)
                eval_loss(*st, lss[size_t(r)], loss_mask(loss, seg, nseg), loss_out.p + size_t(r) * nseg + seg, seg,
                          substep_index);
        }
    }
    allreduce(loss_out.p, size_t(a->n_segments), DType::F64, ROp::Sum);
    std::vector<double> per(size_t(nrep) * nseg);
    CK(cudaMemcpyAsync(per.data(), loss_out.p, per.size() * 8, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    if (keep_final) {  // the context continues from the final state (rollout_loss's final_state)
        put_state(cur);
        cur = st;
    } else {
        put_state(st);
        substep_index = s0;
        time = time0;
        n_active = na0;
        n_stored = ns0;
        park_base = pb0;
        eff = eff0;
        inactive_ids = inact0;
        pending = pend0;
    }
    check_error();
    double total0 = 0;
    for (int r = nrep - 1; r >= 0; r--) {
        double total = 0;
        for (int s = 0; s < nseg; s++) {
            const double v = per[size_t(r) * nseg + s];
            if (per_seg) per_seg[size_t(r) * nseg + s] = v;
            if (long(s + 1) * a->segment_length <= window) total += v;
        }
        if (!std::isfinite(total)) throw FlumeError(FLUME_E_ENGINE, "rollout produced a non-finite loss");
        if (rep_total) rep_total[r] = total;
        total0 = total;
    }
    return total0;
}

// reverse one substep: bars_post (store order of state[t+1]) -> bars_pre (store order of state[t])
void Ctx::adjoint_step(StateBuf& pre, StateBuf& post_st, Record& r, DevArr<float>& bars_post, DevArr<float>& bars_pre,
                       int t_slot) {
    Geom& g = geom;
    BarBuf post{bars_post.p, N}, out{bars_pre.p, N};
    // slabs: cotangents of the particles that migrated in after this substep go home first
    if (slab()) PROF(K_COMM, return_bars(r, post));
    // the forward recorded this substep's grid (r.gridv, r.gridv0, r.cmask) and block map
    RigidDev rd = rigid_dev(r);
    if (nbody > 0) {
        launch_adj_rigid_gather(post, rd, mbar.p, stream);
        if (slab()) allreduce(mbar.p, size_t(nmem) * 6, DType::F64, ROp::Sum);
        PROF(K_RIGID, launch_adj_rigid(g, post, rd, int(chunk_body.size()), d_chunk_body.p, d_chunk_m0.p,
                                       d_chunk_m1.p, mbar.p, rig_partial.p, start_bar.p, abar.p, stream));
        launches += 4;
    }
    PROF(K_ADJ_G2P, dual([&](bool hv, int* w, cudaStream_t s) {
             launch_adj_g2p(g, pre.p, r.perm, r.recs, r.n_blocks, r.celltab, hv ? heavy_grid(grid_adj_h) : light_grid(grid_adj, r.n_active), d_cls.p,
                            r.gridv, post_st.p, post, xbar_tmp.p, Fbar_tmp.p, rd, start_bar.p, staging_bar.p, hv ? hvar : 0, w, s);
         }));
    const int es = eslots();
    double* ep = eff_partial.p + size_t(t_slot % kEffRing) * eff_rows() * es * 18;
    if (slab()) {
        // as in the forward: the halo planes of the v_bar tiles travel while the interior node
        // columns run their adjoint; the edge columns' effector-bar partials take the second
        // half of the substep's rows
        const int c0 = rank > 0 ? geom.sx0 : -1, c1 = rank + 1 < nranks ? geom.sx1 : -1;
        CK(cudaEventRecord(ev_halo_fork, stream));
        CK(cudaStreamWaitEvent(s_comm, ev_halo_fork, 0));
        halo_exchange(r.blockmap, staging_bar.p, nullptr, s_comm);
        CK(cudaEventRecord(ev_halo_join, s_comm));
        PROF(K_ADJ_GRID, launch_adj_grid(g, r.nb_list, r.n_nb, r.blockmap, staging_bar.p, r.gridv0, gridbar.p, r.effk,
                                         ep, r.cmask, eff_blocks, es * 18, stream, 1, c0, c1));
        PROF(K_COMM, CK(cudaStreamWaitEvent(stream, ev_halo_join, 0)));
        PROF(K_ADJ_GRID, launch_adj_grid(g, r.nb_list, r.n_nb, r.blockmap, staging_bar.p, r.gridv0, gridbar.p, r.effk,
                                         ep + size_t(eff_blocks) * es * 18, r.cmask, eff_blocks, es * 18, stream, 2, c0,
                                         c1));
        launches++;
    } else {
        PROF(K_ADJ_GRID, launch_adj_grid(g, r.nb_list, r.n_nb, r.blockmap, staging_bar.p, r.gridv0, gridbar.p, r.effk,
                                         ep, r.cmask, eff_blocks, es * 18, stream));
    }
    eff_pending(t_slot);
    PROF(K_ADJ_P2G, dual([&](bool hv, int* w, cudaStream_t s) {
             launch_adj_p2g(g, pre.p, r.perm, r.recs, r.n_blocks, hv ? heavy_grid(grid_ap_h) : light_grid(grid_ap, r.n_active), d_cls.p, gridbar.p,
                            xbar_tmp.p, Fbar_tmp.p, out, d_nonfinite.p + t_slot, hv ? hvar : 0, w, s);
         }));
    const int* rc = slab() ? r.dcnt : nullptr;
    PROF(K_OTHER, launch_tail_bars(post, out, r.perm, dn(r.n_active, rc ? rc + RC_ACTIVE : nullptr),
                                   dn(r.n_keep, rc ? rc + RC_KEEP : nullptr), dn(r.n_stored, rc ? rc + RC_STORED : nullptr),
                                   stream));
    launches += 1 + (r.n_stored > r.n_active ? 1 : 0);  // grid adjoint, tail bars (dual() counts the rest)
    check_launch();
    if (!r.emit.empty()) {
        double* eo = em_out.p + size_t(t_slot) * es * 12;
        if (r.emit.size() <= size_t(kEmitInline)) {
            launch_adj_emit_inline(out, r.emit.data(), int(r.emit.size()), eo, int(eff.size()),
                                   slab() ? r.dcnt + RC_PARK : nullptr, stream);
        } else {
            d_emit_list.alloc(r.emit.size());
            CK(cudaMemcpyAsync(d_emit_list.p, r.emit.data(), r.emit.size() * sizeof(EmitAdjEntry),
                               cudaMemcpyHostToDevice, stream));
            launch_adj_emit(out, d_emit_list.p, int(r.emit.size()), eo, int(eff.size()),
                            slab() ? r.dcnt + RC_PARK : nullptr, stream);
            CK(cudaStreamSynchronize(stream));
        }
        launches++;
    }
}

void Ctx::grad_trajectory(const flume_actions* a, const flume_loss_desc* loss, long stride, long window,
                          double* grad, double* loss_out_h, double* full_loss, double* per_seg, long* snapshots) {
    // replica contexts: grad = n_rep x n_segments x 6, loss_out_h / full_loss n_rep,
    // per_seg n_rep x n_segments
    const long T = long(a->n_segments) * a->segment_length;
    if (stride <= 0) stride = T;
    if (window <= 0) window = T;
    const int nseg = a->n_segments, seglen = a->segment_length;
    std::vector<std::shared_ptr<void>> keep;
    const std::vector<LossSet> lss = replica_lossets(loss, keep);
    loss_out.alloc(size_t(nrep) * nseg);
    const int es = eslots();
    eff_out.alloc(size_t(T) * es * 18);
    em_out.alloc(size_t(T) * es * 12);
    d_nonfinite.alloc(T);
    xbar_tmp.alloc(size_t(N) * 3);
    Fbar_tmp.alloc(size_t(N) * 9);
    CK(cudaMemsetAsync(em_out.p, 0, em_out.n * 8, stream));
    CK(cudaMemsetAsync(d_nonfinite.p, 0, size_t(T) * sizeof(int), stream));

    for (auto& e : tev)
        if (!e) CK(cudaEventCreate(&e));
    cudaEvent_t ev0 = tev[0], ev1 = tev[1], ev2 = tev[2];
    long launches0 = launches;

    // host-side replay context per substep start
    struct HostSnap {
        long substep;
        double time;
        int n_active, n_stored, park_base;
        std::vector<EffState> eff;
        std::vector<uint32_t> inactive;
        std::map<long, std::vector<int>> pending;
    };
    const long s0 = substep_index;
    const double time0 = time;
    auto take_host = [&]() {
        return HostSnap{substep_index, time, n_active, n_stored, park_base, eff, inactive_ids, pending};
    };
    auto restore_host = [&](const HostSnap& h) {
        substep_index = h.substep;
        time = h.time;
        n_active = h.n_active;
        n_stored = h.n_stored;
        park_base = h.park_base;
        eff = h.eff;
        inactive_ids = h.inactive;
        pending = h.pending;
    };
    const HostSnap host0 = take_host();
    std::vector<std::vector<EffState>> eff_pre(T), eff_post(T);

    // ---------------- forward with snapshots ----------------
    CK(cudaEventRecord(ev0, stream));
    std::map<long, StatePtr> snaps;
    std::map<long, HostSnap> host_snaps;
    const long last_base = ((T - 1) / stride) * stride;  // segment replayed first in the backward
    std::vector<StatePtr> cache_states;                   // indices [cache_base, ...]
    std::vector<RecordPtr> cache_recs;
    long cache_base = -1;

    std::map<long, HostPtr> hsnaps;  // snapshots spilled to pinned host memory
    struct FileSnap {
        off_t off;
        size_t bytes;
        int n;
    };
    std::map<long, FileSnap> fsnaps;  // snapshots spilled to the file tier
    if (spill == 2) {
        if (!fspill || fspill->slot_bytes() != cur->bytes) fspill.reset(new FileSpill(spill_dir, cur->bytes));
        fspill->reset();
    }
    // device buffers of spilled snapshots go back to the pool once their D2H finished
    std::vector<std::pair<StatePtr, cudaEvent_t>> spilling;
    std::vector<cudaEvent_t> own_events;  // (file tier: per-snapshot D2H events)
    auto retire_spilled = [&](bool all) {
        for (size_t i = 0; i < spilling.size();) {
            if (all || cudaEventQuery(spilling[i].second) == cudaSuccess || spilling.size() > 2) {
                CK(cudaStreamWaitEvent(stream, spilling[i].second, 0));
                put_state(spilling[i].first);
                spilling.erase(spilling.begin() + long(i));
            } else {
                i++;
            }
        }
    };
    auto take_snapshot = [&](long at, StatePtr s) {  // s stays the input of the next substep
        if (spill == 2 && at < last_base) {
            if (!cstream) {
                CK(cudaStreamCreateWithFlags(&cstream, cudaStreamNonBlocking));
                CK(cudaEventCreateWithFlags(&ev_snap, cudaEventDisableTiming));
            }
            CK(cudaEventRecord(ev_snap, stream));
            CK(cudaStreamWaitEvent(cstream, ev_snap, 0));
            fsnaps[at] = FileSnap{fspill->put(s->mem, s->bytes, cstream), s->bytes, s->n};
            cudaEvent_t e;
            CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            CK(cudaEventRecord(e, cstream));
            own_events.push_back(e);
            spilling.push_back({s, e});
        } else if (spill == 1 && at < last_base) {
            HostPtr h = spill_state(*s);
            hsnaps[at] = h;
            spilling.push_back({s, h->done});
        } else {
            snaps[at] = s;
        }
        host_snaps[at] = take_host();
    };
    StatePtr st = get_state();
    copy_state(*st, *cur);
    take_snapshot(0, st);
    for (long t = 0; t < T; t++) {
        const bool in_last = t >= last_base;
        if (in_last && cache_base < 0) {
            cache_base = t;
            cache_states.push_back(st);
        }
        if (!in_last) next_scratch();
        RecordPtr rec = in_last ? get_record() : scratch_rec;
        StatePtr nxt = get_state();
        eff_pre[t] = eff;
        forward_substep(a->values + act_stride() * (t / seglen), st, nxt, *rec);
        eff_post[t] = eff;
        if (in_last) {
            cache_recs.push_back(rec);
            cache_states.push_back(nxt);
        } else if (!snaps.count(t) && !hsnaps.count(t) && !fsnaps.count(t)) {
            put_state(st);
        }
        st = nxt;
        retire_spilled(false);
        if ((t + 1) % stride == 0) take_snapshot(t + 1, st);
        if ((t + 1) % seglen == 0) {
            int seg = int((t + 1) / seglen) - 1;
            for (int rp = 0; rp < nrep; rp++)
                eval_loss(*st, lss[size_t(rp)], loss_mask(loss, seg, nseg), loss_out.p + size_t(rp) * nseg + seg, seg,
                          substep_index);
        }
    }
    retire_spilled(true);
    const size_t n_snap = snaps.size() + hsnaps.size() + fsnaps.size();
    allreduce(loss_out.p, size_t(nseg), DType::F64, ROp::Sum);
    CK(cudaEventRecord(ev1, stream));
    std::vector<double> per(size_t(nrep) * nseg);
    CK(cudaMemcpyAsync(per.data(), loss_out.p, per.size() * 8, cudaMemcpyDeviceToHost, stream));
    check_error();
    std::vector<double> lsum(nrep, 0.0), fsum(nrep, 0.0);
    for (int rp = 0; rp < nrep; rp++) {
        for (int s = 0; s < nseg; s++) {
            fsum[rp] += per[size_t(rp) * nseg + s];
            if (long(s + 1) * seglen <= window) lsum[rp] += per[size_t(rp) * nseg + s];
        }
        if (!std::isfinite(lsum[rp])) throw FlumeError(FLUME_E_ENGINE, "grad_trajectory: non-finite forward loss");
    }

    // ---------------- backward ----------------
    
    barsA.alloc(size_t(N) * 24);
    barsB.alloc(size_t(N) * 24);
    CK(cudaMemsetAsync(barsA.p, 0, barsA.n * 4, stream));
    auto release_cache = [&]() {
        for (auto& s : cache_states) {
            bool is_snap = false;
            for (auto& kv : snaps)
                if (kv.second == s) is_snap = true;
            if (!is_snap) put_state(s);
        }
        for (auto& r : cache_recs) put_record(r);
        cache_states.clear();
        cache_recs.clear();
        cache_base = -1;
    };
    auto ensure_cached = [&](long t) {
        if (cache_base >= 0 && t >= cache_base && t < cache_base + long(cache_recs.size())) return;
        release_cache();
        const long base = (t / stride) * stride;
        long end = std::min(base + stride, T);
        restore_host(host_snaps[base]);
        StatePtr s;
        if (hsnaps.count(base)) {  // spilled: back into HBM (released with the cache)
            s = get_state();
            unspill(*hsnaps[base], *s);
        } else if (fsnaps.count(base)) {  // file tier: read back, and start reading the next older one
            const FileSnap& f = fsnaps[base];
            s = get_state();
            fspill->get(f.off, s->mem, f.bytes, stream);
            s->n = f.n;
            if (fsnaps.count(base - stride)) fspill->prefetch(fsnaps[base - stride].off, fsnaps[base - stride].bytes);
        } else {
            s = snaps.at(base);
        }
        cache_base = base;
        cache_states.push_back(s);
        for (long q = base; q < end; q++) {
            RecordPtr rec = get_record();
            StatePtr nxt = get_state();
            forward_substep(a->values + act_stride() * (q / seglen), s, nxt, *rec);
            cache_recs.push_back(rec);
            cache_states.push_back(nxt);
            s = nxt;
        }
    };
    for (long t = T - 1; t >= 0; t--) {
        if ((t + 1) % seglen == 0 && t + 1 <= window) {
            int seg = int((t + 1) / seglen) - 1;
            ensure_cached(t);
            StateBuf& boundary = *cache_states[size_t(t + 1 - cache_base)];
            for (int rp = 0; rp < nrep; rp++) {  // (replicas: disjoint particles, one pass each)
                const LossSet lsb = at_substep(lss[size_t(rp)], s0 + t + 1);
                launch_loss_grad(boundary.p, dn(boundary.n, slab() ? boundary.cnt + SC_STORED : nullptr), d_cls.p,
                                 lsb, loss_mask(loss, seg, nseg), BarBuf{barsA.p, N}, geom.key_inactive, stream);
                launches++;
                BarBuf bb{barsA.p, N};
                point_losses(boundary, lsb, loss_mask(loss, seg, nseg), seg, nullptr, &bb);
            }
        }
        ensure_cached(t);
        const size_t k = size_t(t - cache_base);
        adjoint_step(*cache_states[k], *cache_states[k + 1], *cache_recs[k], barsA, barsB, int(t));
        std::swap(barsA.p, barsB.p);
        std::swap(barsA.n, barsB.n);
    }
    release_cache();
    for (auto& kv : snaps) put_state(kv.second);
    for (auto& kv : hsnaps) host_pool.push_back(kv.second);
    for (cudaEvent_t e : own_events) cudaEventDestroy(e);
    eff_flush();
    if (slab()) {  // per-slab effector / spawn bars and non-finite flags
        allreduce(eff_out.p, size_t(T) * es * 18, DType::F64, ROp::Sum);
        allreduce(em_out.p, size_t(T) * es * 12, DType::F64, ROp::Sum);
        allreduce(d_nonfinite.p, size_t(T), DType::I32, ROp::Max);
    }
    CK(cudaEventRecord(ev2, stream));

    // ---------------- effector pose chain (host, fp64) ----------------
    std::vector<double> eb(size_t(T) * es * 18), em(size_t(T) * es * 12);
    std::vector<int> nonf(T);
    CK(cudaMemcpyAsync(eb.data(), eff_out.p, eb.size() * 8, cudaMemcpyDeviceToHost, stream));
    CK(cudaMemcpyAsync(em.data(), em_out.p, em.size() * 8, cudaMemcpyDeviceToHost, stream));
    CK(cudaMemcpyAsync(nonf.data(), d_nonfinite.p, nonf.size() * 4, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    check_error();
    float fms = 0, bms = 0;
    CK(cudaEventElapsedTime(&fms, ev0, ev1));
    CK(cudaEventElapsedTime(&bms, ev1, ev2));
    restore_host(host0);
    substep_index = s0;
    time = time0;

    const size_t ne = eff.size();
    const double dt = cfg.dt_substep;
    std::vector<V3<double>> et(ne, V3<double>{0, 0, 0});
    std::vector<M3<double>> eR(ne, mzero<double>());
    for (int s = 0; s < nrep * nseg; s++)
        for (int k2 = 0; k2 < 6; k2++) grad[6 * s + k2] = 0.0;
    for (long t = T - 1; t >= 0; t--) {
        const int seg = int(t / seglen);
        double echeck = 0;
        for (size_t e = 0; e < ne; e++) {
            const double* b = &eb[(size_t(t) * es + e) * 18];
            const double* m = &em[(size_t(t) * es + e) * 12];
            double* gs = grad + 6 * (size_t(nrep > 1 ? e / e1 : 0) * nseg + seg);  // replica-major
            for (int q = 0; q < 3; q++) et[e][q] += m[q];
            for (int q = 0; q < 9; q++) eR[e].m[q] += m[3 + q];
            V3<double> t_bar = et[e] + V3<double>{b[0], b[1], b[2]};
            M3<double> r_bar = eR[e];
            for (int q = 0; q < 9; q++) r_bar.m[q] += b[3 + q];
            V3<double> vlin_bar = V3<double>{b[12], b[13], b[14]} + t_bar * dt;
            V3<double> w_bar = {b[15], b[16], b[17]};
            M3<double> r_pre_bar = mzero<double>();
            advance_rotation_vjp(eff_pre[t][e].R, eff_post[t][e].w, dt, r_bar, r_pre_bar, w_bar);
            et[e] = t_bar;
            eR[e] = r_pre_bar;
            const int* mask = eff_shapes[e].action_mask;
            for (int q = 0; q < 3; q++)
                if (mask[q]) gs[q] += vlin_bar[q];
            for (int q = 0; q < 3; q++)
                if (mask[3 + q]) gs[3 + q] += w_bar[q];
            echeck += t_bar.x;
        }
        if (nonf[t] || !std::isfinite(echeck)) {
            FlumeError e(FLUME_E_ADJOINT, "non-finite adjoint at substep " + std::to_string(t));
            e.substep = t;
            throw e;
        }
    }
    for (int rp = 0; rp < nrep; rp++) {
        if (loss_out_h) loss_out_h[rp] = lsum[size_t(rp)];
        if (full_loss) full_loss[rp] = fsum[size_t(rp)];
    }
    if (per_seg)
        for (size_t s = 0; s < per.size(); s++) per_seg[s] = per[s];
    if (snapshots) *snapshots = long(n_snap);
    timing.forward_ms = fms;
    timing.backward_ms = bms;
    timing.substeps = T;
    timing.particle_substeps = T * long(N);
    timing.launches = launches - launches0;
}

void Ctx::adjoint_substep_api(const double* action, double* xb, double* vb, double* Fb, double* Cb, double* ebars,
                              double* abar_out) {
    require_single("adjoint_substep");
    if (slab()) throw FlumeError(FLUME_E_ARG, "adjoint_substep: single-rank contexts only");
    upload_full = true;  // the pre-state's liquids are expanded to a full F below (heavy blocks)
    xbar_tmp.alloc(size_t(N) * 3);
    Fbar_tmp.alloc(size_t(N) * 9);
    eff_out.alloc(kMaxEff * 18);
    em_out.alloc(kMaxEff * 12);
    d_nonfinite.alloc(1);
    CK(cudaMemsetAsync(em_out.p, 0, em_out.n * 8, stream));
    CK(cudaMemsetAsync(d_nonfinite.p, 0, sizeof(int), stream));
    const long s0 = substep_index;
    const double time0 = time;
    const int na0 = n_active, ns0 = n_stored, pb0 = park_base;
    const std::vector<EffState> eff0 = eff;
    const std::vector<uint32_t> inact0 = inactive_ids;
    const auto pend0 = pending;
    StatePtr pre = get_state(), post = get_state();
    copy_state(*pre, *cur);
    launch_expand_f(pre->p, pre->n, d_cls.p, stream);  // full F cotangents out, like the reference
    RecordPtr rec = get_record();
    forward_substep(action, pre, post, *rec);
    const std::vector<EffState> eff_stage = eff;
    check_error();
    for (int k = 0; k < 4; k++) d_up[k].alloc(size_t(N) * (k < 2 ? 3 : 9));
    CK(cudaMemcpyAsync(d_up[0].p, xb, size_t(N) * 24, cudaMemcpyHostToDevice, stream));
    CK(cudaMemcpyAsync(d_up[1].p, vb, size_t(N) * 24, cudaMemcpyHostToDevice, stream));
    CK(cudaMemcpyAsync(d_up[2].p, Fb, size_t(N) * 72, cudaMemcpyHostToDevice, stream));
    CK(cudaMemcpyAsync(d_up[3].p, Cb, size_t(N) * 72, cudaMemcpyHostToDevice, stream));
    
    barsA.alloc(size_t(N) * 24);
    barsB.alloc(size_t(N) * 24);
    launch_bars_from_ref(BarBuf{barsA.p, N}, post->p, N, d_up[0].p, d_up[1].p, d_up[2].p, d_up[3].p, d_cls.p,
                         stream);
    adjoint_step(*pre, *post, *rec, barsA, barsB, 0);
    eff_flush();
    launch_bars_to_ref(BarBuf{barsB.p, N}, pre->p, N, d_up[0].p, d_up[1].p, d_up[2].p, d_up[3].p, d_cls.p, stream);
    CK(cudaMemcpyAsync(xb, d_up[0].p, size_t(N) * 24, cudaMemcpyDeviceToHost, stream));
    CK(cudaMemcpyAsync(vb, d_up[1].p, size_t(N) * 24, cudaMemcpyDeviceToHost, stream));
    CK(cudaMemcpyAsync(Fb, d_up[2].p, size_t(N) * 72, cudaMemcpyDeviceToHost, stream));
    CK(cudaMemcpyAsync(Cb, d_up[3].p, size_t(N) * 72, cudaMemcpyDeviceToHost, stream));
    std::vector<double> ebh(kMaxEff * 18), emh(kMaxEff * 12);
    int nonf = 0;
    CK(cudaMemcpyAsync(ebh.data(), eff_out.p, ebh.size() * 8, cudaMemcpyDeviceToHost, stream));
    CK(cudaMemcpyAsync(emh.data(), em_out.p, emh.size() * 8, cudaMemcpyDeviceToHost, stream));
    CK(cudaMemcpyAsync(&nonf, d_nonfinite.p, 4, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    check_error();
    put_state(pre);
    put_state(post);
    put_record(rec);
    substep_index = s0;
    time = time0;
    n_active = na0;
    n_stored = ns0;
    park_base = pb0;
    inactive_ids = inact0;
    pending = pend0;
    const double dt = cfg.dt_substep;
    double echeck = 0;
    for (size_t e = 0; e < eff0.size(); e++) {
        const double* b = &ebh[e * 18];
        const double* m = &emh[e * 12];
        V3<double> t_bar = {ebars[12 * e] + m[0], ebars[12 * e + 1] + m[1], ebars[12 * e + 2] + m[2]};
        M3<double> r_bar;
        for (int q = 0; q < 9; q++) r_bar.m[q] = ebars[12 * e + 3 + q] + m[3 + q] + b[3 + q];
        t_bar = t_bar + V3<double>{b[0], b[1], b[2]};
        V3<double> vlin_bar = V3<double>{b[12], b[13], b[14]} + t_bar * dt;
        V3<double> w_bar = {b[15], b[16], b[17]};
        M3<double> r_pre_bar = mzero<double>();
        advance_rotation_vjp(eff0[e].R, eff_stage[e].w, dt, r_bar, r_pre_bar, w_bar);
        for (int q = 0; q < 3; q++) ebars[12 * e + q] = t_bar[q];
        for (int q = 0; q < 9; q++) ebars[12 * e + 3 + q] = r_pre_bar.m[q];
        const int* mask = eff_shapes[e].action_mask;
        for (int q = 0; q < 3; q++)
            if (mask[q]) abar_out[q] += vlin_bar[q];
        for (int q = 0; q < 3; q++)
            if (mask[3 + q]) abar_out[3 + q] += w_bar[q];
        echeck += t_bar.x;
    }
    eff = eff0;
    if (nonf || !std::isfinite(echeck)) {
        FlumeError e(FLUME_E_ADJOINT, "non-finite adjoint at substep " + std::to_string(s0));
        e.substep = s0;
        throw e;
    }
}

}  // namespace fl

// ===========================================================================
// C ABI
// ===========================================================================
using fl::Ctx;
using fl::FlumeError;

struct flume_ctx {
    Ctx c;
};

namespace {
thread_local flume_error_info g_create_err{};

template <class F>
int guard(flume_ctx* ctx, F&& f) {
    flume_error_info* info = ctx ? &ctx->c.last_err : &g_create_err;
    *info = flume_error_info{};
    info->particle_id = -1;
    info->body_id = -1;
    info->substep = -1;
    try {
        // calls may come from any host thread: make the context's device current
        if (ctx) CK(cudaSetDevice(ctx->c.device));
        f();
        return FLUME_OK;
    } catch (const FlumeError& e) {
        // engine errors are raised identically on every slab rank (error flags and
        // losses are all-reduced first); device failures may hit one rank only,
        // so they release the peers waiting in the group
        if (e.code == FLUME_E_CUDA && ctx && ctx->c.comm) ctx->c.comm->abort();
        info->code = e.code;
        info->particle_id = e.pid;
        info->body_id = e.body;
        info->substep = e.substep;
        std::snprintf(info->message, sizeof(info->message), "%s", e.what());
        return e.code;
    } catch (const std::exception& e) {
        if (ctx && ctx->c.comm) ctx->c.comm->abort();
        info->code = FLUME_E_OTHER;
        std::snprintf(info->message, sizeof(info->message), "%s", e.what());
        return FLUME_E_OTHER;
    }
}
}  // namespace

extern "C" {

int flume_abi_version(void) { return FLUME_B200_ABI_VERSION; }

int flume_ctx_create(const flume_scene_desc* desc, int device, flume_ctx** out) {
    if (!desc || !out) return FLUME_E_ARG;
    *out = nullptr;
    flume_ctx* ctx = new flume_ctx();
    int rc = guard(nullptr, [&] { ctx->c.init(desc, device); });
    if (rc != FLUME_OK) {
        ctx->c.last_err = g_create_err;
        delete ctx;
        return rc;
    }
    *out = ctx;
    return FLUME_OK;
}

// n copies of a scene description for a replica context: particle i of replica r is
// r * n1 + i, effector e is r * e1 + e, body b is r * body_stride + b
struct ReplicaDesc {
    flume_scene_desc d{};
    std::vector<flume_effector_shape> eff;
    std::vector<flume_rigid_body> rig;
    std::vector<std::vector<long>> members;
    std::vector<flume_emitter> emi;
    std::vector<int> mat, body;
    std::vector<double> mass, vol;
    std::vector<long> act;
    int body_stride = 1;
    ReplicaDesc(const flume_scene_desc* s, int R) {
        const long n1 = s->n_particles;
        const int e1 = s->n_effectors;
        for (long i = 0; i < n1; i++) body_stride = std::max(body_stride, s->body_id[i] + 1);
        for (int b = 0; b < s->n_rigid; b++) body_stride = std::max(body_stride, s->rigid[b].body_id + 1);
        d = *s;
        for (int r = 0; r < R; r++) {
            eff.insert(eff.end(), s->effectors, s->effectors + e1);
            for (long i = 0; i < n1; i++) {
                mat.push_back(s->material_id[i]);
                body.push_back(s->body_id[i] < 0 ? s->body_id[i] : s->body_id[i] + r * body_stride);
                mass.push_back(s->mass[i]);
                vol.push_back(s->volume0[i]);
                act.push_back(s->activation_substep ? s->activation_substep[i] : 0);
            }
            for (int b = 0; b < s->n_rigid; b++) {
                flume_rigid_body rb = s->rigid[b];
                std::vector<long> m(rb.members, rb.members + rb.n_members);
                for (long& p : m) p += r * n1;
                members.push_back(std::move(m));
                rb.body_id += r * body_stride;
                rig.push_back(rb);
            }
            for (long k = 0; k < s->n_emitters; k++) {
                flume_emitter em = s->emitters[k];
                em.particle += r * n1;
                if (em.effector >= 0) em.effector += r * e1;
                emi.push_back(em);
            }
        }
        for (size_t b = 0; b < rig.size(); b++) rig[b].members = members[b].data();
        d.n_effectors = R * e1;
        d.effectors = eff.data();
        d.n_rigid = int(rig.size());
        d.rigid = rig.data();
        d.n_emitters = long(emi.size());
        d.emitters = emi.data();
        d.n_particles = R * n1;
        d.material_id = mat.data();
        d.body_id = body.data();
        d.mass = mass.data();
        d.volume0 = vol.data();
        d.activation_substep = act.data();
    }
};

int flume_ctx_create_replicas(const flume_scene_desc* desc, int n_replicas, int device, flume_ctx** out) {
    if (!desc || !out || n_replicas < 1 || desc->n_particles <= 0) return FLUME_E_ARG;
    *out = nullptr;
    flume_ctx* ctx = new flume_ctx();
    int rc = guard(nullptr, [&] {
        if (long(n_replicas) * desc->n_particles >= (1L << 26))
            throw FlumeError(FLUME_E_ARG, "at most 2^26-1 particles per context");
        ReplicaDesc rd(desc, n_replicas);
        ctx->c.body_stride = rd.body_stride;
        ctx->c.init(&rd.d, device, n_replicas);
    });
    if (rc != FLUME_OK) {
        ctx->c.last_err = g_create_err;
        delete ctx;
        return rc;
    }
    *out = ctx;
    return FLUME_OK;
}

int flume_replicas_rollout_loss(flume_ctx* ctx, const flume_actions* actions, const flume_loss_desc* loss,
                                long window, int keep_final, double* loss_out, double* per_segment) {
    if (!ctx || !actions || !loss_out) return FLUME_E_ARG;
    return guard(ctx, [&] {
        ctx->c.require_particles();
        ctx->c.rollout_loss(actions, loss, window, per_segment, keep_final != 0, loss_out);
    });
}

int flume_replicas_info(const flume_ctx* ctx, int* n_replicas, long* particles_per_replica,
                        int* effectors_per_replica, int* body_stride) {
    if (!ctx) return FLUME_E_ARG;
    if (n_replicas) *n_replicas = ctx->c.nrep;
    if (particles_per_replica) *particles_per_replica = ctx->c.n1;
    if (effectors_per_replica) *effectors_per_replica = ctx->c.e1;
    if (body_stride) *body_stride = ctx->c.body_stride;
    return FLUME_OK;
}

int flume_group_create(const flume_scene_desc* desc, int n_ranks, const int* devices, flume_ctx** out) {
    if (!desc || !out || n_ranks < 1) return FLUME_E_ARG;
    for (int r = 0; r < n_ranks; r++) out[r] = nullptr;
    auto grp = std::make_shared<fl::ThreadGroup>(n_ranks);
    // direct NVLink peer copies between the ranks' devices where the topology allows
    for (int a = 0; a < n_ranks; a++)
        for (int b = 0; b < n_ranks; b++) {
            const int da = devices ? devices[a] : 0, db = devices ? devices[b] : 0;
            int can = 0;
            if (da == db || cudaDeviceCanAccessPeer(&can, da, db) != cudaSuccess || !can) continue;
            cudaSetDevice(da);
            const cudaError_t e = cudaDeviceEnablePeerAccess(db, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        }
    for (int r = 0; r < n_ranks; r++) {
        const int dev = devices ? devices[r] : 0;
        flume_ctx* ctx = new flume_ctx();
        int rc = guard(nullptr, [&] {
            ctx->c.init(desc, dev);
            if (n_ranks > 1) ctx->c.set_transport(fl::make_thread_transport(grp, r, dev));
        });
        if (rc != FLUME_OK) {
            delete ctx;
            for (int q = 0; q < r; q++) {
                delete out[q];
                out[q] = nullptr;
            }
            return rc;
        }
        out[r] = ctx;
    }
    return FLUME_OK;
}

int flume_dist_unique_id(unsigned char uid[128]) {
    if (!uid) return FLUME_E_ARG;
    return guard(nullptr, [&] { fl::nccl_unique_id(uid); });
}

int flume_ipc_unique_id(unsigned char uid[128]) {
    if (!uid) return FLUME_E_ARG;
    return guard(nullptr, [&] { fl::ipc_unique_id(uid); });
}

int flume_ctx_create_dist(const flume_scene_desc* desc, int device, int rank, int n_ranks,
                          const unsigned char uid[128], flume_ctx** out) {
    if (!desc || !out || !uid || rank < 0 || rank >= n_ranks) return FLUME_E_ARG;
    *out = nullptr;
    flume_ctx* ctx = new flume_ctx();
    int rc = guard(nullptr, [&] {
        ctx->c.init(desc, device);
        // (a one-rank NCCL group is allowed: it runs the slab code path with a single slab)
        ctx->c.set_transport(fl::is_ipc_unique_id(uid) ? fl::make_ipc_transport(uid, rank, n_ranks, device)
                                                        : fl::make_nccl_transport(uid, rank, n_ranks, device));
    });
    if (rc != FLUME_OK) {
        delete ctx;
        return rc;
    }
    *out = ctx;
    return FLUME_OK;
}

int flume_slab_split(const double* col_weight, int n_cols, int n_ranks, int* cuts) {
    if (!col_weight || !cuts || n_ranks < 1 || n_cols < n_ranks) return FLUME_E_ARG;
    fl::slab_split(col_weight, n_cols, n_ranks, cuts);
    return FLUME_OK;
}

int flume_slab_set_migration_capacity(flume_ctx* ctx, int capacity) {
    if (!ctx || capacity < 1) return FLUME_E_ARG;
    return guard(ctx, [&] {
        if (!ctx->c.slab()) throw FlumeError(FLUME_E_ARG, "not a slab context");
        ctx->c.set_mig_cap(capacity);
    });
}

int flume_slab_migration_stats(const flume_ctx* ctx, int* capacity, long* retries) {
    if (!ctx) return FLUME_E_ARG;
    if (capacity) *capacity = ctx->c.mig_cap;
    if (retries) *retries = ctx->c.mig_retries;
    return FLUME_OK;
}

int flume_slab_info(const flume_ctx* ctx, int* rank, int* n_ranks, int* sx0, int* sx1, long* n_active) {
    if (!ctx) return FLUME_E_ARG;
    const fl::Ctx& c = ctx->c;
    if (rank) *rank = c.rank;
    if (n_ranks) *n_ranks = c.nranks;
    if (sx0) *sx0 = c.geom.sx0;
    if (sx1) *sx1 = c.geom.sx1;
    if (n_active) *n_active = c.n_active;
    return FLUME_OK;
}

int flume_ctx_destroy(flume_ctx* ctx) {
    if (!ctx) return FLUME_OK;
    cudaSetDevice(ctx->c.device);  // the device buffers are freed on their own device
    cudaStreamSynchronize(ctx->c.stream);
    cudaStream_t s = ctx->c.stream, s2 = ctx->c.s2;
    cudaEvent_t e1 = ctx->c.ev_fork, e2 = ctx->c.ev_join, e3 = ctx->c.ev_snap;
    cudaStream_t s3 = ctx->c.cstream;
    cudaStreamSynchronize(s2);
    if (s3) cudaStreamSynchronize(s3);
    if (ctx->c.h_effring) cudaFreeHost(ctx->c.h_effring);
    for (cudaEvent_t e : ctx->c.effring_ev)
        if (e) cudaEventDestroy(e);
    delete ctx;
    if (s) cudaStreamDestroy(s);
    if (s2) cudaStreamDestroy(s2);
    if (s3) cudaStreamDestroy(s3);
    if (e3) cudaEventDestroy(e3);
    if (e1) cudaEventDestroy(e1);
    if (e2) cudaEventDestroy(e2);
    return FLUME_OK;
}

int flume_set_mode(flume_ctx* ctx, int deterministic, int hard_contact) {
    return guard(ctx, [&] {
        if (!deterministic)
            throw FlumeError(FLUME_E_ARG, "only the deterministic mode exists (it is also the fast one)");
        ctx->c.cfg.hard_contact = hard_contact;
        ctx->c.geom.hard = hard_contact;
    });
}

int flume_set_checkpoint_spill(flume_ctx* ctx, int mode) {
    if (!ctx || mode < 0 || mode > 1) return FLUME_E_ARG;
    return guard(ctx, [&] { ctx->c.spill = mode; });
}

int flume_set_checkpoint_spill_dir(flume_ctx* ctx, const char* dir) {
    if (!ctx || !dir || !*dir) return FLUME_E_ARG;
    return guard(ctx, [&] {
        ctx->c.spill_dir = dir;
        ctx->c.fspill.reset();
        ctx->c.spill = 2;
    });
}

int flume_set_chamfer_mode(flume_ctx* ctx, int mode) {
    if (!ctx || mode < 0 || mode > 2) return FLUME_E_ARG;
    return guard(ctx, [&] { ctx->c.chamfer_mode = mode; });
}

int flume_set_incremental_sort(flume_ctx* ctx, int on) {
    if (!ctx || on < 0 || on > 1) return FLUME_E_ARG;
    return guard(ctx, [&] {
        ctx->c.inc_sort = on != 0;
        ctx->c.chain_break();
        ctx->c.counters_clean = false;  // the counts' clearing rule changes with the mode
    });
}

int flume_sort_stats(const flume_ctx* ctx, long* incremental, long* full) {
    if (!ctx) return FLUME_E_ARG;
    if (incremental) *incremental = ctx->c.n_inc_sorts;
    if (full) *full = ctx->c.n_full_sorts;
    return FLUME_OK;
}

int flume_last_error(const flume_ctx* ctx, flume_error_info* info) {
    if (!info) return FLUME_E_ARG;
    *info = ctx ? ctx->c.last_err : g_create_err;
    return FLUME_OK;
}

int flume_get_stream(flume_ctx* ctx, void** s) {
    if (!ctx || !s) return FLUME_E_ARG;
    *s = ctx->c.stream;
    return FLUME_OK;
}

int flume_sync(flume_ctx* ctx) {
    return guard(ctx, [&] { CK(cudaStreamSynchronize(ctx->c.stream)); });
}

int flume_last_timing(const flume_ctx* ctx, flume_timing* out) {
    if (!ctx || !out) return FLUME_E_ARG;
    *out = ctx->c.timing;
    return FLUME_OK;
}

int flume_state_upload(flume_ctx* ctx, const flume_state_view* view) {
    if (!ctx || !view) return FLUME_E_ARG;
    return guard(ctx, [&] { ctx->c.upload(view); });
}

int flume_state_download(flume_ctx* ctx, flume_state_view* view) {
    if (!ctx || !view) return FLUME_E_ARG;
    return guard(ctx, [&] { ctx->c.download(view); });
}

int flume_store_order(flume_ctx* ctx, unsigned* keys, unsigned* ids, long* n_active) {
    if (!ctx) return FLUME_E_ARG;
    return guard(ctx, [&] {
        Ctx& c = ctx->c;
        if (c.empty) {
            if (n_active) *n_active = 0;
            return;
        }
        if (keys) CK(cudaMemcpyAsync(keys, c.cur->p.key, size_t(c.N) * 4, cudaMemcpyDeviceToHost, c.stream));
        if (ids) CK(cudaMemcpyAsync(ids, c.cur->p.id, size_t(c.N) * 4, cudaMemcpyDeviceToHost, c.stream));
        CK(cudaStreamSynchronize(c.stream));
        if (n_active) *n_active = c.n_active;
    });
}

int flume_store_sorted(flume_ctx* ctx, unsigned* keys, unsigned* ids, float* x, long* n_active) {
    if (!ctx) return FLUME_E_ARG;
    using namespace fl;
    return guard(ctx, [&] {
        Ctx& c = ctx->c;
        if (c.empty) {
            if (n_active) *n_active = 0;
            return;
        }
        if (c.slab()) throw FlumeError(FLUME_E_ARG, "flume_store_sorted: one-rank contexts only");
        // the sort the next substep would start with (incremental when the chain holds), then
        // the store gathered through its permutation; the chain is consumed
        Record& r = c.next_scratch();
        r.n_active = c.n_active;
        r.n_keep = c.n_active + c.n_parked();
        r.n_stored = c.n_stored;
        const Record* prev = (c.keep_counts() && c.chain_rec && c.chain_rec != &r && c.chain_out == c.cur.get())
                                 ? c.chain_rec
                                 : nullptr;
        c.sort_and_lists(*c.cur, r, prev);
        StatePtr t = c.get_state();
        launch_gather(c.cur->p, t->p, r.perm, r.n_keep, c.stream);
        if (keys) CK(cudaMemcpyAsync(keys, t->p.key, size_t(r.n_keep) * 4, cudaMemcpyDeviceToHost, c.stream));
        if (ids) CK(cudaMemcpyAsync(ids, t->p.id, size_t(r.n_keep) * 4, cudaMemcpyDeviceToHost, c.stream));
        for (int a = 0; a < 3 && x; a++)
            CK(cudaMemcpyAsync(x + size_t(a) * c.N, t->p.x(a), size_t(r.n_keep) * 4, cudaMemcpyDeviceToHost,
                               c.stream));
        CK(cudaStreamSynchronize(c.stream));
        c.put_state(t);
        c.chain_break();
        if (n_active) *n_active = c.n_active;
    });
}

int flume_store_positions(flume_ctx* ctx, float* x) {
    if (!ctx || !x) return FLUME_E_ARG;
    return guard(ctx, [&] {
        Ctx& c = ctx->c;
        if (c.empty) return;
        CK(cudaMemcpyAsync(x, c.cur->p.f, size_t(c.N) * 3 * 4, cudaMemcpyDeviceToHost, c.stream));
        CK(cudaStreamSynchronize(c.stream));
    });
}

int flume_profile(flume_ctx* ctx, int enable) {
    if (!ctx) return FLUME_E_ARG;
    return guard(ctx, [&] {
        ctx->c.prof.collect(ctx->c.stream);
        ctx->c.prof.on = enable != 0;
        ctx->c.prof.reset();
    });
}

int flume_kernel_times(flume_ctx* ctx, double* ms, long* counts, int n) {
    if (!ctx) return FLUME_E_ARG;
    return guard(ctx, [&] {
        ctx->c.prof.collect(ctx->c.stream);
        for (int k = 0; k < n && k < fl::K_COUNT; k++) {
            if (ms) ms[k] = ctx->c.prof.ms[k];
            if (counts) counts[k] = ctx->c.prof.count[k];
        }
    });
}

int flume_timer_mark(flume_ctx* ctx, int slot) {
    if (!ctx || slot < 0 || slot >= 8) return FLUME_E_ARG;
    return guard(ctx, [&] {
        if (!ctx->c.marks[slot]) CK(cudaEventCreate(&ctx->c.marks[slot]));
        CK(cudaEventRecord(ctx->c.marks[slot], ctx->c.stream));
    });
}

int flume_timer_elapsed(flume_ctx* ctx, int a, int b, double* ms) {
    if (!ctx || !ms || a < 0 || b < 0 || a >= 8 || b >= 8) return FLUME_E_ARG;
    return guard(ctx, [&] {
        CK(cudaEventSynchronize(ctx->c.marks[b]));
        float t = 0;
        CK(cudaEventElapsedTime(&t, ctx->c.marks[a], ctx->c.marks[b]));
        *ms = t;
    });
}

int flume_substep(flume_ctx* ctx, const double action[6], int count) {
    if (!ctx || !action) return FLUME_E_ARG;
    return guard(ctx, [&] { ctx->c.slab_retry(true, [&] { ctx->c.substep(action, count); }); });
}

int flume_stage_grid(flume_ctx* ctx, double* mass, double* vel) {
    if (!ctx) return FLUME_E_ARG;
    return guard(ctx, [&] { ctx->c.stage_grid(mass, vel); });
}

int flume_rollout_loss(flume_ctx* ctx, const flume_actions* actions, const flume_loss_desc* loss, long window,
                       double* loss_out, double* per_segment) {
    if (!ctx || !actions || !loss_out) return FLUME_E_ARG;
    return guard(ctx, [&] {
        ctx->c.require_particles();
        ctx->c.require_single("flume_rollout_loss (flume_replicas_rollout_loss)");
        ctx->c.slab_retry(false, [&] { *loss_out = ctx->c.rollout_loss(actions, loss, window, per_segment); });
    });
}

int flume_rollout_loss_final(flume_ctx* ctx, const flume_actions* actions, const flume_loss_desc* loss, long window,
                             double* loss_out, double* per_segment) {
    if (!ctx || !actions || !loss_out) return FLUME_E_ARG;
    return guard(ctx, [&] {
        ctx->c.require_particles();
        ctx->c.require_single("flume_rollout_loss (flume_replicas_rollout_loss)");
        ctx->c.slab_retry(true, [&] { *loss_out = ctx->c.rollout_loss(actions, loss, window, per_segment, true); });
    });
}

int flume_loss_per_particle(flume_ctx* ctx, const flume_loss_desc* loss, double* out) {
    if (!ctx || !loss || !out) return FLUME_E_ARG;
    return guard(ctx, [&] {
        ctx->c.require_particles();
        ctx->c.per_particle(loss, out);
    });
}

int flume_grad_trajectory(flume_ctx* ctx, const flume_actions* actions, const flume_loss_desc* loss, long stride,
                          long window, double* action_grad, double* loss_out, double* full_loss,
                          double* per_segment, long* snapshots) {
    if (!ctx || !actions || !action_grad) return FLUME_E_ARG;
    return guard(ctx, [&] {
        ctx->c.require_particles();
        ctx->c.require_single("flume_grad_trajectory (flume_replicas_grad_trajectory)");
        ctx->c.slab_retry(false, [&] {
            ctx->c.grad_trajectory(actions, loss, stride, window, action_grad, loss_out, full_loss, per_segment,
                                   snapshots);
        });
    });
}

int flume_replicas_grad_trajectory(flume_ctx* ctx, const flume_actions* actions, const flume_loss_desc* loss,
                                   long stride, long window, double* action_grad, double* loss_out,
                                   double* full_loss, double* per_segment, long* snapshots) {
    if (!ctx || !actions || !action_grad) return FLUME_E_ARG;
    return guard(ctx, [&] {
        ctx->c.require_particles();
        ctx->c.grad_trajectory(actions, loss, stride, window, action_grad, loss_out, full_loss, per_segment,
                               snapshots);
    });
}

int flume_adjoint_substep(flume_ctx* ctx, const double action[6], double* x_bar, double* v_bar, double* F_bar,
                          double* C_bar, double* eff_bars, double* action_bar) {
    if (!ctx || !action || !x_bar || !v_bar || !F_bar || !C_bar || !action_bar) return FLUME_E_ARG;
    return guard(ctx, [&] {
        ctx->c.require_particles();
        std::vector<double> dummy(size_t(fl::kMaxEff) * 12, 0.0);
        ctx->c.adjoint_substep_api(action, x_bar, v_bar, F_bar, C_bar, eff_bars ? eff_bars : dummy.data(),
                                   action_bar);
    });
}

}  // extern "C"
