// fl_kernels.h -- launch wrappers for the sm_100a kernels (host side view).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>
#include <string>
#include <utility>

#include "fl_layout.cuh"

namespace fl {

// role of the next dual-variant launch of this host thread (DualScope, fl_layout.cuh)
inline int& dual_role() {
    static thread_local int role = 0;
    return role;
}

// hot-path launch with programmatic stream serialization (see pdl_wait)
template <typename... KArgs, typename... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = FL_PDL;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
    if (e != cudaSuccess) throw std::runtime_error(std::string("kernel launch failed: ") + cudaGetErrorString(e));
}

// <<<>>> launches report through cudaGetLastError; called after each launch group
inline void check_launch() {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw std::runtime_error(std::string("kernel launch failed: ") + cudaGetErrorString(e));
}

// A particle count a kernel needs.  On one rank the host knows every count exactly (h);
// on x-slabs the migration changes them on the device, so the kernels read d (the state's
// or the record's device counts) and h is only an upper bound that sizes the grid.
struct DN {
    int h;
    const int* d;
    __host__ __device__ int get() const {
#if defined(__CUDA_ARCH__)
        return d ? *d : h;
#else
        return h;
#endif
    }
};
inline DN dn(int h, const int* d = nullptr) { return DN{h, d}; }
// device counts of a state buffer (slab contexts) and of a substep record
enum StateCnt : int { SC_ACTIVE = 0, SC_STORED = 1, SC_PARK = 2, SC_N = 4 };
enum RecCnt : int {
    RC_ACTIVE = 0,   // active particles of the pre-state after this substep's activations
    RC_KEEP = 1,     // active + parked
    RC_STORED = 2,   // all slots of the pre-state (departed holes included)
    RC_PARK = 3,     // first parked slot of the pre-state (activation slots are relative to it)
    RC_SENT = 4,     // [4], [5]: particles sent down / up after G2P
    RC_RECV = 6,     // [6], [7]: particles received from below / above
    RC_ARR = 8,      // first arrival slot of the post-state
    RC_N = 12
};
// grid for a grid-stride loop over up to n items (256 threads, at most `cap` CTAs)
inline int gs_grid(int n, int cap = 148 * 16) { return std::max(1, std::min(cap, (n + 255) / 256)); }

// node-column filter of the grid update and its adjoint (slab halo overlap): cmode 0 every
// listed node block, 1 all but node columns c0/c1 (the interior, updated while the halo
// planes travel), 2 only those columns
struct GridCols {
    int cmode, c0, c1;
};

// rigid-body bookkeeping for one substep (forward record / backward input)
struct RigidDev {
    int nbody;
    int nmem;                 // total members over all bodies
    const int* off;           // [nbody+1] member offsets
    const int* mrank;         // [N] member rank (global, off[body]+j) by particle id, -1 otherwise
    const double* rest;       // [3*nmem] rest offsets (x0 - c0)
    const double* mass;       // [nmem] member masses
    const double* smrest;     // [3*nbody] sum_j m_j rest_j
    const double* total;      // [nbody] total mass
    const int* body_id;       // [nbody] reference body id
    const int* member_body;   // [nmem] body index of each member
    const int* member_id;     // [nmem] particle id of each member
    // per-substep arrays
    int* mslot;               // [nmem] sorted position of the member in the post-g2p buffer (-1 inactive)
    double* mstart;           // [3*nmem] stage-a position (rigid_body_pass start_positions)
    double* mid;              // [3*nmem] post-g2p position
    double* mact;             // [nmem] 1 where mid holds an active member (all-reduced with mid on slabs)
    double* fit;              // [nbody*24]: R[9] c[3] A[9] total skip ok
};

struct ActEntry {
    int slot;
    int has_xv;
    int departed;  // activates inside another rank's slab
    int rep;       // replica (replica contexts)
    float x[3];
    float v[3];
};
// short activation / spawn lists travel as kernel parameters: no host->device copy, so
// no pageable-copy stream sync on the substep (an emitter adds one particle per substep)
constexpr int kActInline = 64;
struct ActBatch {
    int n;
    ActEntry e[kActInline];
};

struct EmitAdjEntry {
    int slot;
    int eff;
    int mask[3];  // 1 when the spawn clamp was active on that axis
    double local_pos[3];
    double local_vel[3];
};

constexpr int kMaxLossTerms = 8;
enum LossKindId : int { LK_TARGET = 0, LK_HOLD = 1, LK_SPREAD = 2, LK_CHAMFER = 3 };
struct LossTermDev {
    int kind;
    int body;
    int squared;
    double weight;
    double goal[3];
    const float* init;    // hold_initial: [3*N] initial positions by particle id
    const double* gpts;   // trajectory_chamfer: all goal points (device)
    const long* goff_h;   // trajectory_chamfer: set offsets (HOST pointer, n_steps + 1)
    int nsteps;
    int last_g0, last_ng; // trajectory_chamfer: the last goal set (per_particle uses it)
};
// attraction term (losses.hpp:104-218, 348-363, 553-564): the gradient-sharing
// surrogate over every member of one body (active or parked), neighbours within
// `radius` found through a hashed grid with cell = radius
struct AttractionDev {
    int on = 0;
    int n_members = 0;
    double weight = 0, radius = 0, tau = 1;
    const double* prev = nullptr;  // previous iterate's per-particle losses, member (id) order
    const int* mrank = nullptr;    // member rank by particle id (-1: not a member)
    int nc[3] = {0, 0, 0};         // hash cells per axis (one pad cell on each side)
    int key_bits = 0;              // cell-index bits of the sort key
};
struct LossSet {
    int n;
    LossTermDev t[kMaxLossTerms];
    AttractionDev attr;
    // a parked (not yet emitted) particle counts as active once the state's substep
    // index reaches its activation substep (types.hpp:109), before its emission
    const int* act;   // activation substep by particle id
    long substep;     // substep index of the evaluated state
    // emission rewrites a particle's slot in place at the start of its activation substep;
    // at that substep a loss uses its parked position (SoA [3][n_all] by id), as the
    // reference's state still holds it when the loss is evaluated
    const float* x0;
    int n_all;
    int count_parked;  // slabs: parked particles are replicated, only rank 0 counts them
};
__host__ __device__ inline float loss_x(const LossSet& ls, const PBuf& st, int i, uint32_t id, int a) {
    return ls.act[id] == ls.substep ? ls.x0[size_t(a) * ls.n_all + id] : st.x(a)[i];
}

constexpr int kLossBlocks = 296;

// point-set losses (fl_loss.cu): scratch for the body compaction and the NN passes
constexpr int kChamferChunks = 512;
// trajectory_chamfer: member x goal pairs above which the nearest-neighbour passes use the
// grid index instead of the brute-force scan (flume_set_chamfer_mode overrides)
constexpr double kChamferBrutePairs = double(1 << 24);
struct PointLossScratch {
    int *flags = nullptr, *pos = nullptr, *idx = nullptr, *arg = nullptr, *carg = nullptr, *garg = nullptr,
        *count = nullptr;
    double *px = nullptr, *best = nullptr, *partial = nullptr, *cbest = nullptr, *gbest = nullptr,
           *scal = nullptr;
    void* cub_tmp = nullptr;
    size_t cub_bytes = 0, cap_g = 0;
    int cap_n = 0;
    // attraction: member positions / exp(-prev / tau) / slots, hash keys, per-member sums
    double *apx = nullptr, *ae = nullptr, *awsum = nullptr, *asi = nullptr, *apart = nullptr;
    int* aslot = nullptr;
    unsigned long long *akey = nullptr, *akey_sorted = nullptr;
    void* asort_tmp = nullptr;
    size_t asort_bytes = 0;
    int cap_a = 0;
    // trajectory_chamfer at scale: uniform-grid nearest-neighbour index (fl_loss.cu nn_build)
    unsigned long long *nn_keys = nullptr, *nn_keys_sorted = nullptr;
    double *nn_spts = nullptr, *nn_gpart = nullptr, *nn_part = nullptr, *nn_idx = nullptr;
    int *nn_sidx = nullptr, *nn_cstart = nullptr, *nn_cend = nullptr;
    void* nn_sort_tmp = nullptr;
    size_t nn_sort_bytes = 0;
    int nn_cap = 0;
    void reserve_nn(int n);
    void reserve(int n_particles, int max_goals);
    void reserve_attraction(int n_members);
    ~PointLossScratch();
};
// attraction term of `ls` (ls.attr.on): eval adds weight * value into *out, grad adds into bars
void launch_attraction(PointLossScratch& w, const PBuf& st, int n, const LossSet& ls, uint32_t key_departed,
                       double* out, BarBuf* bars, cudaStream_t s);
// LossEvaluator::per_particle (losses.hpp:367-390) of the stored state, by particle id
void launch_per_particle(const PBuf& st, int n, const ClassInfo* cls, const LossSet& ls, uint32_t key_departed,
                         double* out, cudaStream_t s);
// eval (bars == nullptr): adds weight * value into *out; grad: adds d/dx into bars
void launch_point_loss(PointLossScratch& w, const PBuf& st, int n, const ClassInfo* cls, const LossSet& ls,
                       const LossTermDev& t, int seg, uint32_t key_inactive, double* out, BarBuf* bars,
                       unsigned long long* err, int mode, cudaStream_t s);
#ifndef FL_EFF_BLOCKS
#define FL_EFF_BLOCKS 3552
#endif
constexpr int kEffBlocks = FL_EFF_BLOCKS;  // largest grid of the grid adjoint = its effector-bar partials
constexpr int kRigidChunk = 2048;

// ---- forward ----
void launch_upload(const Geom& g, PBuf raw, int n, const double* x, const double* v, const double* F,
                   const double* C, const uint32_t* meta, const uint8_t* active, const ClassInfo* cls,
                   int* any_full, cudaStream_t s);
void launch_gather(PBuf in, PBuf out, const uint32_t* perm, int n, cudaStream_t s);
void launch_activate(const Geom& g, PBuf st, const ActEntry* list, int n, const int* slot_base, cudaStream_t s);
void launch_activate_inline(const Geom& g, PBuf st, const ActEntry* host_list, int n, const int* slot_base,
                            cudaStream_t s);
void launch_p2g(const Geom& g, PBuf st, const uint32_t* perm, const BlockRec* recs, const int* n_blocks,
                const uint16_t* celltab, int grid, const ClassInfo* cls, float4* staging, unsigned long long* err,
                uint32_t substep, int variant, int* wq, cudaStream_t s);
// cmode (slab halo overlap): 0 every listed node block, 1 all but node columns c0/c1, 2 only those
void launch_grid_update(const Geom& g, const int* nb_list, const int* n_nb, int grid, const int* blockmap,
                        const float4* staging, float4* gridv, float4* gridv0, const EffSet& eff, uint8_t* cmask,
                        int* clear, int n_clear, cudaStream_t s, int cmode = 0, int c0 = -1, int c1 = -1);
void launch_g2p(const Geom& g, PBuf in, PBuf out, const uint32_t* perm, const BlockRec* recs,
                const int* n_blocks, int grid, const ClassInfo* cls, const float4* gridv, RigidDev rd,
                unsigned long long* err, uint32_t substep, int variant, int* wq, cudaStream_t s);
void launch_tail_copy(const Geom& g, PBuf in, PBuf out, const uint32_t* perm, DN n_active, DN n, int n_parked,
                      cudaStream_t s);
void launch_rigid(const Geom& g, PBuf out, RigidDev rd, int nchunks, const int* chunk_body,
                  const int* chunk_m0, const int* chunk_m1, double* partial, unsigned long long* err,
                  uint32_t substep, cudaStream_t s);
void launch_download(PBuf st, int n, double* x, double* v, double* F, double* C, int write_parked,
                     uint32_t key_inactive, const ClassInfo* cls, cudaStream_t s);
void launch_download_rigid(PBuf st, int nmem, const int* member_id, double* x, cudaStream_t s);
void launch_upload_rigid(PBuf st, int nmem, const int* member_id, const double* x, cudaStream_t s);
void launch_loss(const PBuf& st, DN n, const ClassInfo* cls, const LossSet& ls, uint32_t mask,
                 double* partial, double* out, uint32_t key_inactive, cudaStream_t s);

// ---- backward ----
void launch_loss_grad(const PBuf& st, DN n, const ClassInfo* cls, const LossSet& ls, uint32_t mask,
                      BarBuf bars, uint32_t key_inactive, cudaStream_t s);
void launch_adj_rigid_gather(BarBuf post, RigidDev rd, double* mbar, cudaStream_t s);
void launch_adj_rigid(const Geom& g, BarBuf post, RigidDev rd, int nchunks, const int* chunk_body,
                      const int* chunk_m0, const int* chunk_m1, const double* mbar, double* partial,
                      float* start_bar, double* abar, cudaStream_t s);
void launch_adj_g2p(const Geom& g, PBuf pre, const uint32_t* perm, const BlockRec* recs, const int* n_blocks,
                    const uint16_t* celltab, int grid, const ClassInfo* cls, const float4* gridv, PBuf postst,
                    BarBuf post, float* xbar_tmp, float* Fbar_tmp, RigidDev rd, const float* start_bar,
                    float4* staging_bar, int variant, int* wq, cudaStream_t s);
void launch_adj_grid(const Geom& g, const int* nb_list, const int* n_nb, const int* blockmap,
                     const float4* staging_bar, const float4* gridv0, float4* gridbar, const EffSet& eff,
                     double* eff_partial, const uint8_t* cmask, int nblocks, int pstride, cudaStream_t s,
                     int cmode = 0, int c0 = -1, int c1 = -1);
constexpr int kEffRing = 16;  // substeps whose effector-bar partials wait for one final-sum launch
void launch_eff_final(const double* ring, int nblocks, int n_eff, long t0, int count, double* eff_out, int pstride,
                      cudaStream_t s);
void launch_adj_p2g(const Geom& g, PBuf pre, const uint32_t* perm, const BlockRec* recs, const int* n_blocks,
                    int grid, const ClassInfo* cls, const float4* gridbar, const float* xbar_tmp,
                    const float* Fbar_tmp, BarBuf out, int* nonfinite, int variant, int* wq, cudaStream_t s);
void launch_tail_bars(BarBuf post, BarBuf out, const uint32_t* perm, DN n_active, DN n_keep, DN n_stored,
                      cudaStream_t s);
void launch_adj_emit(BarBuf out, const EmitAdjEntry* list, int n, double* em_out, int n_eff, const int* slot_base,
                     cudaStream_t s);
constexpr int kEmitInline = 32;
void launch_adj_emit_inline(BarBuf out, const EmitAdjEntry* host_list, int n, double* em_out, int n_eff, const int* slot_base,
                            cudaStream_t s);
void launch_bars_from_ref(BarBuf bars, const PBuf& st, int n, const double* xb, const double* vb,
                          const double* Fb, const double* Cb, const ClassInfo* cls, cudaStream_t s);
void launch_bars_to_ref(BarBuf bars, const PBuf& st, int n, double* xb, double* vb, double* Fb, double* Cb,
                        const ClassInfo* cls, cudaStream_t s);
void launch_expand_f(PBuf st, int n, const ClassInfo* cls, cudaStream_t s);

#ifndef FL_INBOX
#define FL_INBOX 16
#endif
constexpr int kInbox = FL_INBOX;  // arrivals per block kept in its inbox (more go to the overflow list)
// incremental sort (fl_sort.cu header): the previous substep's sort tables + context scratch
struct IncSort {
    const BlockRec* orecs;     // previous record: block list
    const int* oblockmap;      // previous record: block map
    const uint16_t* octab;     // previous record: cell tables
    const uint32_t* okey_in;   // [n] the previous sort's key at every sorted position (bit 31: SVD/rigid)
    uint32_t* okey_out;        // [n] this sort's
    int* dirty;                // [nbtot + 2] blocks a particle entered, left or moved inside (zero between sorts)
    int* acnt;                 // [nbtot + 2] arrivals per block (zero between sorts)
    uint32_t* inbox;           // [nbtot + 2][kInbox] the first kInbox arrivals' slots per block
    int* nmov;                 // arrivals beyond a block's inbox (zero between sorts) ...
    int* novf;                 // ... their count for the per-block sort (the list pass moves it here)
    uint32_t* mov;             // [n] their slots
    int4* rold;                // [maxb] per list slot: {clean, previous list slot or -1, its start, its end}
};

void launch_sort_count(const Geom& g, const PBuf& st, DN n, const ClassInfo* cls, int* bcount, int* bheavy,
                       cudaStream_t s);
// cls_bit != nullptr: slot words carry the class bit (for the okey output of launch_sort_blocks)
void launch_sort_scatter(const Geom& g, const PBuf& st, DN n, const int* bstart, int* bfill, uint32_t* skey,
                         uint32_t* sslot, const ClassInfo* cls_bit, cudaStream_t s);
int sort_list_tiles(const Geom& g);
void launch_sort_lists(const Geom& g, int cap, const int* bcount, const int* bheavy, int* bstart, int* nbflag,
                       int* nb_list, int* n_nb, BlockRec* recs, int* blockmap, int* n_blocks, int4* tile_sum,
                       const IncSort* inc, cudaStream_t s);
// (launch_isort_place: the per-block sort; the arrivals sit in the blocks' inboxes)
// meta: the class bit can change (a liquid uploaded with a full F, kMetaFull, loses it in
// G2P): compare it too; otherwise the key alone (the class bit is the particle's own)
void launch_isort_diff(const Geom& g, const PBuf& st, int n, const ClassInfo* cls, int* bcount, int* bheavy,
                       const IncSort& is, bool meta, cudaStream_t s);
void launch_isort_place(const Geom& g, const PBuf& st, const ClassInfo* cls, const int* bcount, const int* bstart,
                        const BlockRec* recs, int* n_blocks, int cap, const IncSort& is, uint32_t* sslot,
                        uint32_t* perm, uint16_t* celltab, uint32_t* gk, uint32_t* gv, int grid, int arrive_grid,
                        cudaStream_t s);
// id-ordered list of the nonzero flags (two-pass tile scan); tile_sum: flag_list_tiles(n) ints
void launch_flag_list(const int* flags, int n, int* list, int* n_list, int* tile_sum, cudaStream_t s);
int flag_list_tiles(int n);
void launch_sort_blocks(const Geom& g, const int* bcount, const int* bstart, const BlockRec* recs,
                        int* n_blocks, int cap, const uint32_t* skey, const uint32_t* sslot, uint32_t* perm,
                        uint16_t* celltab, uint32_t* gk, uint32_t* gv, uint32_t* okey, int grid, cudaStream_t s);

// ---- x-slab decomposition (fl_slab.cu) ----
size_t halo_bytes(const Geom& g);
void launch_halo_pack(const Geom& g, const int* blockmap, const float4* staging, int col, int plane0, void* out,
                      cudaStream_t s);
void launch_halo_unpack(const Geom& g, const void* in, int col, int plane0, int ghost_base, int* blockmap,
                        float4* staging, int* nbflag, int flag_col, cudaStream_t s);
// fixed-size migration messages: a 16-int header (the count) + cap slots of kMigW words
size_t mig_msg_bytes(int cap);
void launch_mig_pack(const Geom& g, PBuf out, DN n, void* send0, void* send1, uint32_t* src, int cap, int* bcnt,
                     int* overflow, cudaStream_t s);
constexpr int kMigCountInts = 2 * 296;  // per-CTA counts of the stable migration compaction
// counts after the exchange: record [sent, recv, arrival base], post-state counts, overflow
void launch_mig_counts(const void* send0, const void* send1, const void* recv0, const void* recv1, int* rec,
                       int* post_cnt, int cap, int n_cap, int* overflow, cudaStream_t s);
void launch_mig_unpack(PBuf out, const void* in, const int* rec, int dir, int cap, cudaStream_t s);
// before a substep: the record's pre-state counts from the state's device counts
void launch_slab_counts_pre(const int* state_cnt, int* rec, int gained, int n_parked, void* send0, void* send1,
                            cudaStream_t s);
void launch_bars_pack(BarBuf bars, const int* rec, int dir, int cap, void* out, cudaStream_t s);
void launch_bars_scatter(BarBuf bars, const void* in, const uint32_t* src, const int* rec, int dir, int cap,
                         cudaStream_t s);

enum KGrid { KG_P2G = 0, KG_G2P = 1, KG_ADJ_G2P = 2, KG_ADJ_P2G = 3 };
// resident CTAs per SM x SMs; variant 0 plain liquid, 1 heavy beside light, 2 heavy-dominated scene
int occupancy_grid(KGrid which, int variant);

}  // namespace fl
