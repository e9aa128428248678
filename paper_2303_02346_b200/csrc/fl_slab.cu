// fl_slab.cu -- data movement of the x-slab decomposition.
//
// Rank r owns the particle blocks of columns [sx0, sx1).  A particle block at
// column bx scatters into node planes [4bx, 4bx + 6), so
//   * the top column's tiles spill two planes (tile x-planes 4,5) into the
//     first node column of rank r+1, and
//   * rank r's G2P of its top column reads the first two node planes of column
//     sx1, which rank r+1 owns.
// One symmetric halo exchange per scatter covers both: rank r sends tile planes
// 4,5 of its top column up and tile planes 0,1 of its bottom column down.  The
// receiver installs them as "ghost" particle blocks (staging slots past maxb,
// registered in the block map) and the unchanged grid-update gather sums the
// same tiles in the same order as a single rank would -- the node values are
// bit-identical.  Each rank also updates the ghost node column sx1 itself
// (planes 0,1 are complete there), so no second exchange returns grid
// velocities.  The messages are dense over the NB1 x NB2 column positions:
// 72 float4 per position plus one flag word, ~1.2 MB per direction at 128^3.
//
// After G2P, particles whose new base cell lies in another slab's column are
// packed (24 floats + class, id, key) into fixed-size messages and appended to the
// neighbour's state; their old slots are marked departed and dropped by the next
// sort.  The counts travel in the message headers and stay on the device.  The
// backward returns the cotangents of those particles along the same path.
#include <cuda_runtime.h>

#include "fl_kernels.h"
#include "fl_scatter.cuh"

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

namespace fl {

constexpr int kHaloNodes = 72;  // 2 x-planes of a 6x6 tile cross-section

size_t halo_bytes(const Geom& g) { return size_t(g.colblocks) * (kHaloNodes * sizeof(float4) + sizeof(int)); }

__global__ void k_halo_pack(Geom g, const int* __restrict__ blockmap, const float4* __restrict__ staging, int col,
                            int plane0, float4* out) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= g.colblocks * kHaloNodes) return;
    const int p = idx / kHaloNodes, t = idx % kHaloNodes;
    const int by = p / g.NB[2], bz = p % g.NB[2];
    const int slot = blockmap[block_lin(g, col, by, bz)] - 1;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (slot >= 0) v = staging[size_t(slot) * kTile + (plane0 + t / 36) * 36 + t % 36];
    out[idx] = v;
    if (t == 0) reinterpret_cast<int*>(out + size_t(g.colblocks) * kHaloNodes)[p] = slot >= 0 ? 1 : 0;
}

// ghost particle block (col, by, bz) -> staging slot ghost_base + p; the two
// received planes land at tile planes [plane0, plane0 + 2), the rest is zero.
// flag_col >= 0: the ghost tile reaches owned node blocks of that column
// (which may have no local particle block), so flag them for the node list.
__global__ void k_halo_unpack(Geom g, const float4* __restrict__ in, int col, int plane0, int ghost_base,
                              int* blockmap, float4* staging, int* nbflag, int flag_col) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= g.colblocks * int(kTile)) return;
    const int p = idx / kTile, t = idx % kTile;
    const int flag = reinterpret_cast<const int*>(in + size_t(g.colblocks) * kHaloNodes)[p];
    const int by = p / g.NB[2], bz = p % g.NB[2];
    const int slot = ghost_base + p;
    if (t == 0) {
        blockmap[block_lin(g, col, by, bz)] = flag ? slot + 1 : 0;
        if (flag && flag_col >= 0 && nbflag)
            for (int d = 0; d < 4; d++) {
                const int y = by + (d >> 1), z = bz + (d & 1);
                if (y < g.NB[1] && z < g.NB[2]) nbflag[block_lin(g, flag_col, y, z)] = 1;
            }
    }
    if (!flag) return;
    const int tx = t / 36;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (tx >= plane0 && tx < plane0 + 2) v = in[size_t(p) * kHaloNodes + (tx - plane0) * 36 + t % 36];
    staging[size_t(slot) * kTile + t] = v;
}

void launch_halo_pack(const Geom& g, const int* blockmap, const float4* staging, int col, int plane0, void* out,
                      cudaStream_t s) {
    const int n = g.colblocks * kHaloNodes;
    k_halo_pack<<<(n + 255) / 256, 256, 0, s>>>(g, blockmap, staging, col, plane0, static_cast<float4*>(out));
}

void launch_halo_unpack(const Geom& g, const void* in, int col, int plane0, int ghost_base, int* blockmap,
                        float4* staging, int* nbflag, int flag_col, cudaStream_t s) {
    const int n = g.colblocks * int(kTile);
    k_halo_unpack<<<(n + 255) / 256, 256, 0, s>>>(g, static_cast<const float4*>(in), col, plane0, ghost_base,
                                                   blockmap, staging, nbflag, flag_col);
}

// ---------------------------------------------------------------------------
// particle migration: fixed-size messages, counts stay on the device
// ---------------------------------------------------------------------------
// A message is a 16-int header (word 0: the number of particles it carries) and `cap`
// slots of kMigW words.  The pack kernel counts into its own send header; after the
// exchange one thread turns the send/receive headers into the record's counts (sent,
// received, arrival base) and the post-state's device counts, so no host round trip
// is needed per substep.  More migrants than `cap` (or more arrivals than the store
// holds) set the overflow flag, which the host checks once per call and answers with
// a re-run at a larger capacity (the canonical order makes the result independent of
// the capacity).
constexpr int kMigW = 27;   // words per migrating particle: 24 floats, class, id, key
constexpr int kMigHdr = 16;  // header words (64 B keeps the slots 16-byte aligned)

size_t mig_msg_bytes(int cap) { return (size_t(kMigHdr) + size_t(cap) * kMigW) * sizeof(uint32_t); }

// The messages are filled in slot order (a stable compaction: chunk per CTA, CTA
// offsets from the counts pass, block scans inside), so the arrival order on the
// receiving slab -- its storage order of the post-state -- is the same in every run.
// The backward relies on that: a segment replayed from its checkpoint must lay out its
// states exactly as the forward did, or the cotangents of migrated particles (indexed
// by storage slot) would land on other particles.
constexpr int kMigBlocks = 296;
constexpr int kMigThreads = 256;

__device__ __forceinline__ int mig_dir(const Geom& g, const PBuf& out, int j) {
    const uint32_t key = out.key[j];
    if (key >= g.key_inactive) return -1;
    const int col = key_col(g, key);
    return col < g.sx0 ? 0 : (col >= g.sx1 ? 1 : -1);
}

__global__ void __launch_bounds__(kMigThreads) k_mig_count(Geom g, PBuf out, DN nn, int* bcnt) {
    using Red = cub::BlockReduce<int2, kMigThreads>;
    __shared__ typename Red::TempStorage tmp;
    const int n = nn.get();
    const int chunk = (n + gridDim.x - 1) / gridDim.x;
    const int j0 = blockIdx.x * chunk, j1 = min(n, j0 + chunk);
    int2 c = make_int2(0, 0);
    for (int j = j0 + threadIdx.x; j < j1; j += kMigThreads) {
        const int d = mig_dir(g, out, j);
        c.x += d == 0;
        c.y += d == 1;
    }
    const int2 t = Red(tmp).Reduce(c, [](int2 a, int2 b) { return make_int2(a.x + b.x, a.y + b.y); });
    if (threadIdx.x == 0) reinterpret_cast<int2*>(bcnt)[blockIdx.x] = t;
}

__global__ void __launch_bounds__(kMigThreads) k_mig_pack(Geom g, PBuf out, DN nn, const int* __restrict__ bcnt,
                                                           uint32_t* send0, uint32_t* send1, uint32_t* src, int cap,
                                                           int* overflow) {
    using Scan = cub::BlockScan<int2, kMigThreads>;
    using Red = cub::BlockReduce<int2, kMigThreads>;
    __shared__ union {
        typename Scan::TempStorage scan;
        typename Red::TempStorage red;
    } tmp;
    __shared__ int2 base;
    auto add = [](int2 a, int2 b) { return make_int2(a.x + b.x, a.y + b.y); };
    const int n = nn.get();
    const int chunk = (n + gridDim.x - 1) / gridDim.x;
    const int j0 = blockIdx.x * chunk, j1 = min(n, j0 + chunk);
    int2 pre = make_int2(0, 0);
    for (int b = threadIdx.x; b < int(blockIdx.x); b += kMigThreads) pre = add(pre, reinterpret_cast<const int2*>(bcnt)[b]);
    pre = Red(tmp.red).Reduce(pre, add);
    if (threadIdx.x == 0) base = pre;
    __syncthreads();
    int2 off = base;
    for (int t0 = j0; t0 < j1; t0 += kMigThreads) {
        const int j = t0 + threadIdx.x;
        const int d = j < j1 ? mig_dir(g, out, j) : -1;
        int2 mine = make_int2(d == 0, d == 1), rank, tot;
        Scan(tmp.scan).ExclusiveScan(mine, rank, make_int2(0, 0), add, tot);
        __syncthreads();
        if (d >= 0) {
            uint32_t* msg = d == 0 ? send0 : send1;
            const int k = d == 0 ? off.x + rank.x : off.y + rank.y;
            const uint32_t key = out.key[j];
            out.key[j] = g.key_departed;
            if (!msg || k >= cap) {  // the particle is lost for this attempt: the call is re-run larger
                atomicMax(overflow, 1);
            } else {
                uint32_t* w = msg + kMigHdr + size_t(k) * kMigW;
                for (int c = 0; c < 24; c++) w[c] = __float_as_uint(out.f[size_t(c) * out.cap + j]);
                w[24] = out.meta[j];
                w[25] = out.id[j];
                w[26] = key;
                src[size_t(d) * cap + k] = uint32_t(j);
            }
        }
        off = add(off, tot);
    }
    // the last CTA knows the totals: message headers
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
        if (send0) *reinterpret_cast<int*>(send0) = off.x;
        if (send1) *reinterpret_cast<int*>(send1) = off.y;
    }
}

// rec: the substep record's device counts (RecCnt); post: the post-state's (StateCnt)
__global__ void k_mig_counts(const int* send0, const int* send1, const int* recv0, const int* recv1, int* rec,
                             int* post, int cap, int n_cap, int* overflow) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int s0 = send0 ? min(*send0, cap) : 0, s1 = send1 ? min(*send1, cap) : 0;
    const int r0 = recv0 ? min(*recv0, cap) : 0, r1 = recv1 ? min(*recv1, cap) : 0;
    const int base = rec[RC_KEEP];  // arrivals follow the parked tail
    rec[RC_SENT] = s0;
    rec[RC_SENT + 1] = s1;
    rec[RC_RECV] = r0;
    rec[RC_RECV + 1] = r1;
    rec[RC_ARR] = base;
    int stored = base + r0 + r1;
    if (stored > n_cap) {  // slab store overflow: more arrivals than slots
        atomicMax(overflow, 1);
        stored = n_cap;
    }
    post[SC_ACTIVE] = rec[RC_ACTIVE] - s0 - s1 + r0 + r1;
    post[SC_STORED] = stored;
    post[SC_PARK] = rec[RC_ACTIVE];
}

__global__ void k_mig_unpack(PBuf out, const uint32_t* __restrict__ in, const int* __restrict__ rec, int dir,
                             int n_cap) {
    const int n = rec[RC_RECV + dir];
    const int pos0 = rec[RC_ARR] + (dir ? rec[RC_RECV] : 0);
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int j = pos0 + k;
        if (j >= n_cap) return;  // (flagged overflow)
        const uint32_t* w = in + kMigHdr + size_t(k) * kMigW;
        for (int c = 0; c < 24; c++) out.f[size_t(c) * out.cap + j] = __uint_as_float(w[c]);
        out.meta[j] = w[24];
        out.id[j] = w[25];
        out.key[j] = w[26];
    }
}

// before a slab substep: the record's pre-state counts (after `gained` activations) and
// zeroed send headers for this substep's migration
__global__ void k_slab_counts_pre(const int* cnt, int* rec, int gained, int n_parked, int* send0, int* send1) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int na = cnt[SC_ACTIVE] + gained;
    rec[RC_ACTIVE] = na;
    rec[RC_KEEP] = na + n_parked;
    rec[RC_STORED] = cnt[SC_STORED];
    rec[RC_PARK] = cnt[SC_PARK];
    for (int q = RC_SENT; q < RC_N; q++) rec[q] = 0;
    if (send0) *send0 = 0;
    if (send1) *send1 = 0;
}

void launch_mig_pack(const Geom& g, PBuf out, DN n, void* send0, void* send1, uint32_t* src, int cap, int* bcnt,
                     int* overflow, cudaStream_t s) {
    k_mig_count<<<kMigBlocks, kMigThreads, 0, s>>>(g, out, n, bcnt);
    k_mig_pack<<<kMigBlocks, kMigThreads, 0, s>>>(g, out, n, bcnt, static_cast<uint32_t*>(send0),
                                                  static_cast<uint32_t*>(send1), src, cap, overflow);
}

void launch_mig_counts(const void* send0, const void* send1, const void* recv0, const void* recv1, int* rec,
                       int* post_cnt, int cap, int n_cap, int* overflow, cudaStream_t s) {
    k_mig_counts<<<1, 32, 0, s>>>(static_cast<const int*>(send0), static_cast<const int*>(send1),
                                  static_cast<const int*>(recv0), static_cast<const int*>(recv1), rec, post_cnt, cap,
                                  n_cap, overflow);
}

void launch_mig_unpack(PBuf out, const void* in, const int* rec, int dir, int cap, cudaStream_t s) {
    k_mig_unpack<<<gs_grid(cap, 148 * 4), 256, 0, s>>>(out, static_cast<const uint32_t*>(in), rec, dir, out.cap);
}

void launch_slab_counts_pre(const int* state_cnt, int* rec, int gained, int n_parked, void* send0, void* send1,
                            cudaStream_t s) {
    k_slab_counts_pre<<<1, 32, 0, s>>>(state_cnt, rec, gained, n_parked, static_cast<int*>(send0),
                                       static_cast<int*>(send1));
}

// cotangents of arrived particles travel back to the slab they came from (same message
// slots, 24 floats each, after a header of the same size)
__global__ void k_bars_pack(BarBuf bars, const int* __restrict__ rec, int dir, float* out) {
    const int n = rec[RC_RECV + dir];
    const int pos0 = rec[RC_ARR] + (dir ? rec[RC_RECV] : 0);
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
        for (int c = 0; c < 24; c++) out[kMigHdr + size_t(k) * 24 + c] = bars.f[size_t(c) * bars.cap + pos0 + k];
}

__global__ void k_bars_scatter(BarBuf bars, const float* __restrict__ in, const uint32_t* __restrict__ src,
                               const int* __restrict__ rec, int dir) {
    const int n = rec[RC_SENT + dir];
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const size_t j = src[k];
        for (int c = 0; c < 24; c++) bars.f[size_t(c) * bars.cap + j] = in[kMigHdr + size_t(k) * 24 + c];
    }
}

void launch_bars_pack(BarBuf bars, const int* rec, int dir, int cap, void* out, cudaStream_t s) {
    k_bars_pack<<<gs_grid(cap, 148 * 4), 256, 0, s>>>(bars, rec, dir, static_cast<float*>(out));
}

void launch_bars_scatter(BarBuf bars, const void* in, const uint32_t* src, const int* rec, int dir, int cap,
                         cudaStream_t s) {
    k_bars_scatter<<<gs_grid(cap, 148 * 4), 256, 0, s>>>(bars, static_cast<const float*>(in), src, rec, dir);
}

}  // namespace fl
