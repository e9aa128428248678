// fl_sort.cu -- canonical particle order: stable by (cell key, particle id).
//
// Block counting sort, device-driven (no host round trip):
//   1. count particles per 4^3 particle block (inactive particles form a
//      virtual block nbtot that sorts last, ordered by id; slots whose
//      particle moved to another slab form a second one, nbtot + 1, that is
//      listed after it and dropped by the next G2P)
//   2. exclusive scan of the counts -> segment starts
//   3. scatter (local cell, id, slot) into the block segments (arbitrary
//      order inside a segment)
//   4. one CTA per non-empty block sorts its segment by (local cell, id)
//      with a bitonic network in shared memory (global-memory network for
//      segments above the shared capacity)
// The resulting permutation is unique, so it is bit-identical to any other
// stable (key, id) sort -- the same order the CPU parity test recomputes.
// The block count array doubles as the particle-block list for the kernels.
#include <cuda_runtime.h>

#include "fl_kernels.h"
#include "fl_scatter.cuh"

namespace fl {

constexpr int kSortThreads = 256;

__global__ void k_sort_count(Geom g, PBuf st, int n, const ClassInfo* __restrict__ cls, int* bcount,
                             int* bheavy) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t key = st.key[i];
    const int b = key >= g.key_inactive ? g.nbtot + int((key - g.key_inactive) >> 6) : int(key >> 6);
    // warp-aggregated: the store order is nearly sorted, so lanes share blocks
    const unsigned peers = __match_any_sync(__activemask(), b);
    const unsigned heavy = __ballot_sync(__activemask(), cls[meta_cls(st.meta[i])].heavy != 0) & peers;
    const int leader = __ffs(peers) - 1;
    if ((threadIdx.x & 31) == leader) {
        atomicAdd(&bcount[b], __popc(peers));
        if (heavy) atomicOr(&bheavy[b], 1);
    }
}

// Also builds the active particle-block list: the warp that claims a block's
// first segment slot appends the block -- plain-liquid blocks from the front of
// recs, SVD/rigid blocks from the back (n_blocks[0] / n_blocks[1] entries).
// Slot assignment is run-dependent but no result depends on it.
__global__ void k_sort_scatter(Geom g, PBuf st, int n, const int* __restrict__ bstart,
                               const int* __restrict__ bcount, const int* __restrict__ bheavy, int* bfill,
                               uint32_t* skey, uint32_t* sslot, BlockRec* recs, int* n_blocks, int* blockmap,
                               int* nbflag, int cap) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t key = st.key[i];
    const bool inact = key >= g.key_inactive;  // parked or departed
    const int b = inact ? g.nbtot + int((key - g.key_inactive) >> 6) : int(key >> 6);
    const unsigned peers = __match_any_sync(__activemask(), b);
    const int leader = __ffs(peers) - 1;
    const int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == leader) {
        base = atomicAdd(&bfill[b], __popc(peers));
        if (base == 0 && !inact) {
            const bool hv = bheavy[b] != 0;
            const int q = hv ? cap - 1 - atomicAdd(&n_blocks[1], 1) : atomicAdd(&n_blocks[0], 1);
            recs[q] = BlockRec{b, bstart[b], bstart[b] + bcount[b]};
            blockmap[b] = q + 1;
            int bx, by, bz;  // node blocks covered by this block's tile
            block_unlin(g, b, bx, by, bz);
            for (int d = 0; d < 8; d++) {
                const int x = bx + (d >> 2), y = by + ((d >> 1) & 1), z = bz + (d & 1);
                if (x < g.NB[0] && y < g.NB[1] && z < g.NB[2]) nbflag[block_lin(g, x, y, z)] = 1;
            }
        }
    }
    base = __shfl_sync(peers, base, leader);
    const int p = bstart[b] + base + __popc(peers & ((1u << lane) - 1));
    skey[p] = ((inact ? 0u : (key & 63u)) << 26) | st.id[i];
    sslot[p] = uint32_t(i);
}

template <class KP, class VP>
__device__ void bitonic(KP k, VP v, int n, int tid, int nth) {
    for (int size = 2; size <= n; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = tid; i < (n >> 1); i += nth) {
                const int lo = 2 * i - (i & (stride - 1));
                const int hi = lo + stride;
                const bool up = ((lo & size) == 0);
                const uint32_t a = k[lo], b = k[hi];
                if ((a > b) == up) {
                    k[lo] = b;
                    k[hi] = a;
                    const uint32_t t = v[lo];
                    v[lo] = v[hi];
                    v[hi] = t;
                }
            }
            __syncthreads();
        }
    }
}

// per-cell start offsets of a sorted segment (first index with local cell >= c)
template <class KP>
__device__ void cell_starts(KP k, int cnt, uint16_t* out, int tid) {
    if (tid > 64) return;
    const uint32_t want = uint32_t(tid) << 26;
    int lo = 0, hi = cnt;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (k[mid] < want)
            lo = mid + 1;
        else
            hi = mid;
    }
    out[tid] = uint16_t(tid == 64 ? cnt : lo);
}

constexpr int kCountCap = 2048;  // particles per block segment sorted by the counting path

// One CTA per non-empty particle block: counting sort of the segment by local
// cell (64 buckets), then each cell's run is insertion-sorted by particle id
// (runs are ~8 long).  The inactive tail and oversized segments use the
// bitonic network instead.
__global__ void __launch_bounds__(kSortThreads) k_sort_blocks(int nbtot, const int* __restrict__ bcount,
                                                              const int* __restrict__ bstart,
                                                              const BlockRec* __restrict__ recs,
                                                              const int* __restrict__ n_blocks, int cap,
                                                              const uint32_t* skey, const uint32_t* sslot,
                                                              uint32_t* perm, uint16_t* celltab, uint32_t* gk,
                                                              uint32_t* gv) {
    __shared__ uint32_t ik[kCountCap], iv[kCountCap], ok[kCountCap], ov[kCountCap];
    __shared__ int hist[64], fill[64];
    __shared__ uint16_t cs[kCellTab];
    const int nl = n_blocks[0], nh = n_blocks[1];
    const int nb = nl + nh;
    const int tid = threadIdx.x;
    for (int w = blockIdx.x; w <= nb + 1; w += gridDim.x) {
        // w < nb: active block (light ones, then heavy ones from the back of recs);
        // w == nb: the inactive tail (ordered by id); w == nb + 1: departed slots (any order)
        const int q = w < nl ? w : cap - 1 - (w - nl);
        const bool act = w < nb;
        const int cnt = act ? recs[q].end - recs[q].start : bcount[nbtot + (w - nb)];
        if (cnt == 0) continue;
        const int s0 = act ? recs[q].start : bstart[nbtot + (w - nb)];
        if (w == nb + 1) {
            for (int i = tid; i < cnt; i += kSortThreads) perm[s0 + i] = sslot[s0 + i];
            continue;
        }
        if (act && cnt <= kCountCap) {
            for (int i = tid; i < cnt; i += kSortThreads) {
                ik[i] = skey[s0 + i];
                iv[i] = sslot[s0 + i];
            }
            if (tid < 64) hist[tid] = 0;
            __syncthreads();
            for (int i = tid; i < cnt; i += kSortThreads) atomicAdd(&hist[ik[i] >> 26], 1);
            __syncthreads();
            if (tid < 32) {  // exclusive scan of 64 counts by one warp
                int a = hist[2 * tid], b = hist[2 * tid + 1];
                int s = a + b, incl = s;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    int t = __shfl_up_sync(0xffffffffu, incl, o);
                    if (tid >= o) incl += t;
                }
                const int ex = incl - s;
                cs[2 * tid] = uint16_t(ex);
                cs[2 * tid + 1] = uint16_t(ex + a);
                fill[2 * tid] = ex;
                fill[2 * tid + 1] = ex + a;
                if (tid == 31) cs[64] = uint16_t(incl);
            }
            __syncthreads();
            for (int i = tid; i < cnt; i += kSortThreads) {
                const int p = atomicAdd(&fill[ik[i] >> 26], 1);
                ok[p] = ik[i];
                ov[p] = iv[i];
            }
            __syncthreads();
            if (tid < 64) {
                const int a = cs[tid], e = cs[tid + 1];
                for (int i = a + 1; i < e; i++) {
                    const uint32_t kk = ok[i], vv = ov[i];
                    int j = i - 1;
                    while (j >= a && ok[j] > kk) {
                        ok[j + 1] = ok[j];
                        ov[j + 1] = ov[j];
                        j--;
                    }
                    ok[j + 1] = kk;
                    ov[j + 1] = vv;
                }
            }
            if (tid < kCellTab) celltab[size_t(q) * kCellTab + tid] = tid <= 64 ? cs[tid] : 0;
            __syncthreads();
            for (int i = tid; i < cnt; i += kSortThreads) perm[s0 + i] = ov[i];
            __syncthreads();
        } else {
            // inactive tail or oversized block: bitonic network on a global scratch copy
            uint16_t* ct = act ? celltab + size_t(q) * kCellTab : nullptr;
            int np = 1;
            while (np < cnt) np <<= 1;
            uint32_t* k = gk + size_t(s0) * 2;
            uint32_t* v = gv + size_t(s0) * 2;
            for (int i = tid; i < np; i += kSortThreads) {
                k[i] = i < cnt ? skey[s0 + i] : 0xffffffffu;
                v[i] = i < cnt ? sslot[s0 + i] : 0u;
            }
            __syncthreads();
            bitonic(k, v, np, tid, kSortThreads);
            for (int i = tid; i < cnt; i += kSortThreads) perm[s0 + i] = v[i];
            if (ct) cell_starts(k, cnt, ct, tid);
            __syncthreads();
        }
    }
}

void launch_sort_count(const Geom& g, const PBuf& st, int n, const ClassInfo* cls, int* bcount, int* bheavy,
                       cudaStream_t s) {
    if (n <= 0) return;  // (an empty slab)
    k_sort_count<<<(n + 255) / 256, 256, 0, s>>>(g, st, n, cls, bcount, bheavy);
}
void launch_sort_scatter(const Geom& g, const PBuf& st, int n, const int* bstart, const int* bcount,
                         const int* bheavy, int* bfill, uint32_t* skey, uint32_t* sslot, BlockRec* recs, int* n_blocks,
                         int* blockmap, int* nbflag, int cap, cudaStream_t s) {
    if (n <= 0) return;
    k_sort_scatter<<<(n + 255) / 256, 256, 0, s>>>(g, st, n, bstart, bcount, bheavy, bfill, skey, sslot, recs,
                                                   n_blocks, blockmap, nbflag, cap);
}

// compact, id-ordered list of touched node blocks
// compact, id-ordered list of touched node blocks; also publishes the
// particle-block list counters (scratch -> record)
__global__ void k_nb_scatter(const int* __restrict__ flags, const int* __restrict__ pos, int n, int* list,
                             int* n_list, const int* __restrict__ cnt_scratch, int* n_blocks) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) {
        n_blocks[0] = cnt_scratch[0];
        n_blocks[1] = cnt_scratch[1];
    }
    if (i >= n) return;
    if (flags[i]) list[pos[i]] = i;
    if (i == n - 1) *n_list = pos[i] + (flags[i] ? 1 : 0);
}

void launch_nb_scatter(const int* flags, const int* pos, int nbtot, int* list, int* n_list, const int* cnt_scratch,
                       int* n_blocks, cudaStream_t s) {
    k_nb_scatter<<<(nbtot + 255) / 256, 256, 0, s>>>(flags, pos, nbtot, list, n_list, cnt_scratch, n_blocks);
}
void launch_sort_blocks(const Geom& g, const int* bcount, const int* bstart, const BlockRec* recs,
                        const int* n_blocks, int cap, const uint32_t* skey, const uint32_t* sslot, uint32_t* perm,
                        uint16_t* celltab, uint32_t* gk, uint32_t* gv, int grid, cudaStream_t s) {
    k_sort_blocks<<<grid, kSortThreads, 0, s>>>(g.nbtot, bcount, bstart, recs, n_blocks, cap, skey, sslot, perm,
                                                celltab, gk, gv);
}
}  // namespace fl
