// fl_sort.cu -- canonical particle order: stable by (cell key, particle id).
//
// Block counting sort, device-driven (no host round trip):
//   1. count particles per 4^3 particle block (inactive particles form a
//      virtual block nbtot that sorts last, ordered by id; slots whose
//      particle moved to another slab form a second one, nbtot + 1, that is
//      listed after it and dropped by the next G2P)
//   2. one CTA scans the counts -> segment starts, and in the same pass the
//      node-block flags (from the counts of the 2x2x2 particle blocks below
//      each node block), the node-block list and the particle-block list
//      (plain-liquid blocks from the front, SVD/rigid blocks from the back)
//   3. scatter (local cell, id, slot) into the block segments (arbitrary
//      order inside a segment)
//   4. one CTA per non-empty block sorts its segment by (local cell, id):
//      counting sort by cell, then rank by id inside each cell run (a bitonic
//      network in global memory for segments above the shared capacity)
// The resulting permutation is unique, so it is bit-identical to any other
// stable (key, id) sort -- the same order the CPU parity test recomputes.
// The block count array doubles as the particle-block list for the kernels.
//
// Incremental sort (one rank, substeps chained by forward_substep).  G2P writes state t+1
// in the sorted order of substep t and a particle moves ~0.003 cells per substep, so
// nearly every key is unchanged.  Each sort also writes `okey`, the key at every sorted
// position (bit 31: an SVD/rigid particle), and keeps the block counts.  The next sort:
//   1. diff: key (+ class bit) against okey; a changed particle marks its old and new
//      block dirty, and one that changed block updates both counts, the heavy counts
//      and the arrival count and joins the mover list.  The class bit only changes for a
//      liquid uploaded with a full F (kMetaFull, dropped by its first G2P); otherwise the
//      key alone is compared (8 bytes per particle).  (Doing this in G2P instead, where
//      the keys are written, cost G2P more than the kernel: c4 +3.7 us, spills.)
//   2. the list scan as above (new segment starts); for every listed block it also
//      records each block's previous list slot and segment (rold) and clears the dirty flags
//   3. (the diff filed each arrival in its new block's inbox, kInbox slots, the rest in an
//      overflow list that only blocks with more arrivals scan)
//   4. one CTA per block: a clean block copies its old segment in order (perm = the old
//      sorted positions, cell table and okey copied); a dirty block collects the
//      stayers of its old segment and its arrivals and sorts them as in step 4 above
// Counts and the permutation are the full sort's by construction (bit-identical,
// tested against it); activation substeps, slabs and the first substep after any
// other state write use the full sort.
#include <cuda_runtime.h>

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "fl_kernels.h"
#include "fl_scatter.cuh"

namespace fl {

#ifndef FL_SORT_THREADS
#define FL_SORT_THREADS 256
#endif
#ifndef FL_COUNT_CAP
#define FL_COUNT_CAP 1024
#endif
constexpr int kSortThreads = FL_SORT_THREADS;

// Both passes handle kSortItems particles per thread (CTA-strided, so a warp still covers
// consecutive slots for the warp aggregation): the loads of all items are issued before
// the first atomic, which turns one dependent load -> atomic -> store chain per particle
// into kSortItems overlapped ones.
#ifndef FL_SORT_ITEMS
#define FL_SORT_ITEMS 4
#endif
constexpr int kSortItems = FL_SORT_ITEMS;

__device__ __forceinline__ uint32_t heavy_bit(const ClassInfo* __restrict__ cls, uint32_t meta) {
    return (cls[meta_cls(meta)].heavy != 0 || (meta & kMetaFull) != 0u) ? kHeavyBit : 0u;
}

__global__ void k_sort_count(Geom g, PBuf st, DN nn, const ClassInfo* __restrict__ cls, int* bcount,
                             int* bheavy) {
    pdl_wait();
    const int n = nn.get();
    const int i0 = blockIdx.x * blockDim.x * kSortItems + threadIdx.x;
    uint32_t key[kSortItems], meta[kSortItems];
#pragma unroll
    for (int q = 0; q < kSortItems; q++) {
        const int i = i0 + q * blockDim.x;
        key[q] = i < n ? st.key[i] : 0u;
        meta[q] = i < n ? st.meta[i] : 0u;
    }
#pragma unroll
    for (int q = 0; q < kSortItems; q++) {
        if (i0 + q * int(blockDim.x) >= n) break;
        const int b = key[q] >= g.key_inactive ? g.nbtot + int((key[q] - g.key_inactive) >> 6) : int(key[q] >> 6);
        // warp-aggregated: the store order is nearly sorted, so lanes share blocks
        const unsigned peers = __match_any_sync(__activemask(), b);
        const unsigned heavy =
            __ballot_sync(__activemask(), cls[meta_cls(meta[q])].heavy != 0 || (meta[q] & kMetaFull) != 0u) & peers;
        const int leader = __ffs(peers) - 1;
        if ((threadIdx.x & 31) == leader) {
            atomicAdd(&bcount[b], __popc(peers));
            if (heavy) atomicAdd(&bheavy[b], __popc(heavy));  // a count: the incremental sort updates it
        }
    }
}

// cls != nullptr: the slot word carries the class bit (kHeavyBit) for the okey output
__global__ void k_sort_scatter(Geom g, PBuf st, DN nn, const int* __restrict__ bstart, int* bfill, uint32_t* skey,
                               uint32_t* sslot, const ClassInfo* __restrict__ cls) {
    pdl_wait();
    const int n = nn.get();
    const int i0 = blockIdx.x * blockDim.x * kSortItems + threadIdx.x;
    uint32_t key[kSortItems], id[kSortItems], hb[kSortItems];
#pragma unroll
    for (int q = 0; q < kSortItems; q++) {
        const int i = i0 + q * blockDim.x;
        key[q] = i < n ? st.key[i] : 0u;
        id[q] = i < n ? st.id[i] : 0u;
        hb[q] = (cls && i < n) ? heavy_bit(cls, st.meta[i]) : 0u;
    }
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int q = 0; q < kSortItems; q++) {
        const int i = i0 + q * blockDim.x;
        if (i >= n) break;
        const bool inact = key[q] >= g.key_inactive;  // parked or departed
        const int b = inact ? g.nbtot + int((key[q] - g.key_inactive) >> 6) : int(key[q] >> 6);
        const unsigned peers = __match_any_sync(__activemask(), b);
        const int leader = __ffs(peers) - 1;
        int base = 0;
        if (lane == leader) base = atomicAdd(&bfill[b], __popc(peers));
        base = __shfl_sync(peers, base, leader);
        const int p = bstart[b] + base + __popc(peers & ((1u << lane) - 1));
        skey[p] = ((inact ? 0u : (key[q] & 63u)) << 26) | id[q];
        sslot[p] = uint32_t(i) | hb[q];
    }
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

constexpr int kCountCap = FL_COUNT_CAP;  // particles per block segment sorted by the counting path

struct SegSmem {
    uint32_t ik[kCountCap], iv[kCountCap], ok[kCountCap], ov[kCountCap];
    int hist[64], fill[64];
    uint16_t cs[kCellTab];
    int n;
};

// Sorts the cnt (key, slot word) pairs in sm.ik / sm.iv (key = local cell << 26 | id,
// slot word = slot | class bit) into the segment at s0: counting sort by cell, then every
// particle ranks itself inside its cell's run by particle id (runs are ~8 long; measured
// 12% faster than a per-cell insertion sort).  Writes perm, the cell table ct and, when
// okey is given, the sorted keys (block word = block << 6).  The caller loaded ik / iv.
__device__ void seg_count_sort(SegSmem& sm, int cnt, int s0, uint32_t bword, uint32_t* perm, uint16_t* ct,
                               uint32_t* okey) {
    const int tid = threadIdx.x;
    if (tid < 64) sm.hist[tid] = 0;
    __syncthreads();
    for (int i = tid; i < cnt; i += kSortThreads) atomicAdd(&sm.hist[sm.ik[i] >> 26], 1);
    __syncthreads();
    if (tid < 32) {  // exclusive scan of 64 counts by one warp
        int a = sm.hist[2 * tid], b = sm.hist[2 * tid + 1];
        int s = a + b, incl = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (tid >= o) incl += t;
        }
        const int ex = incl - s;
        sm.cs[2 * tid] = uint16_t(ex);
        sm.cs[2 * tid + 1] = uint16_t(ex + a);
        sm.fill[2 * tid] = ex;
        sm.fill[2 * tid + 1] = ex + a;
        int mx = a > b ? a : b;  // largest cell: the scatter kernels' pass count
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const int t = __shfl_xor_sync(0xffffffffu, mx, o);
            mx = t > mx ? t : mx;
        }
        if (tid == 31) {
            sm.cs[64] = uint16_t(incl);
            sm.cs[65] = uint16_t(mx);
        }
    }
    __syncthreads();
    for (int i = tid; i < cnt; i += kSortThreads) {
        const int p = atomicAdd(&sm.fill[sm.ik[i] >> 26], 1);
        sm.ok[p] = sm.ik[i];
        sm.ov[p] = sm.iv[i];
    }
    __syncthreads();
    // each particle's place inside its cell run = the number of run members with a
    // smaller key (keys are unique: they carry the particle id); all threads busy
    for (int i = tid; i < cnt; i += kSortThreads) {
        const uint32_t kk = sm.ok[i];
        const int c = int(kk >> 26);
        const int a = sm.cs[c], e = sm.cs[c + 1];
        int rnk = 0;
        for (int j = a; j < e; j++) rnk += sm.ok[j] < kk ? 1 : 0;
        perm[s0 + a + rnk] = sm.ov[i] & ~kHeavyBit;
        if (okey) okey[s0 + a + rnk] = (bword | uint32_t(c)) | (sm.ov[i] & kHeavyBit);
    }
    if (tid < kCellTab) ct[tid] = sm.cs[tid];
    __syncthreads();
}

// The same for a segment above the shared capacity (or the inactive tail, ct == nullptr,
// ordered by id): bitonic network on the global scratch copy k / v (loaded by the caller,
// padded to a power of two with 0xffffffff keys).
__device__ void seg_bitonic_sort(uint32_t* k, uint32_t* v, int cnt, int np, int s0, uint32_t bword, uint32_t* perm,
                                 uint16_t* ct, uint32_t* okey) {
    const int tid = threadIdx.x;
    bitonic(k, v, np, tid, kSortThreads);
    for (int i = tid; i < cnt; i += kSortThreads) {
        perm[s0 + i] = v[i] & ~kHeavyBit;
        if (okey) okey[s0 + i] = (ct ? (bword | (k[i] >> 26)) : bword) | (v[i] & kHeavyBit);
    }
    if (ct) cell_starts(k, cnt, ct, tid);
    __syncthreads();
    if (ct && tid == 0) {
        int mx = 0;
        for (int c = 0; c < 64; c++) mx = max(mx, int(ct[c + 1]) - int(ct[c]));
        ct[65] = uint16_t(mx);
    }
}

// One CTA per non-empty particle block (full sort).  okey != nullptr: also write the
// sorted keys for the next substep's incremental sort.
__global__ void __launch_bounds__(kSortThreads) k_sort_blocks(Geom g, const int* __restrict__ bcount,
                                                              const int* __restrict__ bstart,
                                                              const BlockRec* __restrict__ recs, int* n_blocks,
                                                              int cap, const uint32_t* skey, const uint32_t* sslot,
                                                              uint32_t* perm, uint16_t* celltab, uint32_t* gk,
                                                              uint32_t* gv, uint32_t* okey) {
    pdl_wait();
    __shared__ SegSmem sm;
    const int nl = n_blocks[0], nh = n_blocks[1];
    const int nb = nl + nh;
    const int tid = threadIdx.x;
    for (int w = blockIdx.x; w <= nb + 1; w += gridDim.x) {
        // w < nb: active block (light ones, then heavy ones from the back of recs);
        // w == nb: the inactive tail (ordered by id); w == nb + 1: departed slots (any order)
        const int q = w < nl ? w : cap - 1 - (w - nl);
        const bool act = w < nb;
        const int cnt = act ? recs[q].end - recs[q].start : bcount[g.nbtot + (w - nb)];
        if (cnt == 0) continue;
        const int s0 = act ? recs[q].start : bstart[g.nbtot + (w - nb)];
        if (w == nb + 1) {
            for (int i = tid; i < cnt; i += kSortThreads) {
                perm[s0 + i] = sslot[s0 + i] & ~kHeavyBit;
                if (okey) okey[s0 + i] = g.key_departed | (sslot[s0 + i] & kHeavyBit);
            }
            continue;
        }
        const uint32_t bword = act ? uint32_t(recs[q].block) << 6 : g.key_inactive;
        if (act && cnt <= kCountCap) {
            for (int i = tid; i < cnt; i += kSortThreads) {
                sm.ik[i] = skey[s0 + i];
                sm.iv[i] = sslot[s0 + i];
            }
            seg_count_sort(sm, cnt, s0, bword, perm, celltab + size_t(q) * kCellTab, okey);
            if (tid == 0) work_file(n_blocks, cap, w < nl ? 0 : 1, q, recs[q], sm.cs[65]);
        } else {
            int np = 1;
            while (np < cnt) np <<= 1;
            uint32_t* k = gk + size_t(s0) * 2;
            uint32_t* v = gv + size_t(s0) * 2;
            for (int i = tid; i < np; i += kSortThreads) {
                k[i] = i < cnt ? skey[s0 + i] : 0xffffffffu;
                v[i] = i < cnt ? sslot[s0 + i] : 0u;
            }
            __syncthreads();
            seg_bitonic_sort(k, v, cnt, np, s0, bword, perm, act ? celltab + size_t(q) * kCellTab : nullptr, okey);
            if (act && tid == 0) work_file(n_blocks, cap, w < nl ? 0 : 1, q, recs[q], celltab[size_t(q) * kCellTab + 65]);
        }
    }
}

// ---------------------------------------------------------------------------
// incremental sort (see the header)
// ---------------------------------------------------------------------------
template <bool META>
__global__ void k_isort_diff(Geom g, PBuf st, int n, const ClassInfo* __restrict__ cls,
                             const uint32_t* __restrict__ okey, int* bcount, int* bheavy, int* acnt, int* dirty,
                             uint32_t* inbox, int* nmov, uint32_t* mov) {
    pdl_wait();
    const int i0 = blockIdx.x * blockDim.x * kSortItems + threadIdx.x;
    uint32_t key[kSortItems], meta[kSortItems], ok[kSortItems];
#pragma unroll
    for (int q = 0; q < kSortItems; q++) {
        const int i = i0 + q * blockDim.x;
        key[q] = i < n ? st.key[i] : 0u;
        if (META) meta[q] = i < n ? st.meta[i] : 0u;
        ok[q] = i < n ? okey[i] : 0u;
    }
#pragma unroll
    for (int q = 0; q < kSortItems; q++) {
        const int i = i0 + q * blockDim.x;
        if (i >= n) break;
        const uint32_t nk = key[q] | (META ? heavy_bit(cls, meta[q]) : (ok[q] & kHeavyBit));
        if (nk == ok[q]) continue;
        const int ob = key_block(g, ok[q] & ~kHeavyBit), nb = key_block(g, key[q]);
        const int oh = int(ok[q] >> 31), nh = int(nk >> 31);
        dirty[ob] = 1;
        dirty[nb] = 1;
        if (ob != nb) {
            atomicSub(&bcount[ob], 1);
            atomicAdd(&bcount[nb], 1);
            if (oh) atomicSub(&bheavy[ob], 1);
            if (nh) atomicAdd(&bheavy[nb], 1);
            const int pos = atomicAdd(&acnt[nb], 1);
            if (pos < kInbox)
                inbox[size_t(nb) * kInbox + pos] = uint32_t(i);
            else
                mov[atomicAdd(nmov, 1)] = uint32_t(i);
        } else if (oh != nh) {
            atomicAdd(&bheavy[nb], nh - oh);
        }
    }
}

__global__ void __launch_bounds__(kSortThreads) k_isort_blocks(Geom g, PBuf st, const ClassInfo* __restrict__ cls,
                                                               const int* __restrict__ bcount,
                                                               const int* __restrict__ bstart,
                                                               const BlockRec* __restrict__ recs, int* n_blocks,
                                                               int cap, IncSort is,
                                                               const uint32_t* sslot, uint32_t* perm,
                                                               uint16_t* celltab, uint32_t* gk, uint32_t* gv) {
    pdl_wait();
    __shared__ SegSmem sm;
    const int nl = n_blocks[0], nh = n_blocks[1];
    const int nb = nl + nh;
    const int tid = threadIdx.x;
    for (int w = blockIdx.x; w <= nb; w += gridDim.x) {
        if (w == nb) {  // the inactive tail: unchanged without activation
            const int s0 = bstart[g.nbtot], cnt = bcount[g.nbtot];
            for (int i = tid; i < cnt; i += kSortThreads) {
                perm[s0 + i] = uint32_t(s0 + i);
                is.okey_out[s0 + i] = is.okey_in[s0 + i];
            }
            continue;
        }
        const int q = w < nl ? w : cap - 1 - (w - nl);
        const BlockRec r = recs[q];
        const int cnt = r.end - r.start, s0 = r.start;
        uint16_t* ct = celltab + size_t(q) * kCellTab;
        const int4 ro = is.rold[q];  // {clean, old list slot, old start, old end}
        const int oq = ro.y;
        if (ro.x) {  // clean: the old segment, in order
            const int os0 = ro.z;
            for (int i = tid; i < cnt; i += kSortThreads) {
                perm[s0 + i] = uint32_t(os0 + i);
                is.okey_out[s0 + i] = is.okey_in[os0 + i];
            }
            if (tid < kCellTab) ct[tid] = is.octab[size_t(oq) * kCellTab + tid];
            if (tid == 0) work_file(n_blocks, cap, w < nl ? 0 : 1, q, r, is.octab[size_t(oq) * kCellTab + 65]);
            continue;
        }
        // dirty: the stayers of the old segment + the arrivals, sorted
        const int os0 = oq >= 0 ? ro.z : 0, oe = oq >= 0 ? ro.w : 0;
        const int na = is.acnt[r.block];
        const int nin = min(na, kInbox);
        const int nov = na > kInbox ? *is.novf : 0;  // more arrivals than the inbox: scan the overflow list
        const bool fits = cnt <= kCountCap;
        int np = 1;
        while (np < cnt) np <<= 1;
        uint32_t* k = gk + size_t(s0) * 2;
        uint32_t* v = gv + size_t(s0) * 2;
        if (tid == 0) sm.n = 0;
        __syncthreads();
        const int nold = oe - os0;
        for (int i = tid; i < nold + nin + nov; i += kSortThreads) {
            const uint32_t p = i < nold ? uint32_t(os0 + i)
                                        : (i < nold + nin ? is.inbox[size_t(r.block) * kInbox + (i - nold)]
                                                          : is.mov[i - nold - nin]);
            const uint32_t key = st.key[p];
            if (i < nold && key_block(g, key) != r.block) continue;       // left the block
            if (i >= nold + nin && key_block(g, key) != r.block) continue;  // another block's overflow
            const uint32_t kk = ((key & 63u) << 26) | st.id[p];
            const uint32_t vv = p | heavy_bit(cls, st.meta[p]);
            const int j = atomicAdd(&sm.n, 1);
            if (fits) {
                sm.ik[j] = kk;
                sm.iv[j] = vv;
            } else {
                k[j] = kk;
                v[j] = vv;
            }
        }
        __syncthreads();
        if (tid == 0) {
            if (sm.n != cnt) __trap();  // the counts and the members disagree: cannot happen
            if (na) is.acnt[r.block] = 0;
        }
        const uint32_t bword = uint32_t(r.block) << 6;
        if (fits) {
            seg_count_sort(sm, cnt, s0, bword, perm, ct, is.okey_out);
            if (tid == 0) work_file(n_blocks, cap, w < nl ? 0 : 1, q, r, sm.cs[65]);
        } else {
            for (int i = cnt + tid; i < np; i += kSortThreads) {
                k[i] = 0xffffffffu;
                v[i] = 0u;
            }
            __syncthreads();
            seg_bitonic_sort(k, v, cnt, np, s0, bword, perm, ct, is.okey_out);
            if (tid == 0) work_file(n_blocks, cap, w < nl ? 0 : 1, q, r, ct[65]);
        }
    }
}

// n.h: the slot count (an upper bound on slabs, where the kernels read the device count)
void launch_sort_count(const Geom& g, const PBuf& st, DN n, const ClassInfo* cls, int* bcount, int* bheavy,
                       cudaStream_t s) {
    if (n.h <= 0) return;  // (an empty slab)
    launch_k(k_sort_count, dim3((n.h + 256 * kSortItems - 1) / (256 * kSortItems)), dim3(256), 0, s, g, st, n, cls,
             bcount, bheavy);
}
void launch_sort_scatter(const Geom& g, const PBuf& st, DN n, const int* bstart, int* bfill, uint32_t* skey,
                         uint32_t* sslot, const ClassInfo* cls_bit, cudaStream_t s) {
    if (n.h <= 0) return;
    launch_k(k_sort_scatter, dim3((n.h + 256 * kSortItems - 1) / (256 * kSortItems)), dim3(256), 0, s, g, st, n,
             bstart, bfill, skey, sslot, cls_bit);
}

void launch_isort_diff(const Geom& g, const PBuf& st, int n, const ClassInfo* cls, int* bcount, int* bheavy,
                       const IncSort& is, bool meta, cudaStream_t s) {
    if (n <= 0) return;
    launch_k(meta ? k_isort_diff<true> : k_isort_diff<false>, dim3((n + 256 * kSortItems - 1) / (256 * kSortItems)),
             dim3(256), 0, s, g, st, n, cls, (const uint32_t*)is.okey_in, bcount, bheavy, is.acnt, is.dirty, is.inbox,
             is.nmov, is.mov);
}
void launch_isort_place(const Geom& g, const PBuf& st, const ClassInfo* cls, const int* bcount, const int* bstart,
                        const BlockRec* recs, int* n_blocks, int cap, const IncSort& is, uint32_t* sslot,
                        uint32_t* perm, uint16_t* celltab, uint32_t* gk, uint32_t* gv, int grid, int arrive_grid,
                        cudaStream_t s) {
    (void)sslot;
    (void)arrive_grid;
    launch_k(k_isort_blocks, dim3(grid), dim3(kSortThreads), 0, s, g, st, cls, bcount, bstart, recs, n_blocks, cap, is,
             (const uint32_t*)sslot, perm, celltab, gk, gv);
}

// ---------------------------------------------------------------------------
// step 2: 4-channel scan over the nbtot + 2 block counts (particles, touched
// node blocks, plain-liquid blocks, SVD/rigid blocks) in two passes of
// 256-block tiles: tile sums, then every tile adds its predecessors' sums
// (<= a few hundred) and writes its outputs.  Deterministic, no atomics.  (A one-pass
// decoupled look-back scan was measured slower on c4: 256-block tiles +2 us, 1024-block
// tiles +4 us per sort -- the look-back chain costs more than the kernel boundary.)
// ---------------------------------------------------------------------------
constexpr int kListThreads = 256;
#ifndef FL_LIST_ITEMS
#define FL_LIST_ITEMS 1
#endif
constexpr int kListItems = FL_LIST_ITEMS;  // consecutive blocks per thread
constexpr int kListTile = kListThreads * kListItems;

struct Sum4 {
    __device__ __forceinline__ int4 operator()(const int4& a, const int4& b) const {
        return make_int4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
    }
};

// node block (x,y,z) is touched when any particle block (x-i, y-j, z-k), i,j,k in {0,1}, is occupied
__device__ __forceinline__ int node_touched(const Geom& g, const int* __restrict__ bcount, int b) {
    int x, y, z;
    block_unlin(g, b, x, y, z);
    int f = 0;
#pragma unroll
    for (int d = 0; d < 8; d++) {
        const int xx = x - (d >> 2), yy = y - ((d >> 1) & 1), zz = z - (d & 1);
        if (xx >= 0 && yy >= 0 && zz >= 0) f |= bcount[block_lin(g, xx, yy, zz)];
    }
    return f != 0;
}

// 1 = plain-liquid block, 2 = SVD/rigid block, 0 = empty (or a virtual block)
__device__ __forceinline__ int block_kind(const Geom& g, const int* __restrict__ bcount,
                                          const int* __restrict__ bheavy, int b) {
    if (b >= g.nbtot || bcount[b] == 0) return 0;
    return bheavy[b] != 0 ? 2 : 1;
}

__global__ void __launch_bounds__(kListThreads) k_list_sums(Geom g, const int* __restrict__ bcount,
                                                            const int* __restrict__ bheavy, int* nbflag,
                                                            int4* tile_sum, int* nmov, int* novf) {
    pdl_wait();
    if (nmov && blockIdx.x == 0 && threadIdx.x == 0) {  // incremental sort: the diff is complete
        *novf = *nmov;
        *nmov = 0;
    }
    using Red = cub::BlockReduce<int4, kListThreads>;
    __shared__ typename Red::TempStorage tmp;
    const int n = g.nbtot + 2;
    const int b0 = blockIdx.x * kListTile + threadIdx.x * kListItems;
    int4 mine = make_int4(0, 0, 0, 0);
#pragma unroll
    for (int k = 0; k < kListItems; k++) {
        const int b = b0 + k;
        if (b >= n) break;
        mine.x += bcount[b];
        if (b < g.nbtot) {
            const int f = node_touched(g, bcount, b);
            nbflag[b] = f;
            mine.y += f;
        }
        const int kind = block_kind(g, bcount, bheavy, b);
        mine.z += kind == 1;
        mine.w += kind == 2;
    }
    const int4 tot = Red(tmp).Reduce(mine, Sum4());
    if (threadIdx.x == 0) tile_sum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kListThreads) k_list_write(Geom g, int cap, const int* __restrict__ bcount,
                                                             const int* __restrict__ bheavy,
                                                             const int* __restrict__ nbflag,
                                                             const int4* __restrict__ tile_sum, int* bstart,
                                                             int* nb_list, int* n_nb, BlockRec* recs, int* blockmap,
                                                             int* n_blocks, const int* __restrict__ oblockmap,
                                                             const BlockRec* __restrict__ orecs, int4* rold,
                                                             int* dirty) {
    pdl_wait();
    using Scan = cub::BlockScan<int4, kListThreads>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ int4 base;
    const int n = g.nbtot + 2, tid = threadIdx.x;
    if (tid < 32) {  // predecessors' tile sums: strided lanes + fixed shuffle tree
        int4 s = make_int4(0, 0, 0, 0);
        for (int t = tid; t < int(blockIdx.x); t += 32) s = Sum4()(s, tile_sum[t]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            s.x += __shfl_down_sync(0xffffffffu, s.x, o);
            s.y += __shfl_down_sync(0xffffffffu, s.y, o);
            s.z += __shfl_down_sync(0xffffffffu, s.z, o);
            s.w += __shfl_down_sync(0xffffffffu, s.w, o);
        }
        if (tid == 0) base = s;
    }
    if (blockIdx.x == 0 && tid < 2 * kWorkClasses) n_blocks[4 + tid] = 0;  // work-order class counts
    const int b0 = blockIdx.x * kListTile + tid * kListItems;
    int cnt[kListItems], flag[kListItems], kind[kListItems];
    int4 mine = make_int4(0, 0, 0, 0);
#pragma unroll
    for (int k = 0; k < kListItems; k++) {
        const int b = b0 + k;
        cnt[k] = b < n ? bcount[b] : 0;
        flag[k] = b < g.nbtot ? nbflag[b] : 0;
        kind[k] = b < n ? block_kind(g, bcount, bheavy, b) : 0;
        mine.x += cnt[k];
        mine.y += flag[k];
        mine.z += kind[k] == 1;
        mine.w += kind[k] == 2;
    }
    int4 pre, tot;
    Scan(tmp).ExclusiveScan(mine, pre, make_int4(0, 0, 0, 0), Sum4(), tot);
    __syncthreads();
    pre = Sum4()(pre, base);
#pragma unroll
    for (int k = 0; k < kListItems; k++) {
        const int b = b0 + k;
        if (b >= n) break;
        bstart[b] = pre.x;
        if (b < g.nbtot) {
            if (flag[k]) nb_list[pre.y] = b;
            int slot = 0;  // block-map convention: slot + 1, 0 = none
            if (kind[k] == 1) slot = pre.z + 1;
            if (kind[k] == 2) slot = cap - pre.w;  // SVD/rigid blocks fill recs from the back
            if (slot) recs[slot - 1] = BlockRec{b, pre.x, pre.x + cnt[k]};
            blockmap[b] = slot;
            // incremental sort: a clean block copies its old segment (its previous list slot)
            if (rold && slot) {
                const int oq = oblockmap[b] - 1;
                const BlockRec o = oq >= 0 ? orecs[oq] : BlockRec{0, 0, 0};
                rold[slot - 1] = make_int4(dirty[b] ? 0 : 1, oq, o.start, o.end);
            }
        }
        if (dirty) dirty[b] = 0;
        pre.x += cnt[k];
        pre.y += flag[k];
        pre.z += kind[k] == 1;
        pre.w += kind[k] == 2;
    }
    if (blockIdx.x == gridDim.x - 1 && tid == 0) {
        const int4 all = Sum4()(base, tot);
        *n_nb = all.y;
        n_blocks[0] = all.z;
        n_blocks[1] = all.w;
    }
}

int sort_list_tiles(const Geom& g) { return (g.nbtot + 2 + kListTile - 1) / kListTile; }

void launch_sort_lists(const Geom& g, int cap, const int* bcount, const int* bheavy, int* bstart, int* nbflag,
                       int* nb_list, int* n_nb, BlockRec* recs, int* blockmap, int* n_blocks, int4* tile_sum,
                       const IncSort* inc, cudaStream_t s) {
    const int tiles = sort_list_tiles(g);
    launch_k(k_list_sums, dim3(tiles), dim3(kListThreads), 0, s, g, bcount, bheavy, nbflag, tile_sum,
             inc ? inc->nmov : nullptr, inc ? inc->novf : nullptr);
    launch_k(k_list_write, dim3(tiles), dim3(kListThreads), 0, s, g, cap, bcount, bheavy, nbflag, tile_sum, bstart,
             nb_list, n_nb, recs, blockmap, n_blocks, inc ? inc->oblockmap : nullptr, inc ? inc->orecs : nullptr,
             inc ? inc->rold : nullptr,
             inc ? inc->dirty : nullptr);
}

// Slabs: the node-block list again after the halo unpack flagged the blocks reached
// only by ghost tiles -- the same two-pass tile scan as the list pass above, over the
// flags alone: per-tile sums, then every tile adds its predecessors' sums and writes
// its part of the id-ordered list (deterministic, no atomics, no library scan).
__global__ void __launch_bounds__(kListThreads) k_flag_sums(const int* __restrict__ flags, int n, int* tile_sum) {
    using Red = cub::BlockReduce<int, kListThreads>;
    __shared__ typename Red::TempStorage tmp;
    const int b = blockIdx.x * kListThreads + threadIdx.x;
    const int t = Red(tmp).Sum(b < n ? (flags[b] != 0) : 0);
    if (threadIdx.x == 0) tile_sum[blockIdx.x] = t;
}

__global__ void __launch_bounds__(kListThreads) k_flag_write(const int* __restrict__ flags, int n,
                                                             const int* __restrict__ tile_sum, int* list,
                                                             int* n_list) {
    using Scan = cub::BlockScan<int, kListThreads>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ int base;
    const int tid = threadIdx.x;
    if (tid < 32) {
        int s = 0;
        for (int t = tid; t < int(blockIdx.x); t += 32) s += tile_sum[t];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
        if (tid == 0) base = s;
    }
    const int b = blockIdx.x * kListThreads + tid;
    const int f = b < n ? (flags[b] != 0) : 0;
    int pre, tot;
    Scan(tmp).ExclusiveSum(f, pre, tot);
    __syncthreads();
    if (f) list[base + pre] = b;
    if (blockIdx.x == gridDim.x - 1 && tid == 0) *n_list = base + tot;
}

void launch_flag_list(const int* flags, int n, int* list, int* n_list, int* tile_sum, cudaStream_t s) {
    const int tiles = (n + kListThreads - 1) / kListThreads;
    k_flag_sums<<<tiles, kListThreads, 0, s>>>(flags, n, tile_sum);
    k_flag_write<<<tiles, kListThreads, 0, s>>>(flags, n, tile_sum, list, n_list);
}
int flag_list_tiles(int n) { return (n + kListThreads - 1) / kListThreads; }

void launch_sort_blocks(const Geom& g, const int* bcount, const int* bstart, const BlockRec* recs,
                        int* n_blocks, int cap, const uint32_t* skey, const uint32_t* sslot, uint32_t* perm,
                        uint16_t* celltab, uint32_t* gk, uint32_t* gv, uint32_t* okey, int grid, cudaStream_t s) {
    launch_k(k_sort_blocks, dim3(grid), dim3(kSortThreads), 0, s, g, bcount, bstart, recs, n_blocks, cap, skey, sslot,
             perm, celltab, gk, gv, okey);
}
}  // namespace fl
