// fl_scatter.cuh -- block-local deterministic scatter and tile gather helpers.
//
// A particle's contribution to node base+o (o in {0,1,2}^3) is
//     w_o(fx) * (m, a + Bm o)                       (P2G, NCH = 4)
//     w_o(fx) * (a + Bm o)                          (G2P adjoint, NCH = 3)
// because rel = node*dx - x = dx (o - fx) (mpm.hpp:281).  Each CTA stages the
// per-particle payload (fx, [m], a, Bm) for its particle block in shared
// memory; thread (cell c, plane ox) then sums the 9 nodes of plane ox over the
// particles of base cell c in sorted order, and the cell partials are folded
// into the 6^3 node tile in a fixed order.  No atomics anywhere.
#pragma once

#include "fl_layout.cuh"

namespace fl {

// threads per scatter CTA: 64 cells x 3 planes accumulate; more threads (FL_SC_THREADS =
// 256) only widen the payload phase (the extra ones idle in the accumulate phase)
#ifndef FL_SC_THREADS
#define FL_SC_THREADS 192
#endif
constexpr int kScThreads = FL_SC_THREADS;
static_assert(kScThreads >= 192 && kScThreads % 64 == 0, "scatter CTA: 64 cells x 3 planes at least");

// resident CTAs per SM requested from ptxas for the plain-liquid variants (register caps)
#ifndef FL_LB_P2G
#define FL_LB_P2G 5
#endif
#ifndef FL_LB_G2P
#define FL_LB_G2P 7  // (8 capped it at 64 registers with spills; round-2 end: G2P 42.5 -> 40.6 us on c4)
#endif
#ifndef FL_LB_ADJG2P
#define FL_LB_ADJG2P 4  // (256-thread CTAs: 64 registers)
#endif
#ifndef FL_LB_ADJP2G
#define FL_LB_ADJP2G 5
#endif
// ... and for the SVD / rigid ("heavy") variants (re-swept after the heavy-first pairs:
// c5 -0.7%, c3 -1.7%, c2 -0.8%)
#ifndef FL_LBH_P2G
#define FL_LBH_P2G 2
#endif
#ifndef FL_LBH_G2P
#define FL_LBH_G2P 5
#endif
#ifndef FL_LBH_ADJG2P
#define FL_LBH_ADJG2P 2
#endif
#ifndef FL_LBH_ADJP2G
#define FL_LBH_ADJP2G 4
#endif
// ... and for a few SVD/rigid blocks (fewer than the SMs) beside a liquid scene (variant 3):
// 256-thread CTAs for the thread-per-particle kernels, 128 registers
#ifndef FL_LBF_G2P
#define FL_LBF_G2P 2
#endif
#ifndef FL_LBF_ADJP2G
#define FL_LBF_ADJP2G 2
#endif
// ... and for the heavy variants when SVD/rigid blocks dominate the scene (launcher variant 2)
#ifndef FL_LBD_P2G
#define FL_LBD_P2G 5
#endif
#ifndef FL_LBD_G2P
#define FL_LBD_G2P 5
#endif
#ifndef FL_LBD_ADJG2P
#define FL_LBD_ADJG2P 3  // (256-thread CTAs)
#endif
#ifndef FL_LBD_ADJP2G
#define FL_LBD_ADJP2G 4
#endif
#ifndef FL_SCR
#define FL_SCR 8
#endif
constexpr int kScR = FL_SCR;     // particle ranks per cell staged per pass (8 = ppc 2^3)
constexpr int kCS = 68;          // rank stride = 4 (mod 32): conflict-free for 8 ranks x 4 cells and 32 cells
constexpr int kPayF = 16;        // payload floats per particle
constexpr int kCellTab = 66;     // per block: 64 cell starts, end, largest cell count (u16)

// Payload staged as pay[f][rank][cell]: the payload phase (lanes = consecutive
// particles of a cell, consecutive ranks) and the accumulate phase (lanes =
// consecutive cells, same rank) both hit distinct banks.  The 6^3 node tile is
// kept as four channel planes; each pass adds the gathered (cell, plane)
// partials of every node in a fixed order (sc_accumulate).
struct alignas(16) ScSmem {
    float pay[kPayF * kScR * kCS];
    float tile[4 * kTile];
    uint16_t cs[kCellTab];
    uint16_t opre[66];  // passes after the first: prefix of the particles each cell still has
};

__device__ __forceinline__ float* pay_slot(ScSmem& sm, int rank, int cell) { return &sm.pay[rank * kCS + cell]; }
constexpr int kPayPlane = kScR * kCS;  // floats between payload fields

// Dynamic block scheduling: a CTA grabs the next list slot from a work counter
// (results do not depend on which CTA processes which block).  Claiming a slot
// one block ahead was measured slower: with a few blocks per CTA the tail
// imbalance it adds outweighs the hidden atomic latency.
__device__ __forceinline__ int next_work(int* counter, int* sh) {
    __syncthreads();
    if (threadIdx.x == 0) *sh = atomicAdd(counter, 1);
    __syncthreads();
    return *sh;
}

// Work order of the persistent block-list kernels: costliest blocks first (longest-processing-
// time first), so a kernel's tail is made of short blocks.  The per-block sort files every
// listed block under (kind, cost class); the record's n_blocks array holds
//   [0] light blocks, [1] SVD/rigid blocks, [4 + kind * 4 + class] blocks per class,
//   from int 16 on, int4 entries [(kind * 4 + class) * maxb + i] = {list slot, block, start,
//   end} (any order inside a class): a kernel gets its next block in one load.
// Class 0: cells over kScR particles (a second staging pass); 1: >= 384 particles; 2: >= 192;
// 3: the rest.  Which CTA takes which block does not change any result.
constexpr int kWorkClasses = 4;
__host__ __device__ constexpr int work_order_ints(int maxb) { return 16 + 4 * 2 * kWorkClasses * maxb; }
__device__ __forceinline__ int work_class(int cnt, int maxcell) {
    return maxcell > FL_SCR ? 0 : (cnt >= 384 ? 1 : (cnt >= 192 ? 2 : 3));
}
__device__ __forceinline__ void work_file(int* nb, int maxb, int kind, int q, const BlockRec& r, int maxcell) {
    const int c = kind * kWorkClasses + work_class(r.end - r.start, maxcell);
    reinterpret_cast<int4*>(nb + 16)[size_t(c) * maxb + atomicAdd(&nb[4 + c], 1)] =
        make_int4(q, r.block, r.start, r.end);
}
// the k-th block of `kind` in work order (k < that kind's block count); wc: the kind's
// class counts (shared memory)
__device__ __forceinline__ int4 work_entry(const int* __restrict__ nb, int maxb, int kind, int k, const int* wc) {
    int i = 0;
#pragma unroll
    for (; i < kWorkClasses - 1; i++) {
        if (k < wc[i]) break;
        k -= wc[i];
    }
    return reinterpret_cast<const int4*>(nb + 16)[size_t(kind * kWorkClasses + i) * maxb + k];
}
// every CTA of a persistent block-list kernel: its kind's class counts into shared memory
// (visible after the first next_work barrier)
__device__ __forceinline__ void work_counts_load(const int* __restrict__ nb, int kind, int* wc, int tid) {
    if (tid < kWorkClasses) wc[tid] = nb[4 + kind * kWorkClasses + tid];
}

// local cell (0..63) of the i-th particle of a block from its cell-start table
// (largest c with cs[c] <= i; empty cells have cs[c] == cs[c+1])
__device__ __forceinline__ int cell_of(const uint16_t* cs, int i) {
    int lo = 0;
#pragma unroll
    for (int step = 32; step > 0; step >>= 1)
        if (int(cs[lo + step]) <= i) lo += step;
    return lo;
}

__device__ __forceinline__ void sc_tile_zero(ScSmem& sm, int tid, int nthreads) {
    for (int i = tid; i < 4 * int(kTile); i += nthreads) sm.tile[i] = 0.f;
}

// Thread (cell c, plane ox) sums the 9 nodes (ox, oy, oz) over the particles of
// cell c staged in this pass, in rank (= particle id) order; the partial sums
// are then folded into the tile by sc_fold: they go to shared memory (reusing
// the payload area) and every tile node gathers its <= 27 (cell, plane)
// contributions in a fixed order.  Must be reached by all threads.
// payload fields: [0..2] fx, then (NCH==4 ? m : -), a[3], Bm[9] row-major
template <int NCH>
__device__ __forceinline__ void sc_accumulate(ScSmem& sm, int c, int ox, int nrank, int tid, int nthreads) {
    constexpr int A0 = (NCH == 4) ? 4 : 3;
    float acc[9][4];
#pragma unroll
    for (int k = 0; k < 9; k++)
#pragma unroll
        for (int q = 0; q < 4; q++) acc[k][q] = 0.f;
    const float oxf = float(ox);
    for (int r = 0; r < nrank; r++) {
        const float* p = &sm.pay[r * kCS + c];
#define PF(f) p[(f) * kPayPlane]
        float wy[3], wz[3];
        bspline_w(PF(1), wy);
        bspline_w(PF(2), wz);
        // only this thread's x weight (same operations as bspline_w)
        const float fx0 = PF(0);
        const float tx = ox == 0 ? 1.5f - fx0 : (ox == 1 ? fx0 - 1.0f : fx0 - 0.5f);
        const float wx = ox == 1 ? 0.75f - tx * tx : 0.5f * tx * tx;
        const float m = (NCH == 4) ? PF(3) : 0.f;
        const float b00 = PF(A0 + 3), b01 = PF(A0 + 4), b02 = PF(A0 + 5);
        const float b10 = PF(A0 + 6), b11 = PF(A0 + 7), b12 = PF(A0 + 8);
        const float b20 = PF(A0 + 9), b21 = PF(A0 + 10), b22 = PF(A0 + 11);
        const float a0x = PF(A0) + b00 * oxf, a0y = PF(A0 + 1) + b10 * oxf, a0z = PF(A0 + 2) + b20 * oxf;
#undef PF
        // a + B o with o in {0,1,2} written out (b*0, b*1, b*2 are exact, so the sums are
        // the same as a + b*o; IEEE rules keep the compiler from dropping the multiplies)
#define FL_STEP(base, d, k) ((k) == 0 ? (base) : ((k) == 1 ? (base) + (d) : (base) + 2.f * (d)))
#pragma unroll
        for (int oy = 0; oy < 3; oy++) {
            const float ayx = FL_STEP(a0x, b01, oy), ayy = FL_STEP(a0y, b11, oy), ayz = FL_STEP(a0z, b21, oy);
            const float wxy = wx * wy[oy];
#pragma unroll
            for (int oz = 0; oz < 3; oz++) {
                const float w = wxy * wz[oz];
                const float vx = FL_STEP(ayx, b02, oz), vy = FL_STEP(ayy, b12, oz), vz = FL_STEP(ayz, b22, oz);
                float* ac = acc[oy * 3 + oz];
                if (NCH == 4) {
                    ac[0] += w * m;
                    ac[1] += w * vx;
                    ac[2] += w * vy;
                    ac[3] += w * vz;
                } else {
                    ac[0] += w * vx;
                    ac[1] += w * vy;
                    ac[2] += w * vz;
                }
            }
        }
    }
#undef FL_STEP
    // fold: partial sums -> shared memory -> per-node fixed-order gather
    float4* part = reinterpret_cast<float4*>(sm.pay);  // [64 cells][3 planes][9 nodes]
    __syncthreads();                                   // the payload has been read
    if (ox < 3)
#pragma unroll
        for (int k = 0; k < 9; k++) part[(c * 3 + ox) * 9 + k] = make_float4(acc[k][0], acc[k][1], acc[k][2], acc[k][3]);
    __syncthreads();
    for (int t = tid; t < int(kTile); t += nthreads) {
        const int X = t / 36, Y = (t / 6) % 6, Z = t % 6;
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int px = 0; px < 3; px++) {
            const int cx = X - px;
            if (cx < 0 || cx > 3) continue;
#pragma unroll
            for (int py = 0; py < 3; py++) {
                const int cy = Y - py;
                if (cy < 0 || cy > 3) continue;
#pragma unroll
                for (int pz = 0; pz < 3; pz++) {
                    const int cz = Z - pz;
                    if (cz < 0 || cz > 3) continue;
                    const float4 v = part[(((cx << 4) | (cy << 2) | cz) * 3 + px) * 9 + py * 3 + pz];
                    s.x += v.x;
                    s.y += v.y;
                    s.z += v.z;
                    s.w += v.w;
                }
            }
        }
        sm.tile[t] += s.x;
        sm.tile[kTile + t] += s.y;
        sm.tile[2 * kTile + t] += s.z;
        sm.tile[3 * kTile + t] += s.w;
    }
}

// A pass stages the particles of rank [r0, r0 + kScR) in their cell (after the first
// pass, a few per block): list them densely (prefix over the cells of min(count - r0, kScR)) so whole warps
// work on them instead of walking every particle with most lanes idle.  Returns the item
// count; all threads.
__device__ __forceinline__ int sc_overflow_prefix(ScSmem& sm, int r0, int tid) {
    if (tid < 32) {
        const int o0 = min(max(int(sm.cs[2 * tid + 1]) - int(sm.cs[2 * tid]) - r0, 0), kScR);
        const int o1 = min(max(int(sm.cs[2 * tid + 2]) - int(sm.cs[2 * tid + 1]) - r0, 0), kScR);
        const int s = o0 + o1;
        int incl = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (tid >= o) incl += t;
        }
        sm.opre[2 * tid] = uint16_t(incl - s);
        sm.opre[2 * tid + 1] = uint16_t(incl - s + o0);
        if (tid == 31) sm.opre[64] = uint16_t(incl);
    }
    __syncthreads();
    return int(sm.opre[64]);
}

// item -> (cell, rank within the pass) of the dense list above
__device__ __forceinline__ void sc_overflow_item(const ScSmem& sm, int item, int& c, int& rank) {
    int lo = 0;
#pragma unroll
    for (int step = 32; step > 0; step >>= 1)
        if (lo + step < 64 && int(sm.opre[lo + step]) <= item) lo += step;
    // skip cells with nothing left (equal prefixes): the item belongs to the last of them
    c = lo;
    rank = item - int(sm.opre[lo]);
}

// load the block's cell table (64 cell starts, end, largest cell count); returns
// the pass count ceil(max cell count / kScR)
__device__ __forceinline__ int sc_load_cells(ScSmem& sm, const uint16_t* __restrict__ celltab, int slot, int tid) {
    if (tid < kCellTab) sm.cs[tid] = celltab[size_t(slot) * kCellTab + tid];
    __syncthreads();
    return (int(sm.cs[65]) + kScR - 1) / kScR;
}

__device__ __forceinline__ void sc_tile_store(const ScSmem& sm, float4* out, int tid, int nthreads) {
    for (int t = tid; t < int(kTile); t += nthreads)
        out[t] = make_float4(sm.tile[t], sm.tile[kTile + t], sm.tile[2 * kTile + t], sm.tile[3 * kTile + t]);
}

// ---------------------------------------------------------------------------
// TMA-staged node tiles.  The 6^3 tile of particle block (bx,by,bz) lies in the
// 2x2x2 node blocks starting at (bx,by,bz); each node block is 64 contiguous
// float4 (1 KB) of the block-major grid, so one elected thread moves the eight
// of them with 1D bulk copies (cp.async.bulk, the TMA engine; SASS UBLKCP) into
// a raw [8][64] float4 buffer and arms an mbarrier with the byte count.  The
// other threads issue their particle loads meanwhile; after the wait every
// thread repacks its share of the tile into the dense 6^3 layout the gather
// loops index with immediate offsets.  Blocks past the grid edge are not
// copied; their tile nodes read as zero.
// ---------------------------------------------------------------------------
constexpr int kTileRaw = 8 * 64;  // float4 per raw tile buffer

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return uint32_t(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
    }
}

// valid-block mask of the tile (bit d = (dx<<2)|(dy<<1)|dz)
__device__ __forceinline__ uint32_t tile_valid(const Geom& g, int bx, int by, int bz) {
    uint32_t m = 0;
#pragma unroll
    for (int d = 0; d < 8; d++)
        if (bx + (d >> 2) < g.NB[0] && by + ((d >> 1) & 1) < g.NB[1] && bz + (d & 1) < g.NB[2]) m |= 1u << d;
    return m;
}

#ifndef FL_TMA_TILE
#define FL_TMA_TILE 1
#endif
#ifndef FL_TMA_LANES
#define FL_TMA_LANES 8
#endif

// warp 0 (after a CTA barrier that ended every generic access of `raw`): lane 0 arms the
// barrier with the byte count, then lanes 0..7 each issue one node block's bulk copy
__device__ __forceinline__ void tile_tma_issue(const Geom& g, const float4* __restrict__ grid, float4* raw,
                                               uint64_t* bar, int bx, int by, int bz, uint32_t valid, int lane) {
    if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                     "r"(uint32_t(__popc(valid)) * 1024u)
                     : "memory");
    }
    __syncwarp();
#pragma unroll
    for (int d0 = 0; d0 < 8; d0 += FL_TMA_LANES) {
        const int d = d0 + lane;
        if (lane < FL_TMA_LANES && (valid >> d & 1u)) {
            const float4* src = grid + size_t(block_lin(g, bx + (d >> 2), by + ((d >> 1) & 1), bz + (d & 1))) * 64;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 1024, [%2];" ::"r"(
                    smem_u32(raw + d * 64)),
                "l"(src), "r"(smem_u32(bar))
                : "memory");
        }
    }
}

// every thread: wait for the bytes, then repack raw -> dense 6^3 tile (caller syncs after)
__device__ __forceinline__ void tile_tma_finish(const float4* raw, float4* tile, uint64_t* bar, uint32_t& phase,
                                                uint32_t valid, int tid, int nthreads) {
    mbar_wait(bar, phase);
    phase ^= 1u;
    for (int t = tid; t < int(kTile); t += nthreads) {
        const int X = t / 36, Y = (t / 6) % 6, Z = t % 6;
        const int d = ((X >> 2) << 2) | ((Y >> 2) << 1) | (Z >> 2);
        tile[t] = (valid >> d & 1u) ? raw[d * 64 + (((X & 3) << 4) | ((Y & 3) << 2) | (Z & 3))]
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

// 6^3 node tile of a block-major float4 grid into shared memory (plain loads; the
// FL_TMA_TILE = 0 variant, kept for A/B runs)
__device__ __forceinline__ void load_tile(const Geom& g, const float4* __restrict__ grid, float4* tile, int bx,
                                          int by, int bz, int tid, int nthreads) {
    for (int t = tid; t < int(kTile); t += nthreads) {
        const int tx = t / 36, ty = (t / 6) % 6, tz = t % 6;
        const int i = 4 * bx + tx, j = 4 * by + ty, k = 4 * bz + tz;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if ((i >> 2) < g.NB[0] && (j >> 2) < g.NB[1] && (k >> 2) < g.NB[2]) v = grid[node_index(g, i, j, k)];
        tile[t] = v;
    }
}

// Tile staging used by the gather kernels: tile_begin right after the work claim (its
// barriers ended the previous block's reads of `raw` and `tile`), tile_end before the
// first read of `tile` (followed by a CTA barrier).
struct TileStage {
    uint64_t* bar;
    float4* raw;
    uint32_t phase;
    uint32_t valid;
    __device__ __forceinline__ void init(uint64_t* b, float4* r, int tid) {
        bar = b;
        raw = r;
        phase = 0;
        if (FL_TMA_TILE && tid == 0) mbar_init(bar);
    }
    __device__ __forceinline__ void begin(const Geom& g, const float4* __restrict__ grid, int bx, int by, int bz,
                                          int tid) {
        if (FL_TMA_TILE) {
            valid = tile_valid(g, bx, by, bz);
            if (tid < 32) tile_tma_issue(g, grid, raw, bar, bx, by, bz, valid, tid);
        }
    }
    __device__ __forceinline__ void end(const Geom& g, const float4* __restrict__ grid, float4* tile, int bx, int by,
                                        int bz, int tid, int nthreads) {
        if (FL_TMA_TILE)
            tile_tma_finish(raw, tile, bar, phase, valid, tid, nthreads);
        else
            load_tile(g, grid, tile, bx, by, bz, tid, nthreads);
    }
};

struct StencilW {
    int l[3];        // base cell relative to the block origin, in [0,4)
    float fx[3];
    float w[3][3];
    float dw[3][3];  // d w / d fx
};

__device__ __forceinline__ void stencil_weights(const Geom& g, V3<float> x, int bx, int by, int bz, StencilW& s) {
    const int bo[3] = {4 * bx, 4 * by, 4 * bz};
#pragma unroll
    for (int a = 0; a < 3; a++) {
        int b = base_cell(x[a], g.inv_dx, s.fx[a]);
        int l = b - bo[a];
        s.l[a] = l < 0 ? 0 : (l > 3 ? 3 : l);
        bspline_w(s.fx[a], s.w[a]);
        bspline_dw(s.fx[a], s.dw[a]);
    }
}

// v = sum w gv, C = (4/dx^2) sum w gv rel^T with rel = dx (o - fx)  (mpm.hpp:352-361).
// Factored per axis around the middle node: with u = o - 1 in {-1,0,1} and
// f = fx - 1, sum_o w gv (o - fx)_a = M_a - v f_a where M_a = sum_o w gv u_a is
// built up z -> y -> x (~260 FMAs instead of ~430 for the 27-node product).
__device__ __forceinline__ void g2p_gather(const Geom& g, const float4* tile, const StencilW& s, V3<float>& v,
                                           M3<float>& c) {
    V3<float> mx = {0.f, 0.f, 0.f}, my = mx, mz = mx;
    v = mx;
#pragma unroll
    for (int ox = 0; ox < 3; ox++) {
        V3<float> bv = {0.f, 0.f, 0.f}, by = bv, bz = bv;
#pragma unroll
        for (int oy = 0; oy < 3; oy++) {
            const float4* row = tile + (s.l[0] + ox) * 36 + (s.l[1] + oy) * 6 + s.l[2];
            const float4 g0 = row[0], g1 = row[1], g2 = row[2];
            const V3<float> a = {s.w[2][0] * g0.x + s.w[2][1] * g1.x + s.w[2][2] * g2.x,
                                 s.w[2][0] * g0.y + s.w[2][1] * g1.y + s.w[2][2] * g2.y,
                                 s.w[2][0] * g0.z + s.w[2][1] * g1.z + s.w[2][2] * g2.z};
            const V3<float> az = {s.w[2][2] * g2.x - s.w[2][0] * g0.x, s.w[2][2] * g2.y - s.w[2][0] * g0.y,
                                  s.w[2][2] * g2.z - s.w[2][0] * g0.z};
            const float wy = s.w[1][oy];
            bv += a * wy;
            if (oy != 1) by += a * (oy == 0 ? -wy : wy);
            bz += az * wy;
        }
        const float wx = s.w[0][ox];
        v += bv * wx;
        if (ox != 1) mx += bv * (ox == 0 ? -wx : wx);
        my += by * wx;
        mz += bz * wx;
    }
    const float kd = g.k4 * g.dx;
    const float f0 = s.fx[0] - 1.f, f1 = s.fx[1] - 1.f, f2 = s.fx[2] - 1.f;
    c.m[0] = (mx.x - v.x * f0) * kd; c.m[1] = (my.x - v.x * f1) * kd; c.m[2] = (mz.x - v.x * f2) * kd;
    c.m[3] = (mx.y - v.y * f0) * kd; c.m[4] = (my.y - v.y * f1) * kd; c.m[5] = (mz.y - v.y * f2) * kd;
    c.m[6] = (mx.z - v.z * f0) * kd; c.m[7] = (my.z - v.z * f1) * kd; c.m[8] = (mz.z - v.z * f2) * kd;
}

// wall band (mpm.hpp:290-299): zero the inward component near each face
__device__ __forceinline__ V3<float> wall_bc_dev(const Geom& g, int i, int j, int k, V3<float> v) {
    const int n[3] = {i, j, k};
#pragma unroll
    for (int a = 0; a < 3; a++) {
        if (n[a] <= g.bw && v[a] < 0.f) v[a] = 0.f;
        if (n[a] >= g.nd[a] - 1 - g.bw && v[a] > 0.f) v[a] = 0.f;
    }
    return v;
}

}  // namespace fl
