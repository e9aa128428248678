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
// packed (24 floats + class, id, key) and appended to the neighbour's state;
// their old slots are marked departed and dropped by the next sort.  The
// backward returns the cotangents of those particles along the same path.
#include <cuda_runtime.h>

#include "fl_kernels.h"
#include "fl_scatter.cuh"

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
// particle migration
// ---------------------------------------------------------------------------
constexpr int kMigW = 27;  // words per migrating particle: 24 floats, class, id, key

__global__ void k_mig_pack(Geom g, PBuf out, int n, uint32_t* send0, uint32_t* send1, uint32_t* src, int* cnt,
                           int cap) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const uint32_t key = out.key[j];
    if (key >= g.key_inactive) return;
    const int col = key_col(g, key);
    const int d = col < g.sx0 ? 0 : (col >= g.sx1 ? 1 : -1);
    if (d < 0) return;
    const int k = atomicAdd(&cnt[d], 1);
    out.key[j] = g.key_departed;
    if (k >= cap) return;  // overflow: the host sees cnt > cap and raises
    uint32_t* w = (d == 0 ? send0 : send1) + size_t(k) * kMigW;
    for (int c = 0; c < 24; c++) w[c] = __float_as_uint(out.f[size_t(c) * out.cap + j]);
    w[24] = out.meta[j];
    w[25] = out.id[j];
    w[26] = key;
    src[size_t(d) * cap + k] = uint32_t(j);
}

__global__ void k_mig_unpack(PBuf out, const uint32_t* __restrict__ in, int n, int pos0) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const uint32_t* w = in + size_t(k) * kMigW;
    const int j = pos0 + k;
    for (int c = 0; c < 24; c++) out.f[size_t(c) * out.cap + j] = __uint_as_float(w[c]);
    out.meta[j] = w[24];
    out.id[j] = w[25];
    out.key[j] = w[26];
}

size_t mig_bytes(int n) { return size_t(n) * kMigW * sizeof(uint32_t); }

void launch_mig_pack(const Geom& g, PBuf out, int n, void* send0, void* send1, uint32_t* src, int* cnt, int cap,
                     cudaStream_t s) {
    if (n <= 0) return;
    k_mig_pack<<<(n + 255) / 256, 256, 0, s>>>(g, out, n, static_cast<uint32_t*>(send0),
                                               static_cast<uint32_t*>(send1), src, cnt, cap);
}

void launch_mig_unpack(PBuf out, const void* in, int n, int pos0, cudaStream_t s) {
    if (n <= 0) return;
    k_mig_unpack<<<(n + 255) / 256, 256, 0, s>>>(out, static_cast<const uint32_t*>(in), n, pos0);
}

// cotangents of arrived particles travel back to the slab they came from
__global__ void k_bars_pack(BarBuf bars, int pos0, int n, float* out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    for (int c = 0; c < 24; c++) out[size_t(k) * 24 + c] = bars.f[size_t(c) * bars.cap + pos0 + k];
}

__global__ void k_bars_scatter(BarBuf bars, const float* __restrict__ in, const uint32_t* __restrict__ src, int n) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const size_t j = src[k];
    for (int c = 0; c < 24; c++) bars.f[size_t(c) * bars.cap + j] = in[size_t(k) * 24 + c];
}

void launch_bars_pack(BarBuf bars, int pos0, int n, void* out, cudaStream_t s) {
    if (n <= 0) return;
    k_bars_pack<<<(n + 255) / 256, 256, 0, s>>>(bars, pos0, n, static_cast<float*>(out));
}

void launch_bars_scatter(BarBuf bars, const void* in, const uint32_t* src, int n, cudaStream_t s) {
    if (n <= 0) return;
    k_bars_scatter<<<(n + 255) / 256, 256, 0, s>>>(bars, static_cast<const float*>(in), src, n);
}

}  // namespace fl
