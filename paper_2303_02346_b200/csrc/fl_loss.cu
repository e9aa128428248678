// fl_loss.cu -- point-set losses at segment boundaries on the device
// (losses.hpp:15-100, 474-551):
//   trajectory_chamfer   symmetric mean nearest-neighbour distance between the
//                        body's active particles A and the segment's goal set G in
//                        fp64 with exact first-index argmins: a brute-force scan for
//                        small |A| |G|, uniform-grid indexes (shell search) above
//                        2^24 pairs -- both paths give identical bits
//   mixing_spread        -sum_ij |x_i - x_j| over the body, O(|A|^2) in fp64
//   attraction           the optimizer's gradient-sharing surrogate (losses.hpp:104-218):
//                        hashed-grid neighbour sums over every member of one body
// Both first compact the body's active particles in store order (deterministic
// prefix sum), so every sum below has a fixed order.  The evaluation adds
// weight * value into the segment's loss slot; the gradient adds into x_bar
// with the reference's per-particle accumulation order (A-term, then G-terms
// in goal order).
#include <cuda_runtime.h>

#include <algorithm>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "fl_kernels.h"

namespace fl {

constexpr int kLT = 256;      // threads per CTA
constexpr int kTileP = 256;   // points staged per shared-memory tile

// ---------------------------------------------------------------------------
// body compaction
// ---------------------------------------------------------------------------
__global__ void k_body_flags(PBuf st, int n, const ClassInfo* __restrict__ cls, int body, uint32_t key_inactive,
                             const int* __restrict__ act, long substep, int* flags) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t key = st.key[i];
    const bool active = key < key_inactive || (key == key_inactive && act[st.id[i]] <= substep);  // (one rank)
    flags[i] = (active && cls[meta_cls(st.meta[i])].body == body) ? 1 : 0;
}

__global__ void k_body_gather(PBuf st, int n, const int* __restrict__ flags, const int* __restrict__ pos,
                              LossSet ls, int* idx, double* px, int* count) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (i == n - 1) *count = pos[i] + flags[i];
    if (!flags[i]) return;
    const int k = pos[i];
    idx[k] = i;
    for (int a = 0; a < 3; a++) px[3 * size_t(k) + a] = double(loss_x(ls, st, i, st.id[i], a));
}

// ---------------------------------------------------------------------------
// trajectory_chamfer
// ---------------------------------------------------------------------------
// squared distance with a fixed rounding sequence (both nearest-neighbour paths use it)
__device__ __forceinline__ double nn_d2(double ex, double ey, double ez) {
    return __fma_rn(ez, ez, __fma_rn(ey, ey, __dmul_rn(ex, ex)));
}

// A -> G: nearest goal of every member (first index on ties, like the reference's strict <)
__global__ void __launch_bounds__(kLT) k_chamfer_a(const double* __restrict__ px, const int* __restrict__ count,
                                                   const double* __restrict__ g, int ng, double* best, int* arg,
                                                   double* partial) {
    __shared__ double gs[3 * kTileP];
    __shared__ double red[kLT];
    const int na = *count;
    const int k = blockIdx.x * kLT + threadIdx.x;
    const bool in = k < na;
    double p[3] = {0, 0, 0};
    if (in)
        for (int a = 0; a < 3; a++) p[a] = px[3 * size_t(k) + a];
    double bd = 1e300;
    int bi = 0;
    for (int t0 = 0; t0 < ng; t0 += kTileP) {
        const int m = min(kTileP, ng - t0);
        __syncthreads();
        for (int q = threadIdx.x; q < 3 * m; q += kLT) gs[q] = g[3 * size_t(t0) + q];
        __syncthreads();
        if (in)
            for (int j = 0; j < m; j++) {
                const double d2 = nn_d2(p[0] - gs[3 * j], p[1] - gs[3 * j + 1], p[2] - gs[3 * j + 2]);
                if (d2 < bd) {
                    bd = d2;
                    bi = t0 + j;
                }
            }
    }
    const double d = in ? sqrt(bd) : 0.0;
    if (in) {
        best[k] = d;
        arg[k] = bi;
    }
    red[threadIdx.x] = d;
    __syncthreads();
    for (int w = kLT / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

// G -> A, stage 1: per (member chunk, goal) nearest member within the chunk
__global__ void __launch_bounds__(kLT) k_chamfer_g(const double* __restrict__ px, const int* __restrict__ count,
                                                   int chunk, const double* __restrict__ g, int ng, double* cbest,
                                                   int* carg) {
    __shared__ double ps[3 * kTileP];
    const int na = *count;
    const int c0 = blockIdx.x * chunk, c1 = min(na, c0 + chunk);
    for (int gq0 = 0; gq0 < ng; gq0 += kLT) {
        const int gq = gq0 + threadIdx.x;
        double q[3] = {0, 0, 0};
        if (gq < ng)
            for (int a = 0; a < 3; a++) q[a] = g[3 * size_t(gq) + a];
        double bd = 1e300;
        int bi = -1;
        for (int t0 = c0; t0 < c1; t0 += kTileP) {
            const int m = min(kTileP, c1 - t0);
            __syncthreads();
            for (int r = threadIdx.x; r < 3 * m; r += kLT) ps[r] = px[3 * size_t(t0) + r];
            __syncthreads();
            if (gq < ng)
                for (int j = 0; j < m; j++) {
                    const double d2 = nn_d2(q[0] - ps[3 * j], q[1] - ps[3 * j + 1], q[2] - ps[3 * j + 2]);
                    if (d2 < bd) {
                        bd = d2;
                        bi = t0 + j;
                    }
                }
        }
        if (gq < ng) {
            cbest[size_t(blockIdx.x) * ng + gq] = bd;
            carg[size_t(blockIdx.x) * ng + gq] = bi;
        }
    }
}

// G -> A, stage 2 (one CTA): chunks in order per goal, then the loss value:
// weight * (sum_a best_a / |A| + sum_g best_g / |G|) added to *out.  scal[0] = |A|.
__global__ void __launch_bounds__(kLT) k_chamfer_final(const int* __restrict__ count, int nchunks, int ng,
                                                       const double* __restrict__ cbest, const int* __restrict__ carg,
                                                       const double* __restrict__ partial, int npartial,
                                                       double weight, double* gbest, int* garg, double* out,
                                                       double* scal, unsigned long long* err) {
    __shared__ double red[kLT];
    const int na = *count;
    if (na == 0) {  // chamfer_distance: empty point set (losses.hpp:17)
        if (threadIdx.x == 0) atomicMin(err, (unsigned long long)pack_err(0xfffffu, ES_LOSS_EMPTY, 0));
        return;
    }
    double sg = 0.0;
    for (int gq = threadIdx.x; gq < ng; gq += kLT) {
        if (nchunks == 0) {  // grid path: gbest / garg are final already
            sg += gbest[gq];
            continue;
        }
        double bd = 1e300;
        int bi = 0;
        for (int c = 0; c < nchunks; c++) {
            const double d = cbest[size_t(c) * ng + gq];
            if (d < bd) {
                bd = d;
                bi = carg[size_t(c) * ng + gq];
            }
        }
        const double d = sqrt(bd);
        gbest[gq] = d;
        garg[gq] = bi;
        sg += d;
    }
    red[threadIdx.x] = sg;
    __syncthreads();
    for (int w = kLT / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    const double sumg = red[0];
    __syncthreads();
    double sa = 0.0;
    for (int b = threadIdx.x; b < npartial; b += kLT) sa += partial[b];
    red[threadIdx.x] = sa;
    __syncthreads();
    for (int w = kLT / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *out += weight * (red[0] / double(na) + sumg / double(ng));
        scal[0] = double(na);
    }
}

// gradient (losses.hpp:35-63): A-term per member, then G-terms in goal order
__global__ void k_chamfer_grad_a(const double* __restrict__ px, const int* __restrict__ idx,
                                 const int* __restrict__ count, const double* __restrict__ g,
                                 const double* __restrict__ best, const int* __restrict__ arg, double weight,
                                 BarBuf bars) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int na = *count;
    if (k >= na) return;
    const double b = best[k];
    if (!(b > 1e-300)) return;
    const double s = weight / (b * double(na));
    const int j = arg[k], i = idx[k];
    for (int a = 0; a < 3; a++) bars.x(a)[i] += float((px[3 * size_t(k) + a] - g[3 * size_t(j) + a]) * s);
}

__global__ void k_chamfer_grad_g(const double* __restrict__ px, const int* __restrict__ idx,
                                 const double* __restrict__ g, int ng, const double* __restrict__ gbest,
                                 const int* __restrict__ garg, double weight, BarBuf bars) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int q = 0; q < ng; q++) {  // sequential: several goals may share a nearest member
        const double b = gbest[q];
        if (!(b > 1e-300)) continue;
        const double s = weight / (b * double(ng));
        const int k = garg[q], i = idx[k];
        for (int a = 0; a < 3; a++) bars.x(a)[i] += float((px[3 * size_t(k) + a] - g[3 * size_t(q) + a]) * s);
    }
}

// ---------------------------------------------------------------------------
// trajectory_chamfer at scale: exact nearest neighbours through a uniform grid
// ---------------------------------------------------------------------------
// For |A| |G| beyond kChamferBrutePairs the two nearest-neighbour passes query a
// uniform-grid index of the target set instead of scanning it: cells of size h over
// the target bounding box (~1 target per cell, <= 128 per axis), targets sorted by
// (cell, index).  A query visits Chebyshev shells r = 0, 1, ... around its (clamped)
// cell; every target in shells > r is at least r h away, so after shell r the search
// stops once the best squared distance is < (r h)^2.  Candidates are compared on
// (d^2, index): the result is the first-index minimum, exactly what the brute-force
// scan returns (losses.hpp:20-23, 38-45), so both paths give identical bits.
constexpr int kNnMaxDim = 128;

// bounding box partials: [block][lo0 lo1 lo2 hi0 hi1 hi2]
__global__ void __launch_bounds__(kLT) k_nn_bbox(const double* __restrict__ pts, int n_static,
                                                 const int* __restrict__ n_dev, double* partial) {
    __shared__ double red[6][kLT];
    const int n = n_dev ? *n_dev : n_static;
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int i = blockIdx.x * kLT + threadIdx.x; i < n; i += gridDim.x * kLT)
        for (int a = 0; a < 3; a++) {
            const double v = pts[3 * size_t(i) + a];
            lo[a] = fmin(lo[a], v);
            hi[a] = fmax(hi[a], v);
        }
    for (int a = 0; a < 3; a++) {
        red[a][threadIdx.x] = lo[a];
        red[3 + a][threadIdx.x] = hi[a];
    }
    __syncthreads();
    for (int w = kLT / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w)
            for (int a = 0; a < 3; a++) {
                red[a][threadIdx.x] = fmin(red[a][threadIdx.x], red[a][threadIdx.x + w]);
                red[3 + a][threadIdx.x] = fmax(red[3 + a][threadIdx.x], red[3 + a][threadIdx.x + w]);
            }
        __syncthreads();
    }
    if (threadIdx.x < 6) partial[6 * blockIdx.x + threadIdx.x] = red[threadIdx.x][0];
}

// one thread: the grid of the index (idx[0..2] lo, idx[3] h, idx[4..6] dims as doubles)
__global__ void k_nn_setup(const double* __restrict__ partial, int nblocks, int n_static, const int* __restrict__ n_dev,
                           double* idx) {
    const int n = n_dev ? *n_dev : n_static;
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int b = 0; b < nblocks; b++)
        for (int a = 0; a < 3; a++) {
            lo[a] = fmin(lo[a], partial[6 * b + a]);
            hi[a] = fmax(hi[a], partial[6 * b + 3 + a]);
        }
    double ext[3], emax = 0.0;
    for (int a = 0; a < 3; a++) {
        ext[a] = n > 0 ? hi[a] - lo[a] : 0.0;
        emax = fmax(emax, ext[a]);
    }
    // ~1 target per cell over the box (flat axes count as one cell), <= kNnMaxDim per axis
    double vol = 1.0;
    int nflat = 0;
    for (int a = 0; a < 3; a++) {
        if (ext[a] > 1e-12 * (emax + 1e-300)) vol *= ext[a];
        else nflat++;
    }
    double h = emax > 0.0 ? (nflat == 3 ? emax : pow(vol / double(max(n, 1)), 1.0 / double(3 - nflat))) : 1.0;
    h = fmax(h, emax / double(kNnMaxDim - 1));
    if (!(h > 0.0)) h = 1.0;
    for (int a = 0; a < 3; a++) {
        idx[a] = n > 0 ? lo[a] : 0.0;
        idx[4 + a] = double(min(kNnMaxDim, int(floor(ext[a] / h)) + 1));
    }
    idx[3] = h;
}

__device__ __forceinline__ int nn_cell_axis(const double* idx, int a, double x) {
    const int d = int(idx[4 + a]);
    const double f = floor((x - idx[a]) / idx[3]);
    return f < 0.0 ? 0 : (f >= double(d) ? d - 1 : int(f));
}

__global__ void k_nn_keys(const double* __restrict__ pts, int n_static, const int* __restrict__ n_dev,
                          const double* __restrict__ idx, unsigned long long* keys, int n_cap) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int n = n_dev ? *n_dev : n_static;
    if (i >= n_cap) return;
    if (i >= n) {  // past the live count: sorts last
        keys[i] = ~0ull;
        return;
    }
    const int d1 = int(idx[5]), d2 = int(idx[6]);
    const int c = (nn_cell_axis(idx, 0, pts[3 * size_t(i)]) * d1 + nn_cell_axis(idx, 1, pts[3 * size_t(i) + 1])) * d2 +
                  nn_cell_axis(idx, 2, pts[3 * size_t(i) + 2]);
    keys[i] = (static_cast<unsigned long long>(c) << 32) | static_cast<unsigned long long>(i);
}

// sorted targets (cell, index): contiguous coordinates + original index, and per-cell [start, end)
__global__ void k_nn_cells(const unsigned long long* __restrict__ sorted, int n_static, const int* __restrict__ n_dev,
                           const double* __restrict__ pts, double* spts, int* sidx, int* cstart, int* cend) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    const int n = n_dev ? *n_dev : n_static;
    if (s >= n) return;
    const unsigned long long k = sorted[s];
    const int c = int(k >> 32), i = int(k & 0xffffffffull);
    sidx[s] = i;
    for (int a = 0; a < 3; a++) spts[3 * size_t(s) + a] = pts[3 * size_t(i) + a];
    if (s == 0 || int(sorted[s - 1] >> 32) != c) cstart[c] = s;
    if (s == n - 1 || int(sorted[s + 1] >> 32) != c) cend[c] = s + 1;
}

// nearest target of each query (first index on ties), its distance, and CTA partial sums
__global__ void __launch_bounds__(kLT) k_nn_query(const double* __restrict__ q, int nq_static,
                                                  const int* __restrict__ nq_dev, const double* __restrict__ idx,
                                                  const double* __restrict__ spts, const int* __restrict__ sidx,
                                                  const int* __restrict__ cstart, const int* __restrict__ cend,
                                                  double* best, int* arg, double* partial) {
    __shared__ double red[kLT];
    const int nq = nq_dev ? *nq_dev : nq_static;
    const int k = blockIdx.x * kLT + threadIdx.x;
    double d = 0.0;
    if (k < nq) {
        const double p0 = q[3 * size_t(k)], p1 = q[3 * size_t(k) + 1], p2 = q[3 * size_t(k) + 2];
        const int D0 = int(idx[4]), D1 = int(idx[5]), D2 = int(idx[6]);
        const double h = idx[3];
        const int c0 = nn_cell_axis(idx, 0, p0), c1 = nn_cell_axis(idx, 1, p1), c2 = nn_cell_axis(idx, 2, p2);
        const int rmax = max(max(D0, D1), D2);
        double bd = 1e300;
        int bi = 0x7fffffff;
        for (int r = 0; r <= rmax; r++) {
            for (int dz = -r; dz <= r; dz++) {
                const int z = c2 + dz;
                if (z < 0 || z >= D2) continue;
                for (int dy = -r; dy <= r; dy++) {
                    const int y = c1 + dy;
                    if (y < 0 || y >= D1) continue;
                    const bool face = dz == -r || dz == r || dy == -r || dy == r;
                    for (int dx = -r; dx <= r; dx += (face || r == 0) ? 1 : 2 * r) {
                        const int x = c0 + dx;
                        if (x < 0 || x >= D0) continue;
                        const int c = (x * D1 + y) * D2 + z;
                        const int e = cend[c];
                        for (int t = cstart[c]; t < e; t++) {
                            const double d2 = nn_d2(p0 - spts[3 * size_t(t)], p1 - spts[3 * size_t(t) + 1],
                                                    p2 - spts[3 * size_t(t) + 2]);
                            const int ti = sidx[t];
                            if (d2 < bd || (d2 == bd && ti < bi)) {
                                bd = d2;
                                bi = ti;
                            }
                        }
                    }
                }
            }
            const double rh = double(r) * h;
            if (bd < rh * rh) break;
        }
        d = sqrt(bd);
        best[k] = d;
        arg[k] = bi == 0x7fffffff ? 0 : bi;  // (no target at all: the final sum raises the empty-set error)
    }
    red[threadIdx.x] = d;
    __syncthreads();
    for (int w = kLT / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

// ---------------------------------------------------------------------------
// mixing_spread (losses.hpp:76-100)
// ---------------------------------------------------------------------------
// grad == 0: per-member partial sums of -sum_j |x_i - x_j| (CTA partials);
// grad == 1: x_bar_i += -w sum_{j != i} 2 (x_i - x_j) / |x_i - x_j|
__global__ void __launch_bounds__(kLT) k_spread(const double* __restrict__ px, const int* __restrict__ idx,
                                                const int* __restrict__ count, int grad, double weight,
                                                double* partial, BarBuf bars) {
    __shared__ double ps[3 * kTileP];
    __shared__ double red[kLT];
    const int na = *count;
    const int k = blockIdx.x * kLT + threadIdx.x;
    const bool in = k < na;
    double p[3] = {0, 0, 0};
    if (in)
        for (int a = 0; a < 3; a++) p[a] = px[3 * size_t(k) + a];
    double s = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
    for (int t0 = 0; t0 < na; t0 += kTileP) {
        const int m = min(kTileP, na - t0);
        __syncthreads();
        for (int r = threadIdx.x; r < 3 * m; r += kLT) ps[r] = px[3 * size_t(t0) + r];
        __syncthreads();
        if (in)
            for (int j = 0; j < m; j++) {
                const double dx = p[0] - ps[3 * j], dy = p[1] - ps[3 * j + 1], dz = p[2] - ps[3 * j + 2];
                const double d = sqrt(dx * dx + dy * dy + dz * dz);
                if (!grad) {
                    s += d;
                } else if (t0 + j != k && d > 1e-300) {
                    const double c = 2.0 / d;
                    gx += dx * c;
                    gy += dy * c;
                    gz += dz * c;
                }
            }
    }
    if (grad) {
        if (in) {
            const int i = idx[k];
            bars.x(0)[i] += float(gx * -weight);
            bars.x(1)[i] += float(gy * -weight);
            bars.x(2)[i] += float(gz * -weight);
        }
        return;
    }
    red[threadIdx.x] = in ? s : 0.0;
    __syncthreads();
    for (int w = kLT / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

__global__ void __launch_bounds__(kLT) k_spread_final(const int* __restrict__ count, const double* __restrict__ partial,
                                                      int npartial, double weight, double* out,
                                                      unsigned long long* err) {
    __shared__ double red[kLT];
    if (*count < 2) {  // mixing_spread_loss: need at least 2 particles (losses.hpp:77)
        if (threadIdx.x == 0) atomicMin(err, (unsigned long long)pack_err(0xfffffu, ES_LOSS_EMPTY, 1));
        return;
    }
    double s = 0.0;
    for (int b = threadIdx.x; b < npartial; b += kLT) s += partial[b];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = kLT / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out += weight * -red[0];
}

// ---------------------------------------------------------------------------
// attraction (losses.hpp:104-218, 553-564) and per_particle (losses.hpp:367-390)
// ---------------------------------------------------------------------------
// A particle's position in the reference's state at this boundary: parked particles
// keep their parked position until the substep that emits them has run
// (mpm.hpp:435-449), while the store already holds the emitted one at that substep.
__device__ __forceinline__ double member_x(const LossSet& ls, const PBuf& st, int i, uint32_t id, int a) {
    return double(ls.act[id] >= ls.substep ? ls.x0[size_t(a) * ls.n_all + id] : st.x(a)[i]);
}

// |a - b| with the reference's operation order (dot(), core.hpp:104-118; no contraction)
__device__ __forceinline__ double dist3(double dx, double dy, double dz) {
    return sqrt(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
}

constexpr int kMemberBits = 24;  // sort key = cell << 24 | member rank

// members in member (= particle id) order: position, exp(-prev / tau), store slot and
// hash key (SpatialHash::build, losses.hpp:118-126: cell = floor(x / radius))
__global__ void k_attr_gather(PBuf st, int n, LossSet ls, uint32_t key_departed, double* px, double* e, int* slot,
                              unsigned long long* key) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || st.key[i] >= key_departed) return;
    const uint32_t id = st.id[i];
    const AttractionDev& A = ls.attr;
    const int r = A.mrank[id];
    if (r < 0) return;
    unsigned long long c = 0;
    for (int a = 0; a < 3; a++) {
        const double p = member_x(ls, st, i, id, a);
        px[3 * size_t(r) + a] = p;
        const int q = min(max(int(floor(p / A.radius)) + 1, 0), A.nc[a] - 1);
        c = c * (unsigned long long)A.nc[a] + (unsigned long long)q;
    }
    e[r] = exp(-A.prev[r] / A.tau);
    slot[r] = i;
    key[r] = (c << kMemberBits) | (unsigned long long)r;
}

// Thread = one member in hash order.  Neighbours are visited like SpatialHash::neighbors
// (losses.hpp:128-147): the 27 cells with axis 0 fastest, each cell in member order.
//   GRAD = false: wsum_i = sum_j w_ij, si_i = sum_j w_ij r_ij, CTA partials of si / wsum
//   GRAD = true:  x_bar_i += sum_j (g_ij + g_ji) (x_i - x_j) / r_ij, where g_ij is the
//                 reference's weight * dloss_dr of pair (i, j) seen from centre i
//                 (losses.hpp:203-215; its grad[j] -= dir * g is the g_ji term here)
template <bool GRAD>
__global__ void __launch_bounds__(kLT) k_attr_pass(const unsigned long long* __restrict__ keys, int na,
                                                   const double* __restrict__ px, const double* __restrict__ e,
                                                   AttractionDev A, double* wsum, double* si, double* partial,
                                                   const int* __restrict__ slot, BarBuf bars) {
    __shared__ double red[kLT];
    const int t = blockIdx.x * kLT + threadIdx.x;
    double contrib = 0.0;
    if (t < na) {
        const unsigned long long kk = keys[t];
        const int r = int(kk & ((1ull << kMemberBits) - 1));
        unsigned long long c = kk >> kMemberBits;
        const int qz = int(c % (unsigned long long)A.nc[2]);
        c /= (unsigned long long)A.nc[2];
        const int qy = int(c % (unsigned long long)A.nc[1]);
        const int qx = int(c / (unsigned long long)A.nc[1]);
        const double p0 = px[3 * size_t(r)], p1 = px[3 * size_t(r) + 1], p2 = px[3 * size_t(r) + 2];
        const double R = A.radius;
        double ws = 0.0, s = 0.0, g0 = 0.0, g1 = 0.0, g2 = 0.0;
        double wr = 0.0, sr = 0.0, er = 0.0;
        if (GRAD) {
            wr = wsum[r];
            sr = si[r];
            er = e[r];
        }
        for (int q = 0; q < 27; q++) {
            const int cx = qx + q % 3 - 1, cy = qy + (q / 3) % 3 - 1, cz = qz + q / 9 - 1;
            if (cx < 0 || cy < 0 || cz < 0 || cx >= A.nc[0] || cy >= A.nc[1] || cz >= A.nc[2]) continue;
            const unsigned long long cell =
                ((unsigned long long)cx * A.nc[1] + (unsigned long long)cy) * A.nc[2] + (unsigned long long)cz;
            const unsigned long long want = cell << kMemberBits;
            int lo = 0, hi = na;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (keys[mid] < want)
                    lo = mid + 1;
                else
                    hi = mid;
            }
            for (int u = lo; u < na; u++) {
                const unsigned long long kj = keys[u];
                if ((kj >> kMemberBits) != cell) break;
                const int j = int(kj & ((1ull << kMemberBits) - 1));
                if (j == r) continue;
                const double dx = p0 - px[3 * size_t(j)], dy = p1 - px[3 * size_t(j) + 1],
                             dz = p2 - px[3 * size_t(j) + 2];
                const double d = dist3(dx, dy, dz);
                if (d >= R) continue;
                const double tent = 1.0 - d / R;
                if (!GRAD) {
                    const double w = e[j] * tent;
                    ws += w;
                    s = __dadd_rn(s, __dmul_rn(w, d));
                } else {
                    double g = 0.0;
                    if (wr > 0.0) {  // pair (r, j) from centre r
                        const double dwdr = -e[j] / R;
                        const double dnum = __dadd_rn(__dmul_rn(dwdr, d), e[j] * tent);
                        g += A.weight * (dnum / wr - sr * dwdr / (wr * wr));
                    }
                    const double wj = wsum[j];
                    if (wj > 0.0) {  // pair (j, r) from centre j
                        const double dwdr = -er / R;
                        const double dnum = __dadd_rn(__dmul_rn(dwdr, d), er * tent);
                        g += A.weight * (dnum / wj - si[j] * dwdr / (wj * wj));
                    }
                    if (d > 1e-300) {
                        g0 += dx / d * g;
                        g1 += dy / d * g;
                        g2 += dz / d * g;
                    }
                }
            }
        }
        if (!GRAD) {
            wsum[r] = ws;  // ws == 0 also covers "no neighbours"
            si[r] = s;
            if (ws > 0.0) contrib = s / ws;
        } else {
            const int i = slot[r];
            bars.x(0)[i] += float(g0);
            bars.x(1)[i] += float(g1);
            bars.x(2)[i] += float(g2);
        }
    }
    if (GRAD) return;
    red[threadIdx.x] = contrib;
    __syncthreads();
    for (int w = kLT / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

__global__ void __launch_bounds__(kLT) k_attr_final(const double* __restrict__ partial, int npartial, double weight,
                                                    double* out) {
    __shared__ double red[kLT];
    double s = 0.0;
    for (int b = threadIdx.x; b < npartial; b += kLT) s += partial[b];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = kLT / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out += weight * red[0];
}

// per_particle: sum over the terms on the particle's body of its unweighted distance
// (target_point, hold_initial, nearest point of the last chamfer goal set), every member
// active or not; mixing_spread contributes nothing
__global__ void k_per_particle(PBuf st, int n, const ClassInfo* __restrict__ cls, LossSet ls,
                               uint32_t key_departed, double* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || st.key[i] >= key_departed) return;
    const uint32_t id = st.id[i];
    const int body = cls[meta_cls(st.meta[i])].body;
    double p[3];
    for (int a = 0; a < 3; a++) p[a] = member_x(ls, st, i, id, a);
    double v = 0.0;
    for (int k = 0; k < ls.n; k++) {
        const LossTermDev& t = ls.t[k];
        if (t.body != body) continue;
        if (t.kind == LK_TARGET) {
            v += dist3(p[0] - t.goal[0], p[1] - t.goal[1], p[2] - t.goal[2]);
        } else if (t.kind == LK_HOLD) {
            const float* q = t.init + 3 * size_t(id);
            v += dist3(p[0] - double(q[0]), p[1] - double(q[1]), p[2] - double(q[2]));
        } else if (t.kind == LK_CHAMFER) {
            const double* g = t.gpts + 3 * size_t(t.last_g0);
            double best = 1e300;
            for (int q = 0; q < t.last_ng; q++)
                best = fmin(best, dist3(p[0] - g[3 * q], p[1] - g[3 * q + 1], p[2] - g[3 * q + 2]));
            v += best;
        }
    }
    out[id] = v;
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
void PointLossScratch::reserve(int n_particles, int max_goals) {
    if (n_particles > cap_n) {
        for (auto p : {(void*)flags, (void*)pos, (void*)idx, (void*)px, (void*)best, (void*)arg}) cudaFree(p);
        cudaMalloc(&flags, sizeof(int) * size_t(n_particles));
        cudaMalloc(&pos, sizeof(int) * size_t(n_particles));
        cudaMalloc(&idx, sizeof(int) * size_t(n_particles));
        cudaMalloc(&px, sizeof(double) * 3 * size_t(n_particles));
        cudaMalloc(&best, sizeof(double) * size_t(n_particles));
        cudaMalloc(&arg, sizeof(int) * size_t(n_particles));
        cudaFree(partial);
        cudaMalloc(&partial, sizeof(double) * (size_t(n_particles) / kLT + 2));
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, flags, pos, n_particles);
        cudaFree(cub_tmp);
        cudaMalloc(&cub_tmp, tb);
        cub_bytes = tb;
        cap_n = n_particles;
    }
    const size_t need = size_t(kChamferChunks) * size_t(max_goals);
    if (need > cap_g) {
        for (auto p : {(void*)cbest, (void*)carg, (void*)gbest, (void*)garg}) cudaFree(p);
        cudaMalloc(&cbest, sizeof(double) * need);
        cudaMalloc(&carg, sizeof(int) * need);
        cudaMalloc(&gbest, sizeof(double) * size_t(max_goals));
        cudaMalloc(&garg, sizeof(int) * size_t(max_goals));
        cap_g = need;
    }
    if (!count) {
        cudaMalloc(&count, sizeof(int));
        cudaMalloc(&scal, sizeof(double) * 4);
    }
}

void PointLossScratch::reserve_attraction(int n_members) {
    if (n_members <= cap_a) return;
    for (auto p : {(void*)apx, (void*)ae, (void*)awsum, (void*)asi, (void*)aslot, (void*)akey, (void*)akey_sorted,
                   (void*)apart, asort_tmp})
        cudaFree(p);
    cudaMalloc(&apx, sizeof(double) * 3 * size_t(n_members));
    cudaMalloc(&ae, sizeof(double) * size_t(n_members));
    cudaMalloc(&awsum, sizeof(double) * size_t(n_members));
    cudaMalloc(&asi, sizeof(double) * size_t(n_members));
    cudaMalloc(&aslot, sizeof(int) * size_t(n_members));
    cudaMalloc(&akey, sizeof(unsigned long long) * size_t(n_members));
    cudaMalloc(&akey_sorted, sizeof(unsigned long long) * size_t(n_members));
    size_t tb = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb, akey, akey_sorted, n_members, 0, 64);
    cudaMalloc(&asort_tmp, tb);
    asort_bytes = tb;
    cudaMalloc(&apart, sizeof(double) * (size_t(n_members) / kLT + 2));
    cap_a = n_members;
}

PointLossScratch::~PointLossScratch() {
    for (auto p : {(void*)flags, (void*)pos, (void*)idx, (void*)px, (void*)best, (void*)arg, (void*)partial,
                   (void*)cbest, (void*)carg, (void*)gbest, (void*)garg, (void*)count, (void*)scal, cub_tmp,
                   (void*)apx, (void*)ae, (void*)awsum, (void*)asi, (void*)aslot, (void*)akey, (void*)akey_sorted,
                   (void*)apart, asort_tmp, (void*)nn_keys, (void*)nn_keys_sorted, (void*)nn_spts, (void*)nn_sidx,
                   nn_sort_tmp, (void*)nn_gpart, (void*)nn_cstart, (void*)nn_cend, (void*)nn_part, (void*)nn_idx})
        cudaFree(p);
}

void launch_attraction(PointLossScratch& w, const PBuf& st, int n, const LossSet& ls, uint32_t key_departed,
                       double* out, BarBuf* bars, cudaStream_t s) {
    const AttractionDev& A = ls.attr;
    const int na = A.n_members;
    if (!A.on || na < 2 || n <= 0) return;  // attraction_loss: fewer than 2 points -> 0
    k_attr_gather<<<(n + 255) / 256, 256, 0, s>>>(st, n, ls, key_departed, w.apx, w.ae, w.aslot, w.akey);
    cub::DeviceRadixSort::SortKeys(w.asort_tmp, w.asort_bytes, w.akey, w.akey_sorted, na, 0,
                                   kMemberBits + A.key_bits, s);
    const int grid = (na + kLT - 1) / kLT;
    // the gradient needs every member's sums first: pass 1 runs for eval and grad alike
    k_attr_pass<false><<<grid, kLT, 0, s>>>(w.akey_sorted, na, w.apx, w.ae, A, w.awsum, w.asi, w.apart, w.aslot,
                                           BarBuf{});
    if (!bars) {
        k_attr_final<<<1, kLT, 0, s>>>(w.apart, grid, A.weight, out);
    } else {
        k_attr_pass<true><<<grid, kLT, 0, s>>>(w.akey_sorted, na, w.apx, w.ae, A, w.awsum, w.asi, nullptr, w.aslot,
                                              *bars);
    }
}

void launch_per_particle(const PBuf& st, int n, const ClassInfo* cls, const LossSet& ls, uint32_t key_departed,
                         double* out, cudaStream_t s) {
    if (n <= 0) return;
    k_per_particle<<<(n + 255) / 256, 256, 0, s>>>(st, n, cls, ls, key_departed, out);
}

static void compact_body(PointLossScratch& w, const PBuf& st, int n, const ClassInfo* cls, int body,
                         uint32_t key_inactive, const LossSet& ls, cudaStream_t s) {
    const int grid = (n + 255) / 256;
    k_body_flags<<<grid, 256, 0, s>>>(st, n, cls, body, key_inactive, ls.act, ls.substep, w.flags);
    cub::DeviceScan::ExclusiveSum(w.cub_tmp, w.cub_bytes, w.flags, w.pos, n, s);
    k_body_gather<<<grid, 256, 0, s>>>(st, n, w.flags, w.pos, ls, w.idx, w.px, w.count);
}

// number of member chunks for the G -> A stage (<= kChamferChunks)
static int chamfer_chunk(int n) { return (n + kChamferChunks - 1) / kChamferChunks; }

constexpr int kNnBboxBlocks = 592;

void PointLossScratch::reserve_nn(int n) {
    if (n <= nn_cap) return;
    for (auto p : {(void*)nn_keys, (void*)nn_keys_sorted, (void*)nn_spts, (void*)nn_sidx, nn_sort_tmp,
                   (void*)nn_gpart})
        cudaFree(p);
    cudaMalloc(&nn_keys, sizeof(unsigned long long) * size_t(n));
    cudaMalloc(&nn_keys_sorted, sizeof(unsigned long long) * size_t(n));
    cudaMalloc(&nn_spts, sizeof(double) * 3 * size_t(n));
    cudaMalloc(&nn_sidx, sizeof(int) * size_t(n));
    cudaMalloc(&nn_gpart, sizeof(double) * (size_t(n) / kLT + 2));
    size_t tb = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb, nn_keys, nn_keys_sorted, n, 0, 53);
    cudaMalloc(&nn_sort_tmp, tb);
    nn_sort_bytes = tb;
    if (!nn_cstart) {
        const size_t cells = size_t(kNnMaxDim) * kNnMaxDim * kNnMaxDim;
        cudaMalloc(&nn_cstart, sizeof(int) * cells);
        cudaMalloc(&nn_cend, sizeof(int) * cells);
        cudaMalloc(&nn_part, sizeof(double) * 6 * kNnBboxBlocks);
        cudaMalloc(&nn_idx, sizeof(double) * 8);
    }
    nn_cap = n;
}

// uniform-grid index of pts[0 .. n) (n = *n_dev when given, else n_static; n <= n_cap)
static void nn_build(PointLossScratch& w, const double* pts, int n_static, const int* n_dev, int n_cap,
                     cudaStream_t s) {
    w.reserve_nn(n_cap);
    const int nb = std::max(1, std::min(kNnBboxBlocks, (n_cap + kLT - 1) / kLT));
    k_nn_bbox<<<nb, kLT, 0, s>>>(pts, n_static, n_dev, w.nn_part);
    k_nn_setup<<<1, 1, 0, s>>>(w.nn_part, nb, n_static, n_dev, w.nn_idx);
    k_nn_keys<<<(n_cap + 255) / 256, 256, 0, s>>>(pts, n_static, n_dev, w.nn_idx, w.nn_keys, n_cap);
    cub::DeviceRadixSort::SortKeys(w.nn_sort_tmp, w.nn_sort_bytes, w.nn_keys, w.nn_keys_sorted, n_cap, 0, 53, s);
    const size_t cells = size_t(kNnMaxDim) * kNnMaxDim * kNnMaxDim;
    cudaMemsetAsync(w.nn_cstart, 0, sizeof(int) * cells, s);
    cudaMemsetAsync(w.nn_cend, 0, sizeof(int) * cells, s);
    k_nn_cells<<<(n_cap + 255) / 256, 256, 0, s>>>(w.nn_keys_sorted, n_static, n_dev, pts, w.nn_spts, w.nn_sidx,
                                                   w.nn_cstart, w.nn_cend);
}

void launch_point_loss(PointLossScratch& w, const PBuf& st, int n, const ClassInfo* cls, const LossSet& ls,
                       const LossTermDev& t, int seg, uint32_t key_inactive, double* out, BarBuf* bars,
                       unsigned long long* err, int mode, cudaStream_t s) {
    if (n <= 0) return;
    compact_body(w, st, n, cls, t.body, key_inactive, ls, s);
    const int grid_a = (n + kLT - 1) / kLT;  // upper bound on the member count
    if (t.kind == LK_SPREAD) {
        if (!bars) {
            k_spread<<<grid_a, kLT, 0, s>>>(w.px, w.idx, w.count, 0, t.weight, w.partial, BarBuf{});
            k_spread_final<<<1, kLT, 0, s>>>(w.count, w.partial, grid_a, t.weight, out, err);
        } else {
            k_spread<<<grid_a, kLT, 0, s>>>(w.px, w.idx, w.count, 1, t.weight, w.partial, *bars);
        }
        return;
    }
    // trajectory_chamfer: goal set min(seg, n_steps - 1)
    const int step = seg < t.nsteps ? seg : t.nsteps - 1;
    const int g0 = t.goff_h[step], ng = t.goff_h[step + 1] - g0;
    const double* g = t.gpts + 3 * size_t(g0);
    const bool grid = mode == 2 || (mode == 0 && double(n) * double(ng) > kChamferBrutePairs);
    if (grid) {  // exact nearest neighbours through uniform-grid indexes (A -> G, then G -> A)
        nn_build(w, g, ng, nullptr, ng, s);
        k_nn_query<<<grid_a, kLT, 0, s>>>(w.px, 0, w.count, w.nn_idx, w.nn_spts, w.nn_sidx, w.nn_cstart, w.nn_cend,
                                          w.best, w.arg, w.partial);
        nn_build(w, w.px, 0, w.count, n, s);
        k_nn_query<<<(ng + kLT - 1) / kLT, kLT, 0, s>>>(g, ng, nullptr, w.nn_idx, w.nn_spts, w.nn_sidx, w.nn_cstart,
                                                         w.nn_cend, w.gbest, w.garg, w.nn_gpart);
        k_chamfer_final<<<1, kLT, 0, s>>>(w.count, 0, ng, nullptr, nullptr, w.partial, grid_a, t.weight, w.gbest,
                                          w.garg, bars ? w.scal + 1 : out, w.scal, err);
    } else {
        const int chunk = chamfer_chunk(n);
        const int nchunks = (n + chunk - 1) / chunk;
        k_chamfer_a<<<grid_a, kLT, 0, s>>>(w.px, w.count, g, ng, w.best, w.arg, w.partial);
        k_chamfer_g<<<nchunks, kLT, 0, s>>>(w.px, w.count, chunk, g, ng, w.cbest, w.carg);
        k_chamfer_final<<<1, kLT, 0, s>>>(w.count, nchunks, ng, w.cbest, w.carg, w.partial, grid_a, t.weight,
                                          w.gbest, w.garg, bars ? w.scal + 1 : out, w.scal, err);
    }
    if (bars) {
        k_chamfer_grad_a<<<grid_a, kLT, 0, s>>>(w.px, w.idx, w.count, g, w.best, w.arg, t.weight, *bars);
        k_chamfer_grad_g<<<1, 32, 0, s>>>(w.px, w.idx, g, ng, w.gbest, w.garg, t.weight, *bars);
    }
}

}  // namespace fl
