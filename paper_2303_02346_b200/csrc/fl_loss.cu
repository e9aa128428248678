// fl_loss.cu -- point-set losses at segment boundaries on the device
// (losses.hpp:15-100, 474-551):
//   trajectory_chamfer   symmetric mean nearest-neighbour distance between the
//                        body's active particles A and the segment's goal set G,
//                        O(|A| |G|) brute force in fp64 (no hashing: exact argmins)
//   mixing_spread        -sum_ij |x_i - x_j| over the body, O(|A|^2) in fp64
//   attraction           the optimizer's gradient-sharing surrogate (losses.hpp:104-218):
//                        hashed-grid neighbour sums over every member of one body
// Both first compact the body's active particles in store order (deterministic
// prefix sum), so every sum below has a fixed order.  The evaluation adds
// weight * value into the segment's loss slot; the gradient adds into x_bar
// with the reference's per-particle accumulation order (A-term, then G-terms
// in goal order).
#include <cuda_runtime.h>

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
                const double dx = p[0] - gs[3 * j], dy = p[1] - gs[3 * j + 1], dz = p[2] - gs[3 * j + 2];
                const double d2 = dx * dx + dy * dy + dz * dz;
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
                    const double dx = q[0] - ps[3 * j], dy = q[1] - ps[3 * j + 1], dz = q[2] - ps[3 * j + 2];
                    const double d2 = dx * dx + dy * dy + dz * dz;
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
                   (void*)apart, asort_tmp})
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

void launch_point_loss(PointLossScratch& w, const PBuf& st, int n, const ClassInfo* cls, const LossSet& ls,
                       const LossTermDev& t, int seg, uint32_t key_inactive, double* out, BarBuf* bars,
                       unsigned long long* err, cudaStream_t s) {
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
    const int chunk = chamfer_chunk(n);
    const int nchunks = (n + chunk - 1) / chunk;
    k_chamfer_a<<<grid_a, kLT, 0, s>>>(w.px, w.count, g, ng, w.best, w.arg, w.partial);
    k_chamfer_g<<<nchunks, kLT, 0, s>>>(w.px, w.count, chunk, g, ng, w.cbest, w.carg);
    k_chamfer_final<<<1, kLT, 0, s>>>(w.count, nchunks, ng, w.cbest, w.carg, w.partial, grid_a, t.weight, w.gbest,
                                      w.garg, bars ? w.scal + 1 : out, w.scal, err);
    if (bars) {
        k_chamfer_grad_a<<<grid_a, kLT, 0, s>>>(w.px, w.idx, w.count, g, w.best, w.arg, t.weight, *bars);
        k_chamfer_grad_g<<<1, 32, 0, s>>>(w.px, w.idx, g, ng, w.gbest, w.garg, t.weight, *bars);
    }
}

}  // namespace fl
