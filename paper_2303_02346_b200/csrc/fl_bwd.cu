// fl_bwd.cu -- reverse-mode MLS-MPM substep kernels for sm_100a.
//
// Mirrors adjoint_substep (proj/include/flume/adjoint.hpp:476-548) without the
// reference's capture_forward re-run: the pre-state of the substep, its
// permutation/block map and the forward grid (velocities after contact, p/m and
// m before it) are all read from the substep's record in the trajectory store,
// and then
//   adjoint_rigid_pass   (adjoint.hpp:210-279)   k_adj_rigid_*
//   adjoint_g2p          (adjoint.hpp:281-365)   k_adj_g2p   (gather + scatter of grid v_bar)
//   adjoint_grid_update  (adjoint.hpp:367-412)   k_adj_grid  (+ deterministic effector-bar reduction)
//   adjoint_p2g          (adjoint.hpp:414-470)   k_adj_p2g
//   emitter adjoint      (adjoint.hpp:503-520)   k_adj_emit
// Bars of state[t+1] are indexed by sorted position j (= storage slot of
// state[t+1]); bars of state[t] are written at the storage slot perm[j].
#include <cuda_runtime.h>

#include "fl_kernels.h"
#include "fl_scatter.cuh"

namespace fl {

// ---------------------------------------------------------------------------
// loss cotangent injection at segment boundaries (losses.hpp:506-525)
// ---------------------------------------------------------------------------
__global__ void k_loss_grad(PBuf st, DN nn, const ClassInfo* __restrict__ cls, LossSet ls, uint32_t mask,
                            uint32_t key_inactive, BarBuf bars) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nn.get()) return;
    const uint32_t key = st.key[i];
    if (key > key_inactive) return;  // departed slot
    if (key == key_inactive && !ls.count_parked) return;
    const int body = cls[meta_cls(st.meta[i])].body;
    const bool active = key < key_inactive || ls.act[st.id[i]] <= ls.substep;
    double g[3] = {0.0, 0.0, 0.0};
    bool any = false;
    for (int k = 0; k < ls.n; k++) {
        if (!((mask >> k) & 1u) || ls.t[k].body != body || ls.t[k].kind > LK_HOLD) continue;
        const LossTermDev& t = ls.t[k];
        double d[3];
        if (t.kind == LK_TARGET) {
            if (!active) continue;
            for (int a = 0; a < 3; a++) d[a] = double(loss_x(ls, st, i, st.id[i], a)) - t.goal[a];
        } else {
            const uint32_t id = st.id[i];
            for (int a = 0; a < 3; a++) d[a] = double(loss_x(ls, st, i, id, a)) - double(t.init[3 * size_t(id) + a]);
        }
        const double nn = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
        if (t.kind == LK_TARGET && t.squared) {
            for (int a = 0; a < 3; a++) g[a] += d[a] * (2.0 * t.weight);
            any = true;
        } else if (nn > 1e-300) {
            for (int a = 0; a < 3; a++) g[a] += d[a] * (t.weight / nn);
            any = true;
        }
    }
    if (any)
        for (int a = 0; a < 3; a++) bars.x(a)[i] += float(g[a]);
}

void launch_loss_grad(const PBuf& st, DN n, const ClassInfo* cls, const LossSet& ls, uint32_t mask, BarBuf bars,
                      uint32_t key_inactive, cudaStream_t s) {
    if (n.h <= 0) return;
    k_loss_grad<<<(n.h + 255) / 256, 256, 0, s>>>(st, n, cls, ls, mask, key_inactive, bars);
}

// ---------------------------------------------------------------------------
// rigid pass adjoint (adjoint.hpp:210-279)
// ---------------------------------------------------------------------------
constexpr int kAdjRigidQ = 12;  // r_bar[9], c_bar[3]

// member cotangents (x_bar, v_bar of the post-rigid state) by member rank; with
// slabs every rank contributes its own members and the array is all-reduced
// (disjoint support: the sum is exact), so every rank solves identical fits
__global__ void k_adj_rigid_gather(BarBuf post, RigidDev rd, double* mbar) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rd.nmem) return;
    const int body = rd.member_body[r];
    const int j = rd.mslot[r];
    double* o = mbar + 6 * size_t(r);
    for (int q = 0; q < 6; q++) o[q] = 0.0;
    if (rd.fit[24 * size_t(body) + 22] != 0.0 || j < 0) return;
    for (int a = 0; a < 3; a++) {
        o[a] = post.x(a)[j];
        o[3 + a] = post.v(a)[j];
        post.x(a)[j] = 0.f;
        post.v(a)[j] = 0.f;
    }
}

__global__ void __launch_bounds__(256) k_adj_rigid_partial(Geom g, const double* mbar, RigidDev rd,
                                                           const int* chunk_m0, const int* chunk_m1,
                                                           double* partial, float* start_bar) {
    __shared__ double red[256];
    const int c = blockIdx.x;
    const int m0 = chunk_m0[c], m1 = chunk_m1[c];
    double acc[kAdjRigidQ];
    for (int q = 0; q < kAdjRigidQ; q++) acc[q] = 0.0;
    for (int r = m0 + threadIdx.x; r < m1; r += 256) {
        const int body = rd.member_body[r];
        const double* fit = rd.fit + 24 * size_t(body);
        if (fit[22] != 0.0) {
            for (int a = 0; a < 3; a++) start_bar[3 * r + a] = 0.f;
            continue;
        }
        const double inv_dt = 1.0 / double(g.dt);
        double xn_bar[3];
        for (int a = 0; a < 3; a++) {
            const double xb = mbar[6 * size_t(r) + a], vb = mbar[6 * size_t(r) + 3 + a];
            xn_bar[a] = xb + vb * inv_dt;
            start_bar[3 * r + a] = float(-vb * inv_dt);
        }
        const double* re = rd.rest + 3 * size_t(r);
        for (int a = 0; a < 3; a++) {
            const double raw = fit[3 * a] * re[0] + fit[3 * a + 1] * re[1] + fit[3 * a + 2] * re[2] + fit[9 + a];
            const double cl = clamp_ref(raw, double(g.lo[a]), double(g.hi[a]));
            if (raw != cl) xn_bar[a] = 0.0;
        }
        for (int a = 0; a < 3; a++)
            for (int b = 0; b < 3; b++) acc[3 * a + b] += xn_bar[a] * re[b];
        for (int a = 0; a < 3; a++) acc[9 + a] += xn_bar[a];
    }
    for (int q = 0; q < kAdjRigidQ; q++) {
        red[threadIdx.x] = acc[q];
        __syncthreads();
        for (int w = 128; w > 0; w >>= 1) {
            if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
            __syncthreads();
        }
        if (threadIdx.x == 0) partial[size_t(c) * kAdjRigidQ + q] = red[0];
        __syncthreads();
    }
}

// abar per body: A_bar[9], c_total[3], total
__global__ void k_adj_rigid_solve(RigidDev rd, int nchunks, const int* chunk_body, const double* partial,
                                  double* abar) {
    const int body = blockIdx.x * blockDim.x + threadIdx.x;
    if (body >= rd.nbody) return;
    const double* fit = rd.fit + 24 * size_t(body);
    double* o = abar + 13 * size_t(body);
    if (fit[22] != 0.0) {
        for (int q = 0; q < 13; q++) o[q] = 0.0;
        return;
    }
    double s[kAdjRigidQ];
    for (int q = 0; q < kAdjRigidQ; q++) s[q] = 0.0;
    for (int c = 0; c < nchunks; c++) {
        if (chunk_body[c] != body) continue;
        for (int q = 0; q < kAdjRigidQ; q++) s[q] += partial[size_t(c) * kAdjRigidQ + q];
    }
    M3<double> r_bar, A;
    for (int k = 0; k < 9; k++) {
        r_bar.m[k] = s[k];
        A.m[k] = fit[12 + k];
    }
    V3<double> c_bar = {s[9], s[10], s[11]};
    Svd<double> t = svd3(A);
    M3<double> a_bar;
    if (det(A) > 0.0) {
        a_bar = polar_rotation_vjp(t, r_bar);
    } else {
        M3<double> flip = mdiag(V3<double>{1.0, 1.0, -1.0});
        a_bar = svd_vjp(t, r_bar * t.V * flip, V3<double>{0.0, 0.0, 0.0}, transpose(r_bar) * t.U * flip, 1e-8);
    }
    V3<double> smr = {rd.smrest[3 * body], rd.smrest[3 * body + 1], rd.smrest[3 * body + 2]};
    V3<double> ct = c_bar - a_bar * smr;
    for (int k = 0; k < 9; k++) o[k] = a_bar.m[k];
    o[9] = ct.x;
    o[10] = ct.y;
    o[11] = ct.z;
    o[12] = fit[21];
}

__global__ void k_adj_rigid_apply(BarBuf post, RigidDev rd, const double* abar) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rd.nmem) return;
    const int body = rd.member_body[r];
    if (rd.fit[24 * size_t(body) + 22] != 0.0) return;
    const double* o = abar + 13 * size_t(body);
    const int j = rd.mslot[r];
    if (j < 0) return;  // member lives on another slab
    const double* re = rd.rest + 3 * size_t(r);
    const double m = rd.mass[r];
    for (int a = 0; a < 3; a++) {
        const double gv = (o[3 * a] * re[0] + o[3 * a + 1] * re[1] + o[3 * a + 2] * re[2]) * m;
        post.x(a)[j] += float(gv + o[9 + a] * (m / o[12]));
    }
}

void launch_adj_rigid_gather(BarBuf post, RigidDev rd, double* mbar, cudaStream_t s) {
    if (rd.nbody == 0) return;
    k_adj_rigid_gather<<<(rd.nmem + 255) / 256, 256, 0, s>>>(post, rd, mbar);
}

void launch_adj_rigid(const Geom& g, BarBuf post, RigidDev rd, int nchunks, const int* chunk_body,
                      const int* chunk_m0, const int* chunk_m1, const double* mbar, double* partial,
                      float* start_bar, double* abar, cudaStream_t s) {
    if (rd.nbody == 0) return;
    k_adj_rigid_partial<<<nchunks, 256, 0, s>>>(g, mbar, rd, chunk_m0, chunk_m1, partial, start_bar);
    k_adj_rigid_solve<<<(rd.nbody + 31) / 32, 32, 0, s>>>(rd, nchunks, chunk_body, partial, abar);
    k_adj_rigid_apply<<<(rd.nmem + 255) / 256, 256, 0, s>>>(post, rd, abar);
}

// ---------------------------------------------------------------------------
// G2P adjoint (adjoint.hpp:281-365): gather + deterministic scatter of grid v_bar
// ---------------------------------------------------------------------------
// NT threads: 256 stage the payload of a full block (8 particles x 64 cells) in two even
// rounds (192 leave a third round two-thirds idle); the extra 64 idle in the accumulate
// phase.  Measured: c4 109.9 -> 104.6 us, c3 283 -> 262 us (all three variants: with
// 192 threads for the heavy blocks beside a liquid scene c4 keeps its 109.6 us -- those
// few SVD blocks are the kernel's tail)
#ifndef FL_ADJG2P_NT
#define FL_ADJG2P_NT 256
#endif
template <bool HEAVY, int MINB, int NT>
__global__ void __launch_bounds__(NT, MINB) k_adj_g2p(Geom g, PBuf pre, const uint32_t* __restrict__ perm,
                                                        const BlockRec* __restrict__ recs,
                                                        const int* __restrict__ n_blocks,
                                                        const uint16_t* __restrict__ celltab,
                                                        const ClassInfo* __restrict__ cls,
                                                        const float4* __restrict__ gridv, PBuf postst, BarBuf post,
                                                        float* xbar_tmp, float* Fbar_tmp, RigidDev rd,
                                                        const float* __restrict__ start_bar, float4* staging_bar,
                                                        int cap, int* wq, int role) {
    const DualScope dual_scope(role);
    extern __shared__ __align__(16) unsigned char smraw[];
    ScSmem& sm = *reinterpret_cast<ScSmem*>(smraw);
    float4* vt = reinterpret_cast<float4*>(smraw + sizeof(ScSmem));
    float4* raw = reinterpret_cast<float4*>(sm.pay);  // raw TMA tile: the payload area is idle here
    static_assert(sizeof(float) * kPayF * kScR * kCS >= sizeof(float4) * kTileRaw, "raw tile alias");
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x;
    TileStage ts;
    ts.init(&bar, raw, tid);
    const int q0 = HEAVY ? g.maxb - n_blocks[1] : 0, q1 = HEAVY ? g.maxb : n_blocks[0];
    const int my_c = tid & 63, my_ox = tid >> 6;
    __shared__ int sh_next;
    __shared__ int s_wc[kWorkClasses];
    work_counts_load(n_blocks, HEAVY ? 1 : 0, s_wc, tid);
    for (;;) {
        const int k = next_work(wq, &sh_next);
        if (k >= q1 - q0) break;
        const int4 we = work_entry(n_blocks, g.maxb, HEAVY ? 1 : 0, k, s_wc);  // costliest blocks first
        const int b = we.x;
        const BlockRec r{we.y, we.z, we.w};
        int bx, by, bz;
        block_unlin(g, r.block, bx, by, bz);
        ts.begin(g, gridv, bx, by, bz, tid);
        sc_tile_zero(sm, tid, NT);
        const int npass = sc_load_cells(sm, celltab, b, tid);
        // repack before the first pass: its prefix barrier orders these raw reads
        // before the payload writes into the same bytes
        ts.end(g, gridv, vt, bx, by, bz, tid, NT);
        for (int pass = 0; pass < npass; pass++) {
            const int r0 = pass * kScR;
            // every pass walks the dense list of the particles it stages (measured: the
            // sorted walk with idle lanes for ranks beyond the pass is slower here)
            const int lim = sc_overflow_prefix(sm, r0, tid);
            for (int it = tid; it < lim; it += NT) {
                int c, rank;
                sc_overflow_item(sm, it, c, rank);
                const int i = int(sm.cs[c]) + r0 + rank;
                const int j = r.start + i;
                const uint32_t s = perm[j];
                float* pay = pay_slot(sm, rank, c);
                const V3<float> x = {pre.x(0)[s], pre.x(1)[s], pre.x(2)[s]};
                const uint32_t pmeta = pre.meta[s];
                const ClassInfo ci = cls[meta_cls(pmeta)];
                const bool cin = !HEAVY || f_compact(ci, pmeta);  // pre-state F = c I
                const bool cpost = !HEAVY || ci.iso;              // post-state F (and its bar) compact
                StencilW sw;
                stencil_weights(g, x, bx - rep_of_col(g, bx) * g.rstride, by, bz, sw);  // replica-local
                V3<float> vraw, vuse;
                M3<float> cnew;
                bool clamped_v;
                if constexpr (HEAVY) {
                    g2p_gather(g, vt, sw, vraw, cnew);
                    const float vn = norm(vraw);
                    clamped_v = vn > g.vmax;
                    vuse = clamped_v ? vraw * (g.vmax / vn) : vraw;
                } else {
                    // plain liquids: the forward stored C_new and the (clamped) velocity
                    // in the post-state at this sorted position; re-gather only when the
                    // CFL clamp fired (v_raw is then not recoverable)
                    clamped_v = (postst.meta[j] & kMetaCfl) != 0u;
#pragma unroll
                    for (int k = 0; k < 9; k++) cnew.m[k] = postst.C(k)[j];
                    vuse = V3<float>{postst.v(0)[j], postst.v(1)[j], postst.v(2)[j]};
                    vraw = vuse;
                    if (clamped_v) {
                        M3<float> cdummy;
                        g2p_gather(g, vt, sw, vraw, cdummy);
                    }
                }
                const M3<float> ipc = meye<float>() + cnew * g.dt;
                M3<float> F;
                if (cin) {
                    F = meye<float>() * pre.F(0)[s];
                } else {
#pragma unroll
                    for (int k = 0; k < 9; k++) F.m[k] = pre.F(k)[s];
                }
                const M3<float> ftr = cin ? ipc * F.m[0] : ipc * F;
                M3<float> cin_bar;
#pragma unroll
                for (int k = 0; k < 9; k++) cin_bar.m[k] = post.C(k)[j];
                M3<float> ftr_bar;
                if (cpost) {  // (viscous) liquid: only tr(F_post_bar) = dL/dc_post is stored
                    ftr_bar = liquid_project_vjp_c(ftr, post.F(0)[j]);
                } else {
                    M3<float> fpost_bar;
#pragma unroll
                    for (int k = 0; k < 9; k++) fpost_bar.m[k] = post.F(k)[j];
                    switch (ci.kind) {
                        case MK_LIQUID:
                        case MK_VISCOUS: ftr_bar = liquid_project_vjp(ftr, fpost_bar); break;  // (rigid members)
                        case MK_PLASTIC: ftr_bar = box_yield_project_vjp(ftr, ci.theta_c, ci.theta_s, fpost_bar); break;
                        case MK_NONNEWTONIAN:
                            ftr_bar = von_mises_project_vjp(ftr, ci.sigma_y, ci.mu, fpost_bar);
                            break;
                        default: ftr_bar = fpost_bar; break;
                    }
                }
                const M3<float> fpre_bar = transpose(ipc) * ftr_bar;
                const M3<float> c_bar = cin ? cin_bar + ftr_bar * (F.m[0] * g.dt) : cin_bar + ftr_bar * transpose(F) * g.dt;
                V3<float> xnb = {post.x(0)[j], post.x(1)[j], post.x(2)[j]};
                if (!HEAVY || ci.rigid < 0) {
#pragma unroll
                    for (int a = 0; a < 3; a++) {
                        const float xr = x[a] + vuse[a] * g.dt;
                        const float xc = clamp_ref(xr, g.lo[a], g.hi[a]);
                        if (xr != xc) xnb[a] = 0.f;
                    }
                } else {
                    const int mr = rd.mrank[pre.id[s]];
                    for (int a = 0; a < 3; a++) {
                        const double xr = pre.mx[3 * mr + a] + double(vuse[a]) * double(g.dt);
                        const double xc = clamp_ref(xr, double(g.lo[a]), double(g.hi[a]));
                        if (xr != xc) xnb[a] = 0.f;
                    }
                }
                const V3<float> vub = {post.v(0)[j] + xnb.x * g.dt, post.v(1)[j] + xnb.y * g.dt,
                                       post.v(2)[j] + xnb.z * g.dt};
                const V3<float> vrb = clamped_v ? V3<float>{0.f, 0.f, 0.f} : vub;
                // x_bar = x_new_bar + sum_o grad w_o s_o - k4 c_bar^T v_raw
                V3<float> xb = xnb - tmul(c_bar, vraw) * g.k4;
                const float kd = g.k4 * g.dx;
                {
                    // x_bar += sum_o grad w_o (gv_o . (v_raw_bar + k4 c_bar rel_o)), factored per axis:
                    // k4 c_bar rel_o = ax[ox] + ay[oy] + az[oz]; the weight-gradient products are
                    // accumulated per x-plane and scaled by dw_x / w_x once per plane.
                    V3<float> ay[3], az[3];
#pragma unroll
                    for (int o = 0; o < 3; o++) {
                        const float ry = (float(o) - sw.fx[1]) * kd, rz = (float(o) - sw.fx[2]) * kd;
                        ay[o] = V3<float>{c_bar.m[1] * ry, c_bar.m[4] * ry, c_bar.m[7] * ry};
                        az[o] = V3<float>{c_bar.m[2] * rz, c_bar.m[5] * rz, c_bar.m[8] * rz};
                    }
                    float sxx = 0.f, syy = 0.f, szz = 0.f;
#pragma unroll 1
                    for (int ox = 0; ox < 3; ox++) {
                        const float wox = ox == 0 ? sw.w[0][0] : (ox == 1 ? sw.w[0][1] : sw.w[0][2]);
                        const float dox = ox == 0 ? sw.dw[0][0] : (ox == 1 ? sw.dw[0][1] : sw.dw[0][2]);
                        const float rx = (float(ox) - sw.fx[0]) * kd;
                        const V3<float> ax = {vrb.x + c_bar.m[0] * rx, vrb.y + c_bar.m[3] * rx, vrb.z + c_bar.m[6] * rx};
                        float px = 0.f, py = 0.f, pz = 0.f;
                        const float4* row = vt + (sw.l[0] + ox) * 36 + sw.l[1] * 6 + sw.l[2];
#pragma unroll
                        for (int oy = 0; oy < 3; oy++) {
                            const V3<float> axy = ax + ay[oy];
                            float sa = 0.f, sb = 0.f;  // z-weighted and z-gradient-weighted sums
#pragma unroll
                            for (int oz = 0; oz < 3; oz++) {
                                const float4 gv4 = row[oy * 6 + oz];
                                const V3<float> u = axy + az[oz];
                                const float sv = gv4.x * u.x + gv4.y * u.y + gv4.z * u.z;
                                sa += sw.w[2][oz] * sv;
                                sb += sw.dw[2][oz] * sv;
                            }
                            px += sw.w[1][oy] * sa;
                            py += sw.dw[1][oy] * sa;
                            pz += sw.w[1][oy] * sb;
                        }
                        sxx += dox * px;
                        syy += wox * py;
                        szz += wox * pz;
                    }
                    xb.x += sxx * g.inv_dx;
                    xb.y += syy * g.inv_dx;
                    xb.z += szz * g.inv_dx;
                }
                if (HEAVY && ci.rigid >= 0) {
                    const int mr = rd.mrank[pre.id[s]];
                    xb.x += start_bar[3 * mr];
                    xb.y += start_bar[3 * mr + 1];
                    xb.z += start_bar[3 * mr + 2];
                }
                xbar_tmp[j] = xb.x;
                xbar_tmp[size_t(cap) + j] = xb.y;
                xbar_tmp[2 * size_t(cap) + j] = xb.z;
                if (cin) {  // dL/dc of the pre-state's F = c I
                    Fbar_tmp[j] = trace(fpre_bar);
                } else {
#pragma unroll
                    for (int k = 0; k < 9; k++) Fbar_tmp[size_t(k) * cap + j] = fpre_bar.m[k];
                }
                // scatter payload: w (v_raw_bar + k4 c_bar dx (o - fx))
                const M3<float> bm = c_bar * kd;
                const V3<float> f3 = {sw.fx[0], sw.fx[1], sw.fx[2]};
                const V3<float> a = vrb - bm * f3;
                pay[0] = sw.fx[0];
                pay[kPayPlane] = sw.fx[1];
                pay[2 * kPayPlane] = sw.fx[2];
                pay[3 * kPayPlane] = a.x;
                pay[4 * kPayPlane] = a.y;
                pay[5 * kPayPlane] = a.z;
#pragma unroll
                for (int k = 0; k < 9; k++) pay[(6 + k) * kPayPlane] = bm.m[k];
            }
            __syncthreads();
            const int nr = my_ox < 3 ? min(max(int(sm.cs[my_c + 1]) - int(sm.cs[my_c]) - r0, 0), kScR) : 0;
            sc_accumulate<3>(sm, my_c, my_ox, nr, tid, NT);
            __syncthreads();
        }
        __syncthreads();
        sc_tile_store(sm, staging_bar + size_t(b) * kTile, tid, NT);
    }
}

static decltype(&k_adj_g2p<false, FL_LB_ADJG2P, FL_ADJG2P_NT>) adj_g2p_kernel(int v) {
    return v == 0 ? k_adj_g2p<false, FL_LB_ADJG2P, FL_ADJG2P_NT>
                  : (v == 2 ? k_adj_g2p<true, FL_LBD_ADJG2P, FL_ADJG2P_NT>
                            : k_adj_g2p<true, FL_LBH_ADJG2P, FL_ADJG2P_NT>);  // (1 and 3)
}
static int adj_g2p_threads(int) { return FL_ADJG2P_NT; }

void launch_adj_g2p(const Geom& g, PBuf pre, const uint32_t* perm, const BlockRec* recs, const int* n_blocks,
                    const uint16_t* celltab, int grid, const ClassInfo* cls, const float4* gridv, PBuf postst,
                    BarBuf post, float* xbar_tmp, float* Fbar_tmp, RigidDev rd, const float* start_bar,
                    float4* staging_bar, int variant, int* wq, cudaStream_t s) {
    const size_t smem = sizeof(ScSmem) + kTile * sizeof(float4);
    static bool attr[4] = {false, false, false, false};
    if (!attr[variant]) {
        cudaFuncSetAttribute(adj_g2p_kernel(variant), cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        attr[variant] = true;
    }
    launch_k(adj_g2p_kernel(variant), dim3(grid), dim3(adj_g2p_threads(variant)), smem, s, g, pre, perm, recs, n_blocks, celltab,
             cls, gridv, postst, post, xbar_tmp, Fbar_tmp, rd, start_bar, staging_bar, post.cap, wq, dual_role());
}

// ---------------------------------------------------------------------------
// grid update adjoint (adjoint.hpp:367-412) with a deterministic CTA-level
// reduction of the per-effector bars (18 scalars each)
// ---------------------------------------------------------------------------
constexpr int kEffQ = 18;  // t[3] R[9] vlin[3] w[3]
#ifndef FL_ADJGRID_THREADS
#define FL_ADJGRID_THREADS 128
#endif
constexpr int kAdjGridThreads = FL_ADJGRID_THREADS;

__device__ __forceinline__ float4 gather_tile_sum(const Geom& g, const int* __restrict__ blockmap,
                                                  const float4* __restrict__ staging, int bx, int by, int bz, int lx,
                                                  int ly, int lz) {
    // the block-map loads first (independent), then the tile loads and the fixed-order sum
    int slot[8];
#pragma unroll
    for (int d = 0; d < 8; d++) {
        const int ddx = d >> 2, ddy = (d >> 1) & 1, ddz = d & 1;
        const int px = bx - ddx, py = by - ddy, pz = bz - ddz;
        const bool in = !((ddx && lx >= 2) || (ddy && ly >= 2) || (ddz && lz >= 2)) && px >= 0 && py >= 0 && pz >= 0;
        slot[d] = in ? blockmap[block_lin(g, px, py, pz)] - 1 : -1;  // map holds slot + 1
    }
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int d = 0; d < 8; d++) {
        if (slot[d] < 0) continue;
        const int ddx = d >> 2, ddy = (d >> 1) & 1, ddz = d & 1;
        const float4 v = staging[size_t(slot[d]) * kTile + (lx + 4 * ddx) * 36 + (ly + 4 * ddy) * 6 + (lz + 4 * ddz)];
        acc.x += v.x;
        acc.y += v.y;
        acc.z += v.z;
        acc.w += v.w;
    }
    return acc;
}

// NE = number of effectors (compile time).  Effector bars: where any lane of a
// warp touched effector e, the warp reduces the 18 components with a fixed
// shuffle tree and lane 0 adds them to the warp's fp64 accumulator in shared
// memory (static node order per warp, since the list partition is static), then
// one fixed-order CTA reduction per launch.  Nothing effector-sized lives in
// registers across nodes, which keeps the kernel at ~64 registers.
// REP (replica contexts): NE effectors per replica, read from eff.ext; the bars of replica
// rep's effector e accumulate in slot rep * NE + e (of eff.n), so the shared accumulators
// are dynamic (kW x eff.n x 18 doubles) and the partial rows `pstride` doubles long.
template <int NE, bool FILTER, bool REP>  // (the column filter only in slab contexts)
__global__ void __launch_bounds__(kAdjGridThreads, 1024 / kAdjGridThreads) k_adj_grid(Geom g, const int* __restrict__ nb_list,
                                                                 const int* __restrict__ n_nb,
                                                                 const int* __restrict__ blockmap,
                                                                 const float4* __restrict__ staging_bar,
                                                                 const float4* __restrict__ gridv0, float4* gridbar,
                                                                 EffSet eff, double* eff_partial,
                                                                 const uint8_t* __restrict__ cmask, GridCols cols,
                                                                 int pstride) {
    pdl_wait();
    constexpr int kW = kAdjGridThreads / 32;
    constexpr int kQs = NE * kEffQ > 0 ? NE * kEffQ : 1;
    __shared__ double wacc_s[REP ? 1 : kW * kQs];
    extern __shared__ double wacc_d[];
    const int kQ = REP ? eff.n * kEffQ : kQs;
    double* wacc = REP ? wacc_d : wacc_s;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int sub = tid >> 6, l = tid & 63;
    const int lx = l >> 4, ly = (l >> 2) & 3, lz = l & 3;
    const int n = *n_nb;
    constexpr int kPer0 = kAdjGridThreads / 64;
    if (int(blockIdx.x) * kPer0 >= n) {  // no node block for this CTA: its partial row is zero
        for (int q = tid; q < (REP ? kQ : NE * kEffQ); q += kAdjGridThreads)
            eff_partial[size_t(blockIdx.x) * pstride + q] = 0.0;
        return;
    }
    for (int q = lane; q < kQ; q += 32) wacc[warp * kQ + q] = 0.0;
    constexpr int kPer = kAdjGridThreads / 64;
    for (int k = blockIdx.x * kPer + sub; k < n; k += gridDim.x * kPer) {
        const int nbid = nb_list[k];
        int bx, by, bz;
        block_unlin(g, nbid, bx, by, bz);
        if (FILTER) {  // (uniform per node block: both warps skip together)
            const bool edge = bx == cols.c0 || bx == cols.c1;
            if (edge != (cols.cmode == 2)) continue;
        }
        const float4 sb = gather_tile_sum(g, blockmap, staging_bar, bx, by, bz, lx, ly, lz);
        V3<float> bar = {sb.x, sb.y, sb.z};
        const size_t idx = size_t(nbid) * 64 + l;
        const float4 g0 = gridv0[idx];
        const float m = g0.w;
        const V3<float> v0 = {g0.x, g0.y, g0.z};
        const bool live = m > g.mass_eps && (bar.x != 0.f || bar.y != 0.f || bar.z != 0.f);
        // effectors in contact range of this node, recorded by the forward grid update:
        // the others are pass-throughs and cost no SDF evaluation here
        const uint32_t cm = live ? uint32_t(cmask[idx]) : 0u;
        float pb0 = 0.f, pb1 = 0.f, pb2 = 0.f, mb = 0.f;
        if (__any_sync(0xffffffffu, live)) {  // warp-uniform: the effector reductions need all lanes
            const int rep = REP ? rep_of_col(g, bx) : 0;
            const EffK<float>* ek = REP ? eff.ext + rep * NE : eff.e;
            const int i = 4 * (bx - rep * g.rstride) + lx, j = 4 * by + ly, kk = 4 * bz + lz;
            const V3<float> p = {float(i) * g.dx, float(j) * g.dx, float(kk) * g.dx};
            const V3<float> v1 = {v0.x + g.gdt[0], v0.y + g.gdt[1], v0.z + g.gdt[2]};
            const V3<float> v2 = wall_bc_dev(g, i, j, kk, v1);
            V3<float> chain[NE > 0 ? NE : 1];
            V3<float> c = v2;
#pragma unroll
            for (int e = 0; e < NE; e++) {
                chain[e] = c;
                if ((cm >> e) & 1u) c = effector_contact(ek[e], g.inv_dx, g.eps_cells, g.hard != 0, p, c);
            }
            // ghost node column (bx == sx1): computed for this slab's gathers, counted by its owner
            const bool owned = bx < g.sx1;
#pragma unroll
            for (int e = NE - 1; e >= 0; e--) {
                EffBars<float> eb;
                eb.t = V3<float>{0.f, 0.f, 0.f};
                eb.R = mzero<float>();
                eb.vlin = eb.t;
                eb.w = eb.t;
                V3<float> in_bar = bar;  // pass-through unless in contact
                bool hit = false;
                if ((cm >> e) & 1u) {
                    in_bar = V3<float>{0.f, 0.f, 0.f};
                    hit = effector_contact_vjp(ek[e], g.dx, g.inv_dx, g.eps_cells, g.hard != 0, p, chain[e], bar,
                                               in_bar, eb) &&
                          owned;
                }
                if (__any_sync(0xffffffffu, hit)) {
                    float vals[kEffQ] = {eb.t.x, eb.t.y, eb.t.z, eb.R.m[0], eb.R.m[1], eb.R.m[2], eb.R.m[3],
                                         eb.R.m[4], eb.R.m[5], eb.R.m[6], eb.R.m[7], eb.R.m[8], eb.vlin.x,
                                         eb.vlin.y, eb.vlin.z, eb.w.x, eb.w.y, eb.w.z};
#pragma unroll
                    for (int q = 0; q < kEffQ; q++) {
                        float v = hit ? vals[q] : 0.f;
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                        if (lane == 0) wacc[warp * kQ + (rep * NE + e) * kEffQ + q] += double(v);
                    }
                }
                if (live) bar = in_bar;
            }
            if (live) {
                if (v2.x != v1.x) bar.x = 0.f;
                if (v2.y != v1.y) bar.y = 0.f;
                if (v2.z != v1.z) bar.z = 0.f;
                const float inv = 1.0f / m;
                pb0 = bar.x * inv;
                pb1 = bar.y * inv;
                pb2 = bar.z * inv;
                mb = -dot(v0, bar) * inv;
            }
        }
        gridbar[idx] = make_float4(pb0, pb1, pb2, mb);
    }
    __syncthreads();
    // only the effectors' components: the final sums read no further (nq = n_eff * 18)
    for (int q = tid; q < (REP ? kQ : NE * kEffQ); q += kAdjGridThreads) {
        double s = 0.0;
        for (int w = 0; w < kW; w++) s += wacc[w * kQ + q];
        eff_partial[size_t(blockIdx.x) * pstride + q] = s;
    }
}

// final effector-bar sums of `count` consecutive substeps [t0, t0 + count) whose
// CTA partials sit in a ring of kEffRing slots (deferred: one launch per ring,
// not per substep); one CTA per (substep, effector component): strided thread
// sums + fixed shuffle tree
// pstride: doubles per partial row / per substep of out (effector slots x 18)
__global__ void __launch_bounds__(256) k_eff_final(const double* ring, int nblocks, int nq, long t0, double* out,
                                                   int pstride) {
    pdl_wait();
    __shared__ double wsum[8];
    const int q = blockIdx.x % nq, tid = threadIdx.x;
    const long t = t0 + blockIdx.x / nq;
    const double* partial = ring + size_t(t % kEffRing) * nblocks * pstride;
    out += size_t(t) * pstride;
    double s = 0.0;
    for (int b = tid; b < nblocks; b += 256) s += partial[size_t(b) * pstride + q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((tid & 31) == 0) wsum[tid >> 5] = s;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; w++) t += wsum[w];
        out[q] = t;
    }
}

template <bool F, bool R>
static void launch_adj_grid_t(const Geom& g, const int* nb_list, const int* n_nb, const int* blockmap,
                              const float4* staging_bar, const float4* gridv0, float4* gridbar, const EffSet& eff,
                              double* eff_partial, const uint8_t* cmask, int nblocks, cudaStream_t s,
                              const GridCols& cols, int pstride) {
    const dim3 gr(nblocks), bl(kAdjGridThreads);
    const int ne = R ? eff.per_rep : eff.n;
    const size_t smem = R ? size_t(kAdjGridThreads / 32) * eff.n * kEffQ * sizeof(double) : 0;
#define FL_ADJGRID_CASE(NE)                                                                                        \
    {                                                                                                              \
        auto k = k_adj_grid<NE, F, R>;                                                                             \
        if (R) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));                   \
        launch_k(k, gr, bl, smem, s, g, nb_list, n_nb, blockmap, staging_bar, gridv0, gridbar, eff, eff_partial,   \
                 cmask, cols, pstride);                                                                            \
    }
    switch (ne) {
        case 0: FL_ADJGRID_CASE(0) break;
        case 1: FL_ADJGRID_CASE(1) break;
        case 2: FL_ADJGRID_CASE(2) break;
        case 3: FL_ADJGRID_CASE(3) break;
        default: FL_ADJGRID_CASE(kMaxEff)
    }
#undef FL_ADJGRID_CASE
}

// pstride: doubles per CTA partial row (effector slots x 18)
void launch_adj_grid(const Geom& g, const int* nb_list, const int* n_nb, const int* blockmap,
                     const float4* staging_bar, const float4* gridv0, float4* gridbar, const EffSet& eff,
                     double* eff_partial, const uint8_t* cmask, int nblocks, int pstride, cudaStream_t s, int cmode,
                     int c0, int c1) {
    const GridCols cols{cmode, c0, c1};
    if (eff.ext)
        launch_adj_grid_t<false, true>(g, nb_list, n_nb, blockmap, staging_bar, gridv0, gridbar, eff, eff_partial,
                                       cmask, nblocks, s, cols, pstride);
    else if (cmode)
        launch_adj_grid_t<true, false>(g, nb_list, n_nb, blockmap, staging_bar, gridv0, gridbar, eff, eff_partial,
                                       cmask, nblocks, s, cols, pstride);
    else
        launch_adj_grid_t<false, false>(g, nb_list, n_nb, blockmap, staging_bar, gridv0, gridbar, eff, eff_partial,
                                        cmask, nblocks, s, cols, pstride);
}

void launch_eff_final(const double* ring, int nblocks, int n_eff, long t0, int count, double* eff_out, int pstride,
                      cudaStream_t s) {
    if (n_eff <= 0 || count <= 0) return;
    launch_k(k_eff_final, dim3(count * n_eff * kEffQ), dim3(256), 0, s, ring, nblocks, n_eff * kEffQ, t0, eff_out,
             pstride);
}

// ---------------------------------------------------------------------------
// P2G adjoint (adjoint.hpp:414-470)
// ---------------------------------------------------------------------------
// pre-state / partial sources of adj_p2g_particle
struct AdjP2gGlobal {
    const PBuf& pre;
    const float* __restrict__ xbar_tmp;
    const float* __restrict__ Fbar_tmp;
    uint32_t s;
    int j, cap;
    __device__ float x(int a) const { return pre.x(a)[s]; }
    __device__ float v(int a) const { return pre.v(a)[s]; }
    __device__ uint32_t meta() const { return pre.meta[s]; }
    __device__ float C(int k) const { return pre.C(k)[s]; }
    __device__ float F(int k) const { return pre.F(k)[s]; }
    __device__ float xbar(int a) const { return xbar_tmp[size_t(a) * cap + j]; }
    __device__ float fbar(int k) const { return Fbar_tmp[size_t(k) * cap + j]; }
};
// plain-liquid staging: 21 fields per particle, [field][particle] in shared memory
constexpr int kAp2gF = 21;  // x3 v3 meta C9 c xbar3 cbar
#ifndef FL_ADJP2G_STAGE
#define FL_ADJP2G_STAGE 1
#endif
struct AdjP2gStaged {
    const float* sp;  // [kAp2gF][n]
    int k, n;
    __device__ float f(int q) const { return sp[q * n + k]; }
    __device__ float x(int a) const { return f(a); }
    __device__ float v(int a) const { return f(3 + a); }
    __device__ uint32_t meta() const { return __float_as_uint(f(6)); }
    __device__ float C(int q) const { return f(7 + q); }
    __device__ float F(int) const { return f(16); }  // (compact: c)
    __device__ float xbar(int a) const { return f(17 + a); }
    __device__ float fbar(int) const { return f(20); }
};

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}

// the P2G adjoint of one particle (adjoint.hpp:414-470): stress recompute + VJP, gather of
// (p_bar, m_bar) from the block's tile `bt`, bars written at storage slot s.  Src supplies
// the pre-state fields and the G2P adjoint's x_bar / F_bar partials (global memory through
// the permutation, or the CTA's cp.async staging).
template <bool HEAVY, class Src>
__device__ __forceinline__ void adj_p2g_particle(const Geom& g, const Src& src, uint32_t s,
                                                 const ClassInfo* __restrict__ cls, const float4* bt, int bx, int by,
                                                 int bz, BarBuf out, int* nonfinite) {
        const V3<float> x = {src.x(0), src.x(1), src.x(2)};
        const V3<float> v = {src.v(0), src.v(1), src.v(2)};
        const uint32_t pmeta = src.meta();
        const ClassInfo ci = cls[meta_cls(pmeta)];
        const bool cin = !HEAVY || f_compact(ci, pmeta);     // F = c I, F_bar stored as dL/dc
        const bool pressure = !HEAVY || (cin && ci.kind == MK_LIQUID);  // stress_mat = s(c) I
        M3<float> F, C;
#pragma unroll
        for (int k = 0; k < 9; k++) C.m[k] = src.C(k);
        if (cin) {
            F = meye<float>() * src.F(0);
        } else {
#pragma unroll
            for (int k = 0; k < 9; k++) F.m[k] = src.F(k);
        }
        const float cc = g.stress_coeff * ci.vol0;
        const bool visc = HEAVY && ci.kind == MK_VISCOUS;
        const M3<float> ipc = meye<float>() + C * g.dt;
        M3<float> fs, P, affine = C * ci.mass;
        Svd<float> t;
        if (pressure) {  // lambda (J - 1) J I with J = c^3
            const float c = F.m[0], jj = c * c * c;
            const float sm = ci.lambda * (jj - 1.f) * jj * cc;
            affine.m[0] -= sm;
            affine.m[4] -= sm;
            affine.m[8] -= sm;
        } else {
            fs = visc ? ipc * F : F;
            bool ok;
            P = corotated_stress_svd(fs, ci.mu, ci.lambda, ok, t);
            affine -= (P * transpose(fs)) * cc;
        }
        StencilW sw;
        stencil_weights(g, x, bx, by, bz, sw);
        const V3<float> mv = v * ci.mass;
        V3<float> xb = {0.f, 0.f, 0.f}, vbsum = {0.f, 0.f, 0.f};
        M3<float> ab = mzero<float>();
        float wsum_p[3] = {0.f, 0.f, 0.f};
        {
            // contrib_o = mv + affine rel_o with rel_o = dx (o - fx) split per axis;
            // grad-w products accumulated per x-plane; A_bar = sum_o w_o p_bar_o rel_o^T
            // gathered column-wise (x column through the per-plane sum).
            V3<float> ay[3], az[3];
            float ry[3], rz[3];
#pragma unroll
            for (int o = 0; o < 3; o++) {
                ry[o] = (float(o) - sw.fx[1]) * g.dx;
                rz[o] = (float(o) - sw.fx[2]) * g.dx;
                ay[o] = V3<float>{affine.m[1] * ry[o], affine.m[4] * ry[o], affine.m[7] * ry[o]};
                az[o] = V3<float>{affine.m[2] * rz[o], affine.m[5] * rz[o], affine.m[8] * rz[o]};
            }
            const float mm = ci.mass;
            const float wrz[3] = {sw.w[2][0] * rz[0], sw.w[2][1] * rz[1], sw.w[2][2] * rz[2]};
            float sxx = 0.f, syy = 0.f, szz = 0.f;
#pragma unroll 1
            for (int ox = 0; ox < 3; ox++) {
                const float wox = ox == 0 ? sw.w[0][0] : (ox == 1 ? sw.w[0][1] : sw.w[0][2]);
                const float dox = ox == 0 ? sw.dw[0][0] : (ox == 1 ? sw.dw[0][1] : sw.dw[0][2]);
                const float rx = (float(ox) - sw.fx[0]) * g.dx;
                const V3<float> ax = {mv.x + affine.m[0] * rx, mv.y + affine.m[3] * rx, mv.z + affine.m[6] * rx};
                float px = 0.f, py = 0.f, pz = 0.f;
                V3<float> tx = {0.f, 0.f, 0.f};
                const float4* row = bt + (sw.l[0] + ox) * 36 + sw.l[1] * 6 + sw.l[2];
#pragma unroll
                for (int oy = 0; oy < 3; oy++) {
                    const V3<float> axy = ax + ay[oy];
                    // per (x, y) column: z-weighted sums, then one scaling by the x/y weights
                    float sa = 0.f, sb = 0.f;
                    V3<float> tz = {0.f, 0.f, 0.f}, tzr = {0.f, 0.f, 0.f};
#pragma unroll
                    for (int oz = 0; oz < 3; oz++) {
                        const float4 b4 = row[oy * 6 + oz];
                        const V3<float> u = axy + az[oz];
                        const float sv = b4.w * mm + b4.x * u.x + b4.y * u.y + b4.z * u.z;
                        sa += sw.w[2][oz] * sv;
                        sb += sw.dw[2][oz] * sv;
                        tz += V3<float>{b4.x, b4.y, b4.z} * sw.w[2][oz];
                        tzr += V3<float>{b4.x, b4.y, b4.z} * wrz[oz];
                    }
                    px += sw.w[1][oy] * sa;
                    py += sw.dw[1][oy] * sa;
                    pz += sw.w[1][oy] * sb;
                    const float wxy = wox * sw.w[1][oy];
                    const V3<float> wob = tz * wxy;
                    tx += wob;
                    ab.m[1] += wob.x * ry[oy]; ab.m[4] += wob.y * ry[oy]; ab.m[7] += wob.z * ry[oy];
                    ab.m[2] += tzr.x * wxy; ab.m[5] += tzr.y * wxy; ab.m[8] += tzr.z * wxy;
                }
                sxx += dox * px;
                syy += wox * py;
                szz += wox * pz;
                ab.m[0] += tx.x * rx; ab.m[3] += tx.y * rx; ab.m[6] += tx.z * rx;
                wsum_p[0] += tx.x;
                wsum_p[1] += tx.y;
                wsum_p[2] += tx.z;
            }
            xb = V3<float>{sxx * g.inv_dx, syy * g.inv_dx, szz * g.inv_dx};
        }
        const V3<float> wp = {wsum_p[0], wsum_p[1], wsum_p[2]};
        xb -= tmul(affine, wp);
        vbsum = wp * ci.mass;
        const M3<float> sm_bar = ab * (-cc);
        M3<float> Fb, Cb = ab * ci.mass;
        float c_bar = 0.f;  // dL/dc for a compact F
        if (pressure) {
            // d/dc [lambda (c^6 - c^3)] tr(sm_bar) = 3 lambda c^2 (2J - 1) tr(sm_bar)
            const float c = F.m[0], jj = c * c * c;
            c_bar = src.fbar(0) + 3.f * ci.lambda * c * c * (2.f * jj - 1.f) * trace(sm_bar);
        } else {
            const M3<float> p_bar = sm_bar * fs;
            M3<float> fs_bar = transpose(sm_bar) * P;
            fs_bar += corotated_stress_vjp(fs, ci.mu, ci.lambda, p_bar, t);
            M3<float> fb_add = fs_bar;
            if (visc) {
                fb_add = transpose(ipc) * fs_bar;
                Cb += fs_bar * transpose(F) * g.dt;
            }
            if (cin) {
                c_bar = src.fbar(0) + trace(fb_add);
            } else {
#pragma unroll
                for (int k = 0; k < 9; k++) Fb.m[k] = src.fbar(k) + fb_add.m[k];
            }
        }
        const float xo[3] = {src.xbar(0) + xb.x, src.xbar(1) + xb.y, src.xbar(2) + xb.z};
#pragma unroll
        for (int a = 0; a < 3; a++) {
            out.x(a)[s] = xo[a];
            out.v(a)[s] = vbsum[a];
        }
#pragma unroll
        for (int k = 0; k < 9; k++) out.C(k)[s] = Cb.m[k];
        if (cin) {
            out.F(0)[s] = c_bar;
        } else {
#pragma unroll
            for (int k = 0; k < 9; k++) out.F(k)[s] = Fb.m[k];
        }
        if (!isfinite(xo[0]) || !isfinite(vbsum.x) || !isfinite(cin ? c_bar : Fb.m[0])) atomicOr(nonfinite, 1);
}

// a few SVD/rigid P2G-adjoint blocks beside a liquid scene (variant 3) in 256-thread CTAs:
// their stress VJP per particle makes them the dual launch's tail, and a full block then
// takes two rounds instead of four (c4 92.8 -> 82.4 us; c5's many such blocks: variant 1)
#ifndef FL_ADJP2G_NTH
#define FL_ADJP2G_NTH 256
#endif
template <bool HEAVY, int MINB, int NT = 128>
__global__ void __launch_bounds__(NT, MINB) k_adj_p2g(Geom g, PBuf pre, const uint32_t* __restrict__ perm,
                                                 const BlockRec* __restrict__ recs, const int* __restrict__ n_blocks,
                                                 const ClassInfo* __restrict__ cls,
                                                 const float4* __restrict__ gridbar,
                                                 const float* __restrict__ xbar_tmp,
                                                 const float* __restrict__ Fbar_tmp, BarBuf out, int* nonfinite,
                                                 int cap, int* wq, int role) {
    const DualScope dual_scope(role);
    __shared__ float4 bt[kTile];
    __shared__ __align__(128) float4 raw[FL_TMA_TILE ? kTileRaw : 1];
    __shared__ __align__(8) uint64_t bar;
    constexpr int kStageBuf = (!HEAVY && FL_ADJP2G_STAGE) ? 2 * NT : 1;
    __shared__ __align__(16) float sp[kAp2gF * kStageBuf];
    __shared__ uint32_t ps[kStageBuf];
    const int tid = threadIdx.x;
    TileStage ts;
    ts.init(&bar, raw, tid);
    const int q0 = HEAVY ? g.maxb - n_blocks[1] : 0, q1 = HEAVY ? g.maxb : n_blocks[0];
    __shared__ int sh_next;
    __shared__ int s_wc[kWorkClasses];
    work_counts_load(n_blocks, HEAVY ? 1 : 0, s_wc, tid);
    for (;;) {
        const int k = next_work(wq, &sh_next);
        if (k >= q1 - q0) break;
        const int4 we = work_entry(n_blocks, g.maxb, HEAVY ? 1 : 0, k, s_wc);  // costliest blocks first
        const int b = we.x;
        const BlockRec r{we.y, we.z, we.w};
        int bx, by, bz;
        block_unlin(g, r.block, bx, by, bz);
        ts.begin(g, gridbar, bx, by, bz, tid);
        const int bxl = bx - rep_of_col(g, bx) * g.rstride;  // replica-local column (the weights)
        uint32_t s_nx = (HEAVY || !FL_ADJP2G_STAGE) && r.start + tid < r.end ? perm[r.start + tid] : 0u;  // see k_g2p
        ts.end(g, gridbar, bt, bx, by, bz, tid, NT);
        __syncthreads();
        if constexpr (!HEAVY && FL_ADJP2G_STAGE) {
            // plain liquids: chunks of kStage particles -- every thread issues cp.async
            // copies of its particles' 21 fields (independent loads, no register round trip,
            // no perm -> state dependency per use), then the chunk computes from shared memory
            constexpr int kStage = 2 * NT;
            for (int c0 = r.start; c0 < r.end; c0 += kStage) {
                const int cn = min(kStage, r.end - c0);
                __syncthreads();  // the previous chunk's reads are done
                for (int k = tid; k < cn; k += NT) {
                    const int j = c0 + k;
                    const uint32_t s = perm[j];
                    ps[k] = s;
#pragma unroll
                    for (int a = 0; a < 3; a++) {
                        cp_async4(&sp[a * kStage + k], pre.x(a) + s);
                        cp_async4(&sp[(3 + a) * kStage + k], pre.v(a) + s);
                        cp_async4(&sp[(17 + a) * kStage + k], xbar_tmp + size_t(a) * cap + j);
                    }
                    cp_async4(&sp[6 * kStage + k], pre.meta + s);
#pragma unroll
                    for (int q = 0; q < 9; q++) cp_async4(&sp[(7 + q) * kStage + k], pre.C(q) + s);
                    cp_async4(&sp[16 * kStage + k], pre.F(0) + s);
                    cp_async4(&sp[20 * kStage + k], Fbar_tmp + j);
                }
                asm volatile("cp.async.commit_group;\n cp.async.wait_group 0;" ::: "memory");
                __syncthreads();
                for (int k = tid; k < cn; k += NT)
                    adj_p2g_particle<HEAVY>(g, AdjP2gStaged{sp, k, kStage}, ps[k], cls, bt, bxl, by, bz, out,
                                            nonfinite);
            }
        } else {
            for (int j = r.start + tid; j < r.end; j += NT) {
                const uint32_t s = s_nx;
                if (j + NT < r.end) s_nx = perm[j + NT];
                adj_p2g_particle<HEAVY>(g, AdjP2gGlobal{pre, xbar_tmp, Fbar_tmp, s, j, cap}, s, cls, bt, bxl, by, bz,
                                        out, nonfinite);
            }
        }
    }
}


static decltype(&k_adj_p2g<false, FL_LB_ADJP2G>) adj_p2g_kernel(int v) {
    switch (v) {
        case 0: return k_adj_p2g<false, FL_LB_ADJP2G>;
        case 1: return k_adj_p2g<true, FL_LBH_ADJP2G>;
        case 2: return k_adj_p2g<true, FL_LBD_ADJP2G>;
        default: return k_adj_p2g<true, FL_LBF_ADJP2G, FL_ADJP2G_NTH>;
    }
}
static int adj_p2g_threads(int v) { return v == 3 ? FL_ADJP2G_NTH : 128; }

void launch_adj_p2g(const Geom& g, PBuf pre, const uint32_t* perm, const BlockRec* recs, const int* n_blocks,
                    int grid, const ClassInfo* cls, const float4* gridbar, const float* xbar_tmp,
                    const float* Fbar_tmp, BarBuf out, int* nonfinite, int variant, int* wq, cudaStream_t s) {
    launch_k(adj_p2g_kernel(variant), dim3(grid), dim3(adj_p2g_threads(variant)), 0, s, g, pre, perm, recs, n_blocks, cls, gridbar,
             xbar_tmp, Fbar_tmp, out, nonfinite, out.cap, wq, dual_role());
}

// inactive particles pass their bars through untouched
// parked particles pass their cotangents through; departed slots (sorted
// positions [n_keep, n_stored)) get zero -- a migrated particle's cotangent is
// returned by its new slab before the previous substep's adjoint
__global__ void k_tail_bars(BarBuf post, BarBuf out, const uint32_t* __restrict__ perm, DN n0, DN nk, DN ns) {
    pdl_wait();
    const int n_keep = nk.get(), n_stored = ns.get();
    for (int j = n0.get() + blockIdx.x * blockDim.x + threadIdx.x; j < n_stored; j += gridDim.x * blockDim.x) {
        uint32_t s = perm[j];
        if (j < n_keep)
            for (int c = 0; c < 24; c++) out.f[size_t(c) * out.cap + s] = post.f[size_t(c) * post.cap + j];
        else
            for (int c = 0; c < 24; c++) out.f[size_t(c) * out.cap + s] = 0.f;
    }
}

void launch_tail_bars(BarBuf post, BarBuf out, const uint32_t* perm, DN n_active, DN n_keep, DN n_stored,
                      cudaStream_t s) {
    // (slabs: h is an upper bound of the tail length)
    int m = n_stored.h - (n_active.d ? 0 : n_active.h);
    if (m <= 0) return;
    launch_k(k_tail_bars, dim3(gs_grid(m)), dim3(256), 0, s, post, out, perm, n_active, n_keep, n_stored);
}

// emitter spawn adjoint, sequential over the substep's spawns (fixed order)
struct EmitBatch {
    int n;
    EmitAdjEntry e[kEmitInline];
};

__global__ void k_adj_emit(BarBuf out, const EmitAdjEntry* list, int n, double* em_out, int n_eff, EmitBatch inl,
                           const int* slot_base) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int q = 0; q < n_eff * 12; q++) em_out[q] = 0.0;
    const int base = slot_base ? *slot_base : 0;  // slabs: slots relative to the parked tail
    for (int i = 0; i < n; i++) {
        EmitAdjEntry e = list ? list[i] : inl.e[i];
        e.slot += base;
        double xb[3], vb[3];
        for (int a = 0; a < 3; a++) {
            xb[a] = out.x(a)[e.slot];
            vb[a] = out.v(a)[e.slot];
            out.x(a)[e.slot] = 0.f;
            out.v(a)[e.slot] = 0.f;
        }
        if (e.eff < 0) continue;
        for (int a = 0; a < 3; a++)
            if (e.mask[a]) xb[a] = 0.0;
        double* o = em_out + 12 * size_t(e.eff);
        for (int a = 0; a < 3; a++) o[a] += xb[a];
        for (int a = 0; a < 3; a++)
            for (int b = 0; b < 3; b++) o[3 + 3 * a + b] += xb[a] * e.local_pos[b] + vb[a] * e.local_vel[b];
    }
}

void launch_adj_emit(BarBuf out, const EmitAdjEntry* list, int n, double* em_out, int n_eff, const int* slot_base,
                     cudaStream_t s) {
    k_adj_emit<<<1, 32, 0, s>>>(out, list, n, em_out, n_eff, EmitBatch{}, slot_base);
}

void launch_adj_emit_inline(BarBuf out, const EmitAdjEntry* host_list, int n, double* em_out, int n_eff,
                            const int* slot_base, cudaStream_t s) {
    EmitBatch b{};
    b.n = n;
    for (int i = 0; i < n; i++) b.e[i] = host_list[i];
    k_adj_emit<<<1, 32, 0, s>>>(out, nullptr, n, em_out, n_eff, b, slot_base);
}

// ---------------------------------------------------------------------------
// bars <-> reference (particle id) order
// ---------------------------------------------------------------------------
// reference-layout cotangents <-> store order; a compact F's cotangent is dL/dc = tr(F_bar)
__global__ void k_bars_from_ref(BarBuf bars, PBuf st, int n, const double* xb, const double* vb, const double* Fb,
                                const double* Cb, const ClassInfo* __restrict__ cls) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    size_t id = st.id[i];
    const uint32_t meta = st.meta[i];
    const bool cf = f_compact(cls[meta_cls(meta)], meta);
    for (int a = 0; a < 3; a++) {
        bars.x(a)[i] = float(xb[3 * id + a]);
        bars.v(a)[i] = float(vb[3 * id + a]);
    }
    for (int k = 0; k < 9; k++) {
        bars.F(k)[i] = float(Fb[9 * id + k]);
        bars.C(k)[i] = float(Cb[9 * id + k]);
    }
    if (cf) bars.F(0)[i] = float(Fb[9 * id] + Fb[9 * id + 4] + Fb[9 * id + 8]);
}

void launch_bars_from_ref(BarBuf bars, const PBuf& st, int n, const double* xb, const double* vb, const double* Fb,
                          const double* Cb, const ClassInfo* cls, cudaStream_t s) {
    if (n <= 0) return;
    k_bars_from_ref<<<(n + 255) / 256, 256, 0, s>>>(bars, st, n, xb, vb, Fb, Cb, cls);
}

__global__ void k_bars_to_ref(BarBuf bars, PBuf st, int n, double* xb, double* vb, double* Fb, double* Cb,
                              const ClassInfo* __restrict__ cls) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    size_t id = st.id[i];
    const uint32_t meta = st.meta[i];
    const bool cf = f_compact(cls[meta_cls(meta)], meta);
    for (int a = 0; a < 3; a++) {
        xb[3 * id + a] = bars.x(a)[i];
        vb[3 * id + a] = bars.v(a)[i];
    }
    for (int k = 0; k < 9; k++) {
        Fb[9 * id + k] = cf ? (k % 4 == 0 ? double(bars.F(0)[i]) / 3.0 : 0.0) : double(bars.F(k)[i]);
        Cb[9 * id + k] = bars.C(k)[i];
    }
}

void launch_bars_to_ref(BarBuf bars, const PBuf& st, int n, double* xb, double* vb, double* Fb, double* Cb,
                        const ClassInfo* cls, cudaStream_t s) {
    if (n <= 0) return;
    k_bars_to_ref<<<(n + 255) / 256, 256, 0, s>>>(bars, st, n, xb, vb, Fb, Cb, cls);
}

// adjoint_substep API: every compact F of the pre-state in full (kMetaFull), so
// the substep's F cotangent comes out as the reference's full 3x3
__global__ void k_expand_f(PBuf st, int n, const ClassInfo* __restrict__ cls) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t meta = st.meta[i];
    if (!f_compact(cls[meta_cls(meta)], meta)) return;
    const float c = st.F(0)[i];
    for (int k = 1; k < 9; k++) st.F(k)[i] = k % 4 == 0 ? c : 0.f;
    st.meta[i] = meta | kMetaFull;
}

void launch_expand_f(PBuf st, int n, const ClassInfo* cls, cudaStream_t s) {
    if (n <= 0) return;
    k_expand_f<<<(n + 255) / 256, 256, 0, s>>>(st, n, cls);
}

int occupancy_grid_fwd(KGrid which, int variant);

int occupancy_grid(KGrid which, int variant) {
    if (which == KG_P2G || which == KG_G2P) return occupancy_grid_fwd(which, variant);
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (which == KG_ADJ_G2P) {
        const size_t smem = sizeof(ScSmem) + kTile * sizeof(float4);
        cudaFuncSetAttribute(adj_g2p_kernel(variant), cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, adj_g2p_kernel(variant), adj_g2p_threads(variant), smem);
    } else {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, adj_p2g_kernel(variant), adj_p2g_threads(variant), 0);
    }
    if (per < 1) per = 1;
    return sms * per;
}

}  // namespace fl
