// fl_fwd.cu -- forward MLS-MPM substep kernels for sm_100a.
//
// One substep (proj/include/flume/mpm.hpp:455-473) is
//   activate -> keys/sort -> P2G -> grid update -> G2P (+projection) -> rigid
// with the particle store kept in canonical (cell key, id) order.  P2G and the
// G2P-adjoint scatter are deterministic without atomics: a CTA owns one 4^3
// particle block, accumulates each base cell's 27 node contributions in
// registers in sorted-particle order, folds cells into the block's 6^3 node
// tile in a fixed order and writes the tile to a per-block staging slot.  The
// grid update then sums the (at most 8) staging tiles that cover a node in a
// fixed order.  Every float sum therefore has a run-independent order.
#include <cuda_runtime.h>

#include <cstdio>

#include "fl_kernels.h"
#include "fl_scatter.cuh"

namespace fl {

// ---------------------------------------------------------------------------
// upload / download / permutation
// ---------------------------------------------------------------------------

__global__ void k_upload(Geom g, PBuf raw, int n, const double* __restrict__ x, const double* __restrict__ v,
                         const double* __restrict__ F, const double* __restrict__ C,
                         const uint32_t* __restrict__ meta, const uint8_t* __restrict__ active,
                         const ClassInfo* __restrict__ cls, int* any_full) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int a = 0; a < 3; a++) {
        raw.x(a)[i] = float(x[3 * size_t(i) + a]);
        raw.v(a)[i] = float(v[3 * size_t(i) + a]);
    }
    for (int k = 0; k < 9; k++) {
        raw.F(k)[i] = float(F[9 * size_t(i) + k]);
        raw.C(k)[i] = float(C[9 * size_t(i) + k]);
    }
    // the full F is stored; an isotropic-class particle whose F is not c I keeps
    // it in full (kMetaFull) until its first G2P
    bool isotropic = true;
    for (int k = 0; k < 9; k++)
        if (k % 4 != 0 && raw.F(k)[i] != 0.f) isotropic = false;
    if (raw.F(4)[i] != raw.F(0)[i] || raw.F(8)[i] != raw.F(0)[i]) isotropic = false;
    const bool full = cls[meta[i]].iso && !isotropic;
    raw.meta[i] = meta[i] | (full ? kMetaFull : 0u);
    if (full) *any_full = 1;  // (the host reads it after the upload: heavy paths possible)
    raw.id[i] = uint32_t(i);
    // active: 0 = parked (activates later), 1 = active here, 2 = active on another slab
    uint32_t key = g.key_inactive;
    if (active[i]) cell_key(g, raw.x(0)[i], raw.x(1)[i], raw.x(2)[i], key, cls[meta[i]].rep);
    if (active[i] == 2) key = g.key_departed;
    raw.key[i] = key;
}

void launch_upload(const Geom& g, PBuf raw, int n, const double* x, const double* v, const double* F,
                   const double* C, const uint32_t* meta, const uint8_t* active, const ClassInfo* cls,
                   int* any_full, cudaStream_t s) {
    if (n <= 0) return;
    k_upload<<<(n + 255) / 256, 256, 0, s>>>(g, raw, n, x, v, F, C, meta, active, cls, any_full);
}

__global__ void k_gather(PBuf in, PBuf out, const uint32_t* __restrict__ perm, int n) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    uint32_t s = perm[j];
#pragma unroll
    for (int c = 0; c < 24; c++) out.f[size_t(c) * out.cap + j] = in.f[size_t(c) * in.cap + s];
    out.meta[j] = in.meta[s];
    out.id[j] = in.id[s];
    out.key[j] = in.key[s];
}

void launch_gather(PBuf in, PBuf out, const uint32_t* perm, int n, cudaStream_t s) {
    if (n <= 0) return;
    k_gather<<<(n + 255) / 256, 256, 0, s>>>(in, out, perm, n);
}

// by particle id; departed slots are skipped, parked particles (replicated on
// every slab) only where write_parked is set
__global__ void k_download(PBuf st, int n, double* x, double* v, double* F, double* C, int write_parked,
                           uint32_t key_inactive, const ClassInfo* __restrict__ cls) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t key = st.key[i];
    if (key > key_inactive || (key == key_inactive && !write_parked)) return;
    size_t id = st.id[i];
    const uint32_t meta = st.meta[i];
    const bool cf = f_compact(cls[meta_cls(meta)], meta);
    for (int a = 0; a < 3; a++) {
        if (x) x[3 * id + a] = double(st.x(a)[i]);
        if (v) v[3 * id + a] = double(st.v(a)[i]);
    }
    for (int k = 0; k < 9; k++) {
        if (F) F[9 * id + k] = cf ? (k % 4 == 0 ? double(st.F(0)[i]) : 0.0) : double(st.F(k)[i]);
        if (C) C[9 * id + k] = double(st.C(k)[i]);
    }
}

void launch_download(PBuf st, int n, double* x, double* v, double* F, double* C, int write_parked,
                     uint32_t key_inactive, const ClassInfo* cls, cudaStream_t s) {
    if (n <= 0) return;
    k_download<<<(n + 255) / 256, 256, 0, s>>>(st, n, x, v, F, C, write_parked, key_inactive, cls);
}

__global__ void k_rigid_x(PBuf st, int nmem, const int* member_id, double* x, int dir) {
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nmem) return;
    size_t id = size_t(member_id[r]);
    for (int a = 0; a < 3; a++) {
        if (dir)
            x[3 * id + a] = st.mx[3 * size_t(r) + a];
        else
            st.mx[3 * size_t(r) + a] = x[3 * id + a];
    }
}

void launch_download_rigid(PBuf st, int nmem, const int* member_id, double* x, cudaStream_t s) {
    if (nmem <= 0) return;
    k_rigid_x<<<(nmem + 255) / 256, 256, 0, s>>>(st, nmem, member_id, x, 1);
}

void launch_upload_rigid(PBuf st, int nmem, const int* member_id, const double* x, cudaStream_t s) {
    if (nmem <= 0) return;
    k_rigid_x<<<(nmem + 255) / 256, 256, 0, s>>>(st, nmem, member_id, const_cast<double*>(x), 0);
}

// ---------------------------------------------------------------------------
// emitter activation (mpm.hpp:435-449); positions precomputed on the host in
// fp64 from the stage-a effector pose
// ---------------------------------------------------------------------------

// slot_base (slab contexts): the entries' slots are relative to the parked tail, whose
// first slot the device counts hold
__global__ void k_activate(Geom g, PBuf st, const ActEntry* list, int n, ActBatch inl, const int* slot_base) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const ActEntry e = list ? list[i] : inl.e[i];
    const int slot = e.slot + (slot_base ? *slot_base : 0);
    if (e.has_xv) {
        for (int a = 0; a < 3; a++) {
            st.x(a)[slot] = e.x[a];
            st.v(a)[slot] = e.v[a];
        }
    }
    uint32_t key;
    cell_key(g, st.x(0)[slot], st.x(1)[slot], st.x(2)[slot], key, e.rep);
    st.key[slot] = e.departed ? g.key_departed : key;  // departed: activates on another slab
}

void launch_activate(const Geom& g, PBuf st, const ActEntry* list, int n, const int* slot_base, cudaStream_t s) {
    if (n <= 0) return;
    k_activate<<<(n + 127) / 128, 128, 0, s>>>(g, st, list, n, ActBatch{}, slot_base);
}

void launch_activate_inline(const Geom& g, PBuf st, const ActEntry* host_list, int n, const int* slot_base,
                            cudaStream_t s) {
    if (n <= 0) return;
    ActBatch b{};
    b.n = n;
    for (int i = 0; i < n; i++) b.e[i] = host_list[i];
    k_activate<<<1, 128, 0, s>>>(g, st, nullptr, n, b, slot_base);
}

// ---------------------------------------------------------------------------
// P2G (mpm.hpp:249-287)
// ---------------------------------------------------------------------------

// NT threads: 192 (64 cells x 3 planes) for the plain-liquid blocks, whose accumulate
// phase dominates.  Variant 3: a few SVD/rigid blocks beside a liquid scene (fewer than
// one per SM) are the kernel's tail, and their payload (a polar SVD per particle)
// dominates, so they stage a full block in two even rounds of 256 threads (c4 76.8 ->
// 73.1 us); with many such blocks (c5) 192 threads keep more of them in flight (256:
// 444 -> 508 us), and SVD-dominated scenes (c3, variant 2) are even.
#ifndef FL_P2G_NTH
#define FL_P2G_NTH 256
#endif
template <bool HEAVY, int MINB, int NT>
__global__ void __launch_bounds__(NT, MINB) k_p2g(Geom g, PBuf st, const uint32_t* __restrict__ perm,
                                                    const BlockRec* __restrict__ recs,
                                                    const int* __restrict__ n_blocks,
                                                    const uint16_t* __restrict__ celltab,
                                                    const ClassInfo* __restrict__ cls, float4* staging,
                                                    unsigned long long* err, uint32_t substep, int* wq, int role) {
    const DualScope dual_scope(role);
    extern __shared__ __align__(16) unsigned char smraw[];
    ScSmem& sm = *reinterpret_cast<ScSmem*>(smraw);
    const int tid = threadIdx.x;
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
        bx -= rep_of_col(g, bx) * g.rstride;  // replica-local column (positions are local)
        __syncthreads();
        const int cnt = r.end - r.start;
        uint32_t s_nx = tid < cnt ? perm[r.start + tid] : 0u;  // overlaps the cell-table barrier
        sc_tile_zero(sm, tid, NT);
        const int npass = sc_load_cells(sm, celltab, b, tid);
        for (int pass = 0; pass < npass; pass++) {
            const int r0 = pass * kScR;
            const int lim = pass == 0 ? cnt : sc_overflow_prefix(sm, r0, tid);
            for (int it = tid; it < lim; it += NT) {
                int c, rank;
                uint32_t s;
                if (pass == 0) {  // every particle in sorted order (prefetching the permutation)
                    c = cell_of(sm.cs, it);
                    s = s_nx;
                    if (it + NT < cnt) s_nx = perm[r.start + it + NT];
                    rank = it - int(sm.cs[c]);
                    if (rank >= kScR) continue;
                } else {  // the dense list of the particles left for this pass
                    sc_overflow_item(sm, it, c, rank);
                    s = perm[r.start + int(sm.cs[c]) + r0 + rank];
                }
                float* pay = pay_slot(sm, rank, c);
                float fx[3];
                int b0 = base_cell(st.x(0)[s], g.inv_dx, fx[0]);
                int b1 = base_cell(st.x(1)[s], g.inv_dx, fx[1]);
                int b2 = base_cell(st.x(2)[s], g.inv_dx, fx[2]);
                uint32_t lc = uint32_t(((b0 - 4 * bx) << 4) | ((b1 - 4 * by) << 2) | (b2 - 4 * bz));
                bool inside = b0 >= 4 * bx && b0 < 4 * bx + 4 && b1 >= 4 * by && b1 < 4 * by + 4 && b2 >= 4 * bz &&
                              b2 < 4 * bz + 4 && lc == uint32_t(c) && b0 + 2 < g.nd[0] && b1 + 2 < g.nd[1] &&
                              b2 + 2 < g.nd[2];
                if (!inside) {
                    atomicMin(err, (unsigned long long)pack_err(substep, ES_P2G_ESCAPE, st.id[s]));
#pragma unroll
                    for (int q = 0; q < kPayF; q++) pay[q * kPayPlane] = 0.f;
                    pay[0] = pay[kPayPlane] = pay[2 * kPayPlane] = 1.f;
                    continue;
                }
                const uint32_t meta = st.meta[s];
                const ClassInfo ci = cls[meta_cls(meta)];
                M3<float> C;
#pragma unroll
                for (int k = 0; k < 9; k++) C.m[k] = st.C(k)[s];
                V3<float> v = {st.v(0)[s], st.v(1)[s], st.v(2)[s]};
                bool ok;
                M3<float> affine = C * ci.mass;
                if (!HEAVY || f_compact(ci, meta)) {
                    const float c = st.F(0)[s];
                    if (!HEAVY || ci.kind == MK_LIQUID) {
                        // F = c I, mu = 0: stress_mat = P F^T = lambda (J - 1) J I, J = c^3
                        const float j = c * c * c;
                        ok = j > 0.f;
                        const float sm = ci.lambda * (j - 1.f) * j * (g.stress_coeff * ci.vol0);
                        affine.m[0] -= sm;
                        affine.m[4] -= sm;
                        affine.m[8] -= sm;
                    } else {  // viscous liquid: Fs = (I + dt C) c
                        const M3<float> fs = (meye<float>() + C * g.dt) * c;
                        const M3<float> P = corotated_stress(fs, ci.mu, ci.lambda, ok);
                        affine -= (P * transpose(fs)) * (g.stress_coeff * ci.vol0);
                    }
                } else {
                    M3<float> F;
#pragma unroll
                    for (int k = 0; k < 9; k++) F.m[k] = st.F(k)[s];
                    M3<float> fs = F;
                    if (ci.kind == MK_VISCOUS) fs = (meye<float>() + C * g.dt) * F;
                    const M3<float> P = corotated_stress(fs, ci.mu, ci.lambda, ok);
                    affine -= (P * transpose(fs)) * (g.stress_coeff * ci.vol0);
                }
                if (!ok) atomicMin(err, (unsigned long long)pack_err(substep, ES_P2G_STRESS, st.id[s]));
                V3<float> f3 = {fx[0], fx[1], fx[2]};
                V3<float> a = v * ci.mass - (affine * f3) * g.dx;
                pay[0] = fx[0];
                pay[kPayPlane] = fx[1];
                pay[2 * kPayPlane] = fx[2];
                pay[3 * kPayPlane] = ci.mass;
                pay[4 * kPayPlane] = a.x;
                pay[5 * kPayPlane] = a.y;
                pay[6 * kPayPlane] = a.z;
#pragma unroll
                for (int k = 0; k < 9; k++) pay[(7 + k) * kPayPlane] = affine.m[k] * g.dx;
            }
            __syncthreads();
            const int nr = my_ox < 3 ? min(max(int(sm.cs[my_c + 1]) - int(sm.cs[my_c]) - r0, 0), kScR) : 0;
            sc_accumulate<4>(sm, my_c, my_ox, nr, tid, NT);
            __syncthreads();
        }
        __syncthreads();
        sc_tile_store(sm, staging + size_t(b) * kTile, tid, NT);
    }
}

// kernel variant: 0 plain liquid, 1 SVD/rigid blocks in a mostly-liquid scene (low
// occupancy, runs beside the light kernel), 2 SVD/rigid-dominated scene
static decltype(&k_p2g<false, FL_LB_P2G, kScThreads>) p2g_kernel(int v) {
    switch (v) {
        case 0: return k_p2g<false, FL_LB_P2G, kScThreads>;
        case 1: return k_p2g<true, FL_LBH_P2G, kScThreads>;
        case 2: return k_p2g<true, FL_LBD_P2G, kScThreads>;
        default: return k_p2g<true, FL_LBH_P2G, FL_P2G_NTH>;
    }
}
static int p2g_threads(int v) { return v == 3 ? FL_P2G_NTH : kScThreads; }

void launch_p2g(const Geom& g, PBuf st, const uint32_t* perm, const BlockRec* recs, const int* n_blocks,
                const uint16_t* celltab, int grid, const ClassInfo* cls, float4* staging, unsigned long long* err,
                uint32_t substep, int variant, int* wq, cudaStream_t s) {
    static bool attr[4] = {false, false, false, false};
    if (!attr[variant]) {
        cudaFuncSetAttribute(p2g_kernel(variant), cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(ScSmem)));
        attr[variant] = true;
    }
    launch_k(p2g_kernel(variant), dim3(grid), dim3(p2g_threads(variant)), sizeof(ScSmem), s, g, st, perm, recs, n_blocks,
             celltab, cls, staging, err, substep, wq, dual_role());
}

// ---------------------------------------------------------------------------
// grid update (mpm.hpp:289-320): one thread per node of each touched node block
// ---------------------------------------------------------------------------

__device__ __forceinline__ float4 gather_staging(const Geom& g, const int* __restrict__ blockmap,
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

#ifndef FL_GRIDUPD_THREADS
#define FL_GRIDUPD_THREADS 256
#endif
constexpr int kGridUpdThreads = FL_GRIDUPD_THREADS;  // 64 nodes (one node block) per 64 threads

// FILTER: the column filter, slab contexts only (it costs the plain path ~2 us); REP: replica
// contexts (local node coordinates, the replica's effectors from device memory; also ~2 us)
template <bool FILTER, bool REP>
__global__ void __launch_bounds__(kGridUpdThreads) k_grid_update(Geom g, const int* __restrict__ nb_list,
                                                     const int* __restrict__ n_nb, const int* __restrict__ blockmap,
                                                     const float4* __restrict__ staging, float4* gridv, float4* gridv0,
                                                     EffSet eff, uint8_t* cmask, int* clear, int n_clear,
                                                     GridCols cols) {
    pdl_wait();
    // the sort's counters are dead by now: clear them for the next substep's sort
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_clear; i += gridDim.x * blockDim.x) clear[i] = 0;
    const int n = *n_nb;
    const int sub = threadIdx.x >> 6, l = threadIdx.x & 63;
    const int lx = l >> 4, ly = (l >> 2) & 3, lz = l & 3;
    constexpr int kPer = kGridUpdThreads / 64;
    for (int k = blockIdx.x * kPer + sub; k < n; k += gridDim.x * kPer) {
        const int nbid = nb_list[k];
        int bx, by, bz;
        block_unlin(g, nbid, bx, by, bz);
        if (FILTER) {
            const bool edge = bx == cols.c0 || bx == cols.c1;
            if (edge != (cols.cmode == 2)) continue;
        }
        const float4 mp = gather_staging(g, blockmap, staging, bx, by, bz, lx, ly, lz);
        const float m = mp.x;
        const size_t idx = size_t(nbid) * 64 + l;
        V3<float> v0 = {0.f, 0.f, 0.f}, v = {0.f, 0.f, 0.f};
        uint32_t hits = 0;  // effectors within contact range of this node (the adjoint skips the rest)
        if (m > g.mass_eps) {
            const float inv = 1.0f / m;
            v0 = V3<float>{mp.y * inv, mp.z * inv, mp.w * inv};
            v = V3<float>{v0.x + g.gdt[0], v0.y + g.gdt[1], v0.z + g.gdt[2]};
            const int rep = REP ? rep_of_col(g, bx) : 0;  // replicas: local node, the replica's effectors
            const int i = 4 * (bx - rep * g.rstride) + lx, j = 4 * by + ly, kk = 4 * bz + lz;
            v = wall_bc_dev(g, i, j, kk, v);
            const V3<float> p = {float(i) * g.dx, float(j) * g.dx, float(kk) * g.dx};
            if (REP) {
                const EffK<float>* er = eff.ext + rep * eff.per_rep;
                for (int e = 0; e < eff.per_rep; e++) {
                    bool hit;
                    v = effector_contact(er[e], g.inv_dx, g.eps_cells, g.hard != 0, p, v, &hit);
                    hits |= uint32_t(hit) << e;
                }
            } else {
                for (int e = 0; e < eff.n; e++) {
                    bool hit;
                    v = effector_contact(eff.e[e], g.inv_dx, g.eps_cells, g.hard != 0, p, v, &hit);
                    hits |= uint32_t(hit) << e;
                }
            }
        }
        gridv[idx] = make_float4(v.x, v.y, v.z, m);
        if (gridv0) gridv0[idx] = make_float4(v0.x, v0.y, v0.z, m);
        if (cmask) cmask[idx] = uint8_t(hits);
    }
}

void launch_grid_update(const Geom& g, const int* nb_list, const int* n_nb, int grid, const int* blockmap,
                        const float4* staging, float4* gridv, float4* gridv0, const EffSet& eff, uint8_t* cmask,
                        int* clear, int n_clear, cudaStream_t s, int cmode, int c0, int c1) {
    launch_k(eff.ext ? k_grid_update<false, true> : cmode ? k_grid_update<true, false> : k_grid_update<false, false>,
             dim3(grid * (256 / kGridUpdThreads)),
             dim3(kGridUpdThreads), 0, s, g, nb_list, n_nb, blockmap, staging, gridv, gridv0, eff, cmask, clear, n_clear,
             GridCols{cmode, c0, c1});
}

// ---------------------------------------------------------------------------
// G2P (mpm.hpp:338-384) with the per-material return map
// ---------------------------------------------------------------------------

// a few SVD/rigid G2P blocks beside a liquid scene (variant 3): 256-thread CTAs took a full
// block in two rounds instead of four when the pair ran on two streams (c4 42.7 -> 40.1 us);
// as a heavy-first pair 128 threads displace fewer light CTAs (c4 -0.2%)
#ifndef FL_G2P_NTH
#define FL_G2P_NTH 128
#endif
template <bool HEAVY, int MINB, int NT = 128>
__global__ void __launch_bounds__(NT, MINB) k_g2p(Geom g, PBuf in, PBuf out, const uint32_t* __restrict__ perm,
                                             const BlockRec* __restrict__ recs, const int* __restrict__ n_blocks,
                                             const ClassInfo* __restrict__ cls, const float4* __restrict__ gridv,
                                             RigidDev rd, unsigned long long* err, uint32_t substep, int* wq,
                                             int role) {
    const DualScope dual_scope(role);
    __shared__ float4 vt[kTile];
    __shared__ __align__(128) float4 raw[FL_TMA_TILE ? kTileRaw : 1];
    __shared__ __align__(8) uint64_t bar;
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
        const int rep = rep_of_col(g, bx);  // replica contexts (0 otherwise)
        ts.begin(g, gridv, bx, by, bz, tid);
        // the perm -> state loads are the kernel's latency chain: the first particle's
        // position/class loads overlap the tile copy, and later ones run one particle
        // ahead (the permutation two ahead)
        const int j0 = r.start + tid;
        uint32_t s_nx = j0 < r.end ? perm[j0] : 0u;
        V3<float> x_nx = {0.f, 0.f, 0.f};
        uint32_t meta_nx = 0u;
        if (j0 < r.end) {
            x_nx = V3<float>{in.x(0)[s_nx], in.x(1)[s_nx], in.x(2)[s_nx]};
            meta_nx = in.meta[s_nx];
        }
        uint32_t s_nx2 = j0 + NT < r.end ? perm[j0 + NT] : 0u;
        ts.end(g, gridv, vt, bx, by, bz, tid, NT);
        __syncthreads();
        for (int j = j0; j < r.end; j += NT) {
            const uint32_t s = s_nx;
            const V3<float> x = x_nx;
            const uint32_t meta = meta_nx;
            if (j + NT < r.end) {
                s_nx = s_nx2;
                x_nx = V3<float>{in.x(0)[s_nx], in.x(1)[s_nx], in.x(2)[s_nx]};
                meta_nx = in.meta[s_nx];
                if (j + 2 * NT < r.end) s_nx2 = perm[j + 2 * NT];
            }
            const uint32_t pid = in.id[s];
            const ClassInfo ci = cls[meta_cls(meta)];
            StencilW sw;
            stencil_weights(g, x, bx - rep * g.rstride, by, bz, sw);
            V3<float> vraw;
            M3<float> cnew;
            g2p_gather(g, vt, sw, vraw, cnew);
            V3<float> vuse = vraw;
            const float vn = norm(vraw);
            if (vn > g.vmax) vuse = vraw * (g.vmax / vn);
            V3<float> xn;
#pragma unroll
            for (int a = 0; a < 3; a++) xn[a] = clamp_ref(x[a] + vuse[a] * g.dt, g.lo[a], g.hi[a]);
            const bool cin = !HEAVY || f_compact(ci, meta);  // input F = c I
            M3<float> ftr;
            if (cin) {
                ftr = (meye<float>() + cnew * g.dt) * in.F(0)[s];
            } else {
                M3<float> F;
#pragma unroll
                for (int k = 0; k < 9; k++) F.m[k] = in.F(k)[s];
                ftr = (meye<float>() + cnew * g.dt) * F;
            }
            M3<float> fnew = ftr;
            bool ok = true;
            if constexpr (HEAVY) {
                switch (ci.kind) {
                    case MK_LIQUID:
                    case MK_VISCOUS: fnew = liquid_project(ftr, ok); break;
                    case MK_PLASTIC: fnew = box_yield_project(ftr, ci.theta_c, ci.theta_s, ok); break;
                    case MK_NONNEWTONIAN: fnew = von_mises_project(ftr, ci.sigma_y, ci.mu, ok); break;
                    default: break;
                }
            } else {
                fnew = liquid_project(ftr, ok);
            }
            if (!ok) atomicMin(err, (unsigned long long)pack_err(substep, ES_G2P_PROJECT, pid));
#pragma unroll
            for (int a = 0; a < 3; a++) {
                out.x(a)[j] = xn[a];
                out.v(a)[j] = vuse[a];
            }
#pragma unroll
            for (int k = 0; k < 9; k++) out.C(k)[j] = cnew.m[k];
            if (!HEAVY || ci.iso) {  // projected to c I: compact store
                out.F(0)[j] = fnew.m[0];
            } else {
#pragma unroll
                for (int k = 0; k < 9; k++) out.F(k)[j] = fnew.m[k];
            }
            out.meta[j] = meta_cls(meta) | (vn > g.vmax ? kMetaCfl : 0u);
            out.id[j] = pid;
            uint32_t key;
            cell_key(g, xn.x, xn.y, xn.z, key, rep);
            out.key[j] = key;
            if (HEAVY && ci.rigid >= 0) {
                // rigid members carry fp64 positions: v = dx/dt in rigid_body_pass
                // (mpm.hpp:412) would otherwise amplify fp32 rounding by 1/dt
                const int mr = rd.mrank[pid];
                rd.mslot[mr] = j;
#pragma unroll
                for (int a = 0; a < 3; a++) {
                    const double sx = in.mx[3 * mr + a];
                    const double xm = clamp_ref(sx + double(vuse[a]) * double(g.dt), double(g.lo[a]), double(g.hi[a]));
                    rd.mstart[3 * mr + a] = sx;
                    rd.mid[3 * mr + a] = xm;
                    if (a == 0) rd.mact[mr] = 1.0;
                    out.mx[3 * mr + a] = xm;
                    out.x(a)[j] = float(xm);
                }
                cell_key(g, out.x(0)[j], out.x(1)[j], out.x(2)[j], key, rep);
                out.key[j] = key;
            }
        }
    }
}

static decltype(&k_g2p<false, FL_LB_G2P>) g2p_kernel(int v) {
    switch (v) {
        case 0: return k_g2p<false, FL_LB_G2P>;
        case 1: return k_g2p<true, FL_LBH_G2P>;
        case 2: return k_g2p<true, FL_LBD_G2P>;
        default: return k_g2p<true, FL_LBF_G2P, FL_G2P_NTH>;
    }
}
static int g2p_threads(int v) { return v == 3 ? FL_G2P_NTH : 128; }

void launch_g2p(const Geom& g, PBuf in, PBuf out, const uint32_t* perm, const BlockRec* recs, const int* n_blocks,
                int grid, const ClassInfo* cls, const float4* gridv, RigidDev rd, unsigned long long* err,
                uint32_t substep, int variant, int* wq, cudaStream_t s) {
    launch_k(g2p_kernel(variant), dim3(grid), dim3(g2p_threads(variant)), 0, s, g, in, out, perm, recs, n_blocks, cls, gridv, rd, err,
             substep, wq, dual_role());
}

__global__ void k_tail_copy(Geom g, PBuf in, PBuf out, const uint32_t* __restrict__ perm, DN n0, DN n1) {
    pdl_wait();
    int j = n0.get() + blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n1.get()) return;
    uint32_t s = perm[j];
    for (int c = 0; c < 24; c++) out.f[size_t(c) * out.cap + j] = in.f[size_t(c) * in.cap + s];
    out.meta[j] = in.meta[s];
    out.id[j] = in.id[s];
    out.key[j] = g.key_inactive;
}

// parked particles: sorted positions [n_active, n) (departed slots beyond n are dropped);
// there are n_parked of them on every rank
void launch_tail_copy(const Geom& g, PBuf in, PBuf out, const uint32_t* perm, DN n_active, DN n, int n_parked,
                      cudaStream_t s) {
    if (n_parked <= 0) return;
    launch_k(k_tail_copy, dim3((n_parked + 255) / 256), dim3(256), 0, s, g, in, out, perm, n_active, n);
}

// ---------------------------------------------------------------------------
// rigid shape matching (mpm.hpp:386-416, materials.hpp:163-202)
// ---------------------------------------------------------------------------

constexpr int kRigidQ = 17;  // m, m x[3], m x r^T[9], m r[3], count

__global__ void __launch_bounds__(256) k_rigid_partial(PBuf out, RigidDev rd, const int* chunk_m0,
                                                       const int* chunk_m1, double* partial) {
    __shared__ double red[256];
    const int c = blockIdx.x;
    const int m0 = chunk_m0[c], m1 = chunk_m1[c];
    double acc[kRigidQ];
#pragma unroll
    for (int q = 0; q < kRigidQ; q++) acc[q] = 0.0;
    for (int r = m0 + threadIdx.x; r < m1; r += 256) {
        if (rd.mact[r] == 0.0) continue;  // member not active (or, with slabs, not reduced yet)
        const double m = rd.mass[r];
        const double x[3] = {rd.mid[3 * size_t(r)], rd.mid[3 * size_t(r) + 1], rd.mid[3 * size_t(r) + 2]};
        const double* re = rd.rest + 3 * size_t(r);
        acc[0] += m;
        for (int a = 0; a < 3; a++) acc[1 + a] += m * x[a];
        for (int a = 0; a < 3; a++)
            for (int b = 0; b < 3; b++) acc[4 + 3 * a + b] += m * x[a] * re[b];
        for (int a = 0; a < 3; a++) acc[13 + a] += m * re[a];
        acc[16] += 1.0;
    }
    for (int q = 0; q < kRigidQ; q++) {
        red[threadIdx.x] = acc[q];
        __syncthreads();
        for (int w = 128; w > 0; w >>= 1) {
            if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
            __syncthreads();
        }
        if (threadIdx.x == 0) partial[size_t(c) * kRigidQ + q] = red[0];
        __syncthreads();
    }
}

// one thread per body: fit = Kabsch(A), recorded for the adjoint
__global__ void k_rigid_solve(RigidDev rd, int nchunks, const int* chunk_body, const double* partial,
                              unsigned long long* err, uint32_t substep) {
    const int body = blockIdx.x * blockDim.x + threadIdx.x;
    if (body >= rd.nbody) return;
    double s[kRigidQ];
    for (int q = 0; q < kRigidQ; q++) s[q] = 0.0;
    for (int c = 0; c < nchunks; c++) {
        if (chunk_body[c] != body) continue;
        for (int q = 0; q < kRigidQ; q++) s[q] += partial[size_t(c) * kRigidQ + q];
    }
    double* fit = rd.fit + 24 * size_t(body);
    const int nmem = rd.off[body + 1] - rd.off[body];
    fit[22] = (double(nmem) == s[16]) ? 0.0 : 1.0;  // skip unless every member is active
    fit[23] = 1.0;
    if (fit[22] != 0.0) return;
    const double total = s[0];
    V3<double> c = {s[1] / total, s[2] / total, s[3] / total};
    M3<double> A;
    for (int a = 0; a < 3; a++)
        for (int b = 0; b < 3; b++) A.m[3 * a + b] = s[4 + 3 * a + b] - c[a] * s[13 + b];
    Svd<double> t = svd3(A);
    double smax = t.s.x > 1e-30 ? t.s.x : 1e-30;
    if (t.s.y < 1e-12 * smax) {
        atomicMin(err, (unsigned long long)pack_err(substep, ES_RIGID, uint32_t(rd.body_id[body])));
        fit[23] = 0.0;
    }
    M3<double> R = t.U * transpose(t.V);
    if (det(A) < 0.0) R = t.U * mdiag(V3<double>{1.0, 1.0, -1.0}) * transpose(t.V);
    for (int k = 0; k < 9; k++) fit[k] = R.m[k];
    for (int a = 0; a < 3; a++) fit[9 + a] = c[a];
    for (int k = 0; k < 9; k++) fit[12 + k] = A.m[k];
    fit[21] = total;
}

__global__ void k_rigid_apply(Geom g, PBuf out, RigidDev rd) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rd.nmem) return;
    const int body = rd.member_body[r];
    const double* fit = rd.fit + 24 * size_t(body);
    const int j = rd.mslot[r];
    // the fp64 member positions are replicated on every slab (mid is all-reduced)
    if (fit[22] != 0.0) {
        if (rd.mact[r] != 0.0)
            for (int a = 0; a < 3; a++) out.mx[3 * size_t(r) + a] = rd.mid[3 * size_t(r) + a];
        return;
    }
    const double* re = rd.rest + 3 * size_t(r);
    double xn[3];
    for (int a = 0; a < 3; a++) {
        double raw = fit[3 * a] * re[0] + fit[3 * a + 1] * re[1] + fit[3 * a + 2] * re[2] + fit[9 + a];
        xn[a] = clamp_ref(raw, double(g.lo[a]), double(g.hi[a]));
        out.mx[3 * size_t(r) + a] = xn[a];
    }
    if (j < 0) return;  // member lives on another slab
    const double inv_dt = 1.0 / double(g.dt);
    for (int a = 0; a < 3; a++) {
        out.x(a)[j] = float(xn[a]);
        out.v(a)[j] = float((xn[a] - rd.mstart[3 * size_t(r) + a]) * inv_dt);
    }
    uint32_t key;
    cell_key(g, out.x(0)[j], out.x(1)[j], out.x(2)[j], key, rep_of_col(g, key_col(g, out.key[j])));
    out.key[j] = key;
}

void launch_rigid(const Geom& g, PBuf out, RigidDev rd, int nchunks, const int* chunk_body, const int* chunk_m0,
                  const int* chunk_m1, double* partial, unsigned long long* err, uint32_t substep, cudaStream_t s) {
    if (rd.nbody == 0) return;  // (with slabs rd.mid / rd.mact were all-reduced first)
    k_rigid_partial<<<nchunks, 256, 0, s>>>(out, rd, chunk_m0, chunk_m1, partial);
    k_rigid_solve<<<(rd.nbody + 31) / 32, 32, 0, s>>>(rd, nchunks, chunk_body, partial, err, substep);
    k_rigid_apply<<<(rd.nmem + 255) / 256, 256, 0, s>>>(g, out, rd);
}

// ---------------------------------------------------------------------------
// target_point / hold_initial losses at segment boundaries (losses.hpp:474-551)
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(256) k_loss_partial(PBuf st, DN nn, const ClassInfo* __restrict__ cls,
                                                      LossSet ls, uint32_t mask, uint32_t key_inactive,
                                                      double* partial) {
    __shared__ double red[256];
    double acc[kMaxLossTerms];
    for (int k = 0; k < kMaxLossTerms; k++) acc[k] = 0.0;
    const int n = nn.get();
    for (int i = blockIdx.x * 256 + threadIdx.x; i < n; i += gridDim.x * 256) {
        const int body = cls[meta_cls(st.meta[i])].body;
        const uint32_t key = st.key[i];
        if (key > key_inactive) continue;  // departed slot: counted on the particle's new slab
        if (key == key_inactive && !ls.count_parked) continue;
        const bool active = key < key_inactive || ls.act[st.id[i]] <= ls.substep;
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
            acc[k] += (t.kind == LK_TARGET && t.squared) ? nn * nn : nn;
        }
    }
    for (int k = 0; k < ls.n; k++) {
        red[threadIdx.x] = acc[k];
        __syncthreads();
        for (int w = 128; w > 0; w >>= 1) {
            if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
            __syncthreads();
        }
        if (threadIdx.x == 0) partial[size_t(blockIdx.x) * kMaxLossTerms + k] = red[0];
        __syncthreads();
    }
}

// warp k sums term k over the block partials (strided lanes + fixed shuffle tree)
__global__ void k_loss_final(const double* partial, int nblocks, LossSet ls, uint32_t mask, double* out) {
    __shared__ double term[kMaxLossTerms];
    const int lane = threadIdx.x & 31, k = threadIdx.x >> 5;
    double s = 0.0;
    if (k < ls.n)
        for (int b = lane; b < nblocks; b += 32) s += partial[size_t(b) * kMaxLossTerms + k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) term[k] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double total = 0.0;
        for (int q = 0; q < ls.n; q++)
            if ((mask >> q) & 1u) total += ls.t[q].weight * term[q];
        *out = total;
    }
}

void launch_loss(const PBuf& st, DN n, const ClassInfo* cls, const LossSet& ls, uint32_t mask, double* partial,
                 double* out, uint32_t key_inactive, cudaStream_t s) {
    k_loss_partial<<<kLossBlocks, 256, 0, s>>>(st, n, cls, ls, mask, key_inactive, partial);
    k_loss_final<<<1, 32 * kMaxLossTerms, 0, s>>>(partial, kLossBlocks, ls, mask, out);
}

int occupancy_grid_fwd(KGrid which, int variant) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (which == KG_P2G) {
        cudaFuncSetAttribute(p2g_kernel(variant), cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(ScSmem)));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, p2g_kernel(variant), p2g_threads(variant), sizeof(ScSmem));
    } else {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, g2p_kernel(variant), g2p_threads(variant), 0);
    }
    if (per < 1) per = 1;
    return sms * per;
}

}  // namespace fl
