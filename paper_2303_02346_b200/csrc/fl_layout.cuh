// fl_layout.cuh -- HBM data layout shared by the kernels and the host engine.
//
// Particles: SoA fp32 (x[3], v[3], F[9], C[9]) plus u32 class / id / cell-key
// per slot; every trajectory state is one such buffer.  The grid is dense but
// block-major: 4x4x4 node blocks, node (i,j,k) lives at
//     block_lin(i>>2, j>>2, k>>2) * 64 + ((i&3)<<4 | (j&3)<<2 | (k&3)).
// Particles are kept in canonical order: stable by (cell key, particle id),
// where the cell key of a particle is
//     block_lin(base>>2) << 6 | (base&3) packed like a node,   base = floor(x/dx - 0.5)
// (the B-spline base cell of quad_weights, proj/include/flume/mpm.hpp:55-71).
// A 4x4x4 block of base cells (a "particle block") scatters into the 6x6x6
// node tile [4B, 4B+6): its own node block plus two planes of the next ones.
#pragma once

#include <cstdint>

#include "fl_physics.cuh"

namespace fl {

constexpr int kMaxEff = 8;
constexpr uint32_t kTile = 216;  // 6^3 nodes per particle-block tile

struct Geom {
    int nd[3];      // node dims (res+1 per axis, types.hpp:84-88)
    int NB[3];      // 4^3 blocks per axis (cover nd)
    int nbtot;      // NB0*NB1*NB2
    int maxb;       // particle-block list capacity: light blocks at [0, n0), heavy at [maxb - n1, maxb)
    uint32_t key_inactive;  // nbtot << 6, sorts after every valid key
    uint32_t key_departed;  // (nbtot + 1) << 6: slot left by a particle that moved to another slab
    int keybits;    // bits needed for key_departed
    int sx0, sx1;   // x-slab of particle-block columns owned by this rank ([0, NB0) for one rank)
    int colblocks;  // NB1 * NB2 blocks per x column
    // replica contexts (a population of one scene side by side in one grid): particle-block
    // x columns per replica including one empty gap column; nd is one replica's node grid and
    // positions stay replica-local.  0: one scene.
    int rstride;
    int idbits;     // bits needed for particle ids
    float dx, inv_dx, dt;
    float lo[3], hi[3];  // clamp_to_interior bounds [dx, L-dx] (mpm.hpp:330-336)
    int bw;              // wall band (types.hpp:61)
    float vmax;          // cfl_fraction * dx / dt (mpm.hpp:322-328)
    float mass_eps;
    float gdt[3];        // gravity * dt
    float eps_cells;
    int hard;
    float k4;            // 4 / dx^2
    float stress_coeff;  // dt * 4 / dx^2 (mpm.hpp:259)
};

// class word of a particle: class index, plus bit 31 set by G2P when the CFL
// clamp (mpm.hpp:322-328) was active in the substep that produced the state
constexpr uint32_t kMetaCfl = 0x80000000u;
// bit 30: an isotropic-class particle whose F is not c*I yet (see f_compact)
constexpr uint32_t kMetaFull = 0x40000000u;
__host__ __device__ inline uint32_t meta_cls(uint32_t m) { return m & 0x3fffffffu; }

// one entry per distinct (material, body, mass, volume0) tuple
struct ClassInfo {
    int kind;
    int body;
    int rigid;   // rigid-body index or -1
    int heavy;   // needs the SVD / rigid code paths (anything but a plain liquid)
    int iso;     // liquid / viscous liquid: the return map makes F = c I (materials.hpp:147-153)
    float mass, vol0;
    float mu, lambda, theta_c, theta_s, sigma_y;
    int rep;     // replica of the class's particles (replica contexts; 0 otherwise)
};

// Compact deformation gradient.  The return map of (viscous) liquids resets F
// to det(F)^(1/3) I every substep, so for those classes the store keeps only
// c = F(0) (F(1..8) are not read or written) and the cotangent likewise only
// dL/dc = tr(F_bar) -- exact, because every consumer of an isotropic F (the
// stress, the trial F, liquid_project_vjp) depends on c alone.  This removes
// 8 of the 24 state floats from every pass over a liquid particle.  A particle
// uploaded with a non-isotropic F carries kMetaFull (full 3x3, heavy path)
// until its first G2P.
__host__ __device__ inline bool f_compact(const ClassInfo& ci, uint32_t meta) {
    return ci.iso != 0 && (meta & kMetaFull) == 0u;
}

struct EffSet {
    int n;
    EffK<float> e[kMaxEff];
    // replica contexts: per_rep effectors per replica, all n of them in device memory (ext)
    int per_rep;
    const EffK<float>* ext;
};

struct PBuf {
    float* f;         // [24][cap]: x0 x1 x2 v0 v1 v2 F00..F22 C00..C22
    uint32_t* meta;   // class index
    uint32_t* id;     // reference particle index
    uint32_t* key;    // cell key (key_inactive for inactive)
    double* mx;       // [3*nmem] fp64 positions of rigid-body members, by member rank
    int cap;
    __host__ __device__ float* x(int a) const { return f + size_t(a) * cap; }
    __host__ __device__ float* v(int a) const { return f + size_t(3 + a) * cap; }
    __host__ __device__ float* F(int k) const { return f + size_t(6 + k) * cap; }
    __host__ __device__ float* C(int k) const { return f + size_t(15 + k) * cap; }
};

// 24-float cotangent buffer with the same component order (x v F C)
struct BarBuf {
    float* f;
    int cap;
    __host__ __device__ float* x(int a) const { return f + size_t(a) * cap; }
    __host__ __device__ float* v(int a) const { return f + size_t(3 + a) * cap; }
    __host__ __device__ float* F(int k) const { return f + size_t(6 + k) * cap; }
    __host__ __device__ float* C(int k) const { return f + size_t(15 + k) * cap; }
};

struct BlockRec {
    int block;  // particle-block linear index
    int start;  // sorted positions [start, end)
    int end;
};

// error record: lexicographic min over (substep, stage, particle/body)
enum ErrStage : uint32_t {
    ES_P2G_ESCAPE = 1,
    ES_P2G_STRESS = 2,
    ES_G2P_PROJECT = 3,
    ES_RIGID = 4,
    ES_LOSS_EMPTY = 5,  // who: 0 chamfer_distance on an empty set, 1 mixing_spread with < 2 particles
};

__host__ __device__ inline uint64_t pack_err(uint32_t substep, uint32_t stage, uint32_t who) {
    return (uint64_t(substep) << 36) | (uint64_t(stage) << 32) | uint64_t(who);
}

__host__ __device__ inline int block_lin(const Geom& g, int bx, int by, int bz) {
    return (bx * g.NB[1] + by) * g.NB[2] + bz;
}
__host__ __device__ inline void block_unlin(const Geom& g, int b, int& bx, int& by, int& bz) {
    bz = b % g.NB[2];
    int r = b / g.NB[2];
    by = r % g.NB[1];
    bx = r / g.NB[1];
}
// Programmatic dependent launch (sm_90+): hot-path kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization (launch_k, fl_kernels.h), so
// a kernel's CTAs are scheduled while its predecessor drains; each such kernel
// waits here, before touching memory, until the predecessor grid has completed.
#ifndef FL_PDL
#define FL_PDL 1
#endif
#ifndef FL_PDL_TRIGGER
#define FL_PDL_TRIGGER 0
#endif
// Every kernel starts with this: wait for the previous grid on the stream (its writes are
// visible afterwards).  FL_PDL_TRIGGER = 1 would also release the next grid right away
// (griddepcontrol.launch_dependents); measured: neutral on c4, but its early CTAs then sit
// in their wait holding SM resources, which costs small scenes 8-16% (c1) and starves
// concurrent contexts of a population, so the dependent launches when this grid exits.
__device__ __forceinline__ void pdl_wait() {
#if defined(__CUDA_ARCH__) && FL_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");
#if FL_PDL_TRIGGER
    asm volatile("griddepcontrol.launch_dependents;" :::);
#endif
#endif
}

// The SVD/rigid and plain-liquid variants of a scatter/gather kernel ("dual" launches) run
// back to back on one stream: the heavy grid (role 1) waits for its predecessor as usual and
// then releases its dependent at once (griddepcontrol.launch_dependents), so the light grid
// (role 2) is placed beside the heavy CTAs already resident instead of filling every SM
// first.  The light grid reads only what the heavy grid's predecessor wrote (complete: the
// heavy grid waited for it before releasing), so it skips the start wait and waits for the
// heavy grid at its end instead -- the next kernel then sees both.  Role 0: a plain launch.
struct DualScope {
    int role;
    __device__ __forceinline__ explicit DualScope(int r) : role(r) {
        if (role != 2) pdl_wait();
#if defined(__CUDA_ARCH__) && FL_PDL
        if (role == 1) asm volatile("griddepcontrol.launch_dependents;" :::);
#endif
    }
    __device__ __forceinline__ ~DualScope() {
#if defined(__CUDA_ARCH__) && FL_PDL
        if (role == 2) asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
    }
};

__host__ __device__ inline int key_col(const Geom& g, uint32_t key) { return int(key >> 6) / g.colblocks; }

// sort block of a key: its particle block, or the virtual parked / departed blocks nbtot, nbtot + 1
__host__ __device__ inline int key_block(const Geom& g, uint32_t key) {
    return key >= g.key_inactive ? g.nbtot + int((key - g.key_inactive) >> 6) : int(key >> 6);
}
// bit 31 of a sorted key word (okey) / sort slot word: the particle takes the SVD/rigid path
constexpr uint32_t kHeavyBit = 0x80000000u;

__host__ __device__ inline size_t node_index(const Geom& g, int i, int j, int k) {
    return size_t(block_lin(g, i >> 2, j >> 2, k >> 2)) * 64 + (((i & 3) << 4) | ((j & 3) << 2) | (k & 3));
}

// Canonical base-cell computation.  Written with explicitly rounded fp32 ops
// (no FMA contraction) so a CPU recomputation from the same fp32 positions is
// bit-identical.
#if defined(__CUDA_ARCH__)
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
#else
inline float mul_rn(float a, float b) { volatile float r = a * b; return r; }
inline float sub_rn(float a, float b) { volatile float r = a - b; return r; }
#endif

__host__ __device__ inline int base_cell(float x, float inv_dx, float& fx) {
    float xs = mul_rn(x, inv_dx);
    float b = floorf(sub_rn(xs, 0.5f));
    fx = sub_rn(xs, b);
    return int(b);
}

// replica of a particle-block x column (replica contexts)
__host__ __device__ inline int rep_of_col(const Geom& g, int bx) { return g.rstride ? bx / g.rstride : 0; }

// returns false when the stencil leaves the grid (mpm.hpp:265-269); rep: the particle's
// replica (its blocks start at x column rep * rstride)
__host__ __device__ inline bool cell_key(const Geom& g, float x0, float x1, float x2, uint32_t& key, int rep = 0) {
    float f;
    int b0 = base_cell(x0, g.inv_dx, f), b1 = base_cell(x1, g.inv_dx, f), b2 = base_cell(x2, g.inv_dx, f);
    bool ok = b0 >= 0 && b1 >= 0 && b2 >= 0 && b0 + 2 < g.nd[0] && b1 + 2 < g.nd[1] && b2 + 2 < g.nd[2];
    if (!ok) {
        b0 = b0 < 0 ? 0 : (b0 > g.nd[0] - 3 ? g.nd[0] - 3 : b0);
        b1 = b1 < 0 ? 0 : (b1 > g.nd[1] - 3 ? g.nd[1] - 3 : b1);
        b2 = b2 < 0 ? 0 : (b2 > g.nd[2] - 3 ? g.nd[2] - 3 : b2);
    }
    key = (uint32_t(block_lin(g, (b0 >> 2) + rep * g.rstride, b1 >> 2, b2 >> 2)) << 6) |
          uint32_t(((b0 & 3) << 4) | ((b1 & 3) << 2) | (b2 & 3));
    return ok;
}

// quadratic B-spline weights (mpm.hpp:63-68) and their d/dfx
__host__ __device__ inline void bspline_w(float fx, float w[3]) {
    float a = 1.5f - fx, b = fx - 1.0f, c = fx - 0.5f;
    w[0] = 0.5f * a * a;
    w[1] = 0.75f - b * b;
    w[2] = 0.5f * c * c;
}
__host__ __device__ inline void bspline_dw(float fx, float dw[3]) {
    dw[0] = fx - 1.5f;
    dw[1] = -2.0f * (fx - 1.0f);
    dw[2] = fx - 0.5f;
}

}  // namespace fl
