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

constexpr int kScThreads = 192;  // 64 cells x 3 planes
constexpr int kScChunk = 512;    // particles staged per pass
constexpr int kPayStride = 17;   // 16 payload floats, odd stride vs. bank conflicts

struct ScSmem {
    union {
        float pay[kScChunk * kPayStride];
        float cellpart[64 * 27 * 4];
    } u;
    uint8_t lc[kScChunk];
    int16_t cs[64], ce[64];
};

__device__ __forceinline__ void sc_ranges(ScSmem& sm, int n, int tid, int nthreads) {
    for (int i = tid; i < n; i += nthreads) {
        const int c = sm.lc[i];
        if (i == 0 || sm.lc[i - 1] != c) sm.cs[c] = int16_t(i);
        if (i == n - 1 || sm.lc[i + 1] != c) sm.ce[c] = int16_t(i + 1);
    }
}

// payload layout: [0..2] fx, then (NCH==4 ? m : -), a[3], Bm[9] row-major
template <int NCH>
__device__ __forceinline__ void sc_accumulate(const ScSmem& sm, int c, int ox, float (&acc)[9][4]) {
    constexpr int A0 = (NCH == 4) ? 4 : 3;
    const float oxf = float(ox);
    for (int i = sm.cs[c]; i < sm.ce[c]; i++) {
        const float* p = &sm.u.pay[i * kPayStride];
        float wxa[3], wy[3], wz[3];
        bspline_w(p[0], wxa);
        bspline_w(p[1], wy);
        bspline_w(p[2], wz);
        const float wx = wxa[ox];
        const float m = (NCH == 4) ? p[3] : 0.f;
        const float b00 = p[A0 + 3], b01 = p[A0 + 4], b02 = p[A0 + 5];
        const float b10 = p[A0 + 6], b11 = p[A0 + 7], b12 = p[A0 + 8];
        const float b20 = p[A0 + 9], b21 = p[A0 + 10], b22 = p[A0 + 11];
        const float a0x = p[A0] + b00 * oxf, a0y = p[A0 + 1] + b10 * oxf, a0z = p[A0 + 2] + b20 * oxf;
#pragma unroll
        for (int oy = 0; oy < 3; oy++) {
            const float oyf = float(oy);
            const float ayx = a0x + b01 * oyf, ayy = a0y + b11 * oyf, ayz = a0z + b21 * oyf;
            const float wxy = wx * wy[oy];
#pragma unroll
            for (int oz = 0; oz < 3; oz++) {
                const float ozf = float(oz);
                const float w = wxy * wz[oz];
                const float vx = ayx + b02 * ozf, vy = ayy + b12 * ozf, vz = ayz + b22 * ozf;
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
}

template <int NCH>
__device__ __forceinline__ void sc_store_cellpart(ScSmem& sm, int c, int ox, const float (&acc)[9][4]) {
#pragma unroll
    for (int k = 0; k < 9; k++) {
        float* d = &sm.u.cellpart[(c * 27 + ox * 9 + k) * 4];
#pragma unroll
        for (int q = 0; q < 4; q++) d[q] = (q < NCH) ? acc[k][q] : 0.f;
    }
}

// fold cell partials into the 6^3 tile (fixed order) and store it
__device__ __forceinline__ void sc_tile(const ScSmem& sm, float4* out, int tid, int nthreads) {
    for (int t = tid; t < int(kTile); t += nthreads) {
        const int tx = t / 36, ty = (t / 6) % 6, tz = t % 6;
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
        const int cx0 = tx > 2 ? tx - 2 : 0, cx1 = tx < 3 ? tx : 3;
        const int cy0 = ty > 2 ? ty - 2 : 0, cy1 = ty < 3 ? ty : 3;
        const int cz0 = tz > 2 ? tz - 2 : 0, cz1 = tz < 3 ? tz : 3;
        for (int cx = cx0; cx <= cx1; cx++)
            for (int cy = cy0; cy <= cy1; cy++)
                for (int cz = cz0; cz <= cz1; cz++) {
                    const int c = cx * 16 + cy * 4 + cz;
                    const int k = (tx - cx) * 9 + (ty - cy) * 3 + (tz - cz);
                    const float* p = &sm.u.cellpart[(c * 27 + k) * 4];
                    s0 += p[0];
                    s1 += p[1];
                    s2 += p[2];
                    s3 += p[3];
                }
        out[t] = make_float4(s0, s1, s2, s3);
    }
}

// 6^3 node tile of a block-major float4 grid into shared memory
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

// v = sum w gv, C = (4/dx^2) sum w gv rel^T with rel = dx (o - fx)  (mpm.hpp:352-361)
__device__ __forceinline__ void g2p_gather(const Geom& g, const float4* tile, const StencilW& s, V3<float>& v,
                                           M3<float>& c) {
    v = V3<float>{0.f, 0.f, 0.f};
    c = mzero<float>();
    const float kd = g.k4 * g.dx;
#pragma unroll
    for (int ox = 0; ox < 3; ox++) {
        const float rx = (float(ox) - s.fx[0]) * kd;
#pragma unroll
        for (int oy = 0; oy < 3; oy++) {
            const float ry = (float(oy) - s.fx[1]) * kd;
            const float wxy = s.w[0][ox] * s.w[1][oy];
#pragma unroll
            for (int oz = 0; oz < 3; oz++) {
                const float rz = (float(oz) - s.fx[2]) * kd;
                const float w = wxy * s.w[2][oz];
                const float4 gv = tile[(s.l[0] + ox) * 36 + (s.l[1] + oy) * 6 + (s.l[2] + oz)];
                const float wx = w * gv.x, wy = w * gv.y, wz = w * gv.z;
                v.x += wx;
                v.y += wy;
                v.z += wz;
                c.m[0] += wx * rx; c.m[1] += wx * ry; c.m[2] += wx * rz;
                c.m[3] += wy * rx; c.m[4] += wy * ry; c.m[5] += wy * rz;
                c.m[6] += wz * rx; c.m[7] += wz * ry; c.m[8] += wz * rz;
            }
        }
    }
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
